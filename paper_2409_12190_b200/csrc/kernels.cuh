// Launch interface of the sm_100a kernels (kernels.cu).
#pragma once

#include <cuda_runtime.h>

#include "comm.hpp"
#include "device.cuh"

namespace bae {

enum WsKind { kWsLin = 0, kWsCost = 1, kWsPrep = 2, kWsSchur = 3, kWsTrial = 4, kWsPrepDir = 5, kWsLinPrep = 6, kWsKinds = 7 };

// Launch shape of one warp-tile kernel: `slice` bytes of shared memory per
// warp (largest small tile of that kind) and `wpb` warps (tiles) per CTA.
struct TileLaunch {
  int slice = 0, wpb = 1;
};
struct SmemSizes {
  TileLaunch lin, cost, prep, schur, trial, prepd, linprep;
};

long long tile_ws_bytes(int kind, int ncam, int npts, int nobs);
void set_smem_limits(int max_bytes);

// Launch wrappers return the number of kernels they launched (the bench's
// gpu_launches). `comm` is null on a single rank; on sharded runs the
// wrapper inserts the cross-rank sums between the tile and camera passes.
int launch_camrec(const Dev& d, bool trial, cudaStream_t s);
int launch_gather_pixels(const double* raw, const int* orig, double* px, long long N, cudaStream_t s);
int launch_points_permute(const double* in, const int* src, double* out, int P, bool to_internal, cudaStream_t s);
int launch_linearize(const Dev& d, const SmemSizes& sm, bool write_jac, cudaStream_t s, Comm* comm);
// Single rank, direct solver, after an accepted step: the linearisation
// and the prep for the damping in d.lam in one pass (k_lin_prep,
// k_cam_lin_prep, k_lin_totals). Needs d.pcg zeroed first.
int launch_lin_prep(const Dev& d, const SmemSizes& sm, double clo, double chi, cudaStream_t s);
// The two halves of launch_lin_prep: the tile pass, then the camera pass + totals
// (on a second stream beside the Schur assembly, single rank).
int launch_lin_prep_tiles(const Dev& d, const SmemSizes& sm, double clo, double chi, cudaStream_t s);
int launch_lin_prep_cams(const Dev& d, double clo, double chi, cudaStream_t s);
int launch_cost(const Dev& d, const SmemSizes& sm, cudaStream_t s, Comm* comm);
// direct = true: the direct solver's prep (RHS, damped H_cc, per-slot W and
// W H~_pp^-1; no block-Jacobi preconditioner and no PCG start state).
int launch_prep(const Dev& d, const SmemSizes& sm, double lambda, double clo, double chi, double tol,
                long long budget, cudaStream_t s, Comm* comm, bool direct);
int launch_pcg_iteration(const Dev& d, const SmemSizes& sm, cudaStream_t s, Comm* comm);
// Cooperative persistent PCG (whole solve, grid barriers between phases; single rank only).
int pcg_persistent_grid(const Dev& d, const SmemSizes& sm);
cudaError_t launch_pcg_persistent(const Dev& d, const SmemSizes& sm, int grid, long long max_iters, cudaStream_t s);
int launch_schur_only(const Dev& d, const SmemSizes& sm, cudaStream_t s);
int launch_trial(const Dev& d, const SmemSizes& sm, cudaStream_t s, Comm* comm);
int launch_commit(const Dev& d, cudaStream_t s);
constexpr int kSchurChunk = 128;  // pairs per k_schur_dense warp (at most)
// defer_hccd: the diagonal blocks leave out H~_cc (launch_add_hccd adds it
// once the camera pass that forms it has run).
int launch_schur_dense(const Dev& d, cudaStream_t s, Comm* comm, bool defer_hccd = false);
int launch_add_hccd(const Dev& d, cudaStream_t s);

}  // namespace bae
