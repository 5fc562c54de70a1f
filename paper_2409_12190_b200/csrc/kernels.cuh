// Launch interface of the sm_100a kernels (kernels.cu).
#pragma once

#include <cuda_runtime.h>

#include "device.cuh"

namespace bae {

enum WsKind { kWsLin = 0, kWsCost = 1, kWsPrep = 2, kWsSchur = 3, kWsTrial = 4, kWsKinds = 5 };

// Launch shape of one warp-tile kernel: `slice` bytes of shared memory per
// warp (largest small tile of that kind) and `wpb` warps (tiles) per CTA.
struct TileLaunch {
  int slice = 0, wpb = 1;
};
struct SmemSizes {
  TileLaunch lin, cost, prep, schur, trial;
};

long long tile_ws_bytes(int kind, int ncam, int npts, int nobs);
void set_smem_limits(int max_bytes);

void launch_camrec(const Dev& d, bool trial, cudaStream_t s);
void launch_linearize(const Dev& d, const SmemSizes& sm, bool write_jac, cudaStream_t s);
void launch_cost(const Dev& d, const SmemSizes& sm, cudaStream_t s);
void launch_prep(const Dev& d, const SmemSizes& sm, double lambda, double clo, double chi, double tol,
                 long long budget, cudaStream_t s);
void launch_pcg_iteration(const Dev& d, const SmemSizes& sm, cudaStream_t s);
// Cooperative persistent PCG (whole solve, grid barriers between phases).
int pcg_persistent_grid(const Dev& d, const SmemSizes& sm);
cudaError_t launch_pcg_persistent(const Dev& d, const SmemSizes& sm, int grid, long long max_iters, cudaStream_t s);
void launch_schur_only(const Dev& d, const SmemSizes& sm, cudaStream_t s);
void launch_trial(const Dev& d, const SmemSizes& sm, cudaStream_t s);
void launch_commit(const Dev& d, cudaStream_t s);
void launch_schur_dense(const Dev& d, cudaStream_t s);

// kernel launches issued per wrapper (for the bench's gpu_launches count)
constexpr int kLaunchesLinearize = 2, kLaunchesCost = 2, kLaunchesPrep = 2, kLaunchesPcgIter = 3,
              kLaunchesTrial = 3, kLaunchesCommit = 1, kLaunchesCamrec = 1;

}  // namespace bae
