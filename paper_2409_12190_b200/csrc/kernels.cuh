// Launch interface of the sm_100a kernels (kernels.cu).
#pragma once

#include <cuda_runtime.h>

#include "device.cuh"

namespace bae {

enum WsKind { kWsLin = 0, kWsCost = 1, kWsPrep = 2, kWsSchur = 3, kWsTrial = 4, kWsKinds = 5 };

// Dynamic shared memory per tile kernel, sized for the largest small tile.
struct SmemSizes {
  int lin = 0, cost = 0, prep = 0, schur = 0, trial = 0;
};

long long tile_ws_bytes(int kind, int ncam, int npts, int nobs);
void set_smem_limits(int max_bytes);

void launch_camrec(const Dev& d, bool trial, cudaStream_t s);
void launch_linearize(const Dev& d, const SmemSizes& sm, bool write_jac, cudaStream_t s);
void launch_cost(const Dev& d, const SmemSizes& sm, bool trial, cudaStream_t s);
void launch_prep(const Dev& d, const SmemSizes& sm, double lambda, double clo, double chi, double tol,
                 long long budget, cudaStream_t s);
void launch_pcg_iteration(const Dev& d, const SmemSizes& sm, cudaStream_t s);
void launch_schur_only(const Dev& d, const SmemSizes& sm, cudaStream_t s);
void launch_trial(const Dev& d, const SmemSizes& sm, cudaStream_t s);
void launch_commit(const Dev& d, cudaStream_t s);

// kernel launches issued per wrapper (for the bench's gpu_launches count)
constexpr int kLaunchesLinearize = 2, kLaunchesCost = 2, kLaunchesPrep = 2, kLaunchesPcgIter = 3,
              kLaunchesTrial = 3, kLaunchesCommit = 1, kLaunchesCamrec = 1;

}  // namespace bae
