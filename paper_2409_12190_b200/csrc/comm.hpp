// Collectives of the landmark-sharded solver.
//
// Each rank owns a contiguous range of points and all their observations;
// cameras are replicated. The only data exchanged are camera-sized partial
// sums (H_cc | g_c after the linearisation, the Schur diagonal blocks and
// RHS after the prep, the 6C reduced-system product once per PCG iteration,
// the dense reduced matrix for the direct solve) plus a few scalars (cost,
// ||g_p||^2, failure flags, the lowest cheirality observation). They are all
// in-place sums on device buffers, issued on the solver stream.
//
// Two backends implement the same interface:
//   * NcclComm  - one process per GPU, ncclAllReduce over NVLink / NVSwitch.
//                 NCCL is loaded at run time (dlopen), so single-GPU use of
//                 the library never needs it. Capturable in CUDA graphs.
//   * GroupComm - ranks that share one process (one host thread per rank),
//                 on one device or several peer-enabled devices. The sum is a
//                 kernel that reads every rank's buffer directly (peer memory
//                 over NVLink when the devices differ) in fixed rank order,
//                 fenced by CUDA events and a host barrier. It lets the whole
//                 sharded path run, and be tested, on a single GPU.
// Both produce bit-identical results on every rank, so every rank takes the
// same control-flow decisions (PCG state machine, LM accept/reject) without
// any further exchange.
#pragma once

#include <cuda_runtime.h>

#include <cstddef>
#include <memory>

#include "bae_b200.h"

struct bae_group;  // opaque in-process rank group (bae_group_create)

namespace bae {

class Comm {
 public:
  Comm(int rank, int world) : rank_(rank), world_(world) {}
  virtual ~Comm() = default;
  int rank() const { return rank_; }
  int world() const { return world_; }
  // In-place element-wise sum of n doubles over all ranks.
  virtual void allreduce_sum(double* buf, std::size_t n, cudaStream_t s) = 0;
  // In-place element-wise minimum of n int32 over all ranks.
  virtual void allreduce_min(int* buf, std::size_t n, cudaStream_t s) = 0;
  // In-place element-wise sum of n doubles over all ranks, valid on `root` only.
  virtual void reduce_sum(double* buf, std::size_t n, int root, cudaStream_t s) = 0;
  // buf (bytes) of `root` into buf of every rank.
  virtual void broadcast(void* buf, std::size_t bytes, int root, cudaStream_t s) = 0;
  // recv[r * bytes .. (r+1) * bytes) = send of rank r.
  virtual void allgather(const void* send, void* recv, std::size_t bytes, cudaStream_t s) = 0;
  // Whether the collectives may be captured into a CUDA graph.
  virtual bool capturable() const = 0;
  virtual const char* kind() const = 0;

 private:
  int rank_, world_;
};

// 128-byte ncclUniqueId (rank 0 creates it, every rank passes it to bae_create_ba).
void nccl_unique_id(void* out128);
std::unique_ptr<Comm> make_nccl_comm(const void* id128, int rank, int world, int device);
std::unique_ptr<Comm> make_group_comm(bae_group* g, int rank, int device);
bae_group* group_create(int world);
void group_destroy(bae_group* g);

}  // namespace bae
