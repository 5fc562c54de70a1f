// Pose-graph optimisation on the device: the
// relative-pose model of make_pgo_problem (problems.hpp:141-188) solved with
// the same LM driver semantics (lm.hpp:115-255) and the tile-sparse Cholesky
// of the direct BA solver (chol.cuh) on the 6x6-block normal matrix.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <vector>

#include "bae_internal.hpp"
#include "chol.cuh"

namespace bae {

bool plateau_stagnation(const double* h, std::size_t n, int patience, double tol);  // lm.hpp:89-98 (problem.cu)

// Device view of a pose graph.
struct PgoDev {
  int n, anchor, nsys;          // poses, anchored first pose (0/1), unknown poses = n - anchor
  long long m;                  // edges
  const int* ei;
  const int* ej;
  const double* meas;           // 7 m
  const double* white;          // 36 m row-major L^T, or null (no information anywhere)
  double* pose;                 // 7 n
  double* pose_t;               // 7 n trial
  double* edge;                 // 28 m: M = J^T J (21 packed), v = J^T r (6), cost (1)
  double* resid;                // 6 m whitened residual rows (export) or null
  double* jexp;                 // 36 m: J_j (export) or null
  const int* inc_ptr;           // nsys + 1: incident edges of each unknown pose
  const int* inc;               // edge id << 1 | (1 if the pose is endpoint j)
  const int* pair_ptr;          // npair + 1: edges between two unknown poses
  const int* pair_edge;         // edge ids, ascending per pair
  int npair;
  const int2* diag_tile;        // nsys: {tile slot, offset}
  const int2* pair_tile;        // npair: {tile slot, row off | col off << 8 | transposed << 16}
  double* tiles;
  double* rhs;                  // 6 nsys
  double* x;                    // 6 nsys
  double* pose_gsq;             // nsys
  double* scal;                 // [cost, grad_sq, new_cost, bad, trial_bad]
};

class PgoProblem {
 public:
  PgoProblem(const double* poses7, int n, const std::int32_t* ei, const std::int32_t* ej, const double* meas7,
             const double* info36, const std::int32_t* has_info, std::int64_t m, bool anchor_first,
             const bae_create_options& opt);
  ~PgoProblem();
  PgoProblem(const PgoProblem&) = delete;
  PgoProblem& operator=(const PgoProblem&) = delete;

  int num_poses() const { return d_.n; }
  std::int64_t num_edges() const { return d_.m; }
  long long launches() const { return launches_; }
  void set_parameters(const double* poses7);
  void get_parameters(double* poses7);
  double evaluate(double* resid6);  // whitened residual rows, edge order
  void jacobian(double* ji36, double* jj36);  // per edge d r_w / d pose_i, d pose_j (row-major 6x6)
  void optimize(const double* poses7, const bae_lm_config& cfg, std::vector<bae_iter_record>& traj,
                bae_lm_report& rep);

 private:
  template <class T>
  T* dalloc(std::size_t n);
  template <class T>
  T* upload(const std::vector<T>& v);
  void sync();
  void read_scal();
  void linearize();
  bool solve(double lambda, const bae_lm_config& cfg);

  bae_create_options opt_;
  PgoDev d_{};
  TileChol tchol_{};
  int chol_grid_ = 0;
  cudaStream_t stream_ = nullptr;
  std::vector<void*> allocs_;
  double* scal_host_ = nullptr;
  int* fail_host_ = nullptr;
  long long launches_ = 0;
};

}  // namespace bae
