// Device-resident BA problem (one GPU / one rank).
#pragma once

#include <cstdlib>

#include <cuda_runtime.h>
#include <cusolverDn.h>

#include <cstdint>
#include <memory>
#include <vector>

#include "bae_internal.hpp"
#include "chol.cuh"
#include "comm.hpp"
#include "kernels.cuh"

namespace bae {

struct TileCholHost;  // problem.cu: the host half of the tile Cholesky's symbolic phase

struct SolveInfo {
  long long iters = 0;
  bool converged = false;
  double rel_residual = 0.0;
  bool pending = false;  // direct solve: the failure word is read after the caller's next synchronisation
};

bool plateau_stagnation(const double* h, std::size_t n, int patience, double tol);

// Device-time breakdown of the LM loop by phase (CUDA events on the solver
// stream, accumulated after each synchronising read-back).
enum Phase : int {
  kPhLinearize = 0,  // K1 + camera reduction
  kPhPrep = 1,       // damping, H~pp^-1, Schur RHS / block-Jacobi
  kPhAssemble = 2,   // dense reduced matrix (direct solver)
  kPhFactor = 3,     // potrf + potrs (direct solver)
  kPhPcg = 4,        // PCG iterations
  kPhTrial = 5,      // retraction, back-substitution, trial cost
  kPhCommit = 6,     // accept
  kPhases = 7
};

// The observation decomposition as it lives in device memory (read back for
// the structure exports: the Jacobian pattern, the transpose plans and the
// normal matrix's block patterns are derived from these arrays, not from the
// host planner's copies).
struct DeviceStructure {
  int C = 0, P = 0, T = 0, E = 0;
  std::int64_t N = 0;
  std::vector<std::int32_t> tile_obs_begin, tile_pt_begin, tile_ent_begin;  // T+1
  std::vector<std::uint32_t> obs_lcpt;                                      // N
  std::vector<std::int32_t> obs_orig;                                       // N
  std::vector<std::int32_t> ent_cam, ent_obs_begin;                         // E, E+1
  std::vector<std::int32_t> cam_ent_ptr, cam_ent;                           // C+1, E
  std::vector<std::int32_t> pt_ptr;                                         // P+1
  std::vector<std::uint16_t> ptobs;                                         // N
  std::vector<std::int32_t> pt_of_internal;                                 // P
  // (camera, point) of slot s of tile t
  int slot_cam(int t, int s) const;
  int slot_pt(int t, int s) const {
    return pt_of_internal[tile_pt_begin[t] + static_cast<int>(obs_lcpt[s] >> 16)];
  }
};

class Problem {
 public:
  Problem(const double* poses7, int C, const double* points3, int P, const double* intr3,
          const std::int32_t* cam_idx, const std::int32_t* pt_idx, const double* px2, std::int64_t N,
          const bae_create_options& opt);
  ~Problem();
  Problem(const Problem&) = delete;
  Problem& operator=(const Problem&) = delete;

  int num_cameras() const { return d_.C; }
  int num_points() const { return P_global_; }
  std::int64_t num_obs() const { return N_global_; }
  // Sharded problem: this rank owns a contiguous range of the
  // points and all their observations; plan() / dev() describe that part.
  bool distributed() const { return comm_ != nullptr; }
  int rank() const { return comm_ ? comm_->rank() : 0; }
  int world() const { return comm_ ? comm_->world() : 1; }
  int local_points() const { return d_.P; }
  std::int64_t local_obs() const { return plan_.N; }
  const Plan& plan() const { return plan_; }
  long long launches() const { return launches_; }
  const Dev& dev() const { return d_; }

  void activate();
  // points_staged: the points are already in pts_user_ (an upload beside the symbolic phase)
  void set_parameters(const double* poses7, const double* points3, bool points_staged = false);
  void get_parameters(double* poses7, double* points3);
  double evaluate(double* resid2);
  void jacobian(double* jpose, double* jpoint, double* resid2);
  DeviceStructure download_structure();
  // The plan's device arrays for parity tests of the two planners
  // (bae_plan_array); returns the element count, copies when out != null.
  std::int64_t plan_array(int which, void* out, std::int64_t cap, int* elem_bytes);
  void block_diagonals(double* hcc36, double* gc6, double* hpp9, double* gp3);
  void solve_step(double lambda, const bae_lm_config& cfg, double* delta, std::int64_t* iters, double* relres);
  void optimize(const double* poses7, const double* points3, const bae_lm_config& cfg,
                std::vector<bae_iter_record>& traj, bae_lm_report& rep);
  double time_kernel(int kind, int reps);
  // [tile columns, stored tiles, tile updates, ordering groups, positions] of the tile Cholesky (0 before use)
  long long direct_pairs() const { return npairs_; }
  long long direct_blocks() const { return d_.nblk; }
  void direct_stats(long long* out5) const {
    out5[0] = tchol_.nt;
    out5[1] = tchol_.nnz;
    out5[2] = chol_updates_;
    out5[3] = chol_groups_;
    out5[4] = tchol_.n / 6;
  }

 private:
  template <class T>
  T* dalloc(std::size_t n);
  template <class T>
  T* upload(const std::vector<T>& v);
  void sync();
  void ensure_point_staging();
  void linearize_async();
  // linearisation fused with the direct prep for `lambda` (single rank); the
  // next solve_direct then starts at the Schur assembly
  void linearize_prep_async(double lambda, const bae_lm_config& cfg);
  bool fuse_lin_prep(const bae_lm_config& cfg) const;
  bool build_lm_graphs(const bae_lm_config& cfg);
  void reset_lm_status(bool keep_err = false);
  void read_lm();
  void linearize();
  bool solve(double lambda, const bae_lm_config& cfg, SolveInfo& info);
  bool solve_pcg(double lambda, const bae_lm_config& cfg, SolveInfo& info);
  bool solve_direct(double lambda, const bae_lm_config& cfg, SolveInfo& info);
  void build_direct();
  void build_pcg_graph();
  void build_tile_chol(const std::vector<int2>& bcam);
  std::vector<long long> camera_graph_keys(const std::vector<int2>& bcam);
  int chol_help_min() const;
  int chol_tail() const;
  void upload_tile_chol(TileCholHost& h);
  void require_single(const char* what) const;
  const char* cheirality_msg() const;
  void ensure_host_obs_orig();
  void unpermute_slots(const std::vector<double>& src, int comps, double* dst) const;
  void phase_begin(int ph);
  void phase_end();
  void phase_collect();

 public:
  void phase_times(double* out) const {
    for (int i = 0; i < kPhases; ++i) out[i] = phase_ms_[i];
  }
  void phase_reset() {
    for (double& v : phase_ms_) v = 0.0;
  }

 private:
  std::vector<cudaEvent_t> ev_pool_;
  std::vector<std::pair<int, int>> ev_open_;  // (phase, index of start event) pending collection
  int ev_next_ = 0, ph_cur_ = -1;
  double phase_ms_[kPhases] = {0, 0, 0, 0, 0, 0, 0};

  bae_create_options opt_;
  std::unique_ptr<Comm> comm_;       // null on a single rank
  int P_global_ = 0;
  std::int64_t N_global_ = 0;
  std::vector<std::int32_t> rank_of_point_;  // sharded: owner of every global point
  std::vector<std::int32_t> local_pts_;      // sharded: global ids of this rank's points, ascending
  int* src_of_internal_ = nullptr;           // single rank: caller id of each internal point (device)
  double* pts_user_ = nullptr;               // single rank: caller-ordered points (device staging)
  LmDev* lm_reset_host_ = nullptr;           // pinned template of the per-evaluation LM flags
  double* lam_host_ = nullptr;               // pinned: the damping of the next direct solve
  bool capturing_ = false;                   // stream capture in progress: no phase events
  // build_lm_graphs: G_solve (a rejected step's retry), G_acc (after an accepted step)
  cudaGraphExec_t lm_graph_solve_ = nullptr, lm_graph_acc_ = nullptr;
  long long graph_solve_launches_ = 0, graph_acc_launches_ = 0;
  bool prep_fused_ = false;  // the pending solve_direct's prep ran with the linearisation
  double graph_clo_ = 0.0, graph_chi_ = 0.0;
  bool lm_graph_failed_ = false;
  long long npairs_ = 0;
  bool check_launch_ = std::getenv("BAE_CHECK_LAUNCH") != nullptr;  // BAE_LAUNCHED (problem.cu)                     // direct solver: (k, l) pairs of the Schur assembly
  bool defer_factor_check_ = false;          // optimize: the direct factorisation's failure word read later
  Plan plan_;
  Dev d_{};
  SmemSizes sm_;
  cudaStream_t stream_ = nullptr;
  // single-rank direct path: the camera pass of the fused linearise + prep
  // runs on side_ beside the Schur assembly (fork ev_fork_, join ev_join_)
  cudaStream_t side_ = nullptr;
  cudaEvent_t ev_fork_ = nullptr, ev_join_ = nullptr;
  bool join_pending_ = false;
  cudaGraphExec_t pcg_graph_ = nullptr;
  std::vector<void*> allocs_;  // arena chunks
  std::vector<std::size_t> alloc_bytes_;
  char* arena_base_ = nullptr;
  std::size_t arena_size_ = 0, arena_used_ = 0;
  std::vector<double> intr_host_;
  PcgDev* pcg_host_ = nullptr;
  LmDev* lm_host_ = nullptr;
  long long launches_ = 0;
  bool use_graph_pcg_ = true;  // BAE_PCG_MODE=persistent: one cooperative launch per solve
  // direct solver state (built on first use of solver = cholesky)
  bool direct_ready_ = false;
  cusolverDnHandle_t solver_ = nullptr;
  double* potrf_work_ = nullptr;
  int potrf_lwork_ = 0;
  int* dev_info_ = nullptr;
  int* host_info_ = nullptr;
  int pcg_grid_ = 0;
  // tile-sparse Cholesky (default direct solver; BAE_DIRECT=cusolver: dense cuSOLVER)
  bool use_tiles_ = true;
  TileChol tchol_{};
  int chol_grid_ = 0;
  int chol_helpers_ = 0;  // helper tasks of the tile Cholesky (plan_chol_tasks)
  long long chol_updates_ = 0;
  int chol_groups_ = 0;
  long long pcg_chunk_launches_ = 0;  // kernels in one captured PCG chunk
};

}  // namespace bae
