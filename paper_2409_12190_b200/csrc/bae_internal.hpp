// Internal host-side declarations shared by the planner, the device solver
// and the C ABI.
#pragma once

#include <algorithm>
#include <cstdint>
#include <cstdlib>
#include <string>
#include <condition_variable>
#include <deque>
#include <functional>
#include <mutex>
#include <thread>
#include <vector>

#include "bae_b200.h"

namespace bae {

// Error carried to the C ABI: code = BAE_ERR_*, index = offending
// observation / position (IndexError, CheiralityError) or pivot, else -1.
struct Error {
  int code;
  std::string msg;
  std::int64_t index;
  Error(int c, std::string m, std::int64_t i = -1) : code(c), msg(std::move(m)), index(i) {}
};

// Static decomposition of one problem into device work units (setup time,
// the B200 counterpart of transpose_symbolic / spgemm_symbolic /
// build_csr_pattern, bsr.hpp:140-160, spgemm.hpp:33-81, assemble.hpp:135-177).
//
// Points are renumbered ("internal" order) so that points seen by nearby
// cameras are adjacent; a tile is a run of consecutive internal points whose
// observations fit one CTA. Inside a tile, observations are ordered by
// (local camera, internal point, observation id), so every camera's
// observations in the tile form one contiguous "entry" segment and every
// point's observations are listed in `ptobs`.
struct Plan {
  int C = 0, P = 0;
  std::int64_t N = 0;
  int tile_obs_target = 0, tile_cam_cap = 0;

  std::vector<std::int32_t> pt_of_internal;  // internal -> original point
  std::vector<std::int32_t> internal_of_pt;  // original -> internal

  int T = 0;
  std::vector<std::int32_t> tile_obs_begin;  // T+1, global observation slots
  std::vector<std::int32_t> tile_pt_begin;   // T+1, internal point ids
  std::vector<std::int32_t> tile_ent_begin;  // T+1, entry ids
  std::vector<std::int32_t> tile_ws;         // T, big-tile workspace slot or -1

  std::vector<std::uint32_t> obs_lcpt;  // N: local camera | local point << 16
  std::vector<std::int32_t> obs_orig;   // N: original observation id
  std::vector<double> obs_px;           // 2N: pixels in slot order

  int E = 0;
  std::vector<std::int32_t> ent_cam;        // E
  std::vector<std::int32_t> ent_obs_begin;  // E+1
  std::vector<std::int32_t> cam_ent_ptr;    // C+1
  std::vector<std::int32_t> cam_ent;        // E, ascending per camera

  std::vector<std::int32_t> pt_ptr;  // P+1 over internal points, into ptobs
  std::vector<std::uint16_t> ptobs;  // N: tile-local slots, ascending obs id per point

  int max_tile_obs = 0, max_tile_cams = 0, max_tile_pts = 0;
  // tiles whose workspace does not fit shared memory run from global scratch
  int n_big = 0, big_obs = 0, big_cams = 0, big_pts = 0;
  bool has_empty_camera = false, has_empty_point = false;
};

// Tile packing segments of the planners (plan.cpp, plan_device.cu): internal
// points [P s / n, P (s + 1) / n) for s < n, n = max(1, P / kPlanSegPts).
constexpr int kPlanSegPts = 2048;
inline int plan_segments(int P) { return P / kPlanSegPts > 1 ? P / kPlanSegPts : 1; }

// Host worker count for the setup passes: BAE_HOST_THREADS, else the
// hardware concurrency, capped at 16.
inline int host_threads() {
  if (const char* e = std::getenv("BAE_HOST_THREADS")) return std::max(1, std::atoi(e));
  return static_cast<int>(std::clamp(std::thread::hardware_concurrency(), 1u, 16u));
}

// Persistent host worker pool behind parallel_chunks: spawning threads per
// call cost more than the planning passes themselves at BAL sizes. Workers
// are created once (leaked at exit, never joined); any number of caller
// threads may submit concurrently; a call made from inside a worker runs
// serially (no nested waits on the pool).
class HostPool {
 public:
  static HostPool& get() {
    static HostPool* p = new HostPool(15);
    return *p;
  }
  static bool in_worker() { return worker_flag(); }
  void submit(std::function<void()> job) {
    {
      std::lock_guard<std::mutex> l(m_);
      q_.push_back(std::move(job));
    }
    cv_.notify_one();
  }

 private:
  explicit HostPool(int n) {
    for (int i = 0; i < n; ++i)
      std::thread([this] {
        worker_flag() = true;
        for (;;) {
          std::function<void()> job;
          {
            std::unique_lock<std::mutex> l(m_);
            cv_.wait(l, [this] { return !q_.empty(); });
            job = std::move(q_.front());
            q_.pop_front();
          }
          job();
        }
      }).detach();
  }
  static bool& worker_flag() {
    static thread_local bool w = false;
    return w;
  }
  std::mutex m_;
  std::condition_variable cv_;
  std::deque<std::function<void()>> q_;
};

// f(chunk, begin, end) over `chunks` contiguous ranges of [0, n) (chunk 0 on
// the calling thread). Chunk boundaries depend only on n and chunks, so a
// caller that combines per-chunk results in chunk order is deterministic.
template <class F>
void parallel_chunks(std::int64_t n, int chunks, F&& f) {
  if (chunks <= 1 || n < 2 || HostPool::in_worker()) {
    for (int c = 0; c < std::max(chunks, 1); ++c) f(c, n * c / std::max(chunks, 1), n * (c + 1) / std::max(chunks, 1));
    return;
  }
  std::mutex dm;
  std::condition_variable dcv;
  int left = chunks - 1;
  for (int c = 1; c < chunks; ++c)
    HostPool::get().submit([&, c] {
      f(c, n * c / chunks, n * (c + 1) / chunks);
      std::lock_guard<std::mutex> l(dm);  // the waiter cannot return before this unlocks
      if (--left == 0) dcv.notify_all();
    });
  f(0, std::int64_t{0}, n / chunks);
  std::unique_lock<std::mutex> l(dm);
  dcv.wait(l, [&] { return left == 0; });
}

// Validation follows make_ba_problem (problems.hpp:90-110): per observation,
// camera index before point index, IndexError carries the position.
// make_ba_problem's checks (problems.hpp:87-136): observation count, then
// (indices = true) the lowest out-of-range camera / point index as
// IndexError(position) -- the device planner checks the indices itself --
// then empty camera / point groups.
void validate_inputs(int C, int P, const std::int32_t* cam_idx, const std::int32_t* pt_idx, std::int64_t N,
                     bool indices = true);

Plan build_plan(int C, int P, const std::int32_t* cam_idx, const std::int32_t* pt_idx, const double* px2,
                std::int64_t N, int tile_obs_target, int tile_cam_cap, int tile_pts_cap, int smem_tile_obs_cap);

void partition_points(int C, int P, const std::int32_t* cam_idx, const std::int32_t* pt_idx, std::int64_t N,
                      int world, std::int32_t* rank_of_point);

void synth_bal_shaped_device(int C, int P, std::int64_t N, std::uint64_t seed, double pixel_sigma, double pose_sigma,
                             double point_sigma, int device, double* poses7, double* points3, double* intr3,
                             std::int32_t* cam_idx, std::int32_t* pt_idx, double* px2, double* true_poses7,
                             double* true_points3);

void synth_bal_shaped(int C, int P, std::int64_t N, std::uint64_t seed, double pixel_sigma, double pose_sigma,
                      double point_sigma, double* poses7, double* points3, double* intr3, std::int32_t* cam_idx,
                      std::int32_t* pt_idx, double* px2, double* true_poses7, double* true_points3);

}  // namespace bae
