// Device-resident BA problem and the Levenberg-Marquardt driver.
//
// Host orchestration mirrors lm_step / optimize (lm.hpp:115-255) while every
// O(N) operation runs on the GPU: linearisation (K1, fused residual +
// Jacobian + block reductions), damping and Schur preparation, the
// implicit-Schur PCG (one CUDA graph per chunk of iterations, device-side
// convergence state), back-substitution, retraction and trial cost. Per LM
// iteration the host reads back one small status record.
#include <algorithm>
#include <chrono>
#include <mutex>
#include <exception>
#include <thread>
#include <map>
#include <climits>
#include <cstddef>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <limits>

#include "pairs.cuh"
#include "plan_device.cuh"
#include "problem.hpp"

// Launch wrappers return their kernel count; BAE_CHECK_LAUNCH=1 also checks
// the runtime's error state before and after every one (a debugging aid: a
// failed launch or API call is named near its call site instead of
// surfacing at a later, unrelated API call).
#define BAE_LAUNCHED(x)                                                 \
  do {                                                                  \
    if (check_launch_) ck(cudaPeekAtLastError(), "before launch: " #x); \
    launches_ += (x);                                                   \
    if (check_launch_) ck(cudaPeekAtLastError(), "launch: " #x);        \
  } while (0)

namespace bae {

namespace {
void ck(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw Error(BAE_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}
constexpr int kSmemLimit = 200 * 1024;
constexpr int kSliceLimit = 48 * 1024;    // per-warp tile workspace
constexpr int kCtaSmemBudget = 113 * 1024; // two CTAs per SM (2 x (113 + 1 reserved) KB = 228 KB)
constexpr int kPcgChunk = 8;

// BAE_HOST_TIMING=1: host-side phase times on stderr (setup profiling).
struct HostTimer {
  bool on = std::getenv("BAE_HOST_TIMING") != nullptr;
  std::chrono::steady_clock::time_point t = std::chrono::steady_clock::now();
  void mark(const char* what) {
    if (!on) return;
    const auto n = std::chrono::steady_clock::now();
    std::fprintf(stderr, "[bae host] %-22s %8.3f ms\n", what, std::chrono::duration<double, std::milli>(n - t).count());
    t = n;
  }
};
}  // namespace

// Device memory of a problem lives in a few large chunks carved by a bump
// allocator (256-byte aligned, so TMA sources stay 16-byte aligned): one
// cudaMalloc / cudaFree per chunk instead of one per array. Chunks of a
// destroyed problem (and the small pinned host words) go to a process-wide
// cache for the next problem on the same device, so a create -> optimise ->
// destroy loop does not pay cudaMalloc / cudaMallocHost each time (bounded;
// the rest is freed).
constexpr std::size_t kArenaChunk = 32u << 20;
// the cache keeps at most a quarter of the device memory (and 48 GB)
std::size_t chunk_cache_limit(int device) {
  static std::mutex m;
  static std::map<int, std::size_t> lim;
  std::lock_guard<std::mutex> l(m);
  auto it = lim.find(device);
  if (it != lim.end()) return it->second;
  std::size_t total = 32ull << 30;
  cudaDeviceProp prop;
  if (cudaGetDeviceProperties(&prop, device) == cudaSuccess) total = prop.totalGlobalMem;
  return lim[device] = std::min<std::size_t>(total / 4, 48ull << 30);
}
constexpr std::size_t kPinnedWord = 4096;

namespace {
struct MemCache {
  std::mutex m;
  std::map<int, std::multimap<std::size_t, void*>> chunks;  // device -> (bytes, chunk)
  std::size_t cached = 0;
  std::vector<void*> pinned;  // kPinnedWord-byte pinned host blocks
};
MemCache& mem_cache() {
  static MemCache* c = new MemCache;  // leaked: never torn down under a live CUDA context
  return *c;
}
void* chunk_take(int device, std::size_t want, std::size_t& got) {
  MemCache& c = mem_cache();
  std::lock_guard<std::mutex> l(c.m);
  auto& mm = c.chunks[device];
  const auto it = mm.lower_bound(want);
  if (it == mm.end() || it->first > 2 * want) return nullptr;
  got = it->first;
  void* p = it->second;
  c.cached -= got;
  mm.erase(it);
  return p;
}
void chunk_give(int device, void* p, std::size_t bytes) {  // the device is current
  MemCache& c = mem_cache();
  std::lock_guard<std::mutex> l(c.m);
  if (c.cached + bytes > chunk_cache_limit(device)) {
    cudaFree(p);
    return;
  }
  c.chunks[device].emplace(bytes, p);
  c.cached += bytes;
}
void* pinned_take() {
  MemCache& c = mem_cache();
  {
    std::lock_guard<std::mutex> l(c.m);
    if (!c.pinned.empty()) {
      void* p = c.pinned.back();
      c.pinned.pop_back();
      return p;
    }
  }
  void* p = nullptr;
  ck(cudaMallocHost(&p, kPinnedWord), "cudaMallocHost");
  return p;
}
void pinned_give(void* p) {
  if (!p) return;
  MemCache& c = mem_cache();
  std::lock_guard<std::mutex> l(c.m);
  c.pinned.push_back(p);
}

// Large host -> device copies of pageable memory. The driver stages pageable
// copies through its own buffer one at a time (≈ 10 GB/s on the GPU box);
// here two pinned staging buffers per device (process-wide, kept) are filled
// by the host worker pool, chunk by chunk, while the other one is in flight.
constexpr std::size_t kStageBytes = 32u << 20;
constexpr std::size_t kStageMin = 64u << 20;  // below: a plain pageable copy
struct PinnedStage {
  std::mutex m;
  void* buf[2] = {nullptr, nullptr};
  cudaEvent_t ev[2] = {nullptr, nullptr};
};
PinnedStage& pinned_stage(int device) {
  static std::mutex gm;
  static std::map<int, PinnedStage*>* stages = new std::map<int, PinnedStage*>;  // leaked, as mem_cache
  std::lock_guard<std::mutex> l(gm);
  PinnedStage*& p = (*stages)[device];
  if (!p) p = new PinnedStage;
  return *p;
}
// Several pageable host ranges through one staging pipeline (the first
// host copy and the last DMA of a call are not overlapped, so consecutive
// arrays share one pipeline instead of one each).
struct UploadSeg {
  void* dst;
  const void* src;
  std::size_t bytes;
};
void upload_pageable_segs(const UploadSeg* seg, int nseg, cudaStream_t s, int device) {
  std::size_t total = 0;
  for (int k = 0; k < nseg; ++k) total += seg[k].bytes;
  if (total < kStageMin) {
    for (int k = 0; k < nseg; ++k)
      ck(cudaMemcpyAsync(seg[k].dst, seg[k].src, seg[k].bytes, cudaMemcpyHostToDevice, s), "H2D");
    return;
  }
  PinnedStage& st = pinned_stage(device);
  std::lock_guard<std::mutex> l(st.m);
  for (int b = 0; b < 2; ++b) {
    if (!st.buf[b]) ck(cudaMallocHost(&st.buf[b], kStageBytes), "cudaMallocHost staging");
    if (!st.ev[b]) ck(cudaEventCreateWithFlags(&st.ev[b], cudaEventDisableTiming), "event");
  }
  const int nth = host_threads();
  std::size_t i = 0;
  for (int k = 0; k < nseg; ++k) {
    for (std::size_t off = 0; off < seg[k].bytes; off += kStageBytes, ++i) {
      const int b = static_cast<int>(i & 1);
      const std::size_t n = std::min(kStageBytes, seg[k].bytes - off);
      if (i >= 2) ck(cudaEventSynchronize(st.ev[b]), "staging reuse");
      char* to = static_cast<char*>(st.buf[b]);
      const char* from = static_cast<const char*>(seg[k].src) + off;
      parallel_chunks(static_cast<std::int64_t>(n), nth, [&](int, std::int64_t a, std::int64_t e) {
        std::memcpy(to + a, from + a, static_cast<std::size_t>(e - a));
      });
      ck(cudaMemcpyAsync(static_cast<char*>(seg[k].dst) + off, to, n, cudaMemcpyHostToDevice, s), "H2D staged");
      ck(cudaEventRecord(st.ev[b], s), "event record");
    }
  }
  for (int b = 0; b < 2; ++b) ck(cudaEventSynchronize(st.ev[b]), "staging");  // buffers free for the next caller
}
void upload_pageable(void* dst, const void* src, std::size_t bytes, cudaStream_t s, int device) {
  const UploadSeg seg{dst, src, bytes};
  upload_pageable_segs(&seg, 1, s, device);
}
// The reverse: DMA into the staging buffers, the host pool copies out
// (synchronises s).
void download_pageable(void* dst, const void* src, std::size_t bytes, cudaStream_t s, int device) {
  if (bytes < kStageMin) {
    ck(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, s), "D2H");
    ck(cudaStreamSynchronize(s), "D2H");
    return;
  }
  PinnedStage& st = pinned_stage(device);
  std::lock_guard<std::mutex> l(st.m);
  for (int b = 0; b < 2; ++b) {
    if (!st.buf[b]) ck(cudaMallocHost(&st.buf[b], kStageBytes), "cudaMallocHost staging");
    if (!st.ev[b]) ck(cudaEventCreateWithFlags(&st.ev[b], cudaEventDisableTiming), "event");
  }
  const int nth = host_threads();
  const std::size_t nchunk = (bytes + kStageBytes - 1) / kStageBytes;
  auto issue = [&](std::size_t i) {
    const int b = static_cast<int>(i & 1);
    const std::size_t off = i * kStageBytes, n = std::min(kStageBytes, bytes - off);
    ck(cudaMemcpyAsync(st.buf[b], static_cast<const char*>(src) + off, n, cudaMemcpyDeviceToHost, s), "D2H staged");
    ck(cudaEventRecord(st.ev[b], s), "event record");
  };
  issue(0);
  for (std::size_t i = 0; i < nchunk; ++i) {
    const int b = static_cast<int>(i & 1);
    ck(cudaEventSynchronize(st.ev[b]), "staging");
    if (i + 1 < nchunk) issue(i + 1);  // the other buffer: its copy-out finished last round
    const std::size_t off = i * kStageBytes, n = std::min(kStageBytes, bytes - off);
    const char* from = static_cast<const char*>(st.buf[b]);
    char* to = static_cast<char*>(dst) + off;
    parallel_chunks(static_cast<std::int64_t>(n), nth, [&](int, std::int64_t a, std::int64_t e) {
      std::memcpy(to + a, from + a, static_cast<std::size_t>(e - a));
    });
  }
}
// A large pageable upload on a helper thread and its own stream, so that it
// overlaps host / device work of the caller (the device planner); wait_on()
// joins and orders a consumer stream after the copy. The destructor joins on
// every path (exceptions included).
struct AsyncUpload {
  std::thread th;
  cudaStream_t s = nullptr;
  cudaEvent_t ev = nullptr;
  std::exception_ptr err;
  void* dst = nullptr;       // owned until wait_on() hands it over
  void* borrowed = nullptr;  // start(..., into): the caller's buffer
  void start(const void* src, std::size_t bytes, int device, void* into = nullptr) {
    ck(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking), "stream");
    ck(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming), "event");
    if (into)
      borrowed = into;  // a caller's buffer (not freed here)
    else
      ck(cudaMallocAsync(&dst, bytes, s), "cudaMallocAsync upload");
    void* to = into ? into : dst;
    th = std::thread([this, src, bytes, device, to] {
      try {
        ck(cudaSetDevice(device), "cudaSetDevice");
        upload_pageable(to, src, bytes, s, device);
        ck(cudaEventRecord(ev, s), "event record");
      } catch (...) {
        err = std::current_exception();
      }
    });
  }
  // the buffer passes to the caller (who frees it, stream-ordered, on `consumer`)
  void* wait_on(cudaStream_t consumer) {
    th.join();
    if (err) std::rethrow_exception(err);
    ck(cudaStreamWaitEvent(consumer, ev, 0), "stream wait");
    void* p = borrowed ? borrowed : dst;
    dst = nullptr;
    return p;
  }
  ~AsyncUpload() {
    if (th.joinable()) th.join();
    if (s) {
      if (dst) cudaFreeAsync(dst, s);
      cudaStreamSynchronize(s);
      cudaStreamDestroy(s);
    }
    if (ev) cudaEventDestroy(ev);
  }
};
}  // namespace

template <class T>
T* Problem::dalloc(std::size_t n) {
  const std::size_t bytes = (std::max<std::size_t>(n, 1) * sizeof(T) + 255) & ~std::size_t{255};
  if (arena_used_ + bytes > arena_size_) {
    const std::size_t sz = std::max(bytes, kArenaChunk);
    std::size_t got = sz;
    void* p = chunk_take(opt_.device, sz, got);
    if (!p) ck(cudaMalloc(&p, sz), "cudaMalloc");
    allocs_.push_back(p);
    alloc_bytes_.push_back(got);
    arena_base_ = static_cast<char*>(p);
    arena_size_ = got;
    arena_used_ = 0;
  }
  T* r = reinterpret_cast<T*>(arena_base_ + arena_used_);
  arena_used_ += bytes;
  return r;
}

template <class T>
T* Problem::upload(const std::vector<T>& v) {
  T* p = dalloc<T>(v.size());
  if (!v.empty())
    ck(cudaMemcpyAsync(p, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice, stream_), "upload");
  return p;
}

Problem::Problem(const double* poses7, int C, const double* points3, int P, const double* intr3,
                 const std::int32_t* cam_idx, const std::int32_t* pt_idx, const double* px2, std::int64_t N,
                 const bae_create_options& opt)
    : opt_(opt) {
  HostTimer ht;
  // The plan: on the device for a single-rank problem large enough to gain
  // (plan_device.cu, which also checks the indices; BAE_PLAN=host / device
  // forces one), else on the host (plan.cpp; sharded ranks plan their own
  // partition there). Both give the same plan element for element.
  const bool sharded = opt.world > 1 || opt.nccl_id != nullptr || opt.group != nullptr;
  bool dev_plan = !sharded && N >= (1 << 17);
  if (const char* e = std::getenv("BAE_PLAN")) dev_plan = !sharded && std::string(e) == "device";
  validate_inputs(C, P, cam_idx, pt_idx, N, !dev_plan);
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
    throw Error(BAE_ERR_CUDA, "no CUDA device available (the B200 path has no CPU fallback)");
  if (opt.device < 0 || opt.device >= ndev) throw Error(BAE_ERR_INVALID_ARGUMENT, "bad device ordinal");
  ck(cudaSetDevice(opt.device), "cudaSetDevice");
  P_global_ = P;
  N_global_ = N;

  // Sharded run: every rank receives the whole problem, as the
  // reference's make_ba_problem does, and keeps the points of its partition
  // (bae_partition_points: contiguous ranges of the camera-sorted point order,
  // balanced by observation count) with all their observations, in ascending
  // observation order. Cameras are replicated.
  const bool dist = opt.world > 1 || opt.nccl_id != nullptr || opt.group != nullptr;
  std::vector<std::int32_t> lcam, lpt, gobs;
  std::vector<double> lpx;
  const std::int32_t* use_cam = cam_idx;
  const std::int32_t* use_pt = pt_idx;
  const double* use_px = px2;
  int use_P = P;
  std::int64_t use_N = N;
  if (dist) {
    if (opt.world < 1 || opt.rank < 0 || opt.rank >= opt.world)
      throw Error(BAE_ERR_INVALID_ARGUMENT, "sharded problem: rank must be in [0, world)");
    if (!opt.group && !opt.nccl_id)
      throw Error(BAE_ERR_INVALID_ARGUMENT, "sharded problem: needs an NCCL unique id or a rank group");
    rank_of_point_.resize(static_cast<std::size_t>(P));
    partition_points(C, P, cam_idx, pt_idx, N, opt.world, rank_of_point_.data());
    std::vector<std::int32_t> owned(static_cast<std::size_t>(opt.world), 0);
    for (int p = 0; p < P; ++p) ++owned[rank_of_point_[p]];
    for (int r = 0; r < opt.world; ++r)
      if (owned[r] == 0) throw Error(BAE_ERR_UNSUPPORTED, "sharded problem: more ranks than point partitions");
    std::vector<std::int32_t> lp_of(static_cast<std::size_t>(P), -1);
    for (int p = 0; p < P; ++p)
      if (rank_of_point_[p] == opt.rank) {
        lp_of[p] = static_cast<std::int32_t>(local_pts_.size());
        local_pts_.push_back(p);
      }
    for (std::int64_t k = 0; k < N; ++k) {
      const int lp = lp_of[pt_idx[k]];
      if (lp < 0) continue;
      lcam.push_back(cam_idx[k]);
      lpt.push_back(lp);
      lpx.push_back(px2[2 * k]);
      lpx.push_back(px2[2 * k + 1]);
      gobs.push_back(static_cast<std::int32_t>(k));
    }
    use_cam = lcam.data();
    use_pt = lpt.data();
    use_px = lpx.data();
    use_P = static_cast<int>(local_pts_.size());
    use_N = static_cast<std::int64_t>(gobs.size());
    comm_ = opt.group ? make_group_comm(opt.group, opt.rank, opt.device)
                      : make_nccl_comm(opt.nccl_id, opt.rank, opt.world, opt.device);
  }
  ck(cudaSetDevice(opt.device), "cudaSetDevice");
  ck(cudaStreamCreateWithFlags(&stream_, cudaStreamNonBlocking), "stream");
  ht.mark("validate+partition");
  int tile_obs = opt.tile_obs > 0 ? opt.tile_obs : kPipeObs;
  if (const char* t = std::getenv("BAE_TILE_OBS")) tile_obs = std::max(8, std::atoi(t));
  int tile_cams = 32;
  if (const char* t = std::getenv("BAE_TILE_CAMS")) tile_cams = std::max(1, std::atoi(t));
  if (const char* m = std::getenv("BAE_PCG_MODE")) use_graph_pcg_ = std::string(m) != "persistent";
  if (comm_) use_graph_pcg_ = true;  // the persistent kernel has no place for the cross-rank sum
  Plan& pl = plan_;
  long long big_stride = 0;
  int nbig = 0;
  TileLaunch* kinds[kWsKinds] = {&sm_.lin, &sm_.cost, &sm_.prep, &sm_.schur, &sm_.trial, &sm_.prepd, &sm_.linprep};
  std::vector<int4> desc;
  std::vector<char> blob;
  std::vector<int> small_tiles, big_tiles;
  DevicePlan dp;
  int* dcam = nullptr;  // raw observation indices on the device (device plan)
  AsyncUpload px_up;    // device plan: the pixels, uploaded beside the planner
  AsyncUpload pts_up;   // and the initial points after them
  if (dev_plan) {
    ck(cudaMallocAsync(reinterpret_cast<void**>(&dcam), 2 * sizeof(int) * static_cast<std::size_t>(use_N), stream_),
       "cudaMallocAsync observation indices");
    const UploadSeg idx[2] = {{dcam, use_cam, sizeof(int) * static_cast<std::size_t>(use_N)},
                              {dcam + use_N, use_pt, sizeof(int) * static_cast<std::size_t>(use_N)}};
    upload_pageable_segs(idx, 2, stream_, opt.device);
    ht.mark("index upload");
    // the pixels travel while the planner runs (its kernels and host steps
    // leave the copy engine idle); gathered into slot order below
    px_up.start(px2, 2 * sizeof(double) * static_cast<std::size_t>(use_N), opt.device);
    // the initial points follow on their own helper (the staging lock puts
    // them after the pixels), into the caller-order buffer set_parameters
    // permutes from
    if (points3 && 3 * sizeof(double) * static_cast<std::size_t>(use_P) >= (64u << 20)) {
      pts_user_ = dalloc<double>(3 * static_cast<std::size_t>(use_P));
      pts_up.start(points3, 3 * sizeof(double) * static_cast<std::size_t>(use_P), opt.device, pts_user_);
    }
    try {
      build_plan_device(C, use_P, dcam, dcam + use_N, use_N, std::min(tile_obs, kPipeObs), std::min(tile_cams, kPipeCams),
                        kPipePts, kSliceLimit, [this](std::size_t n) { return static_cast<void*>(dalloc<char>(n)); },
                        stream_, dp);
    } catch (...) {
      cudaFreeAsync(dcam, stream_);
      throw;
    }
    ck(cudaFreeAsync(dcam, stream_), "cudaFreeAsync");
    if (use_P < 1) throw Error(BAE_ERR_INVALID_ARGUMENT, "track_points: empty group");
    pl.C = C;
    pl.P = use_P;
    pl.N = use_N;
    pl.tile_obs_target = std::min(tile_obs, kPipeObs);
    pl.tile_cam_cap = std::min(tile_cams, kPipeCams);
    pl.T = dp.T;
    pl.E = dp.E;
    pl.max_tile_obs = dp.max_tile_obs;
    pl.max_tile_cams = dp.max_tile_cams;
    pl.max_tile_pts = dp.max_tile_pts;
    pl.n_big = dp.n_big;
    pl.has_empty_camera = dp.has_empty_camera;
    pl.has_empty_point = dp.has_empty_point;
    // the point order for the host-side permutations (obs_orig stays on the
    // device until an export asks for it: host_obs_orig)
    pl.pt_of_internal.resize(static_cast<std::size_t>(use_P));
    ck(cudaMemcpyAsync(pl.pt_of_internal.data(), dp.pt_of_internal, sizeof(int) * use_P, cudaMemcpyDeviceToHost,
                       stream_),
       "D2H point order");
    sync();
    src_of_internal_ = dp.pt_of_internal;
    for (int k = 0; k < kWsKinds; ++k) kinds[k]->slice = dp.kind_slice[k];
    nbig = dp.n_big;
    big_stride = dp.big_need;
    ht.mark("device plan");
  } else {
    // single rank: the pixels go up in the caller's order and are gathered into
    // slot order on the device (a random gather over N on the host otherwise)
    plan_ = build_plan(C, use_P, use_cam, use_pt, dist ? use_px : nullptr, use_N, std::min(tile_obs, kPipeObs),
                       std::min(tile_cams, kPipeCams), kPipePts, 1 << 30);
    ht.mark("build_plan");
    if (dist) {
      // observation ids and the missing-diagonal checks refer to the whole problem
      for (auto& k : plan_.obs_orig) k = gobs[k];
      std::vector<char> cam_seen(static_cast<std::size_t>(C), 0), pt_seen(static_cast<std::size_t>(P), 0);
      for (std::int64_t k = 0; k < N; ++k) {
        cam_seen[cam_idx[k]] = 1;
        pt_seen[pt_idx[k]] = 1;
      }
      plan_.has_empty_camera = std::find(cam_seen.begin(), cam_seen.end(), 0) != cam_seen.end();
      plan_.has_empty_point = std::find(pt_seen.begin(), pt_seen.end(), 0) != pt_seen.end();
    }
    // Tile classes. "Small" tiles (within the kPipe* caps) take the pipelined
    // TMA path of the Schur product and a per-warp shared-memory slice in the
    // other tile kernels; any other tile (one very long track) runs every kind
    // from a global workspace slot.
    desc.assign(static_cast<std::size_t>(pl.T), int4{0, 0, 0, 0});
    // sizes and offsets first (serial, per-tile arithmetic), then the index
    // blobs filled in parallel chunks of tiles
    std::size_t blob_bytes = 0;
    for (int t = 0; t < pl.T; ++t) {
      const int ob = pl.tile_obs_begin[t], pb = pl.tile_pt_begin[t], eb = pl.tile_ent_begin[t];
      const int nobs = pl.tile_obs_begin[t + 1] - ob;
      const int npts = pl.tile_pt_begin[t + 1] - pb;
      const int ncam = pl.tile_ent_begin[t + 1] - eb;
      long long need = 0;
      for (int k = 0; k < kWsKinds; ++k) need = std::max(need, tile_ws_bytes(k, ncam, npts, nobs));
      const bool small = nobs > 0 && nobs <= kPipeObs && ncam <= kPipeCams && npts <= kPipePts && need <= kSliceLimit;
      if (!small) {
        pl.tile_ws[t] = nbig++;
        big_stride = std::max(big_stride, need);
        big_tiles.push_back(t);
        continue;
      }
      pl.tile_ws[t] = -1;
      for (int k = 0; k < kWsKinds; ++k)
        kinds[k]->slice = std::max<int>(kinds[k]->slice, static_cast<int>(tile_ws_bytes(k, ncam, npts, nobs)));
      // index blob: hdr | camid | ent | pptr | lcpt | ptl, padded to 16 bytes
      const int bytes = (32 + 4 * ncam + 4 * (ncam + 1) + 4 * (npts + 1) + 6 * nobs + 15) / 16 * 16;
      desc[t] = int4{static_cast<int>(blob_bytes / 16), bytes, pb, npts};
      blob_bytes += static_cast<std::size_t>(bytes);
      small_tiles.push_back(t);
    }
    blob.assign(blob_bytes, 0);
    parallel_chunks(static_cast<std::int64_t>(small_tiles.size()), small_tiles.size() >= 1024 ? host_threads() : 1,
                    [&](int, std::int64_t i0, std::int64_t i1) {
      for (std::int64_t ii = i0; ii < i1; ++ii) {
        const int t = small_tiles[ii];
        const int ob = pl.tile_obs_begin[t], pb = pl.tile_pt_begin[t], eb = pl.tile_ent_begin[t];
        const int nobs = pl.tile_obs_begin[t + 1] - ob;
        const int npts = pl.tile_pt_begin[t + 1] - pb;
        const int ncam = pl.tile_ent_begin[t + 1] - eb;
        int* w = reinterpret_cast<int*>(blob.data() + 16 * static_cast<std::size_t>(desc[t].x));
        w[0] = ob;
        w[1] = nobs;
        w[2] = pb;
        w[3] = npts;
        w[4] = eb;
        w[5] = ncam;
        int* q = w + 8;
        for (int l = 0; l < ncam; ++l) *q++ = pl.ent_cam[eb + l];
        for (int l = 0; l <= ncam; ++l) *q++ = pl.ent_obs_begin[eb + l] - ob;
        for (int i = 0; i <= npts; ++i) *q++ = pl.pt_ptr[pb + i] - ob;
        std::uint32_t* lc = reinterpret_cast<std::uint32_t*>(q);
        for (int i = 0; i < nobs; ++i) lc[i] = pl.obs_lcpt[ob + i];
        std::uint16_t* ptl = reinterpret_cast<std::uint16_t*>(lc + nobs);
        for (int i = 0; i < nobs; ++i) ptl[i] = pl.ptobs[ob + i];
      }
    });
  }
  // intrinsics as 4 doubles per camera: BAL [f k1 k2 0], pinhole [fx fy cx cy]
  const bool pinhole = opt.camera_model == BAE_CAMERA_PINHOLE;
  if (opt.camera_model != BAE_CAMERA_BAL && !pinhole) throw Error(BAE_ERR_INVALID_ARGUMENT, "unknown camera model");
  const int kw = pinhole ? 4 : 3;
  intr_host_.assign(4 * static_cast<std::size_t>(C), 0.0);
  for (int c = 0; c < C; ++c)
    for (int j = 0; j < kw; ++j) intr_host_[4 * static_cast<std::size_t>(c) + j] = intr3[kw * static_cast<std::size_t>(c) + j];

  int cta_budget = kCtaSmemBudget;
  if (const char* e = std::getenv("BAE_CTA_SMEM_KB")) cta_budget = std::clamp(std::atoi(e), 16, 200) * 1024;
  for (int k = 0; k < kWsKinds; ++k) {
    TileLaunch& tl = *kinds[k];
    tl.slice = std::max(16, (tl.slice + 15) / 16 * 16);
    // up to 8 warp-tiles per CTA, two CTAs per SM within the shared-memory budget
    tl.wpb = std::max(1, std::min(8, cta_budget / tl.slice));
  }
  ht.mark("tile blobs");
  sm_.schur.slice = kPipeWarpBytes;  // pipelined double buffer per warp
  sm_.schur.wpb = kSchurWarps;
  big_stride = (big_stride + 255) / 256 * 256;
  set_smem_limits(kSmemLimit);

  Dev& d = d_;
  d.C = C;
  d.pinhole = pinhole ? 1 : 0;
  d.P = use_P;
  d.T = pl.T;
  d.E = pl.E;
  d.N = static_cast<int>(use_N);
  d.nbig = nbig;
  d.big_stride = big_stride;
  if (dev_plan) {
    d.tile_obs_begin = dp.tile_obs_begin;
    d.tile_pt_begin = dp.tile_pt_begin;
    d.tile_ent_begin = dp.tile_ent_begin;
    d.tile_ws = dp.tile_ws;
    d.obs_lcpt = dp.obs_lcpt;
    d.obs_orig = dp.obs_orig;
    d.ent_cam = dp.ent_cam;
    d.ent_obs_begin = dp.ent_obs_begin;
    d.cam_ent_ptr = dp.cam_ent_ptr;
    d.cam_ent = dp.cam_ent;
    d.pt_ptr = dp.pt_ptr;
    d.ptobs = dp.ptobs;
    d.tile_desc = dp.tile_desc;
    d.tile_blob = dp.tile_blob;
    d.small_tiles = dp.small_tiles;
    d.big_tiles = dp.big_tiles;
    double* px = dalloc<double>(2 * static_cast<std::size_t>(use_N));
    double* raw = static_cast<double*>(px_up.wait_on(stream_));
    BAE_LAUNCHED(launch_gather_pixels(raw, d.obs_orig, px, use_N, stream_));
    ck(cudaFreeAsync(raw, stream_), "cudaFreeAsync");
    d.obs_px = px;
    small_tiles.resize(static_cast<std::size_t>(dp.n_small));  // counts only below
    big_tiles.resize(static_cast<std::size_t>(dp.n_big));
  } else {
    d.tile_obs_begin = upload(pl.tile_obs_begin);
    ht.mark("first chunk + upload");
    d.tile_pt_begin = upload(pl.tile_pt_begin);
    d.tile_ent_begin = upload(pl.tile_ent_begin);
    d.tile_ws = upload(pl.tile_ws);
    d.obs_lcpt = upload(pl.obs_lcpt);
    d.obs_orig = upload(pl.obs_orig);
    if (dist) {
      d.obs_px = upload(pl.obs_px);
    } else {
      double* px = dalloc<double>(2 * static_cast<std::size_t>(use_N));
      double* raw = nullptr;
      ck(cudaMallocAsync(reinterpret_cast<void**>(&raw), 2 * sizeof(double) * use_N, stream_), "cudaMallocAsync");
      ck(cudaMemcpyAsync(raw, px2, 2 * sizeof(double) * use_N, cudaMemcpyHostToDevice, stream_), "H2D pixels");
      BAE_LAUNCHED(launch_gather_pixels(raw, d.obs_orig, px, use_N, stream_));
      ck(cudaFreeAsync(raw, stream_), "cudaFreeAsync");
      d.obs_px = px;
    }
    d.ent_cam = upload(pl.ent_cam);
    d.ent_obs_begin = upload(pl.ent_obs_begin);
    d.cam_ent_ptr = upload(pl.cam_ent_ptr);
    d.cam_ent = upload(pl.cam_ent);
    d.pt_ptr = upload(pl.pt_ptr);
    d.ptobs = upload(pl.ptobs);
    if (blob.empty()) blob.resize(16);
    d.tile_desc = upload(desc);
    d.tile_blob = upload(blob);
    d.small_tiles = upload(small_tiles);
    d.big_tiles = upload(big_tiles);
  }
  ht.mark("uploads");
  d.n_small = static_cast<int>(small_tiles.size());
  d.n_big_tiles = static_cast<int>(big_tiles.size());
  d.bigws = nbig ? dalloc<char>(static_cast<std::size_t>(nbig) * big_stride) : nullptr;
  d.pose = dalloc<double>(7 * static_cast<std::size_t>(C));
  d.intr = upload(intr_host_);
  d.camrec = dalloc<double>(kCamRec * static_cast<std::size_t>(C));
  d.pts = dalloc<double>(3 * static_cast<std::size_t>(use_P) + 2);  // +16 B: TMA point windows
  d.pose_t = dalloc<double>(7 * static_cast<std::size_t>(C));
  d.camrec_t = dalloc<double>(kCamRec * static_cast<std::size_t>(C));
  d.pts_t = dalloc<double>(3 * static_cast<std::size_t>(use_P));
  d.hpp = dalloc<double>(6 * static_cast<std::size_t>(use_P));
  d.gp = dalloc<double>(3 * static_cast<std::size_t>(use_P));
  d.hinv = dalloc<double>(6 * static_cast<std::size_t>(use_P));
  d.dp = dalloc<double>(3 * static_cast<std::size_t>(use_P));
  d.hcc = dalloc<double>(21 * static_cast<std::size_t>(C));
  d.gc = dalloc<double>(6 * static_cast<std::size_t>(C));
  d.hccd = dalloc<double>(21 * static_cast<std::size_t>(C));
  d.minv = dalloc<double>(36 * static_cast<std::size_t>(C));
  d.rhs = dalloc<double>(6 * static_cast<std::size_t>(C));
  d.x = dalloc<double>(6 * static_cast<std::size_t>(C));
  d.r = dalloc<double>(6 * static_cast<std::size_t>(C));
  d.z = dalloc<double>(6 * static_cast<std::size_t>(C));
  d.p = dalloc<double>(6 * static_cast<std::size_t>(C));
  d.y = dalloc<double>(6 * static_cast<std::size_t>(C));
  d.partial = dalloc<double>(27 * static_cast<std::size_t>(std::max(pl.E, 1)));
  d.partial6 = dalloc<double>(6 * static_cast<std::size_t>(std::max(pl.E, 1)));
  d.tile_red = dalloc<double>(2 * static_cast<std::size_t>(pl.T));
  d.cred = dist ? dalloc<double>(27 * static_cast<std::size_t>(C) + 8) : nullptr;
  d.cam_dot = dalloc<double>(2 * static_cast<std::size_t>(C));
  const int max_blocks = std::max((C + kWarpsPerCamBlock - 1) / kWarpsPerCamBlock, (C + 127) / 128) + 1;
  d.block_red = dalloc<double>(4 * static_cast<std::size_t>(std::max(max_blocks, 4096)));
  d.tickets = dalloc<unsigned>(16);
  ck(cudaMemset(d.tickets, 0, 16 * sizeof(unsigned)), "memset");
  d.pcg = dalloc<PcgDev>(1);
  d.lm = dalloc<LmDev>(1);
  d.jstore = nullptr;
  d.resid = nullptr;
  d.trace = nullptr;
  d.wstore = nullptr;
  d.lam = nullptr;
  d.pairs = nullptr;
  d.blk_ptr = nullptr;
  d.blk_cam = nullptr;
  d.blk_ord = nullptr;
  d.chunks = nullptr;
  d.nchunk = 0;
  d.blk_nchunk = nullptr;
  d.blk_ticket = nullptr;
  d.schur_part = nullptr;
  d.nblk = 0;
  d.defer_hccd = 0;
  d.schur = nullptr;
  ht.mark("allocs");
  static_assert(sizeof(PcgDev) <= kPinnedWord && sizeof(LmDev) <= kPinnedWord, "pinned word");
  pcg_host_ = static_cast<PcgDev*>(pinned_take());
  lm_host_ = static_cast<LmDev*>(pinned_take());
  ck(cudaMemset(d.pcg, 0, sizeof(PcgDev)), "memset");

  ht.mark("device alloc+upload");
  if (pts_up.s) {
    pts_up.wait_on(stream_);
    if (!src_of_internal_) {  // (the device plan leaves its own copy)
      std::vector<int> src(plan_.pt_of_internal.begin(), plan_.pt_of_internal.end());
      src_of_internal_ = upload(src);
    }
    set_parameters(poses7, nullptr, /*points_staged=*/true);
  } else {
    set_parameters(poses7, points3);
  }
  ht.mark("set_parameters");
  // Eager forward at construction, as make_ba_problem's graph does
  // (trace.hpp:152,385): cheirality surfaces here with the observation id.
  evaluate(nullptr);
  ht.mark("initial evaluate");
}

Problem::~Problem() {
  cudaSetDevice(opt_.device);
  for (auto& e : ev_pool_) cudaEventDestroy(e);
  if (solver_) cusolverDnDestroy(solver_);
  if (side_) cudaStreamSynchronize(side_);
  if (stream_) cudaStreamSynchronize(stream_);  // the chunks are reused by the next problem
  pinned_give(host_info_);
  if (pcg_graph_) cudaGraphExecDestroy(pcg_graph_);
  if (lm_graph_solve_) cudaGraphExecDestroy(lm_graph_solve_);
  if (lm_graph_acc_) cudaGraphExecDestroy(lm_graph_acc_);
  for (std::size_t i = 0; i < allocs_.size(); ++i) chunk_give(opt_.device, allocs_[i], alloc_bytes_[i]);
  pinned_give(pcg_host_);
  pinned_give(lm_host_);
  pinned_give(lm_reset_host_);
  pinned_give(lam_host_);
  if (side_) cudaStreamDestroy(side_);
  if (ev_fork_) cudaEventDestroy(ev_fork_);
  if (ev_join_) cudaEventDestroy(ev_join_);
  if (stream_) cudaStreamDestroy(stream_);
  comm_.reset();
}

// CheiralityError messages of the two camera models (camera.hpp:36, 52).
const char* Problem::cheirality_msg() const {
  return d_.pinhole ? "pinhole projection: point behind camera" : "bal projection: point on camera plane";
}

int DeviceStructure::slot_cam(int t, int s) const {
  // the entry of slot s: entries of tile t are ordered by local camera and
  // each covers a contiguous slot range
  int lo = tile_ent_begin[t], hi = tile_ent_begin[t + 1] - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) / 2;
    if (ent_obs_begin[mid] <= s) lo = mid; else hi = mid - 1;
  }
  return ent_cam[lo];
}

std::int64_t Problem::plan_array(int which, void* out, std::int64_t cap, int* elem_bytes) {
  require_single("the plan export");
  activate();
  ensure_point_staging();
  sync();
  const std::int64_t T = d_.T, E = d_.E, N = d_.N, C = d_.C, P = d_.P;
  const void* src = nullptr;
  std::int64_t n = 0;
  int eb = 4;
  std::vector<int> meta;
  switch (which) {
    case 0: src = d_.tile_obs_begin; n = T + 1; break;
    case 1: src = d_.tile_pt_begin; n = T + 1; break;
    case 2: src = d_.tile_ent_begin; n = T + 1; break;
    case 3: src = d_.tile_ws; n = T; break;
    case 4: src = d_.obs_lcpt; n = N; break;
    case 5: src = d_.obs_orig; n = N; break;
    case 6: src = d_.ent_cam; n = E; break;
    case 7: src = d_.ent_obs_begin; n = E + 1; break;
    case 8: src = d_.cam_ent_ptr; n = C + 1; break;
    case 9: src = d_.cam_ent; n = E; break;
    case 10: src = d_.pt_ptr; n = P + 1; break;
    case 11: src = d_.ptobs; n = N; eb = 2; break;
    case 12: src = src_of_internal_; n = P; break;
    case 13: src = d_.tile_desc; n = 4 * T; break;
    case 14: src = d_.small_tiles; n = d_.n_small; break;
    case 15: src = d_.big_tiles; n = d_.n_big_tiles; break;
    case 16: src = d_.obs_px; n = 2 * N; eb = 8; break;
    case 17: {  // launch shapes: per kind slice and warps per CTA, big tiles, big stride
      const TileLaunch* k[kWsKinds] = {&sm_.lin, &sm_.cost, &sm_.prep, &sm_.schur, &sm_.trial, &sm_.prepd, &sm_.linprep};
      for (int i = 0; i < kWsKinds; ++i) {
        meta.push_back(k[i]->slice);
        meta.push_back(k[i]->wpb);
      }
      meta.push_back(d_.nbig);
      meta.push_back(static_cast<int>(d_.big_stride));
      meta.push_back(plan_.has_empty_camera ? 1 : 0);
      meta.push_back(plan_.has_empty_point ? 1 : 0);
      meta.push_back(plan_.max_tile_obs);
      n = static_cast<std::int64_t>(meta.size());
      break;
    }
    case 18: {  // the small tiles' index blobs (bytes)
      std::vector<int4> desc(static_cast<std::size_t>(T));
      if (T) ck(cudaMemcpy(desc.data(), d_.tile_desc, T * sizeof(int4), cudaMemcpyDeviceToHost), "D2H");
      for (const int4& q : desc) n = std::max<std::int64_t>(n, 16LL * q.x + q.y);
      src = d_.tile_blob;
      eb = 1;
      break;
    }
    default:
      throw Error(BAE_ERR_INVALID_ARGUMENT, "plan export: unknown array");
  }
  if (elem_bytes) *elem_bytes = eb;
  if (out && n > 0) {
    if (cap < n) throw Error(BAE_ERR_INVALID_ARGUMENT, "plan export: capacity too small");
    if (!meta.empty()) std::memcpy(out, meta.data(), meta.size() * sizeof(int));
    else ck(cudaMemcpy(out, src, static_cast<std::size_t>(n) * eb, cudaMemcpyDeviceToHost), "D2H plan");
  }
  return n;
}

DeviceStructure Problem::download_structure() {
  require_single("the structure export");
  activate();
  ensure_point_staging();
  sync();
  DeviceStructure s;
  s.C = d_.C;
  s.P = d_.P;
  s.T = d_.T;
  s.E = d_.E;
  s.N = d_.N;
  auto get = [&](auto& v, const auto* src, std::size_t n) {
    v.resize(n);
    if (n) ck(cudaMemcpy(v.data(), src, n * sizeof(v[0]), cudaMemcpyDeviceToHost), "D2H structure");
  };
  const std::size_t T = s.T, E = s.E, N = static_cast<std::size_t>(s.N), C = s.C, P = s.P;
  get(s.tile_obs_begin, d_.tile_obs_begin, T + 1);
  get(s.tile_pt_begin, d_.tile_pt_begin, T + 1);
  get(s.tile_ent_begin, d_.tile_ent_begin, T + 1);
  get(s.obs_lcpt, d_.obs_lcpt, N);
  get(s.obs_orig, d_.obs_orig, N);
  get(s.ent_cam, d_.ent_cam, E);
  get(s.ent_obs_begin, d_.ent_obs_begin, E + 1);
  get(s.cam_ent_ptr, d_.cam_ent_ptr, C + 1);
  get(s.cam_ent, d_.cam_ent, E);
  get(s.pt_ptr, d_.pt_ptr, P + 1);
  get(s.ptobs, d_.ptobs, N);
  get(s.pt_of_internal, src_of_internal_, P);
  return s;
}

void Problem::require_single(const char* what) const {
  if (comm_) throw Error(BAE_ERR_UNSUPPORTED, std::string(what) + " is not available on a sharded problem");
}

void Problem::activate() { ck(cudaSetDevice(opt_.device), "cudaSetDevice"); }

void Problem::phase_begin(int ph) {
  if (capturing_) return;  // a captured graph has no host-visible events
  if (ev_pool_.empty()) {
    ev_pool_.resize(512);
    for (auto& e : ev_pool_) ck(cudaEventCreate(&e), "event");
  }
  if (ev_next_ + 2 > static_cast<int>(ev_pool_.size())) phase_collect();
  ph_cur_ = ph;
  ck(cudaEventRecord(ev_pool_[ev_next_], stream_), "event record");
  ev_open_.push_back({ph, ev_next_});
  ev_next_ += 2;
}

void Problem::phase_end() {
  if (capturing_) return;
  ck(cudaEventRecord(ev_pool_[ev_open_.back().second + 1], stream_), "event record");
  ph_cur_ = -1;
}

// Called after a stream synchronisation: accumulates and recycles events.
void Problem::phase_collect() {
  if (ev_open_.empty()) return;
  ck(cudaEventSynchronize(ev_pool_[ev_open_.back().second + 1]), "event sync");
  for (const auto& o : ev_open_) {
    float ms = 0.f;
    ck(cudaEventElapsedTime(&ms, ev_pool_[o.second], ev_pool_[o.second + 1]), "event elapsed");
    phase_ms_[o.first] += ms;
  }
  ev_open_.clear();
  ev_next_ = 0;
}

void Problem::sync() { ck(cudaStreamSynchronize(stream_), "kernel execution"); }

void Problem::set_parameters(const double* poses7, const double* points3, bool points_staged) {
  activate();
  const int C = d_.C, P = d_.P;
  if (poses7)
    ck(cudaMemcpyAsync(d_.pose, poses7, 7 * sizeof(double) * C, cudaMemcpyHostToDevice, stream_), "H2D poses");
  if (points_staged) {  // already in pts_user_ (caller order; the stream is ordered after the copy)
    BAE_LAUNCHED(launch_points_permute(pts_user_, src_of_internal_, d_.pts, P, true, stream_));
  } else if (points3 && !comm_) {  // caller order up, permuted into the internal order on the device
    ensure_point_staging();
    upload_pageable(pts_user_, points3, 3 * sizeof(double) * P, stream_, opt_.device);
    BAE_LAUNCHED(launch_points_permute(pts_user_, src_of_internal_, d_.pts, P, true, stream_));
  } else if (points3) {
    std::vector<double> pts(3 * static_cast<std::size_t>(P));
    for (int i = 0; i < P; ++i) {
      const int p = local_pts_[plan_.pt_of_internal[i]];
      pts[3 * i] = points3[3 * p];
      pts[3 * i + 1] = points3[3 * p + 1];
      pts[3 * i + 2] = points3[3 * p + 2];
    }
    ck(cudaMemcpyAsync(d_.pts, pts.data(), pts.size() * sizeof(double), cudaMemcpyHostToDevice, stream_),
       "H2D points");
    sync();
  }
  BAE_LAUNCHED(launch_camrec(d_, false, stream_));
  sync();
}

// Device staging of the caller-ordered points (single rank): the order
// permutation runs as a kernel instead of a host loop over P.
void Problem::ensure_point_staging() {
  if (pts_user_) return;
  if (!src_of_internal_) {  // the device plan left its own copy
    std::vector<int> src(plan_.pt_of_internal.begin(), plan_.pt_of_internal.end());
    src_of_internal_ = upload(src);
  }
  pts_user_ = dalloc<double>(3 * static_cast<std::size_t>(d_.P));
}

void Problem::get_parameters(double* poses7, double* points3) {
  activate();
  const int C = d_.C, P = d_.P;
  if (poses7) ck(cudaMemcpy(poses7, d_.pose, 7 * sizeof(double) * C, cudaMemcpyDeviceToHost), "D2H poses");
  if (points3 && comm_) {
    // every rank's points in ascending global id, gathered over the ranks
    const int W = comm_->world();
    std::vector<int> owned(static_cast<std::size_t>(W), 0);
    for (int q : rank_of_point_) ++owned[q];
    const std::size_t slot = 3 * static_cast<std::size_t>(*std::max_element(owned.begin(), owned.end()));
    std::vector<double> pts(3 * static_cast<std::size_t>(P)), mine(slot, 0.0), all(slot * W);
    ck(cudaMemcpy(pts.data(), d_.pts, pts.size() * sizeof(double), cudaMemcpyDeviceToHost), "D2H points");
    for (int i = 0; i < P; ++i) {
      const int lp = plan_.pt_of_internal[i];
      for (int a = 0; a < 3; ++a) mine[3 * lp + a] = pts[3 * i + a];
    }
    double* dbuf = nullptr;
    ck(cudaMalloc(&dbuf, sizeof(double) * slot * (W + 1)), "cudaMalloc");
    ck(cudaMemcpyAsync(dbuf, mine.data(), sizeof(double) * slot, cudaMemcpyHostToDevice, stream_), "H2D gather");
    comm_->allgather(dbuf, dbuf + slot, sizeof(double) * slot, stream_);
    ck(cudaMemcpyAsync(all.data(), dbuf + slot, sizeof(double) * slot * W, cudaMemcpyDeviceToHost, stream_),
       "D2H gather");
    sync();
    cudaFree(dbuf);
    std::vector<std::size_t> next(static_cast<std::size_t>(W), 0);
    for (int p = 0; p < P_global_; ++p) {
      const int q = rank_of_point_[p];
      const std::size_t at = q * slot + 3 * next[q]++;
      for (int a = 0; a < 3; ++a) points3[3 * p + a] = all[at + a];
    }
  } else if (points3) {  // permuted back to the caller's order on the device
    ensure_point_staging();
    BAE_LAUNCHED(launch_points_permute(d_.pts, src_of_internal_, pts_user_, P, false, stream_));
    download_pageable(points3, pts_user_, 3 * sizeof(double) * P, stream_, opt_.device);
    sync();
  }
}

// Clears the per-evaluation flags and the trial cost; keeps the cost and
// ||J^T r||^2 of the current linearisation (needed by the next solve).
void Problem::reset_lm_status(bool keep_err) {
  if (!lm_reset_host_) {
    lm_reset_host_ = static_cast<LmDev*>(pinned_take());
    *lm_reset_host_ = LmDev{};
    lm_reset_host_->err_obs = INT_MAX;
  }
  constexpr std::size_t off = offsetof(LmDev, new_cost);
  // keep_err: a linearisation queued ahead of this trial still owns err_obs
  const std::size_t end = keep_err ? offsetof(LmDev, err_obs) : sizeof(LmDev);
  ck(cudaMemcpyAsync(reinterpret_cast<char*>(d_.lm) + off, reinterpret_cast<const char*>(lm_reset_host_) + off,
                     end - off, cudaMemcpyHostToDevice, stream_),
     "H2D lm");
}

void Problem::read_lm() {
  ck(cudaMemcpyAsync(lm_host_, d_.lm, sizeof(LmDev), cudaMemcpyDeviceToHost, stream_), "D2H lm");
  sync();
}

// The original observation id of every slot on the host: the device plan
// keeps it on the device until an export needs it.
void Problem::ensure_host_obs_orig() {
  if (static_cast<std::int64_t>(plan_.obs_orig.size()) == plan_.N) return;
  plan_.obs_orig.resize(static_cast<std::size_t>(plan_.N));
  ck(cudaMemcpy(plan_.obs_orig.data(), d_.obs_orig, sizeof(int) * plan_.N, cudaMemcpyDeviceToHost), "D2H slot ids");
}

void Problem::unpermute_slots(const std::vector<double>& src, int comps, double* dst) const {
  // src: component-major [comp][N] in slot order -> dst: [N][comps] original order
  const std::int64_t N = plan_.N;
  for (std::int64_t s = 0; s < N; ++s) {
    const std::int64_t k = plan_.obs_orig[s];
    for (int j = 0; j < comps; ++j) dst[k * comps + j] = src[static_cast<std::size_t>(j) * N + s];
  }
}

double Problem::evaluate(double* resid2) {
  activate();
  if (resid2) require_single("the residual vector export");
  reset_lm_status();
  double* rbuf = nullptr;
  if (resid2) {
    ck(cudaMalloc(&rbuf, 2 * sizeof(double) * plan_.N), "cudaMalloc");
    d_.resid = rbuf;
  }
  BAE_LAUNCHED(launch_cost(d_, sm_, stream_, comm_.get()));
  d_.resid = nullptr;
  read_lm();
  if (lm_host_->err_obs != INT_MAX) {
    if (rbuf) cudaFree(rbuf);
    throw Error(BAE_ERR_CHEIRALITY, cheirality_msg(), lm_host_->err_obs);
  }
  if (rbuf) {
    std::vector<double> h(2 * static_cast<std::size_t>(plan_.N));
    ck(cudaMemcpy(h.data(), rbuf, h.size() * sizeof(double), cudaMemcpyDeviceToHost), "D2H resid");
    cudaFree(rbuf);
    ensure_host_obs_orig();
    unpermute_slots(h, 2, resid2);
  }
  return lm_host_->cost;
}

void Problem::linearize_async() {
  reset_lm_status();
  phase_begin(kPhLinearize);
  BAE_LAUNCHED(launch_linearize(d_, sm_, false, stream_, comm_.get()));
  phase_end();
}

bool Problem::fuse_lin_prep(const bae_lm_config& cfg) const {
  const char* e = std::getenv("BAE_LIN_PREP");
  return cfg.solver == BAE_SOLVER_CHOLESKY && !comm_ && !(e && e[0] == '0');
}

void Problem::linearize_prep_async(double lambda, const bae_lm_config& cfg) {
  build_direct();
  reset_lm_status();
  *lam_host_ = lambda;  // pinned: a graph replay reads it when the copy executes
  ck(cudaMemcpyAsync(const_cast<double*>(d_.lam), lam_host_, sizeof(double), cudaMemcpyHostToDevice, stream_),
     "H2D lambda");
  ck(cudaMemsetAsync(d_.pcg, 0, sizeof(PcgDev), stream_), "memset pcg");
  phase_begin(kPhLinearize);
  if (side_) {  // the camera pass beside the assembly (joined in solve_direct)
    BAE_LAUNCHED(launch_lin_prep_tiles(d_, sm_, cfg.clamp_min, cfg.clamp_max, stream_));
    ck(cudaEventRecord(ev_fork_, stream_), "event record");
    ck(cudaStreamWaitEvent(side_, ev_fork_, 0), "stream wait");
    BAE_LAUNCHED(launch_lin_prep_cams(d_, cfg.clamp_min, cfg.clamp_max, side_));
    ck(cudaEventRecord(ev_join_, side_), "event record");
    join_pending_ = true;
  } else {
    BAE_LAUNCHED(launch_lin_prep(d_, sm_, cfg.clamp_min, cfg.clamp_max, stream_));
  }
  phase_end();
  prep_fused_ = true;
}

void Problem::linearize() {
  linearize_async();
  read_lm();
  phase_collect();
  if (lm_host_->err_obs != INT_MAX)
    throw Error(BAE_ERR_CHEIRALITY, cheirality_msg(), lm_host_->err_obs);
}

void Problem::jacobian(double* jpose, double* jpoint, double* resid2) {
  activate();
  require_single("the Jacobian export");
  const std::int64_t N = plan_.N;
  double* js = nullptr;
  double* rs = nullptr;
  ck(cudaMalloc(&js, 18 * sizeof(double) * N), "cudaMalloc");
  ck(cudaMalloc(&rs, 2 * sizeof(double) * N), "cudaMalloc");
  d_.jstore = js;
  d_.resid = rs;
  reset_lm_status();
  BAE_LAUNCHED(launch_linearize(d_, sm_, true, stream_, nullptr));
  d_.jstore = nullptr;
  d_.resid = nullptr;
  read_lm();
  std::vector<double> hj(18 * static_cast<std::size_t>(N)), hr(2 * static_cast<std::size_t>(N));
  ck(cudaMemcpy(hj.data(), js, hj.size() * sizeof(double), cudaMemcpyDeviceToHost), "D2H J");
  ck(cudaMemcpy(hr.data(), rs, hr.size() * sizeof(double), cudaMemcpyDeviceToHost), "D2H r");
  cudaFree(js);
  cudaFree(rs);
  if (lm_host_->err_obs != INT_MAX)
    throw Error(BAE_ERR_CHEIRALITY, cheirality_msg(), lm_host_->err_obs);
  ensure_host_obs_orig();
  for (std::int64_t s = 0; s < N; ++s) {
    const std::int64_t k = plan_.obs_orig[s];
    if (jpose)
      for (int j = 0; j < 12; ++j) jpose[k * 12 + j] = hj[static_cast<std::size_t>(j) * N + s];
    if (jpoint)
      for (int j = 0; j < 6; ++j) jpoint[k * 6 + j] = hj[static_cast<std::size_t>(12 + j) * N + s];
    if (resid2) {
      resid2[2 * k] = hr[s];
      resid2[2 * k + 1] = hr[N + s];
    }
  }
}

void Problem::block_diagonals(double* hcc36, double* gc6, double* hpp9, double* gp3) {
  activate();
  require_single("the block-diagonal export");
  linearize();
  const int C = d_.C, P = d_.P;
  std::vector<double> h(21 * static_cast<std::size_t>(C)), g(6 * static_cast<std::size_t>(C));
  std::vector<double> hp(6 * static_cast<std::size_t>(P)), gpv(3 * static_cast<std::size_t>(P));
  ck(cudaMemcpy(h.data(), d_.hcc, h.size() * 8, cudaMemcpyDeviceToHost), "D2H");
  ck(cudaMemcpy(g.data(), d_.gc, g.size() * 8, cudaMemcpyDeviceToHost), "D2H");
  ck(cudaMemcpy(hp.data(), d_.hpp, hp.size() * 8, cudaMemcpyDeviceToHost), "D2H");
  ck(cudaMemcpy(gpv.data(), d_.gp, gpv.size() * 8, cudaMemcpyDeviceToHost), "D2H");
  for (int c = 0; c < C; ++c)
    for (int a = 0; a < 6; ++a) {
      if (gc6) gc6[c * 6 + a] = g[c * 6 + a];
      for (int b = 0; b < 6; ++b)
        if (hcc36) hcc36[c * 36 + a * 6 + b] = h[c * 21 + sym6(a, b)];
    }
  for (int i = 0; i < P; ++i) {
    const int p = plan_.pt_of_internal[i];
    for (int a = 0; a < 3; ++a) {
      if (gp3) gp3[p * 3 + a] = gpv[i * 3 + a];
      for (int b = 0; b < 3; ++b)
        if (hpp9) hpp9[p * 9 + a * 3 + b] = hp[i * 6 + sym3(a, b)];
    }
  }
}

void Problem::build_pcg_graph() {
  if (pcg_graph_) return;
  cudaGraph_t g;
  ck(cudaStreamBeginCapture(stream_, cudaStreamCaptureModeThreadLocal), "begin capture");
  for (int i = 0; i < kPcgChunk; ++i) pcg_chunk_launches_ += launch_pcg_iteration(d_, sm_, stream_, comm_.get());
  ck(cudaStreamEndCapture(stream_, &g), "end capture");
  ck(cudaGraphInstantiate(&pcg_graph_, g, 0), "graph instantiate");
  cudaGraphDestroy(g);
}

// The direct path's LM iteration as one graph launch instead of a few dozen
// API calls: G_solve = damping copy, prep, Schur assembly, tile Cholesky,
// the failure words, the trial and the LM read-back (the retry after a
// rejected step); G_acc = commit of the accepted trial, the linearisation
// fused with the prep (linearize_prep_async), then G_solve's tail. The damping
// is read from pinned memory when the copy node runs; clamps are kernel
// arguments, so a different LmConfig clamp re-captures. Returns false (and
// the caller keeps the plain launches) when capture is not possible.
bool Problem::build_lm_graphs(const bae_lm_config& cfg) {
  if (lm_graph_solve_ && graph_clo_ == cfg.clamp_min && graph_chi_ == cfg.clamp_max) return true;
  if (lm_graph_failed_) return false;
  if (lm_graph_solve_) cudaGraphExecDestroy(lm_graph_solve_);
  if (lm_graph_acc_) cudaGraphExecDestroy(lm_graph_acc_);
  lm_graph_solve_ = lm_graph_acc_ = nullptr;
  auto capture = [&](auto&& body, cudaGraphExec_t& out, long long& nlaunch) {
    cudaGraph_t g = nullptr;
    if (cudaStreamBeginCapture(stream_, cudaStreamCaptureModeThreadLocal) != cudaSuccess) return false;
    capturing_ = true;
    const long long l0 = launches_;
    bool ok = true;
    try {
      body();
    } catch (...) {
      ok = false;
    }
    capturing_ = false;
    nlaunch = launches_ - l0;
    launches_ = l0;
    const cudaError_t e = cudaStreamEndCapture(stream_, &g);
    if (!ok || e != cudaSuccess || !g) {
      if (g) cudaGraphDestroy(g);
      cudaGetLastError();
      return false;
    }
    const cudaError_t ei = cudaGraphInstantiate(&out, g, 0);
    cudaGraphDestroy(g);
    if (ei != cudaSuccess) {
      cudaGetLastError();
      out = nullptr;
      return false;
    }
    return true;
  };
  auto solve_trial = [&] {
    SolveInfo info;
    solve_direct(*lam_host_, cfg, info);  // deferred: no synchronisation inside
    reset_lm_status(true);
    BAE_LAUNCHED(launch_trial(d_, sm_, stream_, nullptr));
    ck(cudaMemcpyAsync(lm_host_, d_.lm, sizeof(LmDev), cudaMemcpyDeviceToHost, stream_), "D2H lm");
  };
  // the solve graph carries no prep: the first iteration's comes fused with
  // the initial linearisation, a rejected step's is launched before the graph
  prep_fused_ = true;
  const bool a = capture(solve_trial, lm_graph_solve_, graph_solve_launches_);
  const bool b = a && capture(
                          [&] {
                            BAE_LAUNCHED(launch_commit(d_, stream_));
                            linearize_prep_async(*lam_host_, cfg);
                            solve_trial();
                          },
                          lm_graph_acc_, graph_acc_launches_);
  prep_fused_ = false;
  if (!b) {
    if (lm_graph_acc_) cudaGraphExecDestroy(lm_graph_acc_);
    if (lm_graph_solve_) cudaGraphExecDestroy(lm_graph_solve_);
    lm_graph_acc_ = lm_graph_solve_ = nullptr;
    lm_graph_failed_ = true;
    return false;
  }
  graph_clo_ = cfg.clamp_min;
  graph_chi_ = cfg.clamp_max;
  return true;
}

// Damped solve for one lambda with the configured solver; returns false when
// the damped system is not SPD or the recurrence broke down, which the LM
// loop turns into a rejected step (lm.hpp:146-152).
bool Problem::solve(double lambda, const bae_lm_config& cfg, SolveInfo& info) {
  return cfg.solver == BAE_SOLVER_CHOLESKY ? solve_direct(lambda, cfg, info) : solve_pcg(lambda, cfg, info);
}

// Maximum reduced-system order for the dense direct solve (8.6 GB of FP64).
constexpr long long kDirectMaxOrder = 32768;

struct TileCholHost {
  int nt = 0, n = 0, npos = 0, ngroups = 0;
  std::vector<int> pos_cam;
  TileCholPlan pl;
  std::vector<int2> blk_tile;
  std::vector<unsigned long long> padmask;
  TileCholTasks tk;
};
static void tile_chol_host(int C, const std::vector<int2>& bcam, const std::vector<long long>& keys, int help_min,
                           int tail, TileCholHost& h);

// Pair list of the reduced camera system: for every point, every ordered pair
// of its observations (k, l) with camera(k) >= camera(l), grouped by camera
// block (two-pass stable counting sort), point-major inside a block.
void Problem::build_direct() {
  if (direct_ready_) return;
  HostTimer ht;
  const long long n = 6LL * d_.C;
  if (const char* m = std::getenv("BAE_DIRECT")) use_tiles_ = std::string(m) != "cusolver";
  if (!use_tiles_ && n > kDirectMaxOrder)
    throw Error(BAE_ERR_UNSUPPORTED, "solver=cholesky: reduced camera system too large for the dense direct solve; "
                                     "use solver=pcg");
  // the pair list on the device (pairs.cu): count, scan, generate, sort by block
  std::vector<int2> bcam;
  std::vector<int> bptr;
  // Single rank: the camera blocks are marked while the pairs are counted,
  // so the tile Cholesky's host symbolic phase (ordering, symbolic
  // factorisation, slots, task queue: ~8 ms at Final-13682) runs on a second
  // host thread while the device generates and sorts the pair list
  // (BAE_SYMB_OVERLAP=0: one after the other)
  const char* so_env = std::getenv("BAE_SYMB_OVERLAP");
  const bool overlap = use_tiles_ && !comm_ && d_.C <= 32768 && !(so_env && so_env[0] == '0');
  std::vector<int2> bcam_pre;
  TileCholHost chol_host;
  std::thread chol_thread;
  std::exception_ptr chol_err;
  struct Joiner {
    std::thread& t;
    ~Joiner() {
      if (t.joinable()) t.join();
    }
  } joiner{chol_thread};
  {
    long long* off = nullptr;
    unsigned* marks = nullptr;
    pairs_pool_setup();
    ck(cudaMallocAsync(reinterpret_cast<void**>(&off), (static_cast<std::size_t>(d_.P) + 1) * sizeof(long long),
                       stream_),
       "cudaMallocAsync pair offsets");
    try {
      if (overlap) {
        const std::size_t words = (static_cast<std::size_t>(d_.C) * d_.C + 31) / 32;
        ck(cudaMallocAsync(reinterpret_cast<void**>(&marks), words * sizeof(unsigned), stream_), "cudaMallocAsync");
        ck(cudaMemsetAsync(marks, 0, words * sizeof(unsigned), stream_), "memset");
      }
      const long long np = count_pairs(d_, off, stream_, marks);
      ht.mark("direct: pair count");
      if (overlap) {
        bcam_pre = marked_blocks(d_, marks, stream_);
        cudaFreeAsync(marks, stream_);
        marks = nullptr;
        const int help = chol_help_min(), tail = chol_tail(), C = d_.C;
        chol_thread = std::thread([&, help, tail, C, keys = camera_graph_keys(bcam_pre)] {
          try {
            tile_chol_host(C, bcam_pre, keys, help, tail, chol_host);
          } catch (...) {
            chol_err = std::current_exception();
          }
        });
        ht.mark("direct: blocks marked");
      }
      if (np >= (1LL << 31) - 1) throw Error(BAE_ERR_UNSUPPORTED, "reduced camera system: too many pairs");
      int2* pairs = dalloc<int2>(static_cast<std::size_t>(std::max(np, 1LL)));
      npairs_ = np;
      build_pairs(d_, off, np, pairs, bcam, bptr, stream_);
      ht.mark("direct: pair generate + sort + blocks");
      d_.pairs = pairs;
    } catch (...) {
      cudaFreeAsync(off, stream_);
      if (marks) cudaFreeAsync(marks, stream_);
      throw;
    }
    cudaFreeAsync(off, stream_);
  }
  d_.blk_ptr = upload(bptr);
  d_.blk_cam = upload(bcam);
  {  // blocks row by row (c1 ascending, c2 ascending): the chunks below keep
     // the long diagonal blocks from stalling a CTA, and the blocks in flight
     // share the V of a few hundred neighbouring cameras, which stays in L2
     // (BAE_SCHUR_ORDER=diagfirst: the diagonal blocks first)
    std::vector<int> ord;
    ord.reserve(bcam.size());
    const char* so = std::getenv("BAE_SCHUR_ORDER");
    if (so && std::string(so) == "diagfirst") {
      for (std::size_t b = 0; b < bcam.size(); ++b)
        if (bcam[b].x == bcam[b].y) ord.push_back(static_cast<int>(b));
      for (std::size_t b = 0; b < bcam.size(); ++b)
        if (bcam[b].x != bcam[b].y) ord.push_back(static_cast<int>(b));
    } else {
      for (std::size_t b = 0; b < bcam.size(); ++b) ord.push_back(static_cast<int>(b));
    }
    d_.blk_ord = upload(ord);
    // work chunks in that block order: about 32 warps' worth per SM, at
    // least kSchurChunk pairs each (short blocks stay whole, long ones split)
    const long long np = bptr.back();
    int nsm = 148;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, opt_.device);
    int ucap = 8 * kSchurChunk;
    if (const char* e = std::getenv("BAE_SCHUR_CHUNK_CAP")) ucap = std::max(kSchurChunk, std::atoi(e));
    const int U = static_cast<int>(std::clamp<long long>(np / (32LL * nsm) / 8 * 8, kSchurChunk, ucap));
    std::vector<int4> chunks;
    std::vector<int> nch(bcam.size(), 0);
    for (int b : ord) {
      const long long q0 = bptr[b], q1 = bptr[b + 1];
      const int first = static_cast<int>(chunks.size());
      // chunk bounds in 64-bit: q + U must not overflow near the 2^31 pair cap
      for (long long q = q0; q < q1 || q == q0; q += U)
        chunks.push_back(int4{b, static_cast<int>(q), static_cast<int>(std::min(q + U, q1)), first});
      nch[b] = static_cast<int>(chunks.size()) - first;
    }
    d_.chunks = upload(chunks);
    d_.nchunk = static_cast<int>(chunks.size());
    d_.blk_nchunk = upload(nch);
    d_.blk_ticket = dalloc<unsigned>(bcam.size());
    d_.schur_part = dalloc<double>(36 * chunks.size());
  }
  d_.nblk = static_cast<int>(bcam.size());
  if (!d_.wstore) d_.wstore = dalloc<double>(12 * static_cast<std::size_t>(plan_.N));  // kVStride
  if (!d_.lam) {
    d_.lam = dalloc<double>(1);
    lam_host_ = static_cast<double*>(pinned_take());
  }
  ht.mark("direct: pair list");
  // single rank: a second stream for the camera pass of the fused
  // linearise + prep, beside the Schur assembly (BAE_FORK=0: one stream)
  const char* fk = std::getenv("BAE_FORK");
  if (!comm_ && !side_ && !(fk && fk[0] == '0')) {
    ck(cudaStreamCreateWithFlags(&side_, cudaStreamNonBlocking), "stream");
    ck(cudaEventCreateWithFlags(&ev_fork_, cudaEventDisableTiming), "event");
    ck(cudaEventCreateWithFlags(&ev_join_, cudaEventDisableTiming), "event");
  }
  if (use_tiles_) {
    if (overlap) {
      chol_thread.join();
      if (chol_err) std::rethrow_exception(chol_err);
      const bool same = bcam.size() == bcam_pre.size() &&
                        std::equal(bcam.begin(), bcam.end(), bcam_pre.begin(),
                                   [](const int2& a, const int2& b) { return a.x == b.x && a.y == b.y; });
      if (same)
        upload_tile_chol(chol_host);
      else  // (the marked blocks are the pair list's blocks by construction)
        build_tile_chol(bcam);
    } else {
      build_tile_chol(bcam);
    }
    ht.mark("direct: tile symbolic");
    direct_ready_ = true;
    return;
  }
  d_.schur = dalloc<double>(static_cast<std::size_t>(n) * static_cast<std::size_t>(n));
  ht.mark("direct: alloc S");
  if (cusolverDnCreate(&solver_) != CUSOLVER_STATUS_SUCCESS) throw Error(BAE_ERR_CUDA, "cusolverDnCreate failed");
  ht.mark("direct: cusolverDnCreate");
  cusolverDnSetStream(solver_, stream_);
  if (cusolverDnDpotrf_bufferSize(solver_, CUBLAS_FILL_MODE_LOWER, static_cast<int>(n), d_.schur,
                                  static_cast<int>(n), &potrf_lwork_) != CUSOLVER_STATUS_SUCCESS)
    throw Error(BAE_ERR_CUDA, "potrf workspace query failed");
  potrf_work_ = dalloc<double>(static_cast<std::size_t>(std::max(potrf_lwork_, 1)));
  dev_info_ = dalloc<int>(1);
  host_info_ = static_cast<int*>(pinned_take());
  direct_ready_ = true;
  ht.mark("direct: alloc+cusolver");
}

// Tile pattern of S (camera blocks -> 48 x 48 tiles, the union over ranks on
// sharded runs), its symbolic factorisation and the device structures. The
// host part (tile_chol_host: ordering, symbolic, slots, task queue) touches
// no device state, so a single-rank problem runs it on a second host thread
// while the device sorts the pair list (build_direct).

// keys: the camera graph's edges c1 * C + c2 (c1 > c2), ascending, unique
static void tile_chol_host(int C, const std::vector<int2>& bcam, const std::vector<long long>& keys, int help_min,
                           int tail, TileCholHost& h) {
  HostTimer ht;
  std::vector<std::pair<int, int>> edges;
  edges.reserve(keys.size());
  for (long long k : keys) edges.emplace_back(static_cast<int>(k / C), static_cast<int>(k % C));
  // elimination order: nested dissection (BAE_ORDER=natural: camera order)
  std::vector<std::vector<int>> groups;
  const char* ord = std::getenv("BAE_ORDER");
  if (ord && std::string(ord) == "natural") {
    groups.emplace_back(C);
    for (int c = 0; c < C; ++c) groups[0][c] = c;
  } else {
    int leaf = 24;  // cameras per nested-dissection leaf (3 tiles)
    if (const char* l = std::getenv("BAE_ND_LEAF")) leaf = std::max(1, std::atoi(l));
    groups = nd_camera_groups(C, edges, leaf);
  }
  ht.mark("chol: nested dissection");
  // positions: groups in order, each padded to whole tiles (8 cameras)
  std::vector<int> pos(static_cast<std::size_t>(C), -1), pos_cam;
  for (const auto& g : groups) {
    for (int c : g) {
      pos[c] = static_cast<int>(pos_cam.size());
      pos_cam.push_back(c);
    }
    while (pos_cam.size() % 8) pos_cam.push_back(-1);
  }
  const int npos = static_cast<int>(pos_cam.size());
  const int n = 6 * npos;
  const int nt = npos / 8;
  h.ngroups = static_cast<int>(groups.size());
  std::vector<std::pair<int, int>> tp;
  tp.reserve(edges.size());
  for (const auto& e : edges) {
    const int a = pos[e.first] / 8, b = pos[e.second] / 8;
    tp.emplace_back(std::max(a, b), std::min(a, b));
  }
  TileCholPlan pl = plan_tile_chol(n, tp);
  ht.mark("chol: symbolic");
  auto slot_of = [&](int ti, int tj) {
    const auto first = pl.rowidx.begin() + pl.colptr[tj], last = pl.rowidx.begin() + pl.colptr[tj + 1];
    const auto it = std::lower_bound(first, last, ti);
    if (it == last || *it != ti) throw Error(BAE_ERR_INVALID_ARGUMENT, "tile pattern misses a camera block");
    return static_cast<int>(it - pl.rowidx.begin());
  };
  // per camera block: its tile slot and where it sits (transposed when the
  // ordering puts camera(k) before camera(l)); then per camera its diagonal slot
  std::vector<int2> blk_tile;
  blk_tile.reserve(bcam.size() + static_cast<std::size_t>(C));
  for (const int2& b : bcam) {
    int p1 = pos[b.x], p2 = pos[b.y];
    const int trans = p1 < p2 ? 1 : 0;
    if (trans) std::swap(p1, p2);
    blk_tile.push_back(int2{slot_of(p1 / 8, p2 / 8), 6 * (p1 % 8) | (6 * (p2 % 8)) << 8 | trans << 16});
  }
  for (int c = 0; c < C; ++c) blk_tile.push_back(int2{slot_of(pos[c] / 8, pos[c] / 8), 6 * (pos[c] % 8)});
  std::vector<unsigned long long> padmask(static_cast<std::size_t>(nt), 0ull);
  for (int q = 0; q < npos; ++q)
    if (pos_cam[q] < 0) padmask[q / 8] |= 0x3full << (6 * (q % 8));
  h.tk = plan_chol_tasks(pl, help_min, tail);
  ht.mark("chol: task queue");
  h.nt = nt;
  h.n = n;
  h.npos = npos;
  h.pos_cam = std::move(pos_cam);
  h.blk_tile = std::move(blk_tile);
  h.padmask = std::move(padmask);
  h.pl = std::move(pl);
}

// The camera graph's edges from the block list (the union over ranks on
// sharded runs, so that every rank derives the same order)
std::vector<long long> Problem::camera_graph_keys(const std::vector<int2>& bcam) {
  const int C = d_.C;
  std::vector<long long> keys;
  keys.reserve(bcam.size());
  for (const int2& b : bcam)
    if (b.x != b.y) keys.push_back(static_cast<long long>(b.x) * C + b.y);
  if (!std::is_sorted(keys.begin(), keys.end())) {  // the block list is already row by row, each pair once
    std::sort(keys.begin(), keys.end());
    keys.erase(std::unique(keys.begin(), keys.end()), keys.end());
  }
  if (comm_) {
    int* dcnt = nullptr;
    ck(cudaMalloc(&dcnt, sizeof(int)), "cudaMalloc");
    const int neg = -static_cast<int>(keys.size());
    ck(cudaMemcpyAsync(dcnt, &neg, sizeof(int), cudaMemcpyHostToDevice, stream_), "H2D");
    comm_->allreduce_min(dcnt, 1, stream_);  // -max count
    int mx = 0;
    ck(cudaMemcpyAsync(&mx, dcnt, sizeof(int), cudaMemcpyDeviceToHost, stream_), "D2H");
    sync();
    cudaFree(dcnt);
    const std::size_t slot = static_cast<std::size_t>(std::max(-mx, 1));
    std::vector<long long> mine(slot, -1), all(slot * comm_->world());
    std::copy(keys.begin(), keys.end(), mine.begin());
    long long* dbuf = nullptr;
    ck(cudaMalloc(&dbuf, sizeof(long long) * slot * (comm_->world() + 1)), "cudaMalloc");
    ck(cudaMemcpyAsync(dbuf, mine.data(), sizeof(long long) * slot, cudaMemcpyHostToDevice, stream_), "H2D");
    comm_->allgather(dbuf, dbuf + slot, sizeof(long long) * slot, stream_);
    ck(cudaMemcpyAsync(all.data(), dbuf + slot, sizeof(long long) * all.size(), cudaMemcpyDeviceToHost, stream_),
       "D2H");
    sync();
    cudaFree(dbuf);
    keys.clear();
    for (long long k : all)
      if (k >= 0) keys.push_back(k);
    std::sort(keys.begin(), keys.end());
    keys.erase(std::unique(keys.begin(), keys.end()), keys.end());
  }
  return keys;
}

void Problem::build_tile_chol(const std::vector<int2>& bcam) {
  TileCholHost h;
  tile_chol_host(d_.C, bcam, camera_graph_keys(bcam), chol_help_min(), chol_tail(), h);
  upload_tile_chol(h);
}

int Problem::chol_help_min() const {
  // update helpers for tiles with many updates (BAE_CHOL_HELP = minimum
  // count, 0 = off): a separator column's tile updates spread over CTAs
  int help_min = 2;
  if (const char* e = std::getenv("BAE_CHOL_HELP")) help_min = std::max(0, std::atoi(e));
  return help_min;
}
int Problem::chol_tail() const {
  // helpers for the queue's last two grids of tasks (one grid: Venice factor
  // 398 us, two: 388 us, all: Final +8 %); BAE_CHOL_TAIL=n overrides
  int tail = 2 * tile_chol_grid(1 << 30);
  if (const char* e = std::getenv("BAE_CHOL_TAIL")) tail = std::max(0, std::atoi(e));
  return tail;
}

void Problem::upload_tile_chol(TileCholHost& h) {
  const TileCholPlan& pl = h.pl;
  const int nt = h.nt, n = h.n;
  chol_groups_ = h.ngroups;
  d_.blk_tile = upload(h.blk_tile);
  d_.stile_count = pl.nnz_tiles();
  d_.stiles = dalloc<double>(static_cast<std::size_t>(pl.nnz_tiles()) * kTT);
  TileChol& t = tchol_;
  t.nt = nt;
  t.n = n;
  t.colptr = upload(pl.colptr);
  t.rowidx = upload(pl.rowidx);
  t.rptr = upload(pl.rptr);
  t.rk = upload(pl.rk);
  t.rslot = upload(pl.rslot);
  t.uptr = upload(pl.uptr);
  t.usrc = upload(pl.usrc);
  t.udst = upload(pl.udst);
  const TileCholTasks& tk = h.tk;
  t.bptr = upload(tk.bptr);
  t.bop = upload(tk.bop);
  t.tasks = upload(tk.tasks);
  t.hmask = upload(tk.hmask);
  t.border = upload(std::vector<int>(tk.order.rbegin(), tk.order.rend()));
  t.ntask = static_cast<int>(tk.tasks.size() / 4);
  chol_helpers_ = tk.helpers;
  t.tiles = d_.stiles;
  t.rhs = d_.rhs;
  t.y = dalloc<double>(static_cast<std::size_t>(nt) * kTB);
  t.x = d_.x;
  t.pos_cam = upload(h.pos_cam);
  t.padmask = upload(h.padmask);
  t.nnz = static_cast<int>(pl.nnz_tiles());
  t.flags = dalloc<unsigned>(2 * static_cast<std::size_t>(t.nnz) + nt);
  t.pflags = t.flags + t.nnz + nt;
  ck(cudaMemsetAsync(t.flags, 0, sizeof(unsigned) * (2 * static_cast<std::size_t>(t.nnz) + nt), stream_),
     "memset flags");
  t.fail = dalloc<int>(1);
  t.next = dalloc<unsigned>(3);
  ck(cudaMemsetAsync(t.next, 0, 3 * sizeof(unsigned), stream_), "memset counters");
  chol_grid_ = tile_chol_grid(t.ntask);
  chol_updates_ = static_cast<long long>(pl.usrc.size());
  if (!host_info_) host_info_ = static_cast<int*>(pinned_take());
}

// Direct solve of the damped reduced camera system (the reference's default
// Cholesky solver on the Schur complement instead of the full system):
// dense S from per-observation W, W H~^-1 (my kernels), LL^T factor and
// triangular solves (cuSOLVER potrf/potrs, FP64). NotSpd -> rejected step.
bool Problem::solve_direct(double lambda, const bae_lm_config& cfg, SolveInfo& info) {
  build_direct();
  const long long n = 6LL * d_.C;
  if (!prep_fused_) {
    *lam_host_ = lambda;  // pinned: a graph replay reads it when the copy executes
    ck(cudaMemcpyAsync(const_cast<double*>(d_.lam), lam_host_, sizeof(double), cudaMemcpyHostToDevice, stream_),
       "H2D lambda");
    ck(cudaMemsetAsync(d_.pcg, 0, sizeof(PcgDev), stream_), "memset pcg");
    phase_begin(kPhPrep);
    BAE_LAUNCHED(launch_prep(d_, sm_, lambda, cfg.clamp_min, cfg.clamp_max, cfg.pcg_tol, 1, stream_, comm_.get(),
                             true));
    phase_end();
  }
  prep_fused_ = false;
  phase_begin(kPhAssemble);
  if (use_tiles_)
    ck(cudaMemsetAsync(d_.stiles, 0, sizeof(double) * kTT * d_.stile_count, stream_), "memset S tiles");
  else
    ck(cudaMemsetAsync(d_.schur, 0, sizeof(double) * n * n, stream_), "memset S");
  BAE_LAUNCHED(launch_schur_dense(d_, stream_, comm_.get(), join_pending_));
  if (join_pending_) {  // the camera pass formed H~_cc and the right-hand side
    ck(cudaStreamWaitEvent(stream_, ev_join_, 0), "stream wait");
    join_pending_ = false;
    BAE_LAUNCHED(launch_add_hccd(d_, stream_));
  }
  phase_end();
  if (use_tiles_) {
    // tile-sparse Cholesky + both substitutions: x = S^-1 rhs straight into d_.x
    info.iters = 0;
    phase_begin(kPhFactor);
    ck(cudaMemsetAsync(tchol_.fail, 0, sizeof(int), stream_), "memset fail");
    std::vector<unsigned long long> trace;
    if (std::getenv("BAE_CHOL_TRACE")) {
      ck(cudaMalloc(&tchol_.trace, 8 * sizeof(unsigned long long) * tchol_.nt), "cudaMalloc");
      ck(cudaMemsetAsync(tchol_.trace, 0, 8 * sizeof(unsigned long long) * tchol_.nt, stream_), "memset");
    }
    // sharded runs: rank 0 holds the summed S, factors it and broadcasts the
    // camera step and its failure word (no redundant factorisations)
    if (!comm_ || comm_->rank() == 0) BAE_LAUNCHED(launch_tile_chol(tchol_, chol_grid_, stream_));
    if (comm_) {
      comm_->broadcast(d_.x, sizeof(double) * static_cast<std::size_t>(n), 0, stream_);
      comm_->broadcast(tchol_.fail, sizeof(int), 0, stream_);
    }
    phase_end();
    if (tchol_.trace) {
      trace.resize(8 * static_cast<std::size_t>(tchol_.nt));
      ck(cudaMemcpyAsync(trace.data(), tchol_.trace, trace.size() * 8, cudaMemcpyDeviceToHost, stream_), "D2H");
      sync();
      cudaFree(tchol_.trace);
      tchol_.trace = nullptr;
      unsigned long long t0 = ~0ull, t1 = 0, tb0 = ~0ull, tb1 = 0;
      double upd = 0, pot = 0, trs = 0, bwd = 0;
      for (int j = 0; j < tchol_.nt; ++j) {
        const unsigned long long* r = &trace[8 * static_cast<std::size_t>(j)];
        t0 = std::min(t0, r[0]);
        t1 = std::max(t1, r[4]);
        tb0 = std::min(tb0, r[6]);
        tb1 = std::max(tb1, r[7]);
        upd += r[1] - r[0];
        pot += r[2] - r[1];
        trs += r[4] - r[2];
        bwd += r[7] - r[6];
      }
      const double nt = tchol_.nt;
      std::fprintf(stderr,
                   "[bae chol] groups %d nt %d tiles %lld updates %lld helpers %d: factor span %.1f us, backward span %.1f us; per column "
                   "mean: wait+update %.2f potrf %.2f below-diagonal %.2f backward %.2f us\n",
                   chol_groups_, tchol_.nt, static_cast<long long>(d_.stile_count), chol_updates_, chol_helpers_,
                   (t1 - t0) * 1e-3,
                   (tb1 - tb0) * 1e-3, upd / nt * 1e-3, pot / nt * 1e-3, trs / nt * 1e-3, bwd / nt * 1e-3);
      if (std::getenv("BAE_CHOL_TRACE")[0] == '2')  // fast-path columns: absolute times from the first start
        for (int j = 0; j < tchol_.nt; ++j) {
          const unsigned long long* r = &trace[8 * static_cast<std::size_t>(j)];
          auto at = [&](int k) { return r[k] ? (r[k] - t0) * 1e-3 : -1.0; };
          std::fprintf(stderr,
                       "  col %4d: start %7.1f last-k seen %7.1f potrf %7.1f..%7.1f first pub %7.1f done %7.1f "
                       "bwd %7.1f..%7.1f\n",
                       j, at(0), at(3), at(1), at(2), at(5), at(4), at(6), at(7));
        }
    }
    ck(cudaMemcpyAsync(host_info_, tchol_.fail, sizeof(int), cudaMemcpyDeviceToHost, stream_), "D2H fail");
    ck(cudaMemcpyAsync(pcg_host_, d_.pcg, sizeof(PcgDev), cudaMemcpyDeviceToHost, stream_), "D2H pcg");
    info.converged = true;
    info.rel_residual = 0.0;
    if (defer_factor_check_ && trace.empty()) {  // checked by the caller after its next synchronisation
      info.pending = true;
      return true;
    }
    sync();
    phase_collect();
    if (*host_info_ == kCholTimeout) throw Error(BAE_ERR_CUDA, "tile Cholesky: dataflow flag wait timed out");
    if (*host_info_ != 0 || pcg_host_->not_spd) return false;  // NotSpdError (cholesky.hpp:229)
    return true;
  }
  ck(cudaMemcpyAsync(d_.x, d_.rhs, sizeof(double) * n, cudaMemcpyDeviceToDevice, stream_), "rhs copy");
  info.iters = 0;
  phase_begin(kPhFactor);
  if (cusolverDnDpotrf(solver_, CUBLAS_FILL_MODE_LOWER, static_cast<int>(n), d_.schur, static_cast<int>(n),
                       potrf_work_, potrf_lwork_, dev_info_) != CUSOLVER_STATUS_SUCCESS)
    throw Error(BAE_ERR_CUDA, "potrf launch failed");
  ck(cudaMemcpyAsync(host_info_, dev_info_, sizeof(int), cudaMemcpyDeviceToHost, stream_), "D2H info");
  ck(cudaMemcpyAsync(pcg_host_, d_.pcg, sizeof(PcgDev), cudaMemcpyDeviceToHost, stream_), "D2H pcg");
  sync();
  if (*host_info_ != 0 || pcg_host_->not_spd) {  // NotSpdError (cholesky.hpp:229)
    phase_end();
    phase_collect();
    return false;
  }
  if (cusolverDnDpotrs(solver_, CUBLAS_FILL_MODE_LOWER, static_cast<int>(n), 1, d_.schur, static_cast<int>(n), d_.x,
                       static_cast<int>(n), dev_info_) != CUSOLVER_STATUS_SUCCESS)
    throw Error(BAE_ERR_CUDA, "potrs launch failed");
  phase_end();
  info.converged = true;
  info.rel_residual = 0.0;
  return true;
}

// Damping + Schur preparation + PCG for one lambda.
bool Problem::solve_pcg(double lambda, const bae_lm_config& cfg, SolveInfo& info) {
  // budget as the reference computes it from the full system's block columns (lm.hpp:139-142)
  const long long budget =
      cfg.pcg_max_iters > 0 ? cfg.pcg_max_iters : std::max<long long>(250, 2LL * (d_.C + P_global_));
  ck(cudaMemsetAsync(d_.pcg, 0, sizeof(PcgDev), stream_), "memset pcg");
  phase_begin(kPhPrep);
  BAE_LAUNCHED(launch_prep(d_, sm_, lambda, cfg.clamp_min, cfg.clamp_max, cfg.pcg_tol, budget, stream_, comm_.get(),
                           false));
  phase_end();
  phase_begin(kPhPcg);
  if (comm_ && !comm_->capturable()) {
    // in-process rank group: host-fenced collectives, plain launches
    for (;;) {
      for (int i = 0; i < kPcgChunk; ++i) launches_ += launch_pcg_iteration(d_, sm_, stream_, comm_.get());
      ck(cudaMemcpyAsync(pcg_host_, d_.pcg, sizeof(PcgDev), cudaMemcpyDeviceToHost, stream_), "D2H pcg");
      sync();
      if (pcg_host_->state >= kPcgDone) break;
    }
  } else if (use_graph_pcg_) {
    build_pcg_graph();
    for (;;) {
      ck(cudaGraphLaunch(pcg_graph_, stream_), "graph launch");
      BAE_LAUNCHED(pcg_chunk_launches_);
      ck(cudaMemcpyAsync(pcg_host_, d_.pcg, sizeof(PcgDev), cudaMemcpyDeviceToHost, stream_), "D2H pcg");
      sync();
      if (pcg_host_->state >= kPcgDone) break;
    }
  } else {
    if (pcg_grid_ == 0) pcg_grid_ = pcg_persistent_grid(d_, sm_);
    for (;;) {
      ck(launch_pcg_persistent(d_, sm_, pcg_grid_, 4096, stream_), "cooperative launch");
      BAE_LAUNCHED(1);
      ck(cudaMemcpyAsync(pcg_host_, d_.pcg, sizeof(PcgDev), cudaMemcpyDeviceToHost, stream_), "D2H pcg");
      sync();
      if (pcg_host_->state >= kPcgDone) break;
    }
  }
  phase_end();
  phase_collect();
  info.iters = pcg_host_->iters;
  info.converged = pcg_host_->converged != 0;
  info.rel_residual = pcg_host_->bnorm > 0 ? (pcg_host_->converged ? pcg_host_->true_norm : pcg_host_->rnorm) /
                                                 pcg_host_->bnorm
                                           : 0.0;
  return pcg_host_->state == kPcgDone && !pcg_host_->not_spd;
}

void Problem::solve_step(double lambda, const bae_lm_config& cfg, double* delta, std::int64_t* iters,
                         double* relres) {
  activate();
  require_single("solve_step (a full-length step export)");
  linearize();
  SolveInfo info;
  if (!solve(lambda, cfg, info)) throw Error(BAE_ERR_NUMERICAL_BREAKDOWN, "damped system not SPD or PCG breakdown");
  reset_lm_status();
  BAE_LAUNCHED(launch_trial(d_, sm_, stream_, comm_.get()));
  sync();
  const int C = d_.C, P = d_.P;
  ck(cudaMemcpy(delta, d_.x, 6 * sizeof(double) * C, cudaMemcpyDeviceToHost), "D2H dc");
  std::vector<double> dp(3 * static_cast<std::size_t>(P));
  ck(cudaMemcpy(dp.data(), d_.dp, dp.size() * 8, cudaMemcpyDeviceToHost), "D2H dp");
  for (int i = 0; i < P; ++i) {
    const int p = plan_.pt_of_internal[i];
    for (int a = 0; a < 3; ++a) delta[6 * static_cast<std::size_t>(C) + 3 * p + a] = dp[3 * i + a];
  }
  if (iters) *iters = info.iters;
  if (relres) *relres = info.rel_residual;
}

static void validate_config(const bae_lm_config& c) {  // lm.hpp:39-45
  if (!(c.damping_min <= c.initial_damping && c.initial_damping <= c.damping_max))
    throw Error(BAE_ERR_INVALID_ARGUMENT, "LmConfig: damping out of bounds");
  if (!(c.damping_up > 0.0 && c.damping_down > 0.0))
    throw Error(BAE_ERR_INVALID_ARGUMENT, "LmConfig: damping factors must be positive");
  if (c.plateau_patience < 1) throw Error(BAE_ERR_INVALID_ARGUMENT, "LmConfig: patience must be >= 1");
}

bool plateau_stagnation(const double* h, std::size_t n, int patience, double tol) {  // lm.hpp:89-98
  if (n < static_cast<std::size_t>(patience) + 1) return false;
  for (std::size_t i = n - static_cast<std::size_t>(patience); i < n; ++i) {
    const double prev = h[i - 1];
    const double imp = prev > 0.0 ? (prev - h[i]) / prev : 0.0;
    if (imp >= tol) return false;
  }
  return true;
}

void Problem::optimize(const double* poses7, const double* points3, const bae_lm_config& cfg,
                       std::vector<bae_iter_record>& traj, bae_lm_report& rep) {
  activate();
  validate_config(cfg);
  if (cfg.solver != BAE_SOLVER_PCG && cfg.solver != BAE_SOLVER_CHOLESKY)
    throw Error(BAE_ERR_INVALID_ARGUMENT, "LmConfig: unknown solver");
  // The first direct solve's symbolic phase (pair list, nested dissection,
  // tile symbolic) is host-heavy: the initial points travel on a helper
  // thread meanwhile (single rank, large problems)
  AsyncUpload pts_up;
  const std::size_t pts_bytes = 3 * sizeof(double) * static_cast<std::size_t>(d_.P);
  if (cfg.solver == BAE_SOLVER_CHOLESKY && !direct_ready_ && points3 && !comm_ && pts_bytes >= (64u << 20)) {
    ensure_point_staging();
    pts_up.start(points3, pts_bytes, opt_.device, pts_user_);
  }
  if (cfg.solver == BAE_SOLVER_CHOLESKY) build_direct();
  if (plan_.has_empty_camera || plan_.has_empty_point)
    throw Error(BAE_ERR_INVALID_ARGUMENT, "diagonal op: missing diagonal entry");  // csr.hpp:53
  if (pts_up.s) {
    pts_up.wait_on(stream_);
    set_parameters(poses7, nullptr, /*points_staged=*/true);
  } else if (poses7 || points3) {
    set_parameters(poses7, points3);
  }
  const double n_obs = static_cast<double>(N_global_);

  cudaEvent_t ev0, ev1;
  ck(cudaEventCreate(&ev0), "event");
  ck(cudaEventCreate(&ev1), "event");
  ck(cudaEventRecord(ev0, stream_), "event record");
  // Direct solves leave the factorisation's failure word and the next
  // linearisation's cost / gradient in flight: the trial's read-back is the
  // one host synchronisation of an LM iteration (a failed factorisation
  // rejects the step as before; its trial result is ignored). On a single
  // rank the iteration runs as captured graphs (build_lm_graphs), the commit
  // of an accepted trial riding with the next linearisation.
  defer_factor_check_ = cfg.solver == BAE_SOLVER_CHOLESKY;
  struct DeferReset {
    bool& f;
    ~DeferReset() { f = false; }
  } defer_reset{defer_factor_check_};
  const char* lg = std::getenv("BAE_LM_GRAPH");
  prep_fused_ = false;
  const bool graphs = defer_factor_check_ && use_tiles_ && fuse_lin_prep(cfg) && !std::getenv("BAE_CHOL_TRACE") &&
                      !(lg && lg[0] == '0') && build_lm_graphs(cfg);
  // Initial evaluate (lm.hpp:217-220); the linearisation computes the cost
  // together with the first step's normal-equation blocks -- with the graphs,
  // fused with the first step's prep at the initial damping (the same bits as
  // the separate passes), so the first solve graph needs no prep of its own.
  bool first_fused = false;
  const char* ff = std::getenv("BAE_FIRST_FUSED");
  if (graphs && !(ff && ff[0] == '0')) {
    linearize_prep_async(cfg.initial_damping, cfg);
    if (join_pending_) {  // the cost and gradient come from the camera pass
      ck(cudaStreamWaitEvent(stream_, ev_join_, 0), "stream wait");
      join_pending_ = false;
    }
    read_lm();
    if (lm_host_->err_obs != INT_MAX) throw Error(BAE_ERR_CHEIRALITY, cheirality_msg(), lm_host_->err_obs);
    first_fused = true;
    prep_fused_ = false;  // (the graph replays do not consult it; later host-side solves must prep)
  } else {
    linearize();
  }
  double cost = lm_host_->cost;
  double grad = std::sqrt(lm_host_->grad_sq);
  std::vector<double> history{cost};
  double lambda = cfg.initial_damping;
  traj.clear();
  traj.push_back({0, 1, cost, cost / n_obs, lambda, 0.0, 0, grad, cost});
  int iterations = 0, accepted_steps = 0, rejected_steps = 0;
  long long total_pcg = 0;
  bool need_lin = false;
  rep = bae_lm_report{};
  rep.reason = BAE_TERM_MAX_ITERS;
  const auto t0 = std::chrono::steady_clock::now();
  bool lin_pending = false, commit_pending = false;
  while (iterations < cfg.max_iterations) {
    const double lambda_used = lambda;
    const bool saturated = lambda >= cfg.damping_max;
    SolveInfo info;
    bool ok = true;
    if (graphs) {
      *lam_host_ = lambda_used;
      if (need_lin) {  // commit of the accepted trial + the next linearisation and solve
        ck(cudaGraphLaunch(lm_graph_acc_, stream_), "graph launch");
        BAE_LAUNCHED(graph_acc_launches_);
        commit_pending = false;
        lin_pending = true;
        need_lin = false;
      } else {
        if (!first_fused) {  // a rejected step (or the first, unfused): the prep, then the solve graph
          ck(cudaMemcpyAsync(const_cast<double*>(d_.lam), lam_host_, sizeof(double), cudaMemcpyHostToDevice, stream_),
             "H2D lambda");
          ck(cudaMemsetAsync(d_.pcg, 0, sizeof(PcgDev), stream_), "memset pcg");
          BAE_LAUNCHED(launch_prep(d_, sm_, lambda_used, cfg.clamp_min, cfg.clamp_max, cfg.pcg_tol, 1, stream_,
                                   nullptr, true));
        }
        ck(cudaGraphLaunch(lm_graph_solve_, stream_), "graph launch");
        BAE_LAUNCHED(graph_solve_launches_);
      }
      first_fused = false;
      sync();
      info.pending = true;
    } else {
      if (need_lin) {
        if (defer_factor_check_) {
          if (fuse_lin_prep(cfg))
            linearize_prep_async(lambda_used, cfg);
          else
            linearize_async();
          lin_pending = true;
        } else {
          linearize();
          grad = std::sqrt(lm_host_->grad_sq);
        }
        need_lin = false;
      }
      ok = solve(lambda_used, cfg, info);
    }
    total_pcg += info.iters;
    bool accepted = false;
    double trial_cost = std::numeric_limits<double>::quiet_NaN();
    if (!graphs && (ok || lin_pending)) {
      if (ok) {
        reset_lm_status(lin_pending);
        phase_begin(kPhTrial);
        BAE_LAUNCHED(launch_trial(d_, sm_, stream_, comm_.get()));
        phase_end();
      }
      read_lm();
      phase_collect();
    }
    if (lin_pending) {
      lin_pending = false;
      if (lm_host_->err_obs != INT_MAX) throw Error(BAE_ERR_CHEIRALITY, cheirality_msg(), lm_host_->err_obs);
      grad = std::sqrt(lm_host_->grad_sq);
    }
    if (info.pending && use_tiles_ && *host_info_ == kCholTimeout)
      throw Error(BAE_ERR_CUDA, "tile Cholesky: dataflow flag wait timed out");
    if (info.pending && (*host_info_ != 0 || pcg_host_->not_spd)) ok = false;  // NotSpdError (cholesky.hpp:229)
    if (ok) {
      trial_cost = (lm_host_->retract_bad || lm_host_->trial_bad) ? std::numeric_limits<double>::infinity()
                                                                   : lm_host_->new_cost;
      if (trial_cost < cost) {
        if (graphs) {
          commit_pending = true;  // with the next linearisation (G_lin), or after the loop
        } else {
          phase_begin(kPhCommit);
          BAE_LAUNCHED(launch_commit(d_, stream_));
          phase_end();
        }
        cost = trial_cost;
        history.push_back(cost);
        ++accepted_steps;
        accepted = true;
        need_lin = true;
      }
    }
    if (accepted) {
      lambda = std::max(lambda * cfg.damping_down, cfg.damping_min);
    } else {
      ++rejected_steps;
      lambda = std::min(lambda * cfg.damping_up, cfg.damping_max);
    }
    ++iterations;
    const double el = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    traj.push_back({iterations, accepted ? 1 : 0, history.back(), history.back() / n_obs, lambda_used, el,
                    info.iters, grad, trial_cost});
    if (!accepted && saturated) {
      rep.reason = BAE_TERM_SOLVER_FAILURE;
      break;
    }
    if (history.back() == 0.0 ||
        plateau_stagnation(history.data(), history.size(), cfg.plateau_patience, cfg.plateau_rel_tol)) {
      rep.reason = BAE_TERM_PLATEAU;
      break;
    }
  }
  if (commit_pending) launches_ += launch_commit(d_, stream_);  // the last accepted trial
  ck(cudaEventRecord(ev1, stream_), "event record");
  sync();
  phase_collect();
  float dev_ms = 0.f;
  ck(cudaEventElapsedTime(&dev_ms, ev0, ev1), "event elapsed");
  cudaEventDestroy(ev0);
  cudaEventDestroy(ev1);
  rep.device_seconds = dev_ms * 1e-3;
  rep.iterations = iterations;
  rep.final_cost = history.back();
  rep.final_mse = rep.final_cost / n_obs;
  rep.accepted_steps = accepted_steps;
  rep.rejected_steps = rejected_steps;
  rep.final_lambda = lambda;
  rep.solve_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  rep.total_pcg_iters = total_pcg;
}

double Problem::time_kernel(int kind, int reps) {
  activate();
  if (reps < 1) reps = 1;
  cudaEvent_t a, b;
  ck(cudaEventCreate(&a), "event");
  ck(cudaEventCreate(&b), "event");
  bae_lm_config cfg;
  bae_lm_config_default(&cfg);
  if (kind == 1 || kind == 2) {
    linearize();
    SolveInfo info;
    cfg.solver = BAE_SOLVER_PCG;  // the PCG state machine, whatever the default solver
    cfg.pcg_max_iters = 1;
    solve(1e-4, cfg, info);
    // force the state machine to keep iterating on the current direction
    PcgDev s = *pcg_host_;
    s.state = kPcgIter;
    s.dir = kDirZBetaP;
    s.budget = LLONG_MAX;
    s.tol = 0.0;
    ck(cudaMemcpy(d_.pcg, &s, sizeof(PcgDev), cudaMemcpyHostToDevice), "H2D pcg");
  }
  if (kind >= 4 && kind <= 8) {  // one damped direct solve first: S assembled, plan built
    linearize();
    SolveInfo info;
    bae_lm_config c2 = cfg;
    c2.solver = BAE_SOLVER_CHOLESKY;
    solve(1e-4, c2, info);
    if (!use_tiles_) throw Error(BAE_ERR_UNSUPPORTED, "time_kernel 4..8 need the tile solver");
    if (kind == 7 && comm_) throw Error(BAE_ERR_UNSUPPORTED, "time_kernel 7: single rank only");
  }
  double* js = nullptr;
  if (kind == 3) {
    ck(cudaMalloc(&js, 18 * sizeof(double) * plan_.N), "cudaMalloc");
    d_.jstore = js;
  }
  auto launch = [&]() {
    switch (kind) {
      case 0:
        BAE_LAUNCHED(launch_linearize(d_, sm_, false, stream_, comm_.get()));
        break;
      case 1:
        BAE_LAUNCHED(launch_schur_only(d_, sm_, stream_));
        break;
      case 2:
        BAE_LAUNCHED(launch_pcg_iteration(d_, sm_, stream_, comm_.get()));
        break;
      case 3:
        BAE_LAUNCHED(launch_linearize(d_, sm_, true, stream_, comm_.get()));
        break;
      case 4:  // tile Cholesky factor + both substitutions (re-factors the factor: same work)
        BAE_LAUNCHED(launch_tile_chol(tchol_, chol_grid_, stream_));
        break;
      case 5:  // direct prep: damped point blocks, V = W L^-T, Schur right-hand side
        BAE_LAUNCHED(launch_prep(d_, sm_, 1e-4, cfg.clamp_min, cfg.clamp_max, cfg.pcg_tol, 1, stream_, nullptr, true));
        break;
      case 6:  // Schur assembly of the reduced camera matrix into its tiles
        BAE_LAUNCHED(launch_schur_dense(d_, stream_, nullptr));
        break;
      case 7:  // linearisation fused with the direct prep (the step after an accepted trial)
        BAE_LAUNCHED(launch_lin_prep(d_, sm_, cfg.clamp_min, cfg.clamp_max, stream_));
        break;
      case 8:  // retraction, point back-substitution and trial cost of the solved step
        BAE_LAUNCHED(launch_trial(d_, sm_, stream_, comm_.get()));
        break;
      default:
        throw Error(BAE_ERR_INVALID_ARGUMENT, "time_kernel: unknown kind");
    }
  };
  launch();  // warm-up
  sync();
  if (kind == 1 && std::getenv("BAE_TRACE")) {
    unsigned long long* tr = nullptr;
    ck(cudaMalloc(&tr, sizeof(unsigned long long) * 8 * d_.T), "cudaMalloc");
    ck(cudaMemset(tr, 0, sizeof(unsigned long long) * 8 * d_.T), "memset");
    d_.trace = tr;
    launch();
    sync();
    d_.trace = nullptr;
    std::vector<unsigned long long> h(8 * static_cast<std::size_t>(d_.T));
    ck(cudaMemcpy(h.data(), tr, h.size() * 8, cudaMemcpyDeviceToHost), "D2H trace");
    cudaFree(tr);
    unsigned long long t0 = ~0ULL, t1 = 0;
    double ph[5] = {0, 0, 0, 0, 0};
    for (int t = 0; t < d_.T; ++t) {
      const unsigned long long* r = &h[8 * static_cast<std::size_t>(t)];
      t0 = std::min(t0, r[0]);
      t1 = std::max(t1, r[5]);
      for (int k = 0; k < 5; ++k) ph[k] += double(r[k + 1] - r[k]);
    }
    std::fprintf(stderr, "trace: span %.1f us, mean per tile: load %.2f ph1 %.2f pt %.2f ph3 %.2f ent %.2f us\n",
                 (t1 - t0) * 1e-3, ph[0] / d_.T * 1e-3, ph[1] / d_.T * 1e-3, ph[2] / d_.T * 1e-3,
                 ph[3] / d_.T * 1e-3, ph[4] / d_.T * 1e-3);
  }
  ck(cudaEventRecord(a, stream_), "record");
  for (int i = 0; i < reps; ++i) launch();
  ck(cudaEventRecord(b, stream_), "record");
  sync();
  float ms = 0.f;
  ck(cudaEventElapsedTime(&ms, a, b), "elapsed");
  d_.jstore = nullptr;
  if (js) cudaFree(js);
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  return ms / reps;
}

}  // namespace bae
