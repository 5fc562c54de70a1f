// The symbolic phase on the device (single-rank problems): the same plan as
// the host planner (plan.cpp build_plan + the tile blobs of problem.cu),
// built from the raw observation arrays with sorts, scans and one greedy
// packing thread per segment. At Final-13682 size this replaces ~0.55 s of
// host work. Every step is deterministic (stable radix sorts, integer
// atomics for counts only), and the result equals the host plan element for
// element (tests/test_gpu_plan.py compares every array).
//
// Orders (as the reference's transpose plans, bsr.hpp:140-160, and plan.cpp):
//   point lists : a point's observations in ascending observation id;
//   internal    : points stably sorted by their lowest observing camera;
//   tiles       : greedy runs of internal points (obs / camera / point caps);
//   slots       : inside a tile, (camera, internal point, observation id).
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_reduce.cuh>
#include <cub/device/device_run_length_encode.cuh>
#include <cub/device/device_scan.cuh>

#include <algorithm>
#include <chrono>
#include <climits>
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <string>
#include <vector>

#include "bae_internal.hpp"
#include "device.cuh"
#include "plan_device.cuh"

namespace bae {

namespace {

void ck(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw Error(BAE_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

constexpr int kNT = 256;
inline unsigned blocks_for(long long n) { return static_cast<unsigned>((n + kNT - 1) / kNT); }
inline int bits_for(unsigned long long maxkey) {
  int b = 1;
  while (b < 64 && (maxkey >> b) != 0) ++b;
  return b;
}

// Stream-ordered scratch freed at scope exit.
struct Scratch {
  cudaStream_t s;
  std::vector<void*> ptrs;
  explicit Scratch(cudaStream_t st) : s(st) {}
  ~Scratch() {
    for (void* p : ptrs) cudaFreeAsync(p, s);
  }
  template <class T>
  T* get(std::size_t n) {
    void* p = nullptr;
    ck(cudaMallocAsync(&p, std::max<std::size_t>(n, 1) * sizeof(T), s), "cudaMallocAsync plan scratch");
    ptrs.push_back(p);
    return static_cast<T*>(p);
  }
};

// ---- validation and counts ----
// err[0] = lowest observation with a camera or point index out of range
// (make_ba_problem's IndexError position, problems.hpp:105-110).
__global__ void k_validate_count(const int* __restrict__ cam, const int* __restrict__ pt, long long N, int C, int P,
                                 int* __restrict__ err, int* __restrict__ pcnt, int* __restrict__ ccnt) {
  for (long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x; k < N; k += (long long)gridDim.x * blockDim.x) {
    const int c = cam[k], p = pt[k];
    if (c < 0 || c >= C || p < 0 || p >= P) {
      atomicMin(err, static_cast<int>(k));
      continue;
    }
    atomicAdd(pcnt + p, 1);
    atomicAdd(ccnt + c, 1);
  }
}

// flags[0] |= 1 for an empty camera, 2 for an empty point, 4 for a point
// with more than 65535 observations.
__global__ void k_count_flags(const int* __restrict__ pcnt, int P, const int* __restrict__ ccnt, int C,
                              int* __restrict__ flags) {
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  int f = 0;
  if (i < C && ccnt[i] == 0) f |= 1;
  if (i < P && pcnt[i] == 0) f |= 2;
  if (i < P && pcnt[i] > 65535) f |= 4;
  if (f) atomicOr(flags, f);
}

__global__ void k_iota(int* __restrict__ v, long long n) {
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i < n) v[i] = static_cast<int>(i);
}

__global__ void k_gather_int(const int* __restrict__ src, const int* __restrict__ idx, long long n,
                             int* __restrict__ out) {
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i < n) out[i] = src[idx[i]];
}

// Lowest observing camera of each point (C for a point without observations).
__global__ void k_mincam(const int* __restrict__ pstart, const int* __restrict__ pcam, int P, int C,
                         int* __restrict__ mincam) {
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= P) return;
  int m = C;
  for (int j = pstart[p]; j < pstart[p + 1]; ++j) m = min(m, pcam[j]);
  mincam[p] = m;
}

__global__ void k_internal_counts(const int* __restrict__ pt_of_internal, const int* __restrict__ pcnt, int P,
                                  int* __restrict__ icnt) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < P) icnt[i] = pcnt[pt_of_internal[i]];
}

// Observations in internal point order: position istart[i] + a holds the
// a-th observation (ascending id) of internal point i; its camera and point.
__global__ void k_internal_obs(const int* __restrict__ pt_of_internal, const int* __restrict__ pstart,
                               const int* __restrict__ istart, const int* __restrict__ pobs,
                               const int* __restrict__ pcam, int P, int* __restrict__ lobs, int* __restrict__ lcam,
                               int* __restrict__ lpt) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= P) return;
  const int p = pt_of_internal[i], b = pstart[p], m = pstart[p + 1] - b, o = istart[i];
  for (int a = 0; a < m; ++a) {
    lobs[o + a] = pobs[b + a];
    lcam[o + a] = pcam[b + a];
    lpt[o + a] = i;
  }
}

// ---- greedy tile packing, one thread per segment (plan.cpp's loop) ----
// A point joins the open tile unless the tile already holds points and the
// point would exceed the observation, camera or point cap; the first point
// of a tile always joins. The open tile's camera set is kept exactly up to
// the camera cap (kPipeCams) and as "over the cap" beyond, which decides
// every later point the same way as the host's exact set. The set lives in
// registers: a shift register (insertion at slot 0) scanned with unrolled
// compares. Tiles go to the segment's scratch range [i0, i1) (a segment has
// at most one tile per point) and are compacted afterwards.
__device__ __forceinline__ bool in_set(const int (&v)[kPipeCams + 1], int n, int c) {
  bool hit = false;
#pragma unroll
  for (int q = 0; q < kPipeCams + 1; ++q) hit |= (q < n) & (v[q] == c);
  return hit;
}
__device__ __forceinline__ void push_set(int (&v)[kPipeCams + 1], int c) {
#pragma unroll
  for (int q = kPipeCams; q > 0; --q) v[q] = v[q - 1];
  v[0] = c;
}

// One warp per segment. The open tile's camera set lives in lanes 16..31
// (slot q in lane 16 + q; ncur slots, or ncur = cam_cap + 1 once over the
// cap) and a point's cameras in lanes 0..15, so one __match_any_sync tells
// each point lane whether its camera is in the set and whether a lower lane
// of the point has it too; the fresh cameras are appended in lane order. A
// point with more than 16 observations runs the register path of one lane on
// a gathered copy of the set. Decisions equal plan.cpp's exact set.
__global__ void k_pack(const int* __restrict__ istart, const int* __restrict__ lcam, int P, int nseg, int obs_cap,
                       int cam_cap, int pts_cap, int* __restrict__ seg_tiles, int* __restrict__ tmp_pt,
                       int* __restrict__ tmp_nobs) {
  static_assert(kPipeCams <= 16, "the set fits lanes 16..31");
  const int sg = blockIdx.x;
  if (sg >= nseg) return;
  const int lane = threadIdx.x & 31;
  const unsigned full = 0xffffffffu;
  const int i0 = static_cast<int>(static_cast<long long>(P) * sg / nseg);
  const int i1 = static_cast<int>(static_cast<long long>(P) * (sg + 1) / nseg);
  if (i1 <= i0) {
    if (lane == 0) seg_tiles[sg] = 0;
    return;
  }
  const bool set_lane = lane >= 16;
  const int empty = -100 - lane;  // a value no camera and no other lane has
  int val = set_lane ? empty : -2 - lane;  // set lanes: slot value; point lanes: this point's camera
  int ncur = 0, t_obs = 0, t_pts = 0, out = i0;
  if (lane == 0) tmp_pt[out] = i0;
  int b = istart[i0];
  for (int i = i0; i < i1; ++i) {
    const int e = istart[i + 1], m = e - b;
    bool close = t_pts > 0 && (t_obs + m > obs_cap || t_pts + 1 > pts_cap || ncur > cam_cap);
    if (m <= 16) {
      if (!set_lane) val = lane < m ? lcam[b + lane] : -2 - lane;
      auto fresh_of = [&]() {  // point lanes whose camera is new to the set and first in the point
        const unsigned same = __match_any_sync(full, val);
        const bool f = !set_lane && lane < m && (same >> 16) == 0u && (__ffs(same) - 1) == lane;
        return __ballot_sync(full, f);
      };
      unsigned fresh = 0u;
      if (t_pts > 0 && !close) {
        fresh = fresh_of();
        close = ncur + __popc(fresh) > cam_cap;
      }
      if (close || t_pts == 0) {  // the point opens a tile: all its distinct cameras are fresh
        if (set_lane) val = empty;
        fresh = fresh_of();
      }
      if (close) {
        if (lane == 0) tmp_nobs[out] = t_obs;
        ++out;
        if (lane == 0) tmp_pt[out] = i;
        t_obs = 0;
        t_pts = 0;
        ncur = 0;
      }
      const int nnew = __popc(fresh);
      if (ncur + nnew > cam_cap) {
        ncur = cam_cap + 1;
      } else {  // set slot ncur + r takes the camera of the r-th fresh lane
        const int r = lane - 16 - ncur;
        const bool take = set_lane && r >= 0 && r < nnew;
        const int v = __shfl_sync(full, val, take ? static_cast<int>(__fns(fresh, 0, r + 1)) : 0);
        if (take) val = v;
        ncur += nnew;
      }
    } else {  // a long track: lane 0 on a gathered copy of the set
      int cams[kPipeCams + 1];
#pragma unroll
      for (int q = 0; q < kPipeCams; ++q) cams[q] = __shfl_sync(full, val, 16 + q);
      cams[kPipeCams] = -1;
      int dec = 0;  // lane 0: close | set size << 1
      if (lane == 0) {
        int n = ncur;
        bool cl = close;
        if (t_pts > 0 && !cl) {
          int fr[kPipeCams + 1];
          int nf = 0;
          for (int a = b; a < e && !cl; ++a) {
            const int cc = lcam[a];
            if (!in_set(cams, n, cc) && !in_set(fr, nf, cc)) {
              if (n + nf + 1 > cam_cap) cl = true;
              else push_set(fr, cc), ++nf;
            }
          }
        }
        if (cl || t_pts == 0) n = 0;
        for (int a = b; a < e && n <= cam_cap; ++a) {  // the point joins: its distinct cameras
          const int cc = lcam[a];
          if (!in_set(cams, n, cc)) {
            if (n == cam_cap) n = cam_cap + 1;
            else push_set(cams, cc), ++n;
          }
        }
        dec = (cl ? 1 : 0) | (n << 1);
      }
      dec = __shfl_sync(full, dec, 0);
      close = dec & 1;
      const int n = dec >> 1;
#pragma unroll
      for (int q = 0; q < kPipeCams; ++q) {
        const int v = __shfl_sync(full, cams[q], 0);
        if (lane == 16 + q) val = q < n ? v : empty;
      }
      if (close) {
        if (lane == 0) tmp_nobs[out] = t_obs;
        ++out;
        if (lane == 0) tmp_pt[out] = i;
        t_obs = 0;
        t_pts = 0;
      }
      ncur = n;
    }
    t_obs += m;
    ++t_pts;
    b = e;
  }
  if (lane == 0) {
    tmp_nobs[out] = t_obs;
    seg_tiles[sg] = out - i0 + 1;
  }
}

// Segment scratch ranges -> the tile list (tile_pt_begin, tile observations).
__global__ void k_pack_compact(const int* __restrict__ seg_first, const int* __restrict__ seg_tiles, int P, int nseg,
                               const int* __restrict__ tmp_pt, const int* __restrict__ tmp_nobs,
                               int* __restrict__ tile_pt, int* __restrict__ tile_nobs) {
  const int sg = blockIdx.x;
  if (sg >= nseg) return;
  const int i0 = static_cast<int>(static_cast<long long>(P) * sg / nseg);
  for (int k = threadIdx.x; k < seg_tiles[sg]; k += blockDim.x) {
    tile_pt[seg_first[sg] + k] = tmp_pt[i0 + k];
    tile_nobs[seg_first[sg] + k] = tmp_nobs[i0 + k];
  }
}

// tile of every internal-order observation position, and per tile its first
// observation (the exclusive scan of tile_nobs gives tile_obs_begin)
__global__ void k_tile_of_pos(const int* __restrict__ tile_obs_begin, int T, int* __restrict__ tile_of) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= T) return;
  for (int j = tile_obs_begin[t]; j < tile_obs_begin[t + 1]; ++j) tile_of[j] = t;
}

__global__ void k_slot_keys(const int* __restrict__ tile_of, const int* __restrict__ lcam, long long N, int C,
                            unsigned long long* __restrict__ keys) {
  const long long j = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (j < N) keys[j] = static_cast<unsigned long long>(tile_of[j]) * static_cast<unsigned long long>(C) + lcam[j];
}

// Entry (tile, camera) runs: entry of every slot and the entry table.
__global__ void k_entries(const unsigned long long* __restrict__ ukeys, const int* __restrict__ run_start, int E,
                          int C, int* __restrict__ ent_cam, int* __restrict__ ent_obs_begin,
                          int* __restrict__ ent_of_slot, const int* __restrict__ run_len) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= E) return;
  ent_cam[e] = static_cast<int>(ukeys[e] % static_cast<unsigned long long>(C));
  const int b = run_start[e];
  ent_obs_begin[e] = b;
  for (int s = b; s < b + run_len[e]; ++s) ent_of_slot[s] = e;
}

// First entry of every tile (entries are tile-major).
__global__ void k_tile_ent_begin(const unsigned long long* __restrict__ ukeys, int E, int C, int T,
                                 int* __restrict__ tile_ent_begin) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t > T) return;
  const unsigned long long key = static_cast<unsigned long long>(t) * static_cast<unsigned long long>(C);
  int lo = 0, hi = E;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (ukeys[mid] < key) lo = mid + 1;
    else hi = mid;
  }
  tile_ent_begin[t] = lo;
}

// Per slot: original observation id, local camera | local point << 16, and
// the inverse slot map of the internal-order positions.
__global__ void k_slots(const int* __restrict__ spos, const int* __restrict__ lobs, const int* __restrict__ lpt,
                        const int* __restrict__ tile_of, const int* __restrict__ ent_of_slot,
                        const int* __restrict__ tile_ent_begin, const int* __restrict__ tile_pt_begin, long long N,
                        int* __restrict__ obs_orig, std::uint32_t* __restrict__ obs_lcpt, int* __restrict__ slot_of_pos) {
  const long long s = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (s >= N) return;
  const int j = spos[s], t = tile_of[j];
  obs_orig[s] = lobs[j];
  obs_lcpt[s] = static_cast<std::uint32_t>(ent_of_slot[s] - tile_ent_begin[t]) |
                (static_cast<std::uint32_t>(lpt[j] - tile_pt_begin[t]) << 16);
  slot_of_pos[j] = static_cast<int>(s);
}

__global__ void k_ptobs(const int* __restrict__ slot_of_pos, const int* __restrict__ tile_of,
                        const int* __restrict__ tile_obs_begin, long long N, std::uint16_t* __restrict__ ptobs) {
  const long long j = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (j < N) ptobs[j] = static_cast<std::uint16_t>(slot_of_pos[j] - tile_obs_begin[tile_of[j]]);
}

// cam_ent_ptr[c] = first entry of camera c in the camera-sorted entry list.
__global__ void k_lower_bound_int(const int* __restrict__ sorted, int n, int m, int* __restrict__ out) {
  const int v = blockIdx.x * blockDim.x + threadIdx.x;
  if (v > m) return;
  int lo = 0, hi = n;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (sorted[mid] < v) lo = mid + 1;
    else hi = mid;
  }
  out[v] = lo;
}

// ---- tile classes (problem.cu): small tiles get a per-warp shared-memory
// slice and an index blob; the others run from global scratch ----
__global__ void k_tile_class(const int* __restrict__ tile_obs_begin, const int* __restrict__ tile_pt_begin,
                             const int* __restrict__ tile_ent_begin, int T, long long slice_limit,
                             int* __restrict__ is_small, int* __restrict__ blob_bytes, int* __restrict__ is_big,
                             int* __restrict__ kind_max, int* __restrict__ stats) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= T) return;
  const int nobs = tile_obs_begin[t + 1] - tile_obs_begin[t];
  const int npts = tile_pt_begin[t + 1] - tile_pt_begin[t];
  const int ncam = tile_ent_begin[t + 1] - tile_ent_begin[t];
  long long need = 0;
  for (int k = 0; k < kWsKindCount; ++k) need = max(need, kind_ws_bytes(k, ncam, npts, nobs));
  const bool small = nobs > 0 && nobs <= kPipeObs && ncam <= kPipeCams && npts <= kPipePts && need <= slice_limit;
  is_small[t] = small ? 1 : 0;
  is_big[t] = small ? 0 : 1;
  blob_bytes[t] = small ? (32 + 4 * ncam + 4 * (ncam + 1) + 4 * (npts + 1) + 6 * nobs + 15) / 16 * 16 : 0;
  if (small) {
    for (int k = 0; k < kWsKindCount; ++k)
      atomicMax(kind_max + k, static_cast<int>(kind_ws_bytes(k, ncam, npts, nobs)));
  } else {
    atomicMax(stats + 3, static_cast<int>(min(need, static_cast<long long>(INT_MAX))));
  }
  atomicMax(stats + 0, nobs);
  atomicMax(stats + 1, ncam);
  atomicMax(stats + 2, npts);
}

// Tile lists, workspace slots and descriptors from the scans of the class flags.
__global__ void k_tile_lists(const int* __restrict__ is_small, const int* __restrict__ small_rank,
                             const int* __restrict__ big_rank, const int* __restrict__ blob_off,
                             const int* __restrict__ blob_bytes, const int* __restrict__ tile_pt_begin, int T,
                             int* __restrict__ small_tiles, int* __restrict__ big_tiles, int* __restrict__ tile_ws,
                             int4* __restrict__ desc) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= T) return;
  if (is_small[t]) {
    small_tiles[small_rank[t]] = t;
    tile_ws[t] = -1;
    desc[t] = int4{blob_off[t] / 16, blob_bytes[t], tile_pt_begin[t], tile_pt_begin[t + 1] - tile_pt_begin[t]};
  } else {
    big_tiles[big_rank[t]] = t;
    tile_ws[t] = big_rank[t];
    desc[t] = int4{0, 0, 0, 0};
  }
}

// Index blob of every small tile (warp per tile): hdr | camid | ent | pptr |
// lcpt | ptl (device.cuh, kPipe* caps).
__global__ void k_tile_blobs(const int* __restrict__ small_tiles, int n_small, const int4* __restrict__ desc,
                             const int* __restrict__ tile_obs_begin, const int* __restrict__ tile_pt_begin,
                             const int* __restrict__ tile_ent_begin, const int* __restrict__ ent_cam,
                             const int* __restrict__ ent_obs_begin, const int* __restrict__ pt_ptr,
                             const std::uint32_t* __restrict__ obs_lcpt, const std::uint16_t* __restrict__ ptobs,
                             char* __restrict__ blob) {
  const int w = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (w >= n_small) return;
  const int t = small_tiles[w];
  const int ob = tile_obs_begin[t], pb = tile_pt_begin[t], eb = tile_ent_begin[t];
  const int nobs = tile_obs_begin[t + 1] - ob, npts = tile_pt_begin[t + 1] - pb, ncam = tile_ent_begin[t + 1] - eb;
  char* base = blob + 16LL * desc[t].x;
  int* hw = reinterpret_cast<int*>(base);
  if (lane < 8) {
    const int h[8] = {ob, nobs, pb, npts, eb, ncam, 0, 0};
    hw[lane] = h[lane];
  }
  int* q = hw + 8;
  for (int l = lane; l < ncam; l += 32) q[l] = ent_cam[eb + l];
  q += ncam;
  for (int l = lane; l <= ncam; l += 32) q[l] = ent_obs_begin[eb + l] - ob;
  q += ncam + 1;
  for (int i = lane; i <= npts; i += 32) q[i] = pt_ptr[pb + i] - ob;
  q += npts + 1;
  std::uint32_t* lc = reinterpret_cast<std::uint32_t*>(q);
  for (int i = lane; i < nobs; i += 32) lc[i] = obs_lcpt[ob + i];
  std::uint16_t* pl = reinterpret_cast<std::uint16_t*>(lc + nobs);
  for (int i = lane; i < nobs; i += 32) pl[i] = ptobs[ob + i];
  // zero padding up to the 16-byte boundary
  char* end = reinterpret_cast<char*>(pl + nobs);
  char* stop = base + desc[t].y;
  for (char* c = end + lane; c < stop; c += 32) *c = 0;
}

template <class KeyT, class ValT>
void sort_pairs(Scratch& sc, const KeyT* kin, KeyT* kout, const ValT* vin, ValT* vout, long long n, int bits,
                cudaStream_t s) {
  std::size_t tb = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, tb, kin, kout, vin, vout, n, 0, bits, s);
  void* tmp = sc.get<char>(tb);
  ck(cub::DeviceRadixSort::SortPairs(tmp, tb, kin, kout, vin, vout, n, 0, bits, s), "plan sort");
}

template <class T>
void excl_scan(Scratch& sc, const T* in, T* out, long long n, cudaStream_t s) {
  std::size_t tb = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, tb, in, out, n, s);
  void* tmp = sc.get<char>(tb);
  ck(cub::DeviceScan::ExclusiveSum(tmp, tb, in, out, n, s), "plan scan");
}

template <class T>
T read1(const T* d, cudaStream_t s) {
  T h{};
  ck(cudaMemcpyAsync(&h, d, sizeof(T), cudaMemcpyDeviceToHost, s), "D2H");
  ck(cudaStreamSynchronize(s), "plan");
  return h;
}

}  // namespace

// BAE_HOST_TIMING=1: stage times of the device planner on stderr (each
// stage synchronised; setup profiling only).
struct StageClock {
  bool on = std::getenv("BAE_HOST_TIMING") != nullptr;
  cudaStream_t s;
  std::chrono::steady_clock::time_point t = std::chrono::steady_clock::now();
  explicit StageClock(cudaStream_t st) : s(st) {}
  void mark(const char* what) {
    if (!on) return;
    cudaStreamSynchronize(s);
    const auto n = std::chrono::steady_clock::now();
    std::fprintf(stderr, "[bae dplan] %-22s %8.3f ms\n", what, std::chrono::duration<double, std::milli>(n - t).count());
    t = n;
  }
};

void build_plan_device(int C, int P, const int* cam, const int* pt, long long N, int tile_obs_cap, int tile_cam_cap,
                       int tile_pts_cap, long long slice_limit, const std::function<void*(std::size_t)>& alloc,
                       cudaStream_t s, DevicePlan& out) {
  StageClock clk(s);
  clk.mark("inputs");
  Scratch sc(s);
  // 1. validation, per-point and per-camera counts
  int* err = sc.get<int>(4);
  int* flags = err + 1;
  const int imax = INT_MAX;
  ck(cudaMemcpyAsync(err, &imax, sizeof(int), cudaMemcpyHostToDevice, s), "H2D");
  ck(cudaMemsetAsync(flags, 0, sizeof(int), s), "memset");
  int* pcnt = sc.get<int>(static_cast<std::size_t>(P) + 1);
  int* ccnt = sc.get<int>(static_cast<std::size_t>(C));
  ck(cudaMemsetAsync(pcnt, 0, sizeof(int) * (static_cast<std::size_t>(P) + 1), s), "memset");
  ck(cudaMemsetAsync(ccnt, 0, sizeof(int) * static_cast<std::size_t>(C), s), "memset");
  k_validate_count<<<std::min<unsigned>(blocks_for(N), 148 * 16), kNT, 0, s>>>(cam, pt, N, C, P, err, pcnt, ccnt);
  ck(cudaGetLastError(), "validate");
  const int bad = read1(err, s);
  if (bad != INT_MAX) {
    int hc = 0;
    ck(cudaMemcpy(&hc, cam + bad, sizeof(int), cudaMemcpyDeviceToHost), "D2H");
    if (hc < 0 || hc >= C) throw Error(BAE_ERR_INDEX, "make_ba_problem: camera index out of range", bad);
    throw Error(BAE_ERR_INDEX, "make_ba_problem: point index out of range", bad);
  }
  k_count_flags<<<blocks_for(std::max(C, P)), kNT, 0, s>>>(pcnt, P, ccnt, C, flags);
  const int fl = read1(flags, s);
  if (fl & 4) throw Error(BAE_ERR_UNSUPPORTED, "a point has more than 65535 observations");
  out.has_empty_camera = (fl & 1) != 0;
  out.has_empty_point = (fl & 2) != 0;
  clk.mark("validate+counts");
  // 2. point lists: observation ids stably sorted by point (ascending id
  //    inside a point), their cameras, point starts
  int* kiota = sc.get<int>(static_cast<std::size_t>(N));
  int* ptsorted = sc.get<int>(static_cast<std::size_t>(N));
  int* pobs = sc.get<int>(static_cast<std::size_t>(N));
  int* pcam = sc.get<int>(static_cast<std::size_t>(N));
  int* pstart = sc.get<int>(static_cast<std::size_t>(P) + 1);
  k_iota<<<blocks_for(N), kNT, 0, s>>>(kiota, N);
  sort_pairs(sc, pt, ptsorted, kiota, pobs, N, bits_for(static_cast<unsigned long long>(P)), s);
  k_gather_int<<<blocks_for(N), kNT, 0, s>>>(cam, pobs, N, pcam);
  excl_scan(sc, pcnt, pstart, static_cast<long long>(P) + 1, s);
  clk.mark("point lists");
  // 3. internal order: points stably sorted by their lowest observing camera
  int* mincam = sc.get<int>(static_cast<std::size_t>(P));
  int* mincam_sorted = sc.get<int>(static_cast<std::size_t>(P));
  int* piota = sc.get<int>(static_cast<std::size_t>(P));
  out.pt_of_internal = static_cast<int*>(alloc(sizeof(int) * static_cast<std::size_t>(P)));
  k_mincam<<<blocks_for(P), kNT, 0, s>>>(pstart, pcam, P, C, mincam);
  k_iota<<<blocks_for(P), kNT, 0, s>>>(piota, P);
  sort_pairs(sc, mincam, mincam_sorted, piota, out.pt_of_internal, P, bits_for(static_cast<unsigned long long>(C)), s);
  // observations in internal order; istart = pt_ptr (a tile's slots are the
  // contiguous run of its points' observations)
  int* icnt = sc.get<int>(static_cast<std::size_t>(P) + 1);
  out.pt_ptr = static_cast<int*>(alloc(sizeof(int) * (static_cast<std::size_t>(P) + 1)));
  ck(cudaMemsetAsync(icnt + P, 0, sizeof(int), s), "memset");
  k_internal_counts<<<blocks_for(P), kNT, 0, s>>>(out.pt_of_internal, pcnt, P, icnt);
  excl_scan(sc, icnt, out.pt_ptr, static_cast<long long>(P) + 1, s);
  int* lobs = sc.get<int>(static_cast<std::size_t>(N));
  int* lcam = sc.get<int>(static_cast<std::size_t>(N));
  int* lpt = sc.get<int>(static_cast<std::size_t>(N));
  k_internal_obs<<<blocks_for(P), kNT, 0, s>>>(out.pt_of_internal, pstart, out.pt_ptr, pobs, pcam, P, lobs, lcam, lpt);
  ck(cudaGetLastError(), "point lists");
  clk.mark("internal order");
  // 4. tiles: greedy packing per segment into scratch, then compacted
  const int nseg = plan_segments(P);
  int* seg_tiles = sc.get<int>(static_cast<std::size_t>(nseg) + 1);
  int* seg_first = sc.get<int>(static_cast<std::size_t>(nseg) + 1);
  int* tmp_pt = sc.get<int>(static_cast<std::size_t>(P));
  int* tmp_nobs = sc.get<int>(static_cast<std::size_t>(P));
  ck(cudaMemsetAsync(seg_tiles + nseg, 0, sizeof(int), s), "memset");
  k_pack<<<nseg, 32, 0, s>>>(out.pt_ptr, lcam, P, nseg, tile_obs_cap, tile_cam_cap, tile_pts_cap, seg_tiles,
                                         tmp_pt, tmp_nobs);
  ck(cudaGetLastError(), "tile packing");
  excl_scan(sc, seg_tiles, seg_first, static_cast<long long>(nseg) + 1, s);
  const int T = read1(seg_first + nseg, s);
  if (T < 1) throw Error(BAE_ERR_INVALID_ARGUMENT, "plan: no tiles");
  out.T = T;
  out.tile_pt_begin = static_cast<int*>(alloc(sizeof(int) * (static_cast<std::size_t>(T) + 1)));
  out.tile_obs_begin = static_cast<int*>(alloc(sizeof(int) * (static_cast<std::size_t>(T) + 1)));
  int* tile_nobs = sc.get<int>(static_cast<std::size_t>(T) + 1);
  k_pack_compact<<<nseg, 128, 0, s>>>(seg_first, seg_tiles, P, nseg, tmp_pt, tmp_nobs, out.tile_pt_begin, tile_nobs);
  ck(cudaMemcpyAsync(out.tile_pt_begin + T, &P, sizeof(int), cudaMemcpyHostToDevice, s), "H2D");
  ck(cudaMemsetAsync(tile_nobs + T, 0, sizeof(int), s), "memset");
  excl_scan(sc, tile_nobs, out.tile_obs_begin, static_cast<long long>(T) + 1, s);
  clk.mark("tile packing");
  int* tile_of = sc.get<int>(static_cast<std::size_t>(N));
  k_tile_of_pos<<<blocks_for(T), kNT, 0, s>>>(out.tile_obs_begin, T, tile_of);
  // 5. slots: stable sort of the internal-order positions by (tile, camera)
  unsigned long long* skeys = sc.get<unsigned long long>(2 * static_cast<std::size_t>(N));
  int* spos = sc.get<int>(static_cast<std::size_t>(N));
  k_slot_keys<<<blocks_for(N), kNT, 0, s>>>(tile_of, lcam, N, C, skeys);
  sort_pairs(sc, skeys, skeys + N, kiota, spos, N,
             bits_for(static_cast<unsigned long long>(T) * static_cast<unsigned long long>(C)), s);
  clk.mark("slot sort");
  // entries: runs of equal (tile, camera)
  unsigned long long* ukeys = sc.get<unsigned long long>(static_cast<std::size_t>(N));
  int* run_len = sc.get<int>(static_cast<std::size_t>(N) + 1);
  int* nruns = sc.get<int>(1);
  {
    std::size_t tb = 0;
    cub::DeviceRunLengthEncode::Encode(nullptr, tb, skeys + N, ukeys, run_len, nruns, N, s);
    void* tmp = sc.get<char>(tb);
    ck(cub::DeviceRunLengthEncode::Encode(tmp, tb, skeys + N, ukeys, run_len, nruns, N, s), "entries");
  }
  const int E = read1(nruns, s);
  out.E = E;
  int* run_start = sc.get<int>(static_cast<std::size_t>(E) + 1);
  ck(cudaMemsetAsync(run_len + E, 0, sizeof(int), s), "memset");
  excl_scan(sc, run_len, run_start, static_cast<long long>(E) + 1, s);
  out.ent_cam = static_cast<int*>(alloc(sizeof(int) * static_cast<std::size_t>(E)));
  out.ent_obs_begin = static_cast<int*>(alloc(sizeof(int) * (static_cast<std::size_t>(E) + 1)));
  out.tile_ent_begin = static_cast<int*>(alloc(sizeof(int) * (static_cast<std::size_t>(T) + 1)));
  int* ent_of_slot = sc.get<int>(static_cast<std::size_t>(N));
  k_entries<<<blocks_for(E), kNT, 0, s>>>(ukeys, run_start, E, C, out.ent_cam, out.ent_obs_begin, ent_of_slot, run_len);
  ck(cudaMemcpyAsync(out.ent_obs_begin + E, &N, sizeof(int), cudaMemcpyHostToDevice, s), "H2D");
  k_tile_ent_begin<<<blocks_for(static_cast<long long>(T) + 1), kNT, 0, s>>>(ukeys, E, C, T, out.tile_ent_begin);
  // per slot: original id, local camera | local point; ptobs
  out.obs_orig = static_cast<int*>(alloc(sizeof(int) * static_cast<std::size_t>(N)));
  out.obs_lcpt = static_cast<std::uint32_t*>(alloc(sizeof(std::uint32_t) * static_cast<std::size_t>(N)));
  out.ptobs = static_cast<std::uint16_t*>(alloc(sizeof(std::uint16_t) * static_cast<std::size_t>(N)));
  int* slot_of_pos = sc.get<int>(static_cast<std::size_t>(N));
  k_slots<<<blocks_for(N), kNT, 0, s>>>(spos, lobs, lpt, tile_of, ent_of_slot, out.tile_ent_begin, out.tile_pt_begin,
                                        N, out.obs_orig, out.obs_lcpt, slot_of_pos);
  k_ptobs<<<blocks_for(N), kNT, 0, s>>>(slot_of_pos, tile_of, out.tile_obs_begin, N, out.ptobs);
  ck(cudaGetLastError(), "slots");
  clk.mark("entries+slots");
  // 6. entries of each camera in ascending entry order
  int* eiota = sc.get<int>(static_cast<std::size_t>(E));
  int* ecam_sorted = sc.get<int>(static_cast<std::size_t>(E));
  out.cam_ent = static_cast<int*>(alloc(sizeof(int) * static_cast<std::size_t>(E)));
  out.cam_ent_ptr = static_cast<int*>(alloc(sizeof(int) * (static_cast<std::size_t>(C) + 1)));
  k_iota<<<blocks_for(E), kNT, 0, s>>>(eiota, E);
  sort_pairs(sc, out.ent_cam, ecam_sorted, eiota, out.cam_ent, E, bits_for(static_cast<unsigned long long>(C)), s);
  k_lower_bound_int<<<blocks_for(static_cast<long long>(C) + 1), kNT, 0, s>>>(ecam_sorted, E, C, out.cam_ent_ptr);
  clk.mark("camera entries");
  // 7. tile classes, lists, descriptors and index blobs
  int* cls = sc.get<int>(5 * (static_cast<std::size_t>(T) + 1));
  int* is_small = cls;
  int* is_big = cls + (T + 1);
  int* blob_bytes = cls + 2 * (T + 1);
  int* small_rank = cls + 3 * (T + 1);
  int* big_rank = cls + 4 * (T + 1);
  int* blob_off = sc.get<int>(static_cast<std::size_t>(T) + 1);
  int* kmax = sc.get<int>(kWsKindCount + 4);
  int* stats = kmax + kWsKindCount;
  ck(cudaMemsetAsync(kmax, 0, sizeof(int) * (kWsKindCount + 4), s), "memset");
  ck(cudaMemsetAsync(is_small + T, 0, sizeof(int), s), "memset");
  ck(cudaMemsetAsync(is_big + T, 0, sizeof(int), s), "memset");
  ck(cudaMemsetAsync(blob_bytes + T, 0, sizeof(int), s), "memset");
  k_tile_class<<<blocks_for(T), kNT, 0, s>>>(out.tile_obs_begin, out.tile_pt_begin, out.tile_ent_begin, T, slice_limit,
                                             is_small, blob_bytes, is_big, kmax, stats);
  excl_scan(sc, is_small, small_rank, static_cast<long long>(T) + 1, s);
  excl_scan(sc, is_big, big_rank, static_cast<long long>(T) + 1, s);
  excl_scan(sc, blob_bytes, blob_off, static_cast<long long>(T) + 1, s);
  int hk[kWsKindCount + 4];
  int nsb[3];
  ck(cudaMemcpyAsync(hk, kmax, sizeof(hk), cudaMemcpyDeviceToHost, s), "D2H");
  ck(cudaMemcpyAsync(nsb + 0, small_rank + T, sizeof(int), cudaMemcpyDeviceToHost, s), "D2H");
  ck(cudaMemcpyAsync(nsb + 1, big_rank + T, sizeof(int), cudaMemcpyDeviceToHost, s), "D2H");
  ck(cudaMemcpyAsync(nsb + 2, blob_off + T, sizeof(int), cudaMemcpyDeviceToHost, s), "D2H");
  ck(cudaStreamSynchronize(s), "tile classes");
  for (int k = 0; k < kWsKindCount; ++k) out.kind_slice[k] = hk[k];
  out.max_tile_obs = hk[kWsKindCount];
  out.max_tile_cams = hk[kWsKindCount + 1];
  out.max_tile_pts = hk[kWsKindCount + 2];
  out.big_need = hk[kWsKindCount + 3];
  if (out.max_tile_obs > 65536) throw Error(BAE_ERR_UNSUPPORTED, "tile exceeds 65536 observations");
  out.n_small = nsb[0];
  out.n_big = nsb[1];
  out.blob_bytes = nsb[2];
  out.small_tiles = static_cast<int*>(alloc(sizeof(int) * static_cast<std::size_t>(std::max(out.n_small, 1))));
  out.big_tiles = static_cast<int*>(alloc(sizeof(int) * static_cast<std::size_t>(std::max(out.n_big, 1))));
  out.tile_ws = static_cast<int*>(alloc(sizeof(int) * static_cast<std::size_t>(T)));
  out.tile_desc = static_cast<int4*>(alloc(sizeof(int4) * static_cast<std::size_t>(T)));
  out.tile_blob = static_cast<char*>(alloc(static_cast<std::size_t>(std::max(out.blob_bytes, 16))));
  k_tile_lists<<<blocks_for(T), kNT, 0, s>>>(is_small, small_rank, big_rank, blob_off, blob_bytes, out.tile_pt_begin,
                                             T, out.small_tiles, out.big_tiles, out.tile_ws, out.tile_desc);
  if (out.n_small)
    k_tile_blobs<<<(out.n_small + 7) / 8, 256, 0, s>>>(out.small_tiles, out.n_small, out.tile_desc,
                                                        out.tile_obs_begin, out.tile_pt_begin, out.tile_ent_begin,
                                                        out.ent_cam, out.ent_obs_begin, out.pt_ptr, out.obs_lcpt,
                                                        out.ptobs, out.tile_blob);
  ck(cudaGetLastError(), "tile blobs");
  ck(cudaStreamSynchronize(s), "device plan");
  clk.mark("tile blobs");
}

}  // namespace bae
