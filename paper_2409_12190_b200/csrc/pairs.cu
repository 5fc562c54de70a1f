// The direct solver's pair list on the device (DESIGN.md §5.3 step 3): for
// every point, every ordered pair (k, l) of its observations with
// c(k) >= c(l), grouped by camera block (c(k), c(l)) ascending and, inside a
// block, in generation order (internal point, k, l) -- a count pass, a scan,
// a generation pass, a stable radix sort on the block key and a run-length
// encode (CUB, library code). Replaces a host counting sort that took
// milliseconds at Trafalgar and seconds at Final-13682.
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_run_length_encode.cuh>
#include <cub/device/device_scan.cuh>

#include <algorithm>
#include <functional>
#include <cstdint>
#include <mutex>
#include <string>
#include <vector>

#include "bae_internal.hpp"
#include "pairs.cuh"

namespace bae {

namespace {

void ck(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw Error(BAE_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

__device__ __forceinline__ int slot_camera(const Dev& d, const TileGeom& g, int slot) {
  return d.ent_cam[g.eb + static_cast<int>(d.obs_lcpt[slot] & 0xffffu)];
}

// One warp per tile, a lane per point: pairs of each internal point.
__global__ void k_pair_count(Dev d, long long* cnt) {
  const int t = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (t >= d.T) return;
  const TileGeom g = tile_geom(d, t);
  for (int lp = threadIdx.x & 31; lp < g.npts; lp += 32) {
    const int i = g.pb + lp, j0 = d.pt_ptr[i], m = d.pt_ptr[i + 1] - j0;
    long long n = 0;
    for (int a = 0; a < m; ++a) {
      const int ca = slot_camera(d, g, g.ob + d.ptobs[j0 + a]);
      for (int b = 0; b < m; ++b) n += ca >= slot_camera(d, g, g.ob + d.ptobs[j0 + b]) ? 1 : 0;
    }
    cnt[i] = n;
  }
}

template <class K>
__global__ void k_pair_gen(Dev d, const long long* off, K* keys, int2* vals) {
  const int t = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (t >= d.T) return;
  const TileGeom g = tile_geom(d, t);
  for (int lp = threadIdx.x & 31; lp < g.npts; lp += 32) {
    const int i = g.pb + lp, j0 = d.pt_ptr[i], m = d.pt_ptr[i + 1] - j0;
    long long at = off[i];
    for (int a = 0; a < m; ++a) {
      const int sa = g.ob + d.ptobs[j0 + a], ca = slot_camera(d, g, sa);
      for (int b = 0; b < m; ++b) {
        const int sb = g.ob + d.ptobs[j0 + b], cb = slot_camera(d, g, sb);
        if (ca >= cb) {
          keys[at] = static_cast<K>(ca) * static_cast<K>(d.C) + static_cast<K>(cb);
          vals[at] = int2{sa, sb};
          ++at;
        }
      }
    }
  }
}

template <class K>
void sort_and_encode(const Dev& d, const long long* off, long long np, int2* pairs, std::vector<int2>& bcam,
                     std::vector<int>& bptr, cudaStream_t s) {
  const int C = d.C;
  int bits = 1;
  while (bits < 64 && (static_cast<unsigned long long>(C) * static_cast<unsigned long long>(C) >> bits) != 0) ++bits;
  K *keys = nullptr, *keys2 = nullptr, *uniq = nullptr;
  int2* vals = nullptr;
  int *runs = nullptr, *nruns = nullptr;
  void* tmp = nullptr;
  std::size_t tsort = 0, trle = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, tsort, keys, keys2, vals, pairs, np, 0, bits, s);
  cub::DeviceRunLengthEncode::Encode(nullptr, trle, keys2, uniq, runs, nruns, np, s);
  try {
    // stream-ordered scratch: the device pool keeps it for the next problem
    ck(cudaMallocAsync(reinterpret_cast<void**>(&keys), 2 * np * sizeof(K), s), "cudaMallocAsync pair keys");
    keys2 = keys + np;
    ck(cudaMallocAsync(reinterpret_cast<void**>(&vals), np * sizeof(int2), s), "cudaMallocAsync pair values");
    ck(cudaMallocAsync(reinterpret_cast<void**>(&uniq), np * sizeof(K), s), "cudaMallocAsync block keys");
    ck(cudaMallocAsync(reinterpret_cast<void**>(&runs), (np + 1) * sizeof(int), s), "cudaMallocAsync counts");
    nruns = runs + np;
    ck(cudaMallocAsync(&tmp, std::max(tsort, trle), s), "cudaMallocAsync CUB scratch");
    k_pair_gen<K><<<(d.T + 7) / 8, 256, 0, s>>>(d, off, keys, vals);
    ck(cudaGetLastError(), "pair generation");
    ck(cub::DeviceRadixSort::SortPairs(tmp, tsort, keys, keys2, vals, pairs, np, 0, bits, s), "pair sort");
    ck(cub::DeviceRunLengthEncode::Encode(tmp, trle, keys2, uniq, runs, nruns, np, s), "block encode");
    int nb = 0;
    ck(cudaMemcpyAsync(&nb, nruns, sizeof(int), cudaMemcpyDeviceToHost, s), "D2H");
    ck(cudaStreamSynchronize(s), "pair list");
    std::vector<K> hk(static_cast<std::size_t>(nb));
    std::vector<int> hc(static_cast<std::size_t>(nb));
    ck(cudaMemcpy(hk.data(), uniq, nb * sizeof(K), cudaMemcpyDeviceToHost), "D2H");
    ck(cudaMemcpy(hc.data(), runs, nb * sizeof(int), cudaMemcpyDeviceToHost), "D2H");
    bcam.resize(static_cast<std::size_t>(nb));
    bptr.assign(static_cast<std::size_t>(nb) + 1, 0);
    for (int b = 0; b < nb; ++b) {
      bcam[b] = int2{static_cast<int>(hk[b] / static_cast<K>(C)), static_cast<int>(hk[b] % static_cast<K>(C))};
      bptr[b + 1] = bptr[b] + hc[b];
    }
  } catch (...) {
    for (void* q : {static_cast<void*>(keys), static_cast<void*>(vals), static_cast<void*>(uniq),
                    static_cast<void*>(runs), tmp})
      if (q) cudaFreeAsync(q, s);
    throw;
  }
  for (void* q : {static_cast<void*>(keys), static_cast<void*>(vals), static_cast<void*>(uniq),
                  static_cast<void*>(runs), tmp})
    cudaFreeAsync(q, s);
}

// The stream-ordered scratch comes from the device's default pool; keep what
// it grows to (the default release threshold of 0 hands it back to the
// driver at every synchronisation, and the next problem maps it again).
void keep_pool() {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return;
  static std::mutex m;
  static std::vector<int> done;
  std::lock_guard<std::mutex> l(m);
  if (std::find(done.begin(), done.end(), dev) != done.end()) return;
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
    std::uint64_t thr = ~0ull;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
  }
  done.push_back(dev);
}

}  // namespace

void pairs_pool_setup() { keep_pool(); }

long long count_pairs(const Dev& d, long long* off, cudaStream_t s) {
  // off: P + 1 entries; counts per internal point, then an exclusive scan
  ck(cudaMemsetAsync(off, 0, (static_cast<std::size_t>(d.P) + 1) * sizeof(long long), s), "memset");
  k_pair_count<<<(d.T + 7) / 8, 256, 0, s>>>(d, off);
  ck(cudaGetLastError(), "pair count");
  void* tmp = nullptr;
  std::size_t tb = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, tb, off, off, d.P + 1, s);
  ck(cudaMallocAsync(&tmp, tb, s), "cudaMallocAsync CUB scratch");
  const cudaError_t e = cub::DeviceScan::ExclusiveSum(tmp, tb, off, off, d.P + 1, s);
  cudaFreeAsync(tmp, s);
  long long np = 0;
  if (e == cudaSuccess) cudaMemcpyAsync(&np, off + d.P, sizeof(long long), cudaMemcpyDeviceToHost, s);
  const cudaError_t e2 = cudaStreamSynchronize(s);
  ck(e, "pair scan");
  ck(e2, "pair count");
  return np;
}

void build_pairs(const Dev& d, const long long* off, long long np, int2* pairs, std::vector<int2>& bcam,
                 std::vector<int>& bptr, cudaStream_t s) {
  if (static_cast<unsigned long long>(d.C) * static_cast<unsigned long long>(d.C) < (1ull << 32))
    sort_and_encode<unsigned>(d, off, np, pairs, bcam, bptr, s);
  else
    sort_and_encode<unsigned long long>(d, off, np, pairs, bcam, bptr, s);
}

// ---------------------------------------------------------------------------
// Supertiles (k_schur_super)
// ---------------------------------------------------------------------------
namespace {

// Warp per camera block: key = supertile * nblk + block for each of its pairs
// (the supertile of the pair's first slot, by binary search of the
// supertiles' first slots).
__global__ void k_super_keys(const int2* __restrict__ pairs, const int* __restrict__ bptr, int nblk,
                             const int* __restrict__ sup_slot0, int nsup, unsigned long long* __restrict__ keys) {
  const int b = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (b >= nblk) return;
  for (int q = bptr[b] + (threadIdx.x & 31); q < bptr[b + 1]; q += 32) {
    const int k = pairs[q].x;
    int lo = 0, hi = nsup;  // last supertile with first slot <= k
    while (hi - lo > 1) {
      const int mid = (lo + hi) >> 1;
      if (sup_slot0[mid] <= k) lo = mid;
      else hi = mid;
    }
    keys[q] = static_cast<unsigned long long>(lo) * static_cast<unsigned long long>(nblk) +
              static_cast<unsigned long long>(b);
  }
}

// Pairs in (supertile, block) order -> supertile-local words (k_schur_single)
// and, per pair, the chunk sort key chunk * kSupKeyStride + unit thread with
// the chunk-local word.
__global__ void k_super_local(const int2* __restrict__ sorted, const unsigned long long* __restrict__ keys, int nblk,
                              const int* __restrict__ sup_slot0, const int* __restrict__ chunk_slot0, int nchunk,
                              const unsigned short* __restrict__ uthread, long long np, unsigned* __restrict__ out,
                              unsigned* __restrict__ ckey, unsigned* __restrict__ cval) {
  const long long q = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (q >= np) return;
  const int sup = static_cast<int>(keys[q] / static_cast<unsigned long long>(nblk));
  const int2 pr = sorted[q];
  const unsigned base = static_cast<unsigned>(sup_slot0[sup]);
  out[q] = (static_cast<unsigned>(pr.x) - base) | ((static_cast<unsigned>(pr.y) - base) << 16);
  int lo = 0, hi = nchunk;  // last chunk with first slot <= k
  while (hi - lo > 1) {
    const int mid = (lo + hi) >> 1;
    if (chunk_slot0[mid] <= pr.x) lo = mid;
    else hi = mid;
  }
  const unsigned cb = static_cast<unsigned>(chunk_slot0[lo]);
  ckey[q] = static_cast<unsigned>(lo) * kSupKeyStride + uthread[q];
  // chunk-local byte offsets of the two V records (kSupChunkObs * 144 < 65536)
  cval[q] = (static_cast<unsigned>(pr.x) - cb) * (kVRec * 8) | ((static_cast<unsigned>(pr.y) - cb) * (kVRec * 8)) << 16;
}

// Warp per regular run (one camera block of one supertile): pair j of the
// run belongs to unit j % R; its consumer thread for every pair.
__global__ void k_unit_thread(const int4* __restrict__ runs, const unsigned short* __restrict__ thr, long long nrun,
                              unsigned short* __restrict__ out) {
  const long long i = static_cast<long long>(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (i >= nrun) return;
  const int4 rr = runs[i];
  for (int j = threadIdx.x & 31; j < rr.y; j += 32) out[rr.x + j] = thr[rr.w + j % rr.z];
}

__device__ __forceinline__ long long lower_bound_u32(const unsigned* __restrict__ k, long long n, unsigned v) {
  long long lo = 0, hi = n;
  while (lo < hi) {
    const long long mid = (lo + hi) >> 1;
    if (k[mid] < v) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}

// Block per chunk: the pair range of every unit thread inside the sorted
// chunk keys; count[c] = the chunk's pairs, first[c] = its first pair.
__global__ void k_chunk_counts(const unsigned* __restrict__ ckey, long long np, const unsigned char* __restrict__ staged,
                               unsigned short* __restrict__ offs, long long* __restrict__ first,
                               long long* __restrict__ bytes) {
  const int c = blockIdx.x;
  __shared__ long long base;
  if (threadIdx.x == 0) base = lower_bound_u32(ckey, np, static_cast<unsigned>(c) * kSupKeyStride);
  __syncthreads();
  for (int u = threadIdx.x; u <= kSupUnits; u += blockDim.x) {
    const long long at = lower_bound_u32(ckey, np, static_cast<unsigned>(c) * kSupKeyStride + u);
    offs[static_cast<long long>(c) * (kSupUnits + 1) + u] = static_cast<unsigned short>(at - base);
    if (u == kSupUnits) {
      first[c] = base;
      bytes[c] = staged[c] ? kSupOffBytes + (4 * (at - base) + 15) / 16 * 16 : 0;
    }
  }
}

// Block per staged chunk: its blob = unit offsets (u16), then its pairs.
__global__ void k_chunk_blobs(const unsigned short* __restrict__ offs, const long long* __restrict__ first,
                              const long long* __restrict__ boff, const long long* __restrict__ bytes,
                              const unsigned* __restrict__ cval, char* __restrict__ blob, int2* __restrict__ desc) {
  const int c = blockIdx.x;
  const long long nb = bytes[c];
  if (threadIdx.x == 0) desc[c] = int2{static_cast<int>(boff[c] / 16), static_cast<int>(nb)};
  if (nb == 0) return;
  char* o = blob + boff[c];
  unsigned short* ob = reinterpret_cast<unsigned short*>(o);
  for (int u = threadIdx.x; u < kSupOffBytes / 2; u += blockDim.x)
    ob[u] = u <= kSupUnits ? offs[static_cast<long long>(c) * (kSupUnits + 1) + u] : 0;
  const int n = offs[static_cast<long long>(c) * (kSupUnits + 1) + kSupUnits];
  unsigned* op = reinterpret_cast<unsigned*>(o + kSupOffBytes);
  for (int q = threadIdx.x; q < (static_cast<int>(nb) - kSupOffBytes) / 4; q += blockDim.x)
    op[q] = q < n ? cval[first[c] + q] : 0u;
}

// (m^2 + sum over cameras of d_c^2) / 2: the pairs (k, l) of one point with
// camera(k) >= camera(l), d_c its observations in camera c.
long long point_pairs(const Plan& pl, int t, int i, std::vector<int>& hist) {
  const int ob = pl.tile_obs_begin[t];
  const long long m = pl.pt_ptr[i + 1] - pl.pt_ptr[i];
  long long sq = 0;
  for (int j = pl.pt_ptr[i]; j < pl.pt_ptr[i + 1]; ++j) {
    const int lc = static_cast<int>(pl.obs_lcpt[ob + pl.ptobs[j]] & 0xffffu);
    sq += 2 * hist[lc] + 1;  // (d + 1)^2 - d^2
    ++hist[lc];
  }
  for (int j = pl.pt_ptr[i]; j < pl.pt_ptr[i + 1]; ++j) hist[pl.obs_lcpt[ob + pl.ptobs[j]] & 0xffffu] = 0;
  return (m * m + sq) / 2;
}

}  // namespace

void build_super(const Dev& d, const Plan& pl, const int2* pairs, const int* blk_ptr_dev,
                 const std::vector<int>& bptr, long long np, unsigned* spairs, SuperHost& out, int grid,
                 const std::function<void*(std::size_t)>& alloc, cudaStream_t s) {
  const int nblk = static_cast<int>(bptr.size()) - 1;
  // 1. supertiles over the warp-tiles, in tile order (host): greedy runs of
  //    tiles whose union of cameras stays within kSupCams and whose slots
  //    stay within kSupMaxObs; chunks of whole tiles within kSupChunkObs
  //    observations and kSupChunkPairs pairs. A tile over any cap is a single
  //    supertile of its own.
  std::vector<int> sup_slot0, chunk_slot0;
  std::vector<unsigned char> staged;  // per chunk: 1 = regular (its blob is staged)
  {
    std::vector<int> stamp(static_cast<std::size_t>(pl.C), -1), hist(static_cast<std::size_t>(pl.C) + 1, 0);
    int ncur = 0, cur_obs = 0, t0 = -1, ch_obs = 0;
    long long ch_pairs = 0;
    std::vector<int2> chunks;
    auto close = [&](int t1) {
      if (t0 < 0) return;
      const int a = pl.tile_obs_begin[t0], e = pl.tile_obs_begin[t1];
      out.sup_a.push_back(int4{a, e - a, static_cast<int>(out.sup_chunk.size()), static_cast<int>(chunks.size())});
      out.sup_b.push_back(int4{0, 0, 0, 0});
      for (const int2& c : chunks) {
        out.sup_chunk.push_back(c);
        chunk_slot0.push_back(c.x);
        staged.push_back(1);
      }
      sup_slot0.push_back(a);
      ++out.regular;
      chunks.clear();
      t0 = -1;
      ncur = 0;
      cur_obs = 0;
    };
    int sid = 0;  // stamp of the open supertile
    for (int t = 0; t < pl.T; ++t) {
      const int ob = pl.tile_obs_begin[t], nobs = pl.tile_obs_begin[t + 1] - ob;
      const int eb = pl.tile_ent_begin[t], nc = pl.tile_ent_begin[t + 1] - eb;
      long long tp = 0;
      if (nobs <= kSupChunkObs && nc <= kSupCams)
        for (int i = pl.tile_pt_begin[t]; i < pl.tile_pt_begin[t + 1]; ++i) tp += point_pairs(pl, t, i, hist);
      if (nobs > kSupChunkObs || nc > kSupCams || tp > kSupChunkPairs) {
        close(t);
        out.sup_a.push_back(int4{ob, nobs, static_cast<int>(out.sup_chunk.size()), 1});
        out.sup_b.push_back(int4{0, 0, 1, 0});
        out.sup_chunk.push_back(int2{ob, ob + nobs});
        chunk_slot0.push_back(ob);
        staged.push_back(0);
        sup_slot0.push_back(ob);
        ++out.single;
        ++sid;
        continue;
      }
      int fresh = 0;
      if (t0 >= 0)
        for (int e = eb; e < eb + nc; ++e) fresh += stamp[pl.ent_cam[e]] == sid ? 0 : 1;
      if (t0 >= 0 && (ncur + fresh > kSupCams || cur_obs + nobs > kSupMaxObs)) close(t);
      if (t0 < 0) {
        t0 = t;
        ++sid;
      }
      for (int e = eb; e < eb + nc; ++e)
        if (stamp[pl.ent_cam[e]] != sid) {
          stamp[pl.ent_cam[e]] = sid;
          ++ncur;
        }
      if (chunks.empty() || ch_obs + nobs > kSupChunkObs || ch_pairs + tp > kSupChunkPairs) {
        chunks.push_back(int2{ob, ob});
        ch_obs = 0;
        ch_pairs = 0;
      }
      chunks.back().y = ob + nobs;
      ch_obs += nobs;
      ch_pairs += tp;
      cur_obs += nobs;
    }
    close(pl.T);
  }
  const int nsup = static_cast<int>(out.sup_a.size());
  const int nchunk = static_cast<int>(out.sup_chunk.size());
  if (static_cast<unsigned long long>(nchunk) * kSupKeyStride >= (1ull << 32))
    throw Error(BAE_ERR_UNSUPPORTED, "supertile assembly: too many chunks");
  // 2. pairs into (supertile, block, point) order: stable radix sort on
  //    supertile * nblk + block (the input is block-grouped, point order inside)
  unsigned long long *keys = nullptr, *keys2 = nullptr, *uniq = nullptr;
  int2* sorted = nullptr;
  int *runs = nullptr, *nruns = nullptr, *dslot0 = nullptr;
  void* tmp = nullptr;
  const unsigned long long kmax = static_cast<unsigned long long>(nsup) * static_cast<unsigned long long>(nblk);
  int bits = 1;
  while (bits < 64 && (kmax >> bits) != 0) ++bits;
  std::size_t tsort = 0, trle = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, tsort, keys, keys2, pairs, sorted, np, 0, bits, s);
  cub::DeviceRunLengthEncode::Encode(nullptr, trle, keys2, uniq, runs, nruns, np, s);
  std::vector<unsigned long long> hk;
  std::vector<int> hc;
  int nr = 0;
  auto release = [&]() {
    for (void* q : {static_cast<void*>(keys), static_cast<void*>(uniq), static_cast<void*>(runs), tmp})
      if (q) cudaFreeAsync(q, s);
    keys = uniq = nullptr;
    runs = nullptr;
    tmp = nullptr;
  };
  try {
    ck(cudaMallocAsync(reinterpret_cast<void**>(&keys), 2 * np * sizeof(unsigned long long), s), "cudaMallocAsync");
    keys2 = keys + np;
    ck(cudaMallocAsync(reinterpret_cast<void**>(&uniq), np * sizeof(unsigned long long), s), "cudaMallocAsync");
    ck(cudaMallocAsync(reinterpret_cast<void**>(&sorted), np * sizeof(int2), s), "cudaMallocAsync");
    ck(cudaMallocAsync(reinterpret_cast<void**>(&runs), (np + 1) * sizeof(int), s), "cudaMallocAsync");
    nruns = runs + np;
    ck(cudaMallocAsync(reinterpret_cast<void**>(&dslot0), nsup * sizeof(int), s), "cudaMallocAsync");
    ck(cudaMallocAsync(&tmp, std::max(tsort, trle), s), "cudaMallocAsync CUB scratch");
    ck(cudaMemcpyAsync(dslot0, sup_slot0.data(), nsup * sizeof(int), cudaMemcpyHostToDevice, s), "H2D");
    k_super_keys<<<(nblk + 7) / 8, 256, 0, s>>>(pairs, blk_ptr_dev, nblk, dslot0, nsup, keys);
    ck(cudaGetLastError(), "supertile keys");
    ck(cub::DeviceRadixSort::SortPairs(tmp, tsort, keys, keys2, pairs, sorted, np, 0, bits, s), "supertile sort");
    ck(cub::DeviceRunLengthEncode::Encode(tmp, trle, keys2, uniq, runs, nruns, np, s), "supertile encode");
    ck(cudaMemcpyAsync(&nr, nruns, sizeof(int), cudaMemcpyDeviceToHost, s), "D2H");
    ck(cudaStreamSynchronize(s), "supertile pairs");
    hk.resize(static_cast<std::size_t>(nr));
    hc.resize(static_cast<std::size_t>(nr));
    ck(cudaMemcpy(hk.data(), uniq, nr * sizeof(unsigned long long), cudaMemcpyDeviceToHost), "D2H");
    ck(cudaMemcpy(hc.data(), runs, nr * sizeof(int), cudaMemcpyDeviceToHost), "D2H");
  } catch (...) {
    release();
    if (sorted) cudaFreeAsync(sorted, s);
    if (dslot0) cudaFreeAsync(dslot0, s);
    throw;
  }
  // keys2 (the sorted keys) lives in `keys`: keep it until step 4
  for (void* q : {static_cast<void*>(uniq), static_cast<void*>(runs), tmp})
    if (q) cudaFreeAsync(q, s);
  uniq = nullptr;
  runs = nullptr;
  tmp = nullptr;
  // 3. units. A regular supertile's runs (one per camera block it touches)
  //    are its units: each goes to a consumer warp (slot warp * kSupJ + j),
  //    largest first to the warp with the fewest MMAs so far (ceil(3 n / 4)
  //    per block and chunk, estimated per supertile). A single supertile's
  //    runs are cut into contiguous ranges of 64 (k_schur_single walks
  //    unit_pr). Each block lists its units in supertile order.
  std::vector<std::vector<int>> blk_list(static_cast<std::size_t>(nblk));
  std::vector<long long> sup_pairs;
  std::vector<int4> runs_dev;    // regular runs: {first pair, pairs, R, offset into run_thr}
  std::vector<unsigned short> run_thr;  // per regular run its R unit threads
  long long q = 0;
  int r = 0;
  for (int sp = 0; sp < nsup; ++sp) {
    const int r0 = r;
    long long tot = 0;
    while (r < nr && static_cast<int>(hk[r] / static_cast<unsigned long long>(nblk)) == sp) tot += hc[r++];
    const int nrun = r - r0;
    const bool single = out.sup_b[sp].z != 0;
    const int u0 = static_cast<int>(out.unit_pr.size());
    if (single) {
      int nu = 0;
      for (int i = r0; i < r; ++i) nu += static_cast<int>((hc[i] + 63) / 64);
      out.sup_b[sp].x = u0;
      out.sup_b[sp].y = nu;
      long long qq = q;
      for (int i = r0; i < r; ++i) {
        const int blk = static_cast<int>(hk[i] % static_cast<unsigned long long>(nblk));
        for (long long a0 = 0; a0 < hc[i]; a0 += 64) {
          blk_list[blk].push_back(static_cast<int>(out.unit_pr.size()));
          out.unit_pr.push_back(int2{static_cast<int>(qq + a0), static_cast<int>(qq + std::min<long long>(a0 + 64, hc[i]))});
        }
        qq += hc[i];
      }
      q = qq;
      sup_pairs.push_back(tot);
      continue;
    }
    if (nrun > kSupUnits) throw Error(BAE_ERR_INVALID_ARGUMENT, "supertile: too many camera blocks");
    std::vector<int> ord(static_cast<std::size_t>(nrun));
    for (int i = 0; i < nrun; ++i) ord[i] = i;
    std::stable_sort(ord.begin(), ord.end(), [&](int x, int y) { return hc[r0 + x] > hc[r0 + y]; });
    std::vector<long long> load(kSupConsumerWarps, 0);
    std::vector<int> cnt(kSupConsumerWarps, 0), slot(static_cast<std::size_t>(nrun), 0);
    for (int x : ord) {
      int best = -1;
      for (int w = 0; w < kSupConsumerWarps; ++w)
        if (cnt[w] < kSupJ && (best < 0 || load[w] < load[best])) best = w;
      slot[x] = best * kSupJ + cnt[best]++;
      load[best] += (3LL * hc[r0 + x] + 3) / 4;
    }
    out.sup_b[sp].x = u0;
    out.sup_b[sp].y = kSupUnits;  // kSupJ slots per consumer warp
    out.unit_pr.resize(out.unit_pr.size() + kSupUnits, int2{0, 0});
    long long qq = q;
    for (int i = r0; i < r; ++i) {
      const int blk = static_cast<int>(hk[i] % static_cast<unsigned long long>(nblk));
      runs_dev.push_back(int4{static_cast<int>(qq), hc[i], 1, static_cast<int>(run_thr.size())});
      run_thr.push_back(static_cast<unsigned short>(slot[i - r0]));
      blk_list[blk].push_back(u0 + slot[i - r0]);
      qq += hc[i];
    }
    q = qq;
    sup_pairs.push_back(tot);
  }
  if (q != np) throw Error(BAE_ERR_INVALID_ARGUMENT, "supertile: pair count mismatch");
  out.units = static_cast<long long>(out.unit_pr.size());
  out.blk_uptr.assign(static_cast<std::size_t>(nblk) + 1, 0);
  for (int b = 0; b < nblk; ++b) out.blk_uptr[b + 1] = out.blk_uptr[b] + static_cast<int>(blk_list[b].size());
  out.blk_units.reserve(static_cast<std::size_t>(out.units));
  for (int b = 0; b < nblk; ++b)
    for (int u : blk_list[b]) out.blk_units.push_back(u);
  // persistent k_schur_super: per chunk its supertile and first unit slot;
  // CTA ranges of whole supertiles, balanced by their pairs
  out.chunk_meta.assign(static_cast<std::size_t>(nchunk), int2{-1, 0});
  long long reg_pairs = 0;
  for (int sp = 0; sp < nsup; ++sp) {
    if (out.sup_b[sp].z) continue;
    for (int c = out.sup_a[sp].z; c < out.sup_a[sp].z + out.sup_a[sp].w; ++c) out.chunk_meta[c] = int2{sp, out.sup_b[sp].x};
    reg_pairs += sup_pairs[sp];
  }
  {
    const int G = std::max(1, std::min(grid, out.regular));
    out.cta_chunk.assign(1, 0);
    out.cta_nreg.clear();
    long long acc = 0;
    int nreg = 0;
    for (int sp = 0; sp < nsup; ++sp) {
      if (!out.sup_b[sp].z) {
        acc += sup_pairs[sp];
        nreg += out.sup_a[sp].w;
      }
      const int k = static_cast<int>(out.cta_chunk.size());  // CTA k - 1 is open
      const bool cut = k < G && acc * G >= reg_pairs * k;
      if (cut || sp == nsup - 1) {
        out.cta_chunk.push_back(out.sup_a[sp].z + out.sup_a[sp].w);
        out.cta_nreg.push_back(nreg);
        nreg = 0;
      }
    }
  }
  // 4. supertile-local words; chunk blobs: pairs re-sorted by (chunk, unit
  //    thread) -- stable, so each unit's pairs stay in point order -- then per
  //    staged chunk the unit offsets and the chunk-local pairs
  int4* drun = nullptr;
  unsigned short *dthr = nullptr, *uth = nullptr, *offs = nullptr;
  int* dch0 = nullptr;
  unsigned *ckey = nullptr, *cval = nullptr, *ckey2 = nullptr, *cval2 = nullptr;
  unsigned char* dstaged = nullptr;
  long long *first = nullptr, *bytes = nullptr, *boff = nullptr;  // bytes, boff: inside first's allocation
  auto release2 = [&]() {
    for (void* p : {static_cast<void*>(keys), static_cast<void*>(sorted), static_cast<void*>(dslot0),
                    static_cast<void*>(drun), static_cast<void*>(dthr), static_cast<void*>(uth),
                    static_cast<void*>(offs), static_cast<void*>(dch0), static_cast<void*>(ckey),
                    static_cast<void*>(cval), static_cast<void*>(dstaged), static_cast<void*>(first), tmp})
      if (p) ck(cudaFreeAsync(p, s), "cudaFreeAsync");
  };
  try {
    const long long nrr = static_cast<long long>(runs_dev.size());
    ck(cudaMallocAsync(reinterpret_cast<void**>(&drun), std::max<long long>(nrr, 1) * sizeof(int4), s),
       "cudaMallocAsync");
    ck(cudaMallocAsync(reinterpret_cast<void**>(&dthr), std::max<std::size_t>(run_thr.size(), 1) * 2, s),
       "cudaMallocAsync");
    ck(cudaMallocAsync(reinterpret_cast<void**>(&uth), np * sizeof(unsigned short), s), "cudaMallocAsync");
    ck(cudaMemsetAsync(uth, 0, np * sizeof(unsigned short), s), "memset");
    ck(cudaMallocAsync(reinterpret_cast<void**>(&dch0), nchunk * sizeof(int), s), "cudaMallocAsync");
    ck(cudaMallocAsync(reinterpret_cast<void**>(&ckey), 2 * np * sizeof(unsigned), s), "cudaMallocAsync");
    ckey2 = ckey + np;
    ck(cudaMallocAsync(reinterpret_cast<void**>(&cval), 2 * np * sizeof(unsigned), s), "cudaMallocAsync");
    cval2 = cval + np;
    ck(cudaMallocAsync(reinterpret_cast<void**>(&dstaged), nchunk, s), "cudaMallocAsync");
    ck(cudaMallocAsync(reinterpret_cast<void**>(&offs), static_cast<std::size_t>(nchunk) * (kSupUnits + 1) * 2, s),
       "cudaMallocAsync");
    ck(cudaMallocAsync(reinterpret_cast<void**>(&first), 3 * (static_cast<std::size_t>(nchunk) + 1) * 8, s),
       "cudaMallocAsync");
    bytes = first + nchunk + 1;
    boff = bytes + nchunk + 1;
    if (nrr) {
      ck(cudaMemcpyAsync(drun, runs_dev.data(), nrr * sizeof(int4), cudaMemcpyHostToDevice, s), "H2D");
      ck(cudaMemcpyAsync(dthr, run_thr.data(), run_thr.size() * 2, cudaMemcpyHostToDevice, s), "H2D");
    }
    ck(cudaMemcpyAsync(dch0, chunk_slot0.data(), nchunk * sizeof(int), cudaMemcpyHostToDevice, s), "H2D");
    ck(cudaMemcpyAsync(dstaged, staged.data(), nchunk, cudaMemcpyHostToDevice, s), "H2D");
    if (nrr) {
      k_unit_thread<<<static_cast<unsigned>((nrr + 7) / 8), 256, 0, s>>>(drun, dthr, nrr, uth);
      ck(cudaGetLastError(), "unit threads");
    }
    k_super_local<<<static_cast<unsigned>((np + 255) / 256), 256, 0, s>>>(sorted, keys2, nblk, dslot0, dch0, nchunk,
                                                                        uth, np, spairs, ckey, cval);
    ck(cudaGetLastError(), "supertile pairs");
    int cbits = 1;
    while (cbits < 32 && ((static_cast<unsigned long long>(nchunk) * kSupKeyStride) >> cbits) != 0) ++cbits;
    std::size_t t2 = 0, t3 = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, t2, ckey, ckey2, cval, cval2, np, 0, cbits, s);
    cub::DeviceScan::ExclusiveSum(nullptr, t3, bytes, boff, nchunk + 1, s);
    ck(cudaMallocAsync(&tmp, std::max(t2, t3), s), "cudaMallocAsync CUB scratch");
    ck(cub::DeviceRadixSort::SortPairs(tmp, t2, ckey, ckey2, cval, cval2, np, 0, cbits, s), "chunk sort");
    k_chunk_counts<<<nchunk, 128, 0, s>>>(ckey2, np, dstaged, offs, first, bytes);
    ck(cudaGetLastError(), "chunk counts");
    ck(cudaMemsetAsync(bytes + nchunk, 0, 8, s), "memset");
    ck(cub::DeviceScan::ExclusiveSum(tmp, t3, bytes, boff, nchunk + 1, s), "blob scan");
    long long total = 0;
    ck(cudaMemcpyAsync(&total, boff + nchunk, 8, cudaMemcpyDeviceToHost, s), "D2H");
    ck(cudaStreamSynchronize(s), "chunk blobs");
    if (total / 16 >= (1LL << 31)) throw Error(BAE_ERR_UNSUPPORTED, "supertile assembly: pair blobs too large");
    out.blob_bytes = total;
    out.blob = static_cast<char*>(alloc(static_cast<std::size_t>(std::max(total, 16LL))));
    out.chunk_blob = static_cast<int2*>(alloc(nchunk * sizeof(int2)));
    k_chunk_blobs<<<nchunk, 128, 0, s>>>(offs, first, boff, bytes, cval2, out.blob, out.chunk_blob);
    ck(cudaGetLastError(), "chunk blobs");
    ck(cudaStreamSynchronize(s), "chunk blobs");
  } catch (...) {
    release2();
    throw;
  }
  release2();
  (void)d;
}

}  // namespace bae
