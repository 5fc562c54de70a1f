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

// One warp per tile, a lane per point: pairs of each internal point (and,
// with `blocks`, a bit per camera block that has one).
__global__ void k_pair_count(Dev d, long long* cnt, unsigned* blocks) {
  const int t = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (t >= d.T) return;
  const TileGeom g = tile_geom(d, t);
  for (int lp = threadIdx.x & 31; lp < g.npts; lp += 32) {
    const int i = g.pb + lp, j0 = d.pt_ptr[i], m = d.pt_ptr[i + 1] - j0;
    long long n = 0;
    for (int a = 0; a < m; ++a) {
      const int ca = slot_camera(d, g, g.ob + d.ptobs[j0 + a]);
      for (int b = 0; b < m; ++b) {
        const int cb = slot_camera(d, g, g.ob + d.ptobs[j0 + b]);
        if (ca >= cb) {
          ++n;
          if (blocks) {
            const unsigned long long key = static_cast<unsigned long long>(ca) * d.C + cb;
            const unsigned bit = 1u << (key & 31u);
            unsigned* w = blocks + (key >> 5);
            if (!(*w & bit)) atomicOr(w, bit);  // most blocks are marked early: skip the atomic
          }
        }
      }
    }
    cnt[i] = n;
  }
}

// Marked blocks -> keys c1 * C + c2, ascending: per word its popcount, an
// exclusive scan, then every word writes its keys at its offset.
__global__ void k_bits_count(const unsigned* w, long long nw, int* cnt) {
  const long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < nw) cnt[i] = __popc(w[i]);
}
__global__ void k_bits_emit(const unsigned* w, long long nw, const int* off, int C, int2* out) {
  const long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= nw) return;
  unsigned v = w[i];
  int at = off[i];
  while (v) {
    const int b = __ffs(v) - 1;
    v &= v - 1;
    const unsigned long long key = static_cast<unsigned long long>(i) * 32 + b;
    out[at++] = int2{static_cast<int>(key / C), static_cast<int>(key % C)};
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

long long count_pairs(const Dev& d, long long* off, cudaStream_t s, unsigned* blocks) {
  // off: P + 1 entries; counts per internal point, then an exclusive scan
  ck(cudaMemsetAsync(off, 0, (static_cast<std::size_t>(d.P) + 1) * sizeof(long long), s), "memset");
  k_pair_count<<<(d.T + 7) / 8, 256, 0, s>>>(d, off, blocks);
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

std::vector<int2> marked_blocks(const Dev& d, const unsigned* blocks, cudaStream_t s) {
  const long long nw = (static_cast<long long>(d.C) * d.C + 31) / 32;
  int* cnt = nullptr;
  int2* keys = nullptr;
  void* tmp = nullptr;
  std::size_t tb = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, tb, cnt, cnt, nw + 1, s);
  std::vector<int2> out;
  try {
    ck(cudaMallocAsync(reinterpret_cast<void**>(&cnt), (nw + 1) * sizeof(int), s), "cudaMallocAsync");
    ck(cudaMallocAsync(&tmp, tb, s), "cudaMallocAsync CUB scratch");
    ck(cudaMemsetAsync(cnt + nw, 0, sizeof(int), s), "memset");
    const unsigned nb = static_cast<unsigned>((nw + 255) / 256);
    k_bits_count<<<nb, 256, 0, s>>>(blocks, nw, cnt);
    ck(cub::DeviceScan::ExclusiveSum(tmp, tb, cnt, cnt, nw + 1, s), "block scan");
    int n = 0;
    ck(cudaMemcpyAsync(&n, cnt + nw, sizeof(int), cudaMemcpyDeviceToHost, s), "D2H");
    ck(cudaStreamSynchronize(s), "block count");
    ck(cudaMallocAsync(reinterpret_cast<void**>(&keys), std::max(n, 1) * sizeof(int2), s), "cudaMallocAsync");
    k_bits_emit<<<nb, 256, 0, s>>>(blocks, nw, cnt, d.C, keys);
    out.resize(static_cast<std::size_t>(n));
    ck(cudaMemcpyAsync(out.data(), keys, n * sizeof(int2), cudaMemcpyDeviceToHost, s), "D2H blocks");
    ck(cudaStreamSynchronize(s), "blocks");
  } catch (...) {
    for (void* q : {static_cast<void*>(cnt), tmp, static_cast<void*>(keys)})
      if (q) cudaFreeAsync(q, s);
    throw;
  }
  for (void* q : {static_cast<void*>(cnt), tmp, static_cast<void*>(keys)}) cudaFreeAsync(q, s);
  return out;
}

void build_pairs(const Dev& d, const long long* off, long long np, int2* pairs, std::vector<int2>& bcam,
                 std::vector<int>& bptr, cudaStream_t s) {
  if (static_cast<unsigned long long>(d.C) * static_cast<unsigned long long>(d.C) < (1ull << 32))
    sort_and_encode<unsigned>(d, off, np, pairs, bcam, bptr, s);
  else
    sort_and_encode<unsigned long long>(d, off, np, pairs, bcam, bptr, s);
}

}  // namespace bae
