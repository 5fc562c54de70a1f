// Device-side data layout, tile workspaces and the deterministic reduction
// primitives shared by all kernels.
#pragma once

#include <cstdint>

#include "lie.cuh"

namespace bae {

constexpr int kTileThreads = 256;  // CTA size of the tile kernels (8 warps)
constexpr int kCamRec = 16;        // per camera: R[9] t[3] intrinsics[4] (BAL f k1 k2 0 | pinhole fx fy cx cy)
constexpr int kWarpsPerCamBlock = 8;
constexpr int kSTileElems = 48 * 48;  // one tile of the tile-sparse reduced matrix (chol.cuh kTT)

// PCG state machine (implicit-Schur PCG, restating pcg.hpp:32-129 on the
// reduced camera system).
enum PcgState : int { kPcgIter = 0, kPcgVerify = 1, kPcgDone = 2, kPcgBreakdown = 3 };
enum PcgDir : int { kDirZ = 0, kDirZBetaP = 1, kDirX = 2 };

struct PcgDev {
  double rz, alpha, beta, bnorm, rnorm, true_norm, tol;
  long long iters, budget;
  int state, dir, converged, not_spd;
};

struct LmDev {
  double cost;        // cost at the linearisation point
  double grad_sq;     // ||J^T r||^2 at the linearisation point
  double new_cost;    // trial cost
  int trial_bad;      // cheirality / non-finite in the trial step
  int retract_bad;
  int err_obs;        // lowest observation on the camera plane (INT_MAX: none)
  int pad;
};

// Everything a kernel needs, passed by value.
struct Dev {
  int C, P, T, E, N;
  int pinhole;  // camera variant of the whole problem (problems.hpp:94-98)
  int nbig;
  long long big_stride;  // bytes per big-tile workspace
  const int* tile_obs_begin;
  const int* tile_pt_begin;
  const int* tile_ent_begin;
  const int* tile_ws;
  const std::uint32_t* obs_lcpt;
  const int* obs_orig;
  const double* obs_px;
  const int* ent_cam;
  const int* ent_obs_begin;
  const int* cam_ent_ptr;
  const int* cam_ent;
  const int* pt_ptr;
  const std::uint16_t* ptobs;
  char* bigws;
  // parameters
  double* pose;    // 7C  [t q]
  double* intr;    // 4C  [f k1 k2 0] or [fx fy cx cy]
  double* camrec;  // 16C
  double* pts;     // 3P internal order
  double* pose_t;
  double* camrec_t;
  double* pts_t;
  // linearisation / damping
  double* hpp;    // 6P
  double* gp;     // 3P
  double* hinv;   // 6P
  double* dp;     // 3P
  double* hcc;    // 21C
  double* gc;     // 6C
  double* hccd;   // 21C damped
  double* minv;   // 36C
  double* rhs;    // 6C
  // PCG vectors (6C each)
  double* x;
  double* r;
  double* z;
  double* p;
  double* y;
  double* partial;    // E * 27
  double* partial6;   // E * 6: Schur RHS pieces of the fused linearisation + prep
  double* tile_red;   // T * 2
  // Sharded runs: per-rank camera-sized partial sums that the
  // communicator sums in place between a tile pass and its camera pass;
  // null on a single rank (the camera passes then read the entries directly).
  double* cred;
  double* cam_dot;    // 2C per-camera scalars for fixed-order totals
  double* block_red;  // grid-reduction scratch
  unsigned* tickets;  // grid-reduction tickets
  PcgDev* pcg;
  LmDev* lm;
  // stored-Jacobian mode and exports (slot order, component-major [comp][N])
  double* jstore;  // 18 * N or null
  double* resid;   // 2 * N or null
  // direct solver (dense reduced camera system): per-slot W = J_c^T J_p and
  // W H~_pp^-1 (36 doubles, slot order), pair list grouped by camera block
  double* wstore;           // direct solver: compact V = W L^-T record per slot ([Q | y], 12 doubles)
  const double* lam;        // direct solver: the damping of the current solve (device copy)
  const int2* pairs;       // (slot k, slot l), c(k) >= c(l), grouped by block
  const int* blk_ptr;      // nblk + 1
  const int2* blk_cam;     // (c1, c2), c1 >= c2
  int nblk;
  int defer_hccd;           // k_schur_dense: diagonal blocks without H~_cc (added by k_add_hccd)
  double* schur;           // 6C x 6C, column-major (lower triangle used; cuSOLVER path)
  // tile-sparse storage of S (chol.cuh): per camera block the slot of the
  // 48 x 48 tile holding it (8 cameras per tile), column-major tiles
  // per camera block {tile slot, row offset | col offset << 8 | transposed << 16},
  // then per camera {diagonal tile slot, offset}
  const int* blk_ord;       // direct solver: diagonal blocks first, then row by row
  const int4* chunks;       // k_schur_dense work: (block, first pair, end pair, block's first chunk), blk_ord order
  int nchunk;
  const int* blk_nchunk;    // chunks per block
  unsigned* blk_ticket;     // per block: chunks done (reset before every assembly)
  double* schur_part;       // 36 per chunk: partial 6x6 sums of multi-chunk blocks
  const int2* blk_tile;
  double* stiles;
  long long stile_count;
  unsigned long long* trace;  // per-tile phase timestamps (BAE_TRACE) or null
  // pipelined small tiles: per-tile descriptor {blob offset / 16, blob bytes,
  // first point, point count} and the packed per-tile index blobs
  const int4* tile_desc;
  const char* tile_blob;
  const int* small_tiles;
  const int* big_tiles;
  int n_small, n_big_tiles;
};

// ---- pipelined warp-tiles: fixed caps and the per-warp shared-memory map ----
// A small tile has at most kPipeObs observations, kPipeCams cameras and
// kPipePts points; its index blob is
//   [hdr int x8: ob nobs pb npts eb ncam 0 0 | camid[ncam] | ent[ncam+1] |
//    pptr[npts+1] | lcpt u32[nobs] | ptl u16[nobs] ] padded to 16 bytes.
constexpr int kPipeObs = 96, kPipeCams = 16, kPipePts = 32;
constexpr int kBlobCap = 32 + 4 * kPipeCams + 4 * (kPipeCams + 1) + 4 * (kPipePts + 1) + 6 * kPipeObs + 16;
constexpr int kBufBlob = 0;
constexpr int kBufPts = (kBlobCap + 15) / 16 * 16;                  // point window (+8 B alignment slack)
constexpr int kBufHinv = kBufPts + (kPipePts * 24 + 16 + 15) / 16 * 16;
constexpr int kBufCam = kBufHinv + kPipePts * 48;                   // camera records, 128 B each
constexpr int kBufVz = kBufCam + kPipeCams * 128;                   // direction (x or z), 48 B each
constexpr int kBufVp = kBufVz + kPipeCams * 48;                     // p (for z + beta p)
constexpr int kBufBytes = kBufVp + kPipeCams * 48;
constexpr int kScrStage = 2 * kBufBytes;                            // stage [6][kPipeObs] doubles
constexpr int kScrTp = kScrStage + 6 * kPipeObs * 8;                // t_p [kPipePts][3]
constexpr int kScrBar = kScrTp + kPipePts * 24;                     // 4 mbarriers
constexpr int kPipeWarpBytes = (kScrBar + 32 + 127) / 128 * 128;
// Warp-tiles per CTA of the pipelined Schur product (k_schur_tiles,
// k_pcg_persistent): two such CTAs fill an SM's shared memory.
constexpr int kSchurWarps = 4;
// Their register cap: no spills (the 128 of two 256-thread CTAs spilled),
// 168 measured fastest (200 and 255 schedule worse: Venice tile pass
// 234 vs 296 us).
constexpr int kSchurMaxReg = 168;

// Programmatic dependent launch: wait until the preceding kernel of the
// stream has completed and its writes are visible (a no-op for a kernel not
// launched with the programmatic attribute).
__device__ __forceinline__ void grid_dep_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_fence_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned parity) {
  unsigned ok = 0;
  long long spins = 0;
  do {
    if (++spins > (1ll << 22)) __trap();  // a lost transaction must fail loudly, never hang
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
  } while (!ok);
}
// TMA bulk copy global -> shared (16 B aligned, size a multiple of 16),
// completion counted on the mbarrier.
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, unsigned long long* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

__device__ __forceinline__ unsigned long long global_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// Packed symmetric storage: 6x6 upper triangle row-major (21), 3x3 (6).
__host__ __device__ constexpr int sym6(int a, int b) {
  return a <= b ? a * 6 - a * (a - 1) / 2 + (b - a) : b * 6 - b * (b - 1) / 2 + (a - b);
}
__host__ __device__ constexpr int sym3(int a, int b) {
  return a <= b ? a * 3 - a * (a - 1) / 2 + (b - a) : b * 3 - b * (b - 1) / 2 + (a - b);
}

// clamp-then-scale damping of one diagonal entry (assemble.hpp:94-101).
__host__ __device__ __forceinline__ double damp_diag(double d, double lambda, double lo, double hi) {
  const double c = d < lo ? lo : (hi < d ? hi : d);
  return c * (1.0 + lambda);
}

// Tile workspace: carved from dynamic shared memory, or from global scratch
// for the rare tile that does not fit (one very long point track).
struct Ws {
  double* cam;
  double* pt;
  double* stage;
  double* piece;
  int* ent;                 // ncam + 1 entry boundaries (tile-local slots)
  int* pptr;                // npts + 1 point-list offsets (tile-local)
  std::uint32_t* lcpt;      // nobs local camera | local point << 16
  std::uint16_t* ptl;       // nobs slots grouped by point
  int* camid;               // ncam global camera ids
};
struct WsDims {
  int camw, ptw, stw, pw;
};
__host__ __device__ __forceinline__ long long ws_bytes(WsDims w, int ncam, int npts, int nobs) {
  const long long nchunk = (nobs + 31) / 32;
  const long long dbl = (long long)ncam * w.camw + (long long)npts * w.ptw + (long long)nobs * w.stw +
                        (nchunk + ncam) * w.pw;
  // ints: ent, pptr, lcpt ; shorts: ptl
  return dbl * 8 + (long long)(ncam + 1) * 4 + (long long)(npts + 1) * 4 + (long long)nobs * 4 +
         ((long long)nobs * 2 + 15) / 16 * 16 + (long long)ncam * 4;
}
// Workspace shapes of the warp-tile kernels (doubles per camera, per point,
// per observation, per piece), kernels.cu:
//   lin (K1): cam [t3 q4 k4 R9] pt p3 stage Jc12 Jp6 r2
//   lin+prep (K1+F1): cam + t3 of the record, pt p3 L6 v3
//   cost (K1c), prep (K3/K4; direct: RHS stage only), Schur product (K5),
//   trial (K7/K8)
// Stage rows of an odd number of doubles: lanes writing consecutive rows hit
// distinct bank pairs (20-double rows put every 4th lane on the same banks).
constexpr int kLinStW = 21;  // Jc12 Jp6 r2 + 1 pad
constexpr int kPrepDirStW = 7;  // RHS piece 6 + 1 pad
constexpr WsDims kLinWs{20, 3, kLinStW, 0};
constexpr WsDims kLinPrepWs{23, 12, kLinStW, 0};
constexpr WsDims kCostWs{11, 3, 0, 0};
constexpr WsDims kPrepWs{16, 12, 27, 0};
constexpr WsDims kPrepDirWs{16, 12, kPrepDirStW, 0};
constexpr WsDims kSxWs{24, 3, 6, 0};
constexpr WsDims kTrialWs{29, 6, 3, 0};
// Workspace bytes of one tile for a kernel kind (WsKind order, kernels.cuh:
// lin, cost, prep, schur, trial, prep-direct, lin+prep).
__host__ __device__ __forceinline__ long long kind_ws_bytes(int kind, int ncam, int npts, int nobs) {
  switch (kind) {
    case 0: return ws_bytes(kLinWs, ncam, npts, nobs);
    case 1: return ws_bytes(kCostWs, ncam, npts, nobs);
    case 2: return ws_bytes(kPrepWs, ncam, npts, nobs);
    case 3: return ws_bytes(kSxWs, ncam, npts, nobs);
    case 4: return ws_bytes(kTrialWs, ncam, npts, nobs);
    case 5: return ws_bytes(kPrepDirWs, ncam, npts, nobs);
    default: return ws_bytes(kLinPrepWs, ncam, npts, nobs);
  }
}
constexpr int kWsKindCount = 7;

__device__ __forceinline__ Ws ws_carve(char* base, WsDims w, int ncam, int npts, int nobs) {
  Ws ws;
  double* d = reinterpret_cast<double*>(base);
  const int nchunk = (nobs + 31) / 32;
  ws.cam = d;
  d += (long long)ncam * w.camw;
  ws.pt = d;
  d += (long long)npts * w.ptw;
  ws.stage = d;
  d += (long long)nobs * w.stw;
  ws.piece = d;
  d += (long long)(nchunk + ncam) * w.pw;
  ws.ent = reinterpret_cast<int*>(d);
  ws.pptr = ws.ent + (ncam + 1);
  ws.lcpt = reinterpret_cast<std::uint32_t*>(ws.pptr + (npts + 1));
  ws.ptl = reinterpret_cast<std::uint16_t*>(ws.lcpt + nobs);
  ws.camid = reinterpret_cast<int*>(reinterpret_cast<char*>(ws.ptl) + ((long long)nobs * 2 + 15) / 16 * 16);
  return ws;
}

struct TileGeom {
  int ob, nobs, pb, npts, eb, ncam, big, trace_id;
};
__device__ __forceinline__ TileGeom tile_geom(const Dev& d, int t) {
  TileGeom g;
  g.ob = d.tile_obs_begin[t];
  g.nobs = d.tile_obs_begin[t + 1] - g.ob;
  g.pb = d.tile_pt_begin[t];
  g.npts = d.tile_pt_begin[t + 1] - g.pb;
  g.eb = d.tile_ent_begin[t];
  g.ncam = d.tile_ent_begin[t + 1] - g.eb;
  g.big = d.tile_ws[t];
  g.trace_id = t;
  return g;
}

// L2 prefetch of a byte range (TMA bulk prefetch, 16-byte granules): the
// inputs of a tile that runs about one resident wave later, so that its
// warp's dependent index / field loads hit L2 instead of HBM.
__device__ __forceinline__ void l2_prefetch(const void* p, long long bytes) {
  if (bytes <= 0) return;
  const unsigned long long a = reinterpret_cast<unsigned long long>(p) & ~15ull;
  const unsigned long long e = (reinterpret_cast<unsigned long long>(p) + bytes + 15) & ~15ull;
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(a), "r"(static_cast<unsigned>(e - a)) : "memory");
}
struct TileSpan {
  int ob, oe, pb, pe, eb, ee;
};
// Geometry of tile tn (empty past the last tile); loaded early, used late.
__device__ __forceinline__ TileSpan tile_span(const Dev& d, int tn) {
  TileSpan q{0, 0, 0, 0, 0, 0};
  if (tn < d.T) {
    q.ob = d.tile_obs_begin[tn];
    q.oe = d.tile_obs_begin[tn + 1];
    q.pb = d.tile_pt_begin[tn];
    q.pe = d.tile_pt_begin[tn + 1];
    q.eb = d.tile_ent_begin[tn];
    q.ee = d.tile_ent_begin[tn + 1];
  }
  return q;
}
// The index arrays, pixels and point coordinates of a tile, plus up to two
// per-point arrays of w doubles (e.g. g_p and H~_pp^-1 for the trial pass).
__device__ __forceinline__ void prefetch_tile(const Dev& d, const TileSpan& q, const double* pa = nullptr, int wa = 0,
                                              const double* pb = nullptr, int wb = 0) {
  if (q.oe <= q.ob) return;
  const long long no = q.oe - q.ob, np = q.pe - q.pb, ne = q.ee - q.eb;
  l2_prefetch(d.obs_lcpt + q.ob, no * 4);
  l2_prefetch(d.ptobs + q.ob, no * 2);
  l2_prefetch(d.obs_px + 2LL * q.ob, no * 16);
  l2_prefetch(d.pt_ptr + q.pb, (np + 1) * 4);
  l2_prefetch(d.pts + 3LL * q.pb, np * 24);
  l2_prefetch(d.ent_obs_begin + q.eb, (ne + 1) * 4);
  l2_prefetch(d.ent_cam + q.eb, ne * 4);
  if (pa) l2_prefetch(pa + (long long)wa * q.pb, np * wa * 8);
  if (pb) l2_prefetch(pb + (long long)wb * q.pb, np * wb * 8);
}

// Warp-level segmented reduction over 32 consecutive tile slots. Segments
// are contiguous runs of equal `seg` (the local camera); the head lane of each
// run ends up with the run's sum and stores it as a "piece": lane 0 into its
// chunk slot, any other head into the slot of its camera. The tree shape
// depends only on the segment boundaries, so the result is deterministic.
template <int W>
__device__ __forceinline__ void seg_reduce_pieces(double (&v)[W], int seg, int slot, int nchunk, double* piece) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    const int os = __shfl_down_sync(0xffffffffu, seg, off);
    const bool take = (lane + off < 32) && (os == seg);
#pragma unroll
    for (int j = 0; j < W; ++j) {
      const double o = __shfl_down_sync(0xffffffffu, v[j], off);
      if (take) v[j] += o;
    }
  }
  const int ps = __shfl_up_sync(0xffffffffu, seg, 1);
  if (seg >= 0 && (lane == 0 || ps != seg)) {
    const int at = (lane == 0) ? (slot >> 5) : (nchunk + seg);
#pragma unroll
    for (int j = 0; j < W; ++j) piece[at * W + j] = v[j];
  }
}

// Combine the pieces of every tile camera in slot order and write the
// per-entry partial sums (W doubles per entry).
template <int W>
__device__ __forceinline__ void entries_from_pieces(const Ws& ws, int ncam, int nobs, int eb, double* out) {
  const int nchunk = (nobs + 31) / 32;
  for (int idx = threadIdx.x; idx < ncam * W; idx += blockDim.x) {
    const int e = idx / W, j = idx - e * W;
    const int b = ws.ent[e], en = ws.ent[e + 1];
    double acc = 0.0;
    int m = b >> 5;
    if (b & 31) {
      acc = ws.piece[(nchunk + e) * W + j];
      ++m;
    }
    for (; (m << 5) < en; ++m) acc += ws.piece[m * W + j];
    out[(long long)(eb + e) * W + j] = acc;
  }
}

// Fixed-order block sum of one double per thread (result valid in thread 0).
__device__ __forceinline__ double block_sum(double v, double* scratch) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
  __syncthreads();
  if (lane == 0) scratch[warp] = v;
  __syncthreads();
  double s = 0.0;
  if (threadIdx.x == 0) {
    const int nw = (blockDim.x + 31) >> 5;
    for (int i = 0; i < nw; ++i) s += scratch[i];
  }
  return s;
}

// Last-block-done grid reduction of K doubles per block. Every block calls it
// with its block totals (thread 0's vals); returns true in the last block,
// whose thread 0 receives the grid totals summed in block order.
template <int K>
__device__ __forceinline__ bool grid_reduce(const double (&vals)[K], double* scratch, unsigned* ticket,
                                            double (&tot)[K]) {
  __shared__ bool last;
  if (threadIdx.x == 0) {
#pragma unroll
    for (int k = 0; k < K; ++k) scratch[(long long)blockIdx.x * K + k] = vals[k];
    __threadfence();
    const unsigned t = atomicAdd(ticket, 1u);
    last = (t == gridDim.x - 1);
  }
  __syncthreads();
  if (!last) return false;
  __threadfence();
  if (threadIdx.x == 0) {
#pragma unroll
    for (int k = 0; k < K; ++k) tot[k] = 0.0;
    for (unsigned b = 0; b < gridDim.x; ++b)
#pragma unroll
      for (int k = 0; k < K; ++k) tot[k] += ((volatile double*)scratch)[(long long)b * K + k];
    *ticket = 0u;
  }
  return true;
}

// Cholesky-based inverse of a packed symmetric n x n matrix (n = 3 or 6).
// Returns false unless every pivot is positive and finite (NotSpdError,
// cholesky.hpp:229).
template <int n>
__host__ __device__ __forceinline__ bool spd_inverse(const double* a, double* inv_full) {
  double l[n][n];
#pragma unroll
  for (int i = 0; i < n; ++i)
#pragma unroll
    for (int j = 0; j < n; ++j) l[i][j] = 0.0;
#pragma unroll
  for (int j = 0; j < n; ++j) {
    double dsum = (n == 6) ? a[sym6(j, j)] : a[sym3(j, j)];
#pragma unroll
    for (int k = 0; k < j; ++k) dsum -= l[j][k] * l[j][k];
    if (!(dsum > 0.0) || !isfinite(dsum)) return false;
    const double ljj = sqrt(dsum);
    l[j][j] = ljj;
    const double il = 1.0 / ljj;
#pragma unroll
    for (int i = j + 1; i < n; ++i) {
      double s = (n == 6) ? a[sym6(i, j)] : a[sym3(i, j)];
#pragma unroll
      for (int k = 0; k < j; ++k) s -= l[i][k] * l[j][k];
      l[i][j] = s * il;
    }
  }
  // M = L^-1 (lower triangular)
  double m[n][n];
#pragma unroll
  for (int i = 0; i < n; ++i) {
#pragma unroll
    for (int j = 0; j < n; ++j) m[i][j] = 0.0;
    m[i][i] = 1.0 / l[i][i];
#pragma unroll
    for (int j = 0; j < i; ++j) {
      double s = 0.0;
#pragma unroll
      for (int k = j; k < i; ++k) s += l[i][k] * m[k][j];
      m[i][j] = -s * m[i][i];
    }
  }
  // A^-1 = M^T M
#pragma unroll
  for (int i = 0; i < n; ++i)
#pragma unroll
    for (int j = i; j < n; ++j) {
      double s = 0.0;
#pragma unroll
      for (int k = j; k < n; ++k) s += m[k][i] * m[k][j];
      inv_full[i * n + j] = s;
      inv_full[j * n + i] = s;
    }
  return true;
}

}  // namespace bae
