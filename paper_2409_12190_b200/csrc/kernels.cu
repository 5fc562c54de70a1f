// sm_100a kernels of the BA hot path. FP64 throughout (the reference is FP64,
// SPEC.md:332). All sums are deterministic: fixed-order staged reductions and
// fixed shuffle trees, no floating-point atomics.
//
// Work decomposition. A tile (Plan, bae_internal.hpp) is a run of points and
// their observations, processed by ONE WARP with its own shared-memory
// workspace slice; a CTA hosts several independent warp-tiles. Phases inside a
// tile are separated by __syncwarp only, so a tile never waits on another
// tile, and a tile's global loads are issued in batches (one memory latency
// per dependent stage).
//
// Per-observation algebra (one observation k, camera c, point p, camera-frame
// point y = R p + t, D = d(pixel)/d(y) from camera.hpp:59-71):
//   J_c = D [I | -[y]x]   (2x6, trace.hpp:612-629: up * [I | -skew(y)])
//   J_p = D R             (2x3, trace.hpp:612-629: up * R)
//   J_c v   = D (v_rho + v_omega x y)         J_c^T e = [g ; y x g], g = D^T e
//   J_p t   = D (R t)                         J_p^T u = R^T (D^T u)
#include <cfloat>
#include <climits>
#include <cstdlib>
#include <string>

#include <cooperative_groups.h>

#include "device.cuh"
#include "kernels.cuh"

namespace bae {

// ---------------------------------------------------------------------------
// per-observation math
// ---------------------------------------------------------------------------

// y = R p + t and D for one observation from a camera record
// (R[9] t[3] intrinsics[4]).
__device__ __forceinline__ void obs_geometry(bool pin, const double* cam, const double* pt, P3& y, double* D) {
  const double* R = cam;
  y.x = R[0] * pt[0] + R[1] * pt[1] + R[2] * pt[2] + cam[9];
  y.y = R[3] * pt[0] + R[4] * pt[1] + R[5] * pt[2] + cam[10];
  y.z = R[6] * pt[0] + R[7] * pt[1] + R[8] * pt[2] + cam[11];
  cam_dproj(pin, y, cam + 12, D);
}

// J_c = D [I | -[y]x] (trace.hpp:612-629 with up = D), row-major 2x6.
__device__ __forceinline__ void jac_cam(const double* D, const P3& y, double* Jc) {
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    const double d0 = D[i * 3], d1 = D[i * 3 + 1], d2 = D[i * 3 + 2];
    Jc[i * 6 + 0] = d0;
    Jc[i * 6 + 1] = d1;
    Jc[i * 6 + 2] = d2;
    Jc[i * 6 + 3] = d1 * (-y.z) + d2 * y.y;
    Jc[i * 6 + 4] = d0 * y.z + d2 * (-y.x);
    Jc[i * 6 + 5] = d0 * (-y.y) + d1 * y.x;
  }
}

// J_p = D R, row-major 2x3.
__device__ __forceinline__ void jac_pt(const double* D, const double* R, double* Jp) {
#pragma unroll
  for (int i = 0; i < 2; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j) Jp[i * 3 + j] = D[i * 3] * R[j] + D[i * 3 + 1] * R[3 + j] + D[i * 3 + 2] * R[6 + j];
}

// s = J_p^T J_c v  (3-vector) using the factored forms.
__device__ __forceinline__ void jpt_jc_v(const double* D, const P3& y, const double* R, const double* v, double* s) {
  const double ax = v[0] + (v[4] * y.z - v[5] * y.y);
  const double ay = v[1] + (v[5] * y.x - v[3] * y.z);
  const double az = v[2] + (v[3] * y.y - v[4] * y.x);
  const double u0 = D[0] * ax + D[1] * ay + D[2] * az;
  const double u1 = D[3] * ax + D[4] * ay + D[5] * az;
  const double g0 = D[0] * u0 + D[3] * u1;
  const double g1 = D[1] * u0 + D[4] * u1;
  const double g2 = D[2] * u0 + D[5] * u1;
  s[0] = R[0] * g0 + R[3] * g1 + R[6] * g2;
  s[1] = R[1] * g0 + R[4] * g1 + R[7] * g2;
  s[2] = R[2] * g0 + R[5] * g1 + R[8] * g2;
}

// z = J_c^T J_p t  (6-vector).
__device__ __forceinline__ void jct_jp_t(const double* D, const P3& y, const double* R, const double* t, double* z) {
  const double rt0 = R[0] * t[0] + R[1] * t[1] + R[2] * t[2];
  const double rt1 = R[3] * t[0] + R[4] * t[1] + R[5] * t[2];
  const double rt2 = R[6] * t[0] + R[7] * t[1] + R[8] * t[2];
  const double e0 = D[0] * rt0 + D[1] * rt1 + D[2] * rt2;
  const double e1 = D[3] * rt0 + D[4] * rt1 + D[5] * rt2;
  const double g0 = D[0] * e0 + D[3] * e1;
  const double g1 = D[1] * e0 + D[4] * e1;
  const double g2 = D[2] * e0 + D[5] * e1;
  z[0] = g0;
  z[1] = g1;
  z[2] = g2;
  z[3] = y.y * g2 - y.z * g1;
  z[4] = y.z * g0 - y.x * g2;
  z[5] = y.x * g1 - y.y * g0;
}

// Forward residual exactly as the reference evaluates it: quaternion rotate
// (trace.hpp:439-452, lie.hpp:88-93), bal_project_cam / pinhole_project_cam
// (camera.hpp:33-57), sub as p0 + (-1) p1 (trace.hpp:488-497).
// cam: [t3 q4 intrinsics4].
__device__ __forceinline__ bool residual(bool pin, const double* cam, const double* pt, double2 px, double& r0,
                                         double& r1, P3& y) {
  const P3 yr = quat_rotate({cam[3], cam[4], cam[5], cam[6]}, {pt[0], pt[1], pt[2]});
  y = {yr.x + cam[0], yr.y + cam[1], yr.z + cam[2]};
  double u, w;
  if (!cam_project(pin, y, cam + 7, u, w)) return false;
  r0 = u + -1.0 * px.x;
  r1 = w + -1.0 * px.y;
  return true;
}

// ---------------------------------------------------------------------------
// warp-tile infrastructure
// ---------------------------------------------------------------------------

__device__ __forceinline__ int lane_id() { return threadIdx.x & 31; }

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
  return v;
}

// Batched warp copy global -> workspace: each lane issues up to kBatch
// independent loads before its first store; loads past the end are
// predicated off (no duplicate requests for short arrays).
// `addr(i)` returns the source address of element i.
constexpr int kBatch = 8;
// The tile's thread index in a group of NT threads (a warp, or the warp pair
// of the linearisation: kLinThreads).
template <int NT>
__device__ __forceinline__ int tile_tid() {
  return static_cast<int>(threadIdx.x) & (NT - 1);
}
template <int NT, class T, class Addr, class Store>
__device__ __forceinline__ void group_copy(int n, Addr addr, Store store) {
  for (int base = tile_tid<NT>(); base < n; base += kBatch * NT) {
    T v[kBatch];
#pragma unroll
    for (int b = 0; b < kBatch; ++b)
      if (base + b * NT < n) v[b] = *addr(base + b * NT);
#pragma unroll
    for (int b = 0; b < kBatch; ++b)
      if (base + b * NT < n) store(base + b * NT, v[b]);
  }
}
template <class T, class Addr, class Store>
__device__ __forceinline__ void warp_copy(int n, Addr addr, Store store) {
  group_copy<32, T>(n, addr, store);
}

// Tile index data: entry boundaries, camera ids, point-list offsets, slot
// camera/point codes and the point lists (all independent loads).
template <int NT = 32>
__device__ __forceinline__ void load_tile_index(const Dev& d, const TileGeom& g, const Ws& ws) {
  const int* eo = d.ent_obs_begin + g.eb;
  const int* ec = d.ent_cam + g.eb;
  const int* pp = d.pt_ptr + g.pb;
  const std::uint32_t* lc = d.obs_lcpt + g.ob;
  const std::uint16_t* pl = d.ptobs + g.ob;
  group_copy<NT, int>(g.ncam + 1, [&](int i) { return eo + i; }, [&](int i, int v) { ws.ent[i] = v - g.ob; });
  group_copy<NT, int>(g.ncam, [&](int i) { return ec + i; }, [&](int i, int v) { ws.camid[i] = v; });
  group_copy<NT, int>(g.npts + 1, [&](int i) { return pp + i; }, [&](int i, int v) { ws.pptr[i] = v - g.ob; });
  group_copy<NT, std::uint32_t>(g.nobs, [&](int i) { return lc + i; },
                                [&](int i, std::uint32_t v) { ws.lcpt[i] = v; });
  group_copy<NT, std::uint16_t>(g.nobs, [&](int i) { return pl + i; },
                                [&](int i, std::uint16_t v) { ws.ptl[i] = v; });
}

// W consecutive doubles per point from src[(pb + lp) * W] into ws.pt[lp * ptw + off]
// (kSoA: into ws.pt[(off + k) * npts + lp], see pt_get).
template <int W, int NT = 32, bool kSoA = false>
__device__ __forceinline__ void load_point_fields(const Ws& ws, int ptw, int off, const double* src, int pb,
                                                  int npts) {
  const double* base = src + (long long)pb * W;
  group_copy<NT, double>(
      npts * W, [&](int i) { return base + i; },
      [&](int i, double v) {
        const int lp = i / W;
        if (kSoA)
          ws.pt[(off + i - lp * W) * npts + lp] = v;
        else
          ws.pt[lp * ptw + off + (i - lp * W)] = v;
      });
}

// Structure-of-arrays point area (the 12-double prep rows): field c of local
// point lp at ws.pt[c * npts + lp], so lanes on consecutive points touch
// consecutive bank pairs (12-double rows put every 4th point on one bank).
template <int K>
__device__ __forceinline__ void pt_get(const Ws& ws, int npts, int lp, int c0, double* out) {
#pragma unroll
  for (int k = 0; k < K; ++k) out[k] = ws.pt[(c0 + k) * npts + lp];
}
template <int K>
__device__ __forceinline__ void pt_put(const Ws& ws, int npts, int lp, int c0, const double* in) {
#pragma unroll
  for (int k = 0; k < K; ++k) ws.pt[(c0 + k) * npts + lp] = in[k];
}

// W consecutive doubles per camera from src[camid * stride] into
// ws.cam[l * camw + off]. Needs ws.camid (load_tile_index + a tile barrier).
template <int W, int NT = 32>
__device__ __forceinline__ void load_cam_fields(const Ws& ws, int ncam, int camw, int off, const double* src,
                                                int stride) {
  group_copy<NT, double>(
      ncam * W,
      [&](int i) {
        const int l = i / W;
        return src + (long long)ws.camid[l] * stride + (i - l * W);
      },
      [&](int i, double v) {
        const int l = i / W;
        ws.cam[l * camw + off + (i - l * W)] = v;
      });
}

// Per (tile camera, component): sum of the staged W-vectors over the
// camera's slot range, in slot order (two interleaved partial sums).
template <int W, int SW, int NT = 32>
__device__ __forceinline__ void entries_from_stage(const Ws& ws, int ncam, int eb, double* out) {
  for (int idx = tile_tid<NT>(); idx < ncam * W; idx += NT) {
    const int e = idx / W, j = idx - e * W;
    const int b = ws.ent[e], en = ws.ent[e + 1];
    double a0 = 0.0, a1 = 0.0;
    int q = b;
    for (; q + 1 < en; q += 2) {
      a0 += ws.stage[q * SW + j];
      a1 += ws.stage[(q + 1) * SW + j];
    }
    if (q < en) a0 += ws.stage[q * SW + j];
    out[(long long)(eb + e) * W + j] = a0 + a1;
  }
}

// Workspace base of a tile: this warp's slice of dynamic shared memory, or a
// global slot for the rare tile that does not fit (one very long track).
// kShared is a compile-time constant so the compiler emits LDS/STS.
template <bool kShared>
__device__ __forceinline__ char* ws_base(const Dev& d, const TileGeom& g, char* smem, int slice) {
  return kShared ? smem + (threadIdx.x >> 5) * slice : d.bigws + (long long)g.big * d.big_stride;
}

// Dispatch one warp-tile body on shared or global workspace.
#define BAE_TILE_DISPATCH(body, ...) \
  do {                               \
    if (g.big >= 0)                  \
      body<false>(__VA_ARGS__);      \
    else                             \
      body<true>(__VA_ARGS__);       \
  } while (0)

// ---------------------------------------------------------------------------
// K-rec: camera records (R from the quaternion, lie.hpp:68-70) after any
// pose update.
// ---------------------------------------------------------------------------
__global__ void k_camrec(const double* __restrict__ pose, const double* __restrict__ intr, double* __restrict__ rec,
                         int C) {
  grid_dep_wait();
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= C) return;
  const double* s = pose + (long long)c * 7;
  double* o = rec + (long long)c * kCamRec;
  quat_to_R({s[3], s[4], s[5], s[6]}, o);
  o[9] = s[0];
  o[10] = s[1];
  o[11] = s[2];
  o[12] = intr[c * 4];
  o[13] = intr[c * 4 + 1];
  o[14] = intr[c * 4 + 2];
  o[15] = intr[c * 4 + 3];
}

// Direct solver, per observation slot: V = W L^-T is 6 x 3, but W = J_c^T J_p
// = [M; [y]x M] (J_c = D [I | -[y]x], M = D^T J_p), so V = [Q; [y]x Q] with
// Q = M L^-T: the record keeps Q (row-major 9) and the camera-frame point y
// (3): 96 bytes, three whole 32-byte sectors, instead of 144 (160 aligned).
constexpr int kVStride = 12;
// Direct solver prep, shared by k_prep<true> and the fused k_lin_prep (one
// copy of the arithmetic, so the two agree bit for bit).
// Per point: damped H~_pp, its inverse (d.hinv, for the
// back-substitution), its Cholesky factor L (1/l00, l10, l20, 1/l11, l21,
// 1/l22) into sp[3..8] and v = H~_pp^-1 g_p into sp[9..11]. h: the packed
// H_pp (6), g: g_p (3). Returns false when the damped block is not SPD.
__device__ __forceinline__ bool prep_point_direct(const Dev& d, long long ip, double (&h)[6], const double* g,
                                                  double lambda, double clo, double chi, double* sp) {
  double inv[9];
  h[0] = damp_diag(h[0], lambda, clo, chi);
  h[3] = damp_diag(h[3], lambda, clo, chi);
  h[5] = damp_diag(h[5], lambda, clo, chi);
  const bool pfail = !spd_inverse<3>(h, inv);
  if (pfail) {
#pragma unroll
    for (int j = 0; j < 9; ++j) inv[j] = 0.0;
  }
  const double hi[6] = {inv[0], inv[1], inv[2], inv[4], inv[5], inv[8]};
#pragma unroll
  for (int j = 0; j < 6; ++j) d.hinv[ip * 6 + j] = hi[j];
  double lf[6] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
  if (!pfail) {
    const double l00 = sqrt(h[0]), l10 = h[1] / l00, l20 = h[2] / l00;
    const double l11 = sqrt(h[3] - l10 * l10), l21 = (h[4] - l20 * l10) / l11;
    const double l22 = sqrt(h[5] - l20 * l20 - l21 * l21);
    lf[0] = 1.0 / l00;
    lf[1] = l10;
    lf[2] = l20;
    lf[3] = 1.0 / l11;
    lf[4] = l21;
    lf[5] = 1.0 / l22;
  }
#pragma unroll
  for (int j = 0; j < 6; ++j) sp[3 + j] = lf[j];
  sp[9] = inv[0] * g[0] + inv[1] * g[1] + inv[2] * g[2];
  sp[10] = inv[3] * g[0] + inv[4] * g[1] + inv[5] * g[2];
  sp[11] = inv[6] * g[0] + inv[7] * g[1] + inv[8] * g[2];
  return !pfail;
}

// Direct solver, per observation slot: the compact V record [Q | y] (see
// kVStride) and the Schur right-hand side piece W v into rhs[0..5].
__device__ __forceinline__ void prep_obs_direct(const Dev& d, long long slot, const double (&W)[18], const P3& y,
                                                const double* sp, double* rhs) {
  const double* lf = sp + 3;
  double vv[kVStride];
#pragma unroll
  for (int a = 0; a < 3; ++a) {  // rows of Q = M L^-T (M = the top half of W)
    const double v0 = W[a * 3] * lf[0];
    const double v1 = (W[a * 3 + 1] - lf[1] * v0) * lf[3];
    const double v2 = (W[a * 3 + 2] - lf[2] * v0 - lf[4] * v1) * lf[5];
    vv[a * 3] = v0;
    vv[a * 3 + 1] = v1;
    vv[a * 3 + 2] = v2;
  }
  vv[9] = y.x;
  vv[10] = y.y;
  vv[11] = y.z;
  double* vo = d.wstore + slot * kVStride;
#pragma unroll
  for (int j = 0; j < kVStride / 4; ++j)  // whole 32-byte sectors per store
    asm volatile("st.global.v4.f64 [%0], {%1, %2, %3, %4};" ::"l"(vo + 4 * j), "d"(vv[4 * j]), "d"(vv[4 * j + 1]),
                 "d"(vv[4 * j + 2]), "d"(vv[4 * j + 3])
                 : "memory");
  const double* vp = sp + 9;
#pragma unroll
  for (int a = 0; a < 6; ++a) rhs[a] = W[a * 3] * vp[0] + W[a * 3 + 1] * vp[1] + W[a * 3 + 2] * vp[2];
}

// ---------------------------------------------------------------------------
// K1: fused residual + Jacobian + block reductions (the linearisation).
// Replaces evaluate + sparse_jacobian + the CC/LL SpGEMM quadrants and the
// b = -J^T r SpMVs (trace.hpp:412-806, assemble.hpp:61-84).
//   per point : H_pp (6), g_p (3)          -> hpp, gp
//   per entry : H_cc (21), g_c (6) partial -> partial[e][27]
//   per tile  : sum r^2, sum |g_p|^2       -> tile_red
// The forward residual follows the reference (quaternion rotate); its
// Jacobian uses that forward value y (trace.hpp:612-629).
// cam: [t3 q4 k4 R9] (20) ; pt: p3 ; stage: Jc12 Jp6 r2 (20)
// ---------------------------------------------------------------------------
// fused with the direct prep: camera + t3 of the record, point p3 L6 v3

// kPrep: the direct solver's prep fused in (accepted LM steps: linearise and
// damp in one pass over the tile's data): the point side goes on to the
// damped point block and its factor, each observation to V and its
// right-hand side piece (entries into d.partial6). W comes from the camera
// record's R, t exactly as k_prep forms it, so the fused and the separate
// prep agree bit for bit.
//
// A tile is worked by a warp pair (kLinThreads threads on one workspace
// slice, synchronised by the pair's named barrier): twice the resident warps
// of a warp per tile for the same shared memory. Every per-observation,
// per-point and per-entry result keeps its order (an entry's or a point's
// sum runs on one thread), and the tile totals are SplitSums, so the group
// size does not change a bit.
// k_lin_prep runs warp pairs (kLinThreads); k_linearize, with its smaller
// workspace, is faster with a warp per tile (NT = 32).
// Tile cost / |g|^2 totals in one order for every group size: item i goes to
// partial (i & 32) of its lane, each partial takes the warp's fixed tree,
// total = tree(even runs) + tree(odd runs). A warp pair's thread sees items
// of one parity only, so its warp totals are the two trees.
struct SplitSum {
  double a = 0.0, b = 0.0;
  __device__ __forceinline__ void add(int i, double v) {
    if (i & 32)
      b += v;
    else
      a += v;
  }
  __device__ __forceinline__ double warp_total() const { return warp_sum(a) + warp_sum(b); }
};
constexpr int kLinThreads = 64;
template <int NT>
__device__ __forceinline__ void tile_sync() {
  if constexpr (NT == 32)
    __syncwarp();
  else
    asm volatile("bar.sync %0, %1;" ::"r"(1 + static_cast<int>(threadIdx.x) / NT), "n"(NT) : "memory");
}
template <int NT>
__device__ __forceinline__ int group_tile_index() {
  return blockIdx.x * (blockDim.x / NT) + threadIdx.x / NT;
}

template <bool kShared, bool kPrep, int NT>
__device__ __forceinline__ void lin_tile(const Dev& d, const TileGeom& g, char* smem, int slice, int t,
                                         int write_jac, double clo = 0.0, double chi = 0.0) {
  constexpr int kPtw = kPrep ? 12 : 3, kCw = kPrep ? 23 : 20;
  char* base = kShared ? smem + (threadIdx.x / NT) * slice : d.bigws + (long long)g.big * d.big_stride;
  const Ws ws = ws_carve(base, kPrep ? kLinPrepWs : kLinWs, g.ncam, g.npts, g.nobs);
  const int tt = tile_tid<NT>(), lane = tt & 31, wp = tt >> 5;
  load_point_fields<3, NT, kPrep>(ws, kPtw, 0, d.pts, g.pb, g.npts);
  load_tile_index<NT>(d, g, ws);
  tile_sync<NT>();
  load_cam_fields<7, NT>(ws, g.ncam, kCw, 0, d.pose, 7);
  load_cam_fields<4, NT>(ws, g.ncam, kCw, 7, d.intr, 4);
  load_cam_fields<kPrep ? 12 : 9, NT>(ws, g.ncam, kCw, 11, d.camrec, kCamRec);
  tile_sync<NT>();
  SplitSum cost;
  int bad = INT_MAX;
  for (int s = tt; s < g.nobs; s += NT) {
    const std::uint32_t lcpt = ws.lcpt[s];
    const double* cam = ws.cam + (lcpt & 0xffff) * kCw;
    double pv[3];
    const double* pt = pv;
    if constexpr (kPrep)
      pt_get<3>(ws, g.npts, lcpt >> 16, 0, pv);
    else
      pt = ws.pt + (lcpt >> 16) * kPtw;
    const double2 px = reinterpret_cast<const double2*>(d.obs_px)[g.ob + s];
    double* st = ws.stage + s * kLinStW;
    double r0 = 0.0, r1 = 0.0;
    P3 y;
    if (residual(d.pinhole, cam, pt, px, r0, r1, y)) {
      double D[6];
      cam_dproj(d.pinhole, y, cam + 7, D);
      jac_cam(D, y, st);
      jac_pt(D, cam + 11, st + 12);
      st[18] = r0;
      st[19] = r1;
      cost.add(s, r0 * r0 + r1 * r1);
      if (write_jac && d.jstore) {
        const long long gs = g.ob + s;
#pragma unroll
        for (int j = 0; j < 18; ++j) d.jstore[(long long)j * d.N + gs] = st[j];
      }
      if (d.resid) {
        d.resid[g.ob + s] = r0;
        d.resid[(long long)d.N + g.ob + s] = r1;
      }
    } else {
      bad = min(bad, d.obs_orig[g.ob + s]);
#pragma unroll
      for (int j = 0; j < 20; ++j) st[j] = 0.0;
    }
  }
  if (bad != INT_MAX) atomicMin(&d.lm->err_obs, bad);
  tile_sync<NT>();
  // camera side: lane j < 27 of each warp owns component j (the H_cc upper
  // triangle row-major, then g_c) of the entries e = wp, wp + 2, ... (no
  // per-lane trip counts, no index decoding). Per component:
  // st[a] st[b0] + st[6 + a] st[b1] over the entry's observations in order.
  {
    const int j = min(lane, 26);
    int a = j - 21, b0 = 18, b1 = 19;  // g_c: J_c^T r
    if (j < 21) {
      a = 0;
      int rem = j;
#pragma unroll
      for (int r = 0; r < 5; ++r)
        if (rem >= 6 - a) {
          rem -= 6 - a;
          ++a;
        }
      b0 = a + rem;
      b1 = 6 + b0;
    }
    for (int e = wp; e < g.ncam; e += NT / 32) {
      const int qb = ws.ent[e], qe = ws.ent[e + 1];
      const double* st = ws.stage + qb * kLinStW;
      double acc0 = 0.0, acc1 = 0.0;  // two interleaved partial sums, slot order
      int q = qb;
      for (; q + 1 < qe; q += 2, st += 2 * kLinStW) {
        acc0 += st[a] * st[b0] + st[6 + a] * st[b1];
        acc1 += st[kLinStW + a] * st[kLinStW + b0] + st[kLinStW + 6 + a] * st[kLinStW + b1];
      }
      if (q < qe) acc0 += st[a] * st[b0] + st[6 + a] * st[b1];
      if (lane < 27) d.partial[(long long)(g.eb + e) * 27 + lane] = acc0 + acc1;
    }
  }
  // point side: H_pp (6) and g_p (3) per point, observations in id order
  SplitSum gsq;
  int pfail = 0;
  for (int lp = tt; lp < g.npts; lp += NT) {
    double h[9];
#pragma unroll
    for (int j = 0; j < 9; ++j) h[j] = 0.0;
    for (int q = ws.pptr[lp]; q < ws.pptr[lp + 1]; ++q) {
      const double* st = ws.stage + ws.ptl[q] * kLinStW;
      const double* jp = st + 12;
      int k = 0;
#pragma unroll
      for (int a = 0; a < 3; ++a)
#pragma unroll
        for (int b = a; b < 3; ++b) h[k++] += jp[a] * jp[b] + jp[3 + a] * jp[3 + b];
#pragma unroll
      for (int a = 0; a < 3; ++a) h[6 + a] += jp[a] * st[18] + jp[3 + a] * st[19];
    }
    const long long ip = g.pb + lp;
#pragma unroll
    for (int j = 0; j < 6; ++j) d.hpp[ip * 6 + j] = h[j];
#pragma unroll
    for (int j = 0; j < 3; ++j) d.gp[ip * 3 + j] = h[6 + j];
    gsq.add(lp, h[6] * h[6] + h[7] * h[7] + h[8] * h[8]);
    if (kPrep) {
      double h6[6] = {h[0], h[1], h[2], h[3], h[4], h[5]};
      double spl[12];
      if (!prep_point_direct(d, ip, h6, h + 6, *d.lam, clo, chi, spl)) pfail = 1;
      pt_put<9>(ws, g.npts, lp, 3, spl + 3);
    }
  }
  // tile totals (tile_red): a warp pair adds warp 1's trees to warp 0's
  const double ct = cost.warp_total(), gt = gsq.warp_total();
  if constexpr (NT == 32) {
    if (lane == 0) {
      d.tile_red[t * 2] = ct;
      d.tile_red[t * 2 + 1] = gt;
    }
  } else {
    static_assert(NT == 64, "warp or warp pair");
    // warp 1's trees reach warp 0 through shared memory (a global round trip
    // here stalled warp 0, and with it the pair's next barrier, ~500 cycles)
    __shared__ double pair_red[8][2];  // at most eight pairs per CTA (TileLaunch::wpb)
    double* pr = pair_red[(threadIdx.x / NT) & 7];
    if (wp == 1 && lane == 0) {
      pr[0] = ct;
      pr[1] = gt;
    }
    tile_sync<NT>();
    if (wp == 0 && lane == 0) {
      d.tile_red[t * 2] = ct + pr[0];
      d.tile_red[t * 2 + 1] = gt + pr[1];
    }
  }
  if (kPrep) {
    if (pfail) atomicExch(&d.pcg->not_spd, 1);
    tile_sync<NT>();
    for (int s = tt; s < g.nobs; s += NT) {  // V and the right-hand side pieces
      const std::uint32_t lcpt = ws.lcpt[s];
      const double* cam = ws.cam + (lcpt & 0xffff) * kCw;
      const double* R = cam + 11;  // record R9 t3; intrinsics at cam + 7
      double sp[12];
      pt_get<12>(ws, g.npts, lcpt >> 16, 0, sp);
      P3 y;
      y.x = R[0] * sp[0] + R[1] * sp[1] + R[2] * sp[2] + R[9];
      y.y = R[3] * sp[0] + R[4] * sp[1] + R[5] * sp[2] + R[10];
      y.z = R[6] * sp[0] + R[7] * sp[1] + R[8] * sp[2] + R[11];
      double D[6], Jc[12], Jp[6];
      cam_dproj(d.pinhole, y, cam + 7, D);
      jac_cam(D, y, Jc);
      jac_pt(D, R, Jp);
      double W[18];
#pragma unroll
      for (int a = 0; a < 6; ++a)
#pragma unroll
        for (int j = 0; j < 3; ++j) W[a * 3 + j] = Jc[a] * Jp[j] + Jc[6 + a] * Jp[3 + j];
      double rhs[6];
      prep_obs_direct(d, g.ob + s, W, y, sp, rhs);
      double* st = ws.stage + s * kLinStW;
#pragma unroll
      for (int a = 0; a < 6; ++a) st[a] = rhs[a];
    }
    tile_sync<NT>();
    entries_from_stage<6, kLinStW, NT>(ws, g.ncam, g.eb, d.partial6);
  }
  tile_sync<NT>();
}

// 96 registers: two CTAs of up to 10 warps (5 pairs, the Final-13682 slice)
// per SM; 98 (rounded to 104) left one.
__global__ void __maxnreg__(96) k_lin_prep(Dev d, int slice, double clo, double chi, int pf) {
  grid_dep_wait();
  extern __shared__ __align__(16) char smem[];
  const int t = group_tile_index<kLinThreads>();
  if (t >= d.T) return;
  const bool lead = threadIdx.x % kLinThreads == 0;
  const TileSpan nx = pf > 0 && lead ? tile_span(d, t + pf) : TileSpan{0, 0, 0, 0, 0, 0};
  const TileGeom g = tile_geom(d, t);
  if (lead) prefetch_tile(d, nx);  // one wave ahead
  if (g.big >= 0)
    lin_tile<false, true, kLinThreads>(d, g, smem, slice, t, 0, clo, chi);
  else
    lin_tile<true, true, kLinThreads>(d, g, smem, slice, t, 0, clo, chi);
}

__global__ void __launch_bounds__(256) k_linearize(Dev d, int slice, int write_jac, int pf) {
  grid_dep_wait();
  extern __shared__ __align__(16) char smem[];
  const int t = group_tile_index<32>();
  if (t >= d.T) return;
  const TileSpan nx = pf > 0 && lane_id() == 0 ? tile_span(d, t + pf) : TileSpan{0, 0, 0, 0, 0, 0};
  const TileGeom g = tile_geom(d, t);
  if (lane_id() == 0) prefetch_tile(d, nx);  // one wave ahead
  if (g.big >= 0)
    lin_tile<false, false, 32>(d, g, smem, slice, t, write_jac);
  else
    lin_tile<true, false, 32>(d, g, smem, slice, t, write_jac);
}

// Residual only (evaluate + squared_norm, problems.hpp:66, lm.hpp:81-85) at
// the current parameters; writes resid when requested.

template <bool kShared>
__device__ __forceinline__ void cost_tile(const Dev& d, const TileGeom& g, char* smem, int slice, int t) {
  const Ws ws = ws_carve(ws_base<kShared>(d, g, smem, slice), kCostWs, g.ncam, g.npts, g.nobs);
  const int lane = lane_id();
  load_point_fields<3>(ws, 3, 0, d.pts, g.pb, g.npts);
  load_tile_index(d, g, ws);
  __syncwarp();
  load_cam_fields<7>(ws, g.ncam, 11, 0, d.pose, 7);
  load_cam_fields<4>(ws, g.ncam, 11, 7, d.intr, 4);
  __syncwarp();
  SplitSum cost;
  int bad = INT_MAX;
  for (int s = lane; s < g.nobs; s += 32) {
    const std::uint32_t lcpt = ws.lcpt[s];
    const double2 px = reinterpret_cast<const double2*>(d.obs_px)[g.ob + s];
    double r0, r1;
    P3 y;
    if (residual(d.pinhole, ws.cam + (lcpt & 0xffff) * 11, ws.pt + (lcpt >> 16) * 3, px, r0, r1, y)) {
      if (d.resid) {
        d.resid[g.ob + s] = r0;
        d.resid[(long long)d.N + g.ob + s] = r1;
      }
      cost.add(s, r0 * r0 + r1 * r1);
    } else {
      bad = min(bad, d.obs_orig[g.ob + s]);
    }
  }
  if (bad != INT_MAX) atomicMin(&d.lm->err_obs, bad);
  const double ct = cost.warp_total();
  if (lane == 0) d.tile_red[t * 2] = ct;
  __syncwarp();
}

__global__ void __launch_bounds__(256) k_cost(Dev d, int slice) {
  grid_dep_wait();
  extern __shared__ __align__(16) char smem[];
  const int t = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (t >= d.T) return;
  const TileGeom g = tile_geom(d, t);
  BAE_TILE_DISPATCH(cost_tile, d, g, smem, slice, t);
}

// ---------------------------------------------------------------------------
// Camera-side reductions: warp per camera, lane-strided over the camera's
// entries in entry order, fixed xor tree.
// ---------------------------------------------------------------------------
template <int W>
__device__ __forceinline__ void warp_entry_sum(const Dev& d, int c, double (&acc)[W]) {
  const int lane = lane_id();
#pragma unroll
  for (int j = 0; j < W; ++j) acc[j] = 0.0;
  for (int q = d.cam_ent_ptr[c] + lane; q < d.cam_ent_ptr[c + 1]; q += 32) {
    const double* src = d.partial + (long long)d.cam_ent[q] * W;
#pragma unroll
    for (int j = 0; j < W; ++j) acc[j] += src[j];
  }
#pragma unroll
  for (int j = 0; j < W; ++j) acc[j] = warp_sum(acc[j]);
}

// Block-wide sum of camera c's entries (W doubles each), fixed order. Entry
// slot s = warp * G + lane / W (G = 32 / W slots per warp, S slots per
// block) takes the camera's entries s, s + S, s + 2S, ... with four loads in
// flight per lane and coalesced W-double rows; the S slot sums are then added
// in slot order. out[0..W) (shared) is valid after the call.
// NT is the summation layout's thread count: a larger block runs it with its
// first NT threads (same order, same bits) and joins the barriers.
template <int W, int NT>
__device__ __forceinline__ void block_entry_sum(const Dev& d, int c, double* red, double* out,
                                                const double* __restrict__ src) {
  constexpr int G = 32 / W, S = G * (NT / 32);
  const int lane = lane_id(), warp = threadIdx.x >> 5;
  const int slot = warp * G + lane / W, j = lane % W;
  const bool active = lane < G * W && threadIdx.x < NT;
  const int e = d.cam_ent_ptr[c + 1];
  double acc = 0.0;
  if (active) {
    // entries q, q + S, ... in that order (the sum's order); eight partials
    // in flight, and the next eight entry ids loaded while they land, so a
    // group costs one dependent round trip instead of two
    constexpr int U = 8;
    int q = d.cam_ent_ptr[c] + slot;
    int id[U];
#pragma unroll
    for (int k = 0; k < U; ++k) id[k] = q + k * S < e ? d.cam_ent[q + k * S] : -1;
    while (q < e) {
      double v[U];
#pragma unroll
      for (int k = 0; k < U; ++k) v[k] = id[k] >= 0 ? src[(long long)id[k] * W + j] : 0.0;
      const int qn = q + U * S;
#pragma unroll
      for (int k = 0; k < U; ++k) id[k] = qn + k * S < e ? d.cam_ent[qn + k * S] : -1;
#pragma unroll
      for (int k = 0; k < U; ++k)
        if (q + k * S < e) acc += v[k];
      q = qn;
    }
    red[slot * W + j] = acc;
  }
  __syncthreads();
  if (threadIdx.x < W) {
    double t = 0.0;
    for (int k = 0; k < S; ++k) t += red[k * W + threadIdx.x];
    out[threadIdx.x] = t;
  }
  __syncthreads();
}

// Camera c's W-vector: the rank-summed d.cred on sharded runs, else the
// block entry sum.
template <int W, int NT>
__device__ __forceinline__ void cam_block_acc(const Dev& d, int c, double* red, double* out) {
  if (d.cred) {
    if (threadIdx.x < W) out[threadIdx.x] = d.cred[(long long)c * W + threadIdx.x];
    __syncthreads();
  } else {
    block_entry_sum<W, NT>(d, c, red, out, d.partial);
  }
}

// Sharded runs: this rank's per-camera entry sums into d.cred (block per
// camera), plus trailing scalars computed by one extra block:
//   extra 1 (linearisation): [sum r^2, sum |g_p|^2] over this rank's tiles
//   extra 2 (prep)          : [1 if a local point block was not SPD]
// The W = 6 instance (PCG product) is skipped once the solve has finished,
// like the other kernels of a PCG chunk.
// Thread-strided sums over the per-tile [cost, gradient] pairs in the
// thread's fixed order (tt, tt + blockDim, ...), eight loads in flight (a
// one-block reduction over 316 k tiles waited on one load at a time: 145 us).
template <bool kTwo>
__device__ __forceinline__ void tile_pair_sums(const double* tr, int T, double& a, double& b) {
  const int bd = blockDim.x;
  int tt = threadIdx.x;
  for (; tt + 7 * bd < T; tt += 8 * bd) {
    double va[8], vb[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      va[k] = tr[(tt + k * bd) * 2];
      if (kTwo) vb[k] = tr[(tt + k * bd) * 2 + 1];
    }
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      a += va[k];
      if (kTwo) b += vb[k];
    }
  }
  for (; tt < T; tt += bd) {
    a += tr[tt * 2];
    if (kTwo) b += tr[tt * 2 + 1];
  }
}

template <int W, int NT>
__global__ void __launch_bounds__(NT) k_cam_entry_sums(Dev d, int extra, int pcg_gated) {
  grid_dep_wait();
  __shared__ double red[(32 / W) * (NT / 32) * W];
  __shared__ double acc[W];
  if (pcg_gated && d.pcg->state >= kPcgDone) return;
  if (blockIdx.x == gridDim.x - 1) {
    if (extra == 1) {
      double a = 0.0, b = 0.0;
      tile_pair_sums<true>(d.tile_red, d.T, a, b);
      a = block_sum(a, red);
      __syncthreads();
      b = block_sum(b, red);
      if (threadIdx.x == 0) {
        d.cred[(long long)W * d.C] = a;
        d.cred[(long long)W * d.C + 1] = b;
      }
    } else if (extra == 2 && threadIdx.x == 0) {
      d.cred[(long long)W * d.C] = d.pcg->not_spd ? 1.0 : 0.0;
    }
    return;
  }
  const int c = blockIdx.x;
  block_entry_sum<W, NT>(d, c, red, acc, d.partial);
  if (threadIdx.x < W) d.cred[(long long)c * W + threadIdx.x] = acc[threadIdx.x];
}

// Camera side of the linearisation (block per camera): H_cc (21) and g_c (6)
// from the camera's entries; |g_c|^2 per camera for the totals.
// kCamNT threads per camera block for the LM-loop camera passes (16 slots
// of 27-wide entries, 80 of 6-wide ones): few cameras, so the per-camera
// sums are latency-bound and want many loads in flight.
constexpr int kCamNT = 512;

__global__ void __launch_bounds__(kCamNT) k_cam_linearize(Dev d) {
  grid_dep_wait();
  __shared__ double red[16 * 27];
  __shared__ double acc[27];
  const int c = blockIdx.x;
  cam_block_acc<27, kCamNT>(d, c, red, acc);
  const int t = threadIdx.x;
  if (t < 21) d.hcc[(long long)c * 21 + t] = acc[t];
  else if (t < 27) d.gc[(long long)c * 6 + (t - 21)] = acc[t];
  if (t == 0) {
    double gsq = 0.0;
#pragma unroll
    for (int j = 0; j < 6; ++j) gsq += acc[21 + j] * acc[21 + j];
    d.cam_dot[c] = gsq;
  }
}

// Camera side of the fused linearisation + direct prep (block per camera,
// single rank): k_cam_linearize's H_cc, g_c, |g_c|^2 and
// k_cam_prep_direct's damped H~_cc and Schur RHS, with the same summation
// orders as those two kernels.
__global__ void __launch_bounds__(kCamNT) k_cam_lin_prep(Dev d, double clo, double chi) {
  grid_dep_wait();
  __shared__ double red[80 * 6];  // >= 16 * 27
  __shared__ double acc[27];
  __shared__ double acc6[6];
  const int c = blockIdx.x;
  block_entry_sum<27, kCamNT>(d, c, red, acc, d.partial);
  block_entry_sum<6, kCamNT>(d, c, red, acc6, d.partial6);
  const int t = threadIdx.x;
  if (t < 21) {
    double h = acc[t];
    d.hcc[(long long)c * 21 + t] = h;
    if (t == sym6(0, 0) || t == sym6(1, 1) || t == sym6(2, 2) || t == sym6(3, 3) || t == sym6(4, 4) ||
        t == sym6(5, 5))
      h = damp_diag(h, *d.lam, clo, chi);
    d.hccd[(long long)c * 21 + t] = h;
  } else if (t < 27) {
    d.gc[(long long)c * 6 + (t - 21)] = acc[t];
  } else if (t >= 32 && t < 38) {
    const int a = t - 32;
    d.rhs[(long long)c * 6 + a] = -acc[21 + a] + acc6[a];
  } else if (t == 64) {
    double gsq = 0.0;
#pragma unroll
    for (int j = 0; j < 6; ++j) gsq += acc[21 + j] * acc[21 + j];
    d.cam_dot[c] = gsq;
  }
}

// Cost and ||J^T r||^2 of the linearisation (one block, fixed order): tile
// totals in tile order (sharded: already summed over ranks) + camera |g_c|^2.
__global__ void __launch_bounds__(1024) k_lin_totals(Dev d) {
  grid_dep_wait();
  __shared__ double red[32];
  double a = 0.0, b = 0.0, g = 0.0;
  if (!d.cred) tile_pair_sums<true>(d.tile_red, d.T, a, b);
  for (int c = threadIdx.x; c < d.C; c += blockDim.x) g += d.cam_dot[c];
  a = block_sum(a, red);
  __syncthreads();
  b = block_sum(b, red);
  __syncthreads();
  g = block_sum(g, red);
  if (threadIdx.x == 0) {
    if (d.cred) {
      a = d.cred[27LL * d.C];
      b = d.cred[27LL * d.C + 1];
    }
    d.lm->cost = a;
    d.lm->grad_sq = b + g;
  }
}

// Total of the per-tile costs, fixed order, one block.
__global__ void k_sum_tiles(Dev d, int trial) {
  grid_dep_wait();
  __shared__ double red[32];
  double a = 0.0, unused = 0.0;
  tile_pair_sums<false>(d.tile_red, d.T, a, unused);
  a = block_sum(a, red);
  if (d.cred) {  // sharded: [local cost, local trial failure] go to the cross-rank sum
    if (threadIdx.x == 0) {
      d.cred[0] = a;
      d.cred[1] = (trial && d.lm->trial_bad) ? 1.0 : 0.0;
    }
    return;
  }
  if (threadIdx.x == 0) {
    if (trial)
      d.lm->new_cost = (d.lm->trial_bad || d.lm->retract_bad || !isfinite(a)) ? INFINITY : a;
    else
      d.lm->cost = a;
  }
}

// Sharded runs: the cost (or trial cost) from the rank-summed [cost, failure].
__global__ void k_finish_cost(Dev d, int trial) {
  grid_dep_wait();
  const double a = d.cred[0];
  const bool bad = d.cred[1] > 0.0;
  if (trial) {
    d.lm->trial_bad = bad ? 1 : 0;
    d.lm->new_cost = (bad || d.lm->retract_bad || !isfinite(a)) ? INFINITY : a;
  } else {
    d.lm->cost = a;
  }
}

// ---------------------------------------------------------------------------
// K3/K4 prep for one damping value: per point H~_pp^-1 and v = H~_pp^-1 g_p;
// per entry the Schur right-hand side (J_c^T J_p v) and the block-Jacobi
// blocks (W H~_pp^-1 W^T, W = J_c^T J_p) of S's diagonal.
// cam: R9 t3 k4 (16) ; pt: p3 hinv6 v3 (12) ; stage 27
// Direct solver (kDirect): no block-Jacobi blocks (PCG only), stage 6 (the
// RHS), and W, W H~_pp^-1 of every slot kept for the assembly of S.
// ---------------------------------------------------------------------------

template <bool kShared, bool kDirect>
__device__ __forceinline__ void prep_tile(const Dev& d, const TileGeom& g, char* smem, int slice, double lambda,
                                          double clo, double chi) {
  if (kDirect) lambda = *d.lam;  // direct solves keep lambda on the device (graph-replayed LM iterations)
  constexpr int SW = kDirect ? kPrepDirStW : 27;  // row stride; the direct RHS piece is 6 wide
  const Ws ws = ws_carve(ws_base<kShared>(d, g, smem, slice), kDirect ? kPrepDirWs : kPrepWs, g.ncam, g.npts, g.nobs);
  const int lane = lane_id();
  load_point_fields<3, 32, true>(ws, 12, 0, d.pts, g.pb, g.npts);
  load_tile_index(d, g, ws);
  __syncwarp();
  load_cam_fields<16>(ws, g.ncam, 16, 0, d.camrec, kCamRec);
  int fail = 0;
  for (int lp = lane; lp < g.npts; lp += 32) {
    const long long ip = g.pb + lp;
    double h[6], inv[9];
#pragma unroll
    for (int j = 0; j < 6; ++j) h[j] = d.hpp[ip * 6 + j];
    double sp[12];
    if (kDirect) {  // the Cholesky factor L of H~_pp instead of its inverse (shared with k_lin_prep)
      const double g3[3] = {d.gp[ip * 3], d.gp[ip * 3 + 1], d.gp[ip * 3 + 2]};
      if (!prep_point_direct(d, ip, h, g3, lambda, clo, chi, sp)) fail = 1;
      pt_put<9>(ws, g.npts, lp, 3, sp + 3);
      continue;
    }
    h[0] = damp_diag(h[0], lambda, clo, chi);
    h[3] = damp_diag(h[3], lambda, clo, chi);
    h[5] = damp_diag(h[5], lambda, clo, chi);
    const bool pfail = !spd_inverse<3>(h, inv);
    if (pfail) {
      fail = 1;
#pragma unroll
      for (int j = 0; j < 9; ++j) inv[j] = 0.0;
    }
    const double hi[6] = {inv[0], inv[1], inv[2], inv[4], inv[5], inv[8]};
#pragma unroll
    for (int j = 0; j < 6; ++j) d.hinv[ip * 6 + j] = hi[j];
#pragma unroll
    for (int j = 0; j < 6; ++j) sp[3 + j] = hi[j];
    const double g0 = d.gp[ip * 3], g1 = d.gp[ip * 3 + 1], g2 = d.gp[ip * 3 + 2];
    sp[9] = inv[0] * g0 + inv[1] * g1 + inv[2] * g2;
    sp[10] = inv[3] * g0 + inv[4] * g1 + inv[5] * g2;
    sp[11] = inv[6] * g0 + inv[7] * g1 + inv[8] * g2;
    pt_put<9>(ws, g.npts, lp, 3, sp + 3);
  }
  if (fail) atomicExch(&d.pcg->not_spd, 1);
  __syncwarp();
  for (int s = lane; s < g.nobs; s += 32) {
    const std::uint32_t lcpt = ws.lcpt[s];
    const double* cam = ws.cam + (lcpt & 0xffff) * 16;
    double sp[12];
    pt_get<12>(ws, g.npts, lcpt >> 16, 0, sp);
    P3 y;
    double D[6], Jc[12], Jp[6];
    obs_geometry(d.pinhole, cam, sp, y, D);
    jac_cam(D, y, Jc);
    jac_pt(D, cam, Jp);
    double W[18];  // 6x3
#pragma unroll
    for (int a = 0; a < 6; ++a)
#pragma unroll
      for (int j = 0; j < 3; ++j) W[a * 3 + j] = Jc[a] * Jp[j] + Jc[6 + a] * Jp[3 + j];
    double* st = ws.stage + s * SW;
    if (!kDirect) {
      const double* hi = sp + 3;  // packed xx xy xz yy yz zz
      const double H[9] = {hi[0], hi[1], hi[2], hi[1], hi[3], hi[4], hi[2], hi[4], hi[5]};
      double WH[18];
#pragma unroll
      for (int a = 0; a < 6; ++a)
#pragma unroll
        for (int j = 0; j < 3; ++j)
          WH[a * 3 + j] = W[a * 3] * H[j] + W[a * 3 + 1] * H[3 + j] + W[a * 3 + 2] * H[6 + j];
      int q = 0;
#pragma unroll
      for (int a = 0; a < 6; ++a)
#pragma unroll
        for (int b = a; b < 6; ++b)
          st[q++] = WH[a * 3] * W[b * 3] + WH[a * 3 + 1] * W[b * 3 + 1] + WH[a * 3 + 2] * W[b * 3 + 2];
    } else {  // direct solver: V = W L^-T of this slot and its RHS piece (shared with k_lin_prep)
      prep_obs_direct(d, g.ob + s, W, y, sp, st);
      continue;
    }
    const double* vp = sp + 9;
#pragma unroll
    for (int a = 0; a < 6; ++a) st[SW - 6 + a] = W[a * 3] * vp[0] + W[a * 3 + 1] * vp[1] + W[a * 3 + 2] * vp[2];
  }
  __syncwarp();
  entries_from_stage<kDirect ? 6 : SW, SW>(ws, g.ncam, g.eb, d.partial);
  __syncwarp();
}

template <bool kDirect>
__global__ void __launch_bounds__(256) k_prep(Dev d, int slice, double lambda, double clo, double chi, int pf) {
  grid_dep_wait();
  extern __shared__ __align__(16) char smem[];
  const int t = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (t >= d.T) return;
  const TileSpan nx = pf > 0 && lane_id() == 0 ? tile_span(d, t + pf) : TileSpan{0, 0, 0, 0, 0, 0};
  const TileGeom g = tile_geom(d, t);
  if (lane_id() == 0) prefetch_tile(d, nx, d.hpp, 6, d.gp, 3);  // one wave ahead
  if (g.big >= 0)
    prep_tile<false, kDirect>(d, g, smem, slice, lambda, clo, chi);
  else
    prep_tile<true, kDirect>(d, g, smem, slice, lambda, clo, chi);
}

// Camera side of the direct solver's prep (block per camera): damped H~_cc
// and the Schur RHS b = -g_c + sum_k J_c^T J_p H~_pp^-1 g_p.
__global__ void __launch_bounds__(kCamNT) k_cam_prep_direct(Dev d, double lambda, double clo, double chi) {
  grid_dep_wait();
  lambda = *d.lam;
  __shared__ double red[80 * 6];
  __shared__ double acc[6];
  const int c = blockIdx.x;
  cam_block_acc<6, kCamNT>(d, c, red, acc);
  if (threadIdx.x == 0 && c == 0 && d.cred && d.cred[6LL * d.C] > 0.0)
    atomicExch(&d.pcg->not_spd, 1);  // a point block failed on some rank
  if (threadIdx.x < 21) {
    const int t = threadIdx.x;
    double h = d.hcc[(long long)c * 21 + t];
    if (t == sym6(0, 0) || t == sym6(1, 1) || t == sym6(2, 2) || t == sym6(3, 3) || t == sym6(4, 4) ||
        t == sym6(5, 5))
      h = damp_diag(h, lambda, clo, chi);
    d.hccd[(long long)c * 21 + t] = h;
  } else if (threadIdx.x >= 32 && threadIdx.x < 38) {
    const int a = threadIdx.x - 32;
    d.rhs[(long long)c * 6 + a] = -d.gc[(long long)c * 6 + a] + acc[a];
  }
}

// Camera side of the prep (block per camera): damped H~_cc, block-Jacobi
// inverse of S_cc (falls back to H~_cc^-1 when the 6x6 Schur block is not
// numerically SPD), Schur RHS, and PCG initialisation x = 0, r = b,
// z = M^-1 r; per-camera r.r and r.z for the totals.
__global__ void __launch_bounds__(256) k_cam_prep(Dev d, double lambda, double clo, double chi) {
  grid_dep_wait();
  __shared__ double red[8 * 27];
  __shared__ double acc[27];
  const int c = blockIdx.x;
  cam_block_acc<27, 256>(d, c, red, acc);
  if (threadIdx.x != 0) return;
  double hd[21], s[21], m[36], b[6];
  double rr = 0.0, rz = 0.0;
#pragma unroll
  for (int j = 0; j < 21; ++j) hd[j] = d.hcc[(long long)c * 21 + j];
#pragma unroll
  for (int a = 0; a < 6; ++a) hd[sym6(a, a)] = damp_diag(hd[sym6(a, a)], lambda, clo, chi);
#pragma unroll
  for (int j = 0; j < 21; ++j) {
    d.hccd[(long long)c * 21 + j] = hd[j];
    s[j] = hd[j] - acc[j];
  }
  if (!spd_inverse<6>(s, m)) {
    if (!spd_inverse<6>(hd, m)) {
      atomicExch(&d.pcg->not_spd, 1);
#pragma unroll
      for (int j = 0; j < 36; ++j) m[j] = 0.0;
    }
  }
#pragma unroll
  for (int j = 0; j < 36; ++j) d.minv[(long long)c * 36 + j] = m[j];
#pragma unroll
  for (int a = 0; a < 6; ++a) b[a] = -d.gc[(long long)c * 6 + a] + acc[21 + a];
#pragma unroll
  for (int a = 0; a < 6; ++a) {
    double zz = 0.0;
#pragma unroll
    for (int j = 0; j < 6; ++j) zz += m[a * 6 + j] * b[j];
    const long long o = (long long)c * 6 + a;
    d.rhs[o] = b[a];
    d.x[o] = 0.0;
    d.r[o] = b[a];
    d.z[o] = zz;
    d.p[o] = 0.0;
    rr += b[a] * b[a];
    rz += b[a] * zz;
  }
  d.cam_dot[2LL * c] = rr;
  d.cam_dot[2LL * c + 1] = rz;
}

// PCG start state from the prep totals (one block, fixed order).
__global__ void __launch_bounds__(1024) k_prep_totals(Dev d, double tol, long long budget) {
  grid_dep_wait();
  __shared__ double red[32];
  double rr = 0.0, rz = 0.0;
  for (int c = threadIdx.x; c < d.C; c += blockDim.x) {
    rr += d.cam_dot[2LL * c];
    rz += d.cam_dot[2LL * c + 1];
  }
  rr = block_sum(rr, red);
  __syncthreads();
  rz = block_sum(rz, red);
  if (threadIdx.x != 0) return;
  PcgDev& s = *d.pcg;
  // Tolerance semantics of the reference (pcg.hpp:85): ||r|| <= tol ||b|| with
  // b the FULL right-hand side -J^T r. Back-substitution satisfies the point
  // rows exactly, so the full residual equals the reduced one and the
  // reference's test is applied unchanged to the reduced recurrence.
  s.bnorm = sqrt(d.lm->grad_sq);
  s.rz = rz;
  s.tol = tol;
  s.iters = 0;
  s.budget = budget;
  s.dir = kDirZ;
  s.beta = 0.0;
  s.converged = 0;
  s.true_norm = sqrt(rr);
  if (d.cred && d.cred[27LL * d.C] > 0.0) s.not_spd = 1;  // a point block failed on some rank
  if (s.not_spd) {
    s.state = kPcgBreakdown;
  } else if (s.bnorm == 0.0 || rr == 0.0) {  // x = 0 solves the system exactly
    s.state = kPcgDone;
    s.converged = 1;
  } else {
    s.state = kPcgIter;
  }
}

// ---------------------------------------------------------------------------
// F2: dense reduced camera system for the direct solver (the reference's
// default SolverChoice::cholesky, lm.hpp:132-136). One warp per camera block
// (c1 >= c2):  S[c1,c2] = delta(c1,c2) H~_cc - sum_{points} sum_{k in c1, l in c2}
// V_k V_l^T with V = W L^-T (H~_pp = L L^T, so V_k V_l^T = W_k H~_pp^-1 W_l^T),
// each V from its compact [Q | y] record, pairs in (point, k, l) order, lanes
// strided over the block's pairs, fixed xor tree; column-major lower
// triangle for potrf.
// ---------------------------------------------------------------------------
// 256-bit read-only global load (sm_100: one instruction per 32-byte sector)
__device__ __forceinline__ void ldg_v4(const double* p, double* o) {
  asm volatile("ld.global.nc.v4.f64 {%0, %1, %2, %3}, [%4];"
               : "=d"(o[0]), "=d"(o[1]), "=d"(o[2]), "=d"(o[3])
               : "l"(p));
}
constexpr int kSchurDenseThreads = 128;
// acc += V_a V_b^T from two [Q | y] records (kSame: a and b are one record,
// G = Q Q^T is formed from its six distinct dot products -- x y == y x, so
// the same bits as the general form)
template <bool kSame>
__device__ __forceinline__ void schur_pair(const double (&a)[kVStride], const double (&b)[kVStride], double (&acc)[36]) {
  // V_a V_b^T = [G, G Y_b^T; Y_a G, Y_a G Y_b^T] with G = Q_a Q_b^T and
  // Y = [y]x: row i of G Y_b^T is y_b x (row i of G), column j of Y_a X
  // is y_a x (column j of X)
  const double ya[3] = {a[9], a[10], a[11]}, yb[3] = {b[9], b[10], b[11]};
  double G[9], T[9];
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j) {
      double gij;
      if (kSame && j < i)
        gij = G[j * 3 + i];
      else
        gij = a[3 * i] * b[3 * j] + a[3 * i + 1] * b[3 * j + 1] + a[3 * i + 2] * b[3 * j + 2];
      G[i * 3 + j] = gij;
      acc[i * 6 + j] += gij;
    }
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j) {
      const int j1 = (j + 1) % 3, j2 = (j + 2) % 3;
      const double tij = yb[j1] * G[i * 3 + j2] - yb[j2] * G[i * 3 + j1];
      T[i * 3 + j] = tij;
      acc[i * 6 + 3 + j] += tij;
    }
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    const int i1 = (i + 1) % 3, i2 = (i + 2) % 3;
#pragma unroll
    for (int j = 0; j < 3; ++j) {
      double& bl = acc[(3 + i) * 6 + j];
      bl = fma(ya[i1], G[i2 * 3 + j], bl);
      bl = fma(-ya[i2], G[i1 * 3 + j], bl);
      double& br = acc[(3 + i) * 6 + 3 + j];
      br = fma(ya[i1], T[i2 * 3 + j], br);
      br = fma(-ya[i2], T[i1 * 3 + j], br);
    }
  }
}
__device__ __forceinline__ void ld_rec(const double* w, int r, double (&a)[kVStride]) {
  // three 32-byte loads a record: each touches one whole sector (16-byte
  // loads touch every sector twice, and the L1 pays per sector touched)
  const double* p = w + (long long)r * kVStride;
#pragma unroll
  for (int j = 0; j < kVStride / 4; ++j) ldg_v4(p + 4 * j, a + 4 * j);
}
// 128 registers: four 4-warp CTAs per SM (Final: 3 CTAs at 140 registers 3.25 ms, 4 CTAs 2.95 ms, 5 CTAs
// with spills 3.86 ms; 2.72 ms with the next pair's index loaded ahead)
__global__ void __launch_bounds__(kSchurDenseThreads, 4) k_schur_dense(Dev d) {
  grid_dep_wait();
  // Warp per chunk of at most kSchurChunk pairs of one camera block (a long
  // block -- a diagonal one holds every observation of its camera -- is cut
  // into several, so no warp walks a whole camera's observations alone).
  // Lane = pair slot: each lane forms the whole 6x6 V_k V_l^T of its pairs
  // (both 96-byte [Q | y] records reach its registers once: the LSU writeback of
  // loaded bytes, not L1 or DRAM, bounds this kernel; 128 registers, so
  // 4-warp CTAs, 4 per SM), then a fixed
  // reduce-scatter tree over the 32 slots leaves elements
  // 9 g .. 9 g + 8 of the chunk sum in lane group g = lane >> 3. A block of
  // one chunk is written at once; otherwise each chunk stores its 6x6
  // partial and the block's last chunk to finish (ticket) adds the partials
  // in chunk order. Every order depends only on the block.
  const int wid = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (wid >= d.nchunk) return;
  const int4 ch = d.chunks[wid];  // block, first pair, end pair, index of the block's first chunk
  const int blk = ch.x;
  const int lane = lane_id();
  double acc[36];
#pragma unroll
  for (int j = 0; j < 36; ++j) acc[j] = 0.0;
  // the next pair's index is loaded before this pair's records (a fully
  // prefetched next pair -- its records too -- needs 168 registers and three
  // CTAs per SM: 3.80 vs 2.72 ms at Final)
  int q = ch.y + lane;
  int2 pr = q < ch.z ? d.pairs[q] : make_int2(0, 0);
#pragma unroll 1
  for (; q < ch.z; q += 32) {
    const int2 pn = q + 32 < ch.z ? d.pairs[q + 32] : pr;
    double a[kVStride];
    ld_rec(d.wstore, pr.x, a);
    if (pr.x == pr.y) {  // (k, k): a quarter of the pairs (the diagonal blocks), one record
      schur_pair<true>(a, a, acc);
    } else {
      double b[kVStride];
      ld_rec(d.wstore, pr.y, b);
      schur_pair<false>(a, b, acc);
    }
    pr = pn;
  }
  // reduce-scatter: xor 16 halves the 36 sums (bit 4 keeps [18 b4, +18)),
  // xor 8 halves again (bit 3 keeps the upper 9), xor 4/2/1 finish the 9
  // (a + b == b + a, so the partners agree bit for bit)
  double h18[18];
  {
    const bool up = lane & 16;
#pragma unroll
    for (int i = 0; i < 18; ++i) {
      const double keep = up ? acc[18 + i] : acc[i], give = up ? acc[i] : acc[18 + i];
      h18[i] = keep + __shfl_xor_sync(0xffffffffu, give, 16);
    }
  }
  double v9[9];
  {
    const bool up = lane & 8;
#pragma unroll
    for (int i = 0; i < 9; ++i) {
      const double keep = up ? h18[9 + i] : h18[i], give = up ? h18[i] : h18[9 + i];
      v9[i] = keep + __shfl_xor_sync(0xffffffffu, give, 8);
    }
  }
#pragma unroll
  for (int i = 0; i < 9; ++i)
#pragma unroll
    for (int off = 4; off > 0; off >>= 1) v9[i] += __shfl_xor_sync(0xffffffffu, v9[i], off);
  // lane (g, j = lane & 7) owns element 9 g + j, and j == 0 also 9 g + 8
  const int g9 = 9 * (lane >> 3), j8 = lane & 7;
  double own = v9[0];
#pragma unroll
  for (int i = 1; i < 8; ++i)
    if (j8 == i) own = v9[i];
  const double own8 = v9[8];
  const int first = ch.w, count = d.blk_nchunk[blk];
  double v36 = 0.0;  // multi-chunk: entry (lane / 6, lane % 6) of the block sum, lanes 0..35 -> 0..31 + 4 below
  double v36b = 0.0;
  if (count > 1) {
    double* mine = d.schur_part + 36LL * wid;
    mine[g9 + j8] = own;
    if (j8 == 0) mine[g9 + 8] = own8;
    __threadfence();
    __syncwarp();
    int t = 0;
    if (lane == 0) t = static_cast<int>(atomicAdd(d.blk_ticket + blk, 1u));
    t = __shfl_sync(0xffffffffu, t, 0);
    if (t != count - 1) return;
    __threadfence();  // the other chunks' partials, published before their tickets
    for (int i = 0; i < count; ++i) {  // chunk order
      const double* pp = d.schur_part + 36LL * (first + i);
      v36 += __ldcg(pp + lane);
      if (lane < 4) v36b += __ldcg(pp + 32 + lane);
    }
  }
  const int2 cc = d.blk_cam[blk];
  const long long n = 6LL * d.C;
  const double* h = d.hccd + (long long)cc.x * 21;
  // dense column-major S, or the block's place in its 48 x 48 tile (the
  // camera order of the tile factorisation may put it transposed)
  double* base;
  long long ldr, ldc;  // element (r, c) of the block at base[r * ldr + c * ldc]
  if (d.stiles) {
    const int2 bt = d.blk_tile[blk];
    const int ro = bt.y & 0xff, co = (bt.y >> 8) & 0xff;
    base = d.stiles + (long long)bt.x * kSTileElems + co * 48 + ro;
    const bool tr = (bt.y >> 16) & 1;
    ldr = tr ? 48 : 1;
    ldc = tr ? 1 : 48;
  } else {
    base = d.schur + 6LL * cc.y * n + 6LL * cc.x;
    ldr = 1;
    ldc = n;
  }
  // sharded: H~_cc is added after the rank sum; deferred: after the camera pass
  const bool diag = cc.x == cc.y && !d.cred && !d.defer_hccd;
  if (count == 1) {
    const int e = g9 + j8;
    double v = -own;
    if (diag) v += h[sym6(e / 6, e % 6)];
    base[(e / 6) * ldr + (e % 6) * ldc] = v;
    if (j8 == 0) {
      const int e8 = g9 + 8;
      double v8 = -own8;
      if (diag) v8 += h[sym6(e8 / 6, e8 % 6)];
      base[(e8 / 6) * ldr + (e8 % 6) * ldc] = v8;
    }
    return;
  }
  {
    const int r = lane / 6, c = lane % 6;
    double v = -v36;
    if (diag) v += h[sym6(r, c)];
    base[r * ldr + c * ldc] = v;
  }
  if (lane < 4) {
    const int e = 32 + lane, r = e / 6, c = e % 6;
    double v = -v36b;
    if (diag) v += h[sym6(r, c)];
    base[r * ldr + c * ldc] = v;
  }
}

// Sharded direct solve: the damped camera blocks join the rank-summed S.
__global__ void k_add_hccd(Dev d) {
  grid_dep_wait();
  const long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= 36LL * d.C) return;
  const int c = (int)(idx / 36), r = (int)(idx % 36) / 6, col = (int)(idx % 6);
  const long long n = 6LL * d.C;
  const double h = d.hccd[(long long)c * 21 + sym6(r, col)];
  if (d.stiles) {  // camera c's diagonal block inside its diagonal tile
    const int2 bt = d.blk_tile[d.nblk + c];
    d.stiles[(long long)bt.x * kSTileElems + (bt.y + col) * 48 + bt.y + r] += h;
  }
  else
    d.schur[(6LL * c + col) * n + 6LL * c + r] += h;
}

// ---------------------------------------------------------------------------
// K5: implicit Schur product, tile part. For v = current PCG direction
// (z, z + beta p, or x when verifying the true residual):
//   s_k = J_p^T J_c v_c(k);  w_p = sum_k s_k;  t_p = H~_pp^-1 w_p;
//   partial[e] = sum_{k in e} J_c^T J_p t_p(k)
// The camera part then forms y = H~_cc v - sum partial.
// Only data shared across lanes goes through shared memory: the tile's
// camera records + direction (cam, 24 per camera), the per-observation
// exchange vectors (stage, SoA [6][nobs]) and t_p (pt, 3 per point).
// Observation and point data are read straight from global memory by the
// lane that owns them. D and y of a lane's first kCacheRounds observations
// stay in registers between the two observation phases.
// ---------------------------------------------------------------------------
constexpr int kCacheRounds = 2;

// The PCG direction is formed lazily (p = z + beta p) by both the tile and
// the camera part with the same fused expression, so both see identical bits.
__device__ __forceinline__ double dir_component(const PcgDev& s, const Dev& d, long long o) {
  return s.dir == kDirX ? d.x[o] : (s.dir == kDirZ ? d.z[o] : fma(s.beta, d.p[o], d.z[o]));
}
__device__ __forceinline__ void dir_vector(const PcgDev& s, const Dev& d, long long c, double* v) {
#pragma unroll
  for (int j = 0; j < 6; ++j) v[j] = dir_component(s, d, c * 6 + j);
}

// Copy the 16-double records (and optionally a 6-vector per camera from
// `vec6`) of the tile's cameras into ws.cam[l * ld + ...]; two cameras per
// pass (lane -> camera l0 + lane/16, field lane%16). Small tiles resolve the
// camera id by shuffling it from the lane that loaded it.
template <bool kSmall, class Vec6>
__device__ __forceinline__ void copy_tile_cams(const Dev& d, const TileGeom& g, const Ws& ws, int ld,
                                               const double* rec, int mycam, Vec6 vec6) {
  const int lane = lane_id(), sub = lane >> 4, j = lane & 15;
#pragma unroll 4
  for (int l0 = 0; l0 < g.ncam; l0 += 2) {
    const int l = min(l0 + sub, g.ncam - 1);
    const int c = kSmall ? __shfl_sync(0xffffffffu, mycam, l & 31) : d.ent_cam[g.eb + l];
    const double r = rec[(long long)c * kCamRec + j];
    const double v = j < 6 ? vec6(c, j) : 0.0;
    if (l0 + sub < g.ncam) {
      ws.cam[l * ld + j] = r;
      if (j < 6) ws.cam[l * ld + 16 + j] = v;
    }
  }
}

// Camera records (16 doubles) + the PCG direction (6) of the tile's cameras
// into ws.cam[l * 24]; 16 lanes per camera, two cameras per pass. The
// direction kind is warp-uniform and hoisted out of the loop.
template <bool kSmall>
__device__ __forceinline__ void sx_copy_cams(const Dev& d, const PcgDev& st, const TileGeom& g, const Ws& ws,
                                             int mycam) {
  const int lane = lane_id(), sub = lane >> 4, j = lane & 15;
  const int dir = st.dir;
  const double beta = st.beta;
  const double* va = dir == kDirX ? d.x : d.z;  // first term
#pragma unroll 4
  for (int l0 = 0; l0 < g.ncam; l0 += 2) {
    const int l = min(l0 + sub, g.ncam - 1);
    const int c = kSmall ? __shfl_sync(0xffffffffu, mycam, l & 31) : d.ent_cam[g.eb + l];
    const long long o = (long long)c * 6 + min(j, 5);
    const double r = d.camrec[(long long)c * kCamRec + j];
    double v = va[o];
    if (dir == kDirZBetaP) v = fma(beta, d.p[o], v);  // same fused expression as dir_component
    if (l0 + sub < g.ncam) {
      ws.cam[l * 24 + j] = r;
      if (j < 6) ws.cam[l * 24 + 16 + j] = v;
    }
  }
}

template <bool kSmall>
__device__ __forceinline__ void sx_tile_impl(const Dev& d, const PcgDev& st, const TileGeom& g, char* smem,
                                             int slice) {
  const Ws ws = ws_carve(ws_base<kSmall>(d, g, smem, slice), kSxWs, g.ncam, g.npts, g.nobs);
  const int lane = lane_id();
  const int nobs = g.nobs;
  if (d.trace && lane == 0) d.trace[(long long)g.trace_id * 8 + 0] = global_ns();
  // ---- level-2 loads (depend only on the tile geometry), all in flight together
  std::uint32_t lc[kCacheRounds];
  std::uint16_t pl[kCacheRounds];
#pragma unroll
  for (int r = 0; r < kCacheRounds; ++r) {
    const int s = min(r * 32 + lane, nobs - 1);
    lc[r] = d.obs_lcpt[g.ob + s];
    pl[r] = d.ptobs[g.ob + s];
  }
  const int pp0 = d.pt_ptr[g.pb + min(lane, g.npts)];
  const int pp1 = d.pt_ptr[g.pb + min(lane + 32, g.npts)];
  const int eo0 = d.ent_obs_begin[g.eb + min(lane, g.ncam)];
  const int eo1 = d.ent_obs_begin[g.eb + min(lane + 32, g.ncam)];
  const int mycam = kSmall ? d.ent_cam[g.eb + min(lane, g.ncam - 1)] : 0;
  // ---- level-3 loads: point coordinates of the lane's observations
  double px[kCacheRounds][3];
#pragma unroll
  for (int r = 0; r < kCacheRounds; ++r) {
    const double* p = d.pts + (long long)(g.pb + (lc[r] >> 16)) * 3;
    px[r][0] = p[0];
    px[r][1] = p[1];
    px[r][2] = p[2];
  }
  // index data into the workspace
#pragma unroll
  for (int r = 0; r < kCacheRounds; ++r)
    if (r * 32 + lane < nobs) ws.ptl[r * 32 + lane] = pl[r];
  for (int s = kCacheRounds * 32 + lane; s < nobs; s += 32) ws.ptl[s] = d.ptobs[g.ob + s];
  if (lane <= g.npts) ws.pptr[lane] = pp0 - g.ob;
  if (lane + 32 <= g.npts) ws.pptr[lane + 32] = pp1 - g.ob;
  for (int i = lane + 64; i <= g.npts; i += 32) ws.pptr[i] = d.pt_ptr[g.pb + i] - g.ob;
  if (lane <= g.ncam) ws.ent[lane] = eo0 - g.ob;
  if (lane + 32 <= g.ncam) ws.ent[lane + 32] = eo1 - g.ob;
  for (int i = lane + 64; i <= g.ncam; i += 32) ws.ent[i] = d.ent_obs_begin[g.eb + i] - g.ob;
  sx_copy_cams<kSmall>(d, st, g, ws, mycam);
  __syncwarp();
  if (d.trace && lane == 0) d.trace[(long long)g.trace_id * 8 + 1] = global_ns();
  // phase 1: s_k = J_p^T J_c v
  double cD[kCacheRounds][6];
  P3 cy[kCacheRounds];
#pragma unroll
  for (int r = 0; r < kCacheRounds; ++r) {
    const int s = r * 32 + lane;
    if (s < nobs) {
      const double* cam = ws.cam + (lc[r] & 0xffff) * 24;
      obs_geometry(d.pinhole, cam, px[r], cy[r], cD[r]);
      double sv[3];
      jpt_jc_v(cD[r], cy[r], cam, cam + 16, sv);
      ws.stage[s] = sv[0];
      ws.stage[nobs + s] = sv[1];
      ws.stage[2 * nobs + s] = sv[2];
    }
  }
  for (int s = kCacheRounds * 32 + lane; s < nobs; s += 32) {  // long tiles
    const std::uint32_t l = d.obs_lcpt[g.ob + s];
    const double* cam = ws.cam + (l & 0xffff) * 24;
    const double* p = d.pts + (long long)(g.pb + (l >> 16)) * 3;
    const double pp[3] = {p[0], p[1], p[2]};
    P3 y;
    double D[6], sv[3];
    obs_geometry(d.pinhole, cam, pp, y, D);
    jpt_jc_v(D, y, cam, cam + 16, sv);
    ws.stage[s] = sv[0];
    ws.stage[nobs + s] = sv[1];
    ws.stage[2 * nobs + s] = sv[2];
  }
  __syncwarp();
  if (d.trace && lane == 0) d.trace[(long long)g.trace_id * 8 + 2] = global_ns();
  // point phase: t_p = H~_pp^-1 sum_k s_k (observations in id order)
  for (int lp = lane; lp < g.npts; lp += 32) {
    const long long ip = g.pb + lp;
    const double* hi = d.hinv + ip * 6;
    const double h0 = hi[0], h1 = hi[1], h2 = hi[2], h3 = hi[3], h4 = hi[4], h5 = hi[5];
    double w0 = 0.0, w1 = 0.0, w2 = 0.0;
    const int q1 = ws.pptr[lp + 1];
    for (int q = ws.pptr[lp]; q < q1; ++q) {
      const int s = ws.ptl[q];
      w0 += ws.stage[s];
      w1 += ws.stage[nobs + s];
      w2 += ws.stage[2 * nobs + s];
    }
    ws.pt[lp * 3] = h0 * w0 + h1 * w1 + h2 * w2;
    ws.pt[lp * 3 + 1] = h1 * w0 + h3 * w1 + h4 * w2;
    ws.pt[lp * 3 + 2] = h2 * w0 + h4 * w1 + h5 * w2;
  }
  __syncwarp();
  if (d.trace && lane == 0) d.trace[(long long)g.trace_id * 8 + 3] = global_ns();
  // phase 3: z_k = J_c^T J_p t_p -> stage rows 0..5 (overwrites s_k)
#pragma unroll
  for (int r = 0; r < kCacheRounds; ++r) {
    const int s = r * 32 + lane;
    if (s < nobs) {
      const double* cam = ws.cam + (lc[r] & 0xffff) * 24;
      double z[6];
      jct_jp_t(cD[r], cy[r], cam, ws.pt + (lc[r] >> 16) * 3, z);
#pragma unroll
      for (int j = 0; j < 6; ++j) ws.stage[j * nobs + s] = z[j];
    }
  }
  for (int s = kCacheRounds * 32 + lane; s < nobs; s += 32) {
    const std::uint32_t l = d.obs_lcpt[g.ob + s];
    const double* cam = ws.cam + (l & 0xffff) * 24;
    const double* p = d.pts + (long long)(g.pb + (l >> 16)) * 3;
    const double pp[3] = {p[0], p[1], p[2]};
    P3 y;
    double D[6], z[6];
    obs_geometry(d.pinhole, cam, pp, y, D);
    jct_jp_t(D, y, cam, ws.pt + (l >> 16) * 3, z);
#pragma unroll
    for (int j = 0; j < 6; ++j) ws.stage[j * nobs + s] = z[j];
  }
  __syncwarp();
  if (d.trace && lane == 0) d.trace[(long long)g.trace_id * 8 + 4] = global_ns();
  // one lane per tile camera: its 6-vector summed over its slot range, slot order
  for (int e = lane; e < g.ncam; e += 32) {
    const int b = ws.ent[e], en = ws.ent[e + 1];
    double a[6] = {0, 0, 0, 0, 0, 0};
    for (int q = b; q < en; ++q)
#pragma unroll
      for (int j = 0; j < 6; ++j) a[j] += ws.stage[j * nobs + q];
    double* out = d.partial + (long long)(g.eb + e) * 6;
#pragma unroll
    for (int j = 0; j < 6; ++j) out[j] = a[j];
  }
  __syncwarp();  // the slice is reused by this warp's next tile
}

__device__ __forceinline__ void sx_tile(const Dev& d, const PcgDev& st, int t, char* smem, int slice) {
  const TileGeom g = tile_geom(d, t);
  if (g.nobs == 0) return;
  if (g.big >= 0)
    sx_tile_impl<false>(d, st, g, smem, slice);
  else
    sx_tile_impl<true>(d, st, g, smem, slice);
}

// ---------------------------------------------------------------------------
// K5 pipelined: the same implicit Schur product for small tiles, with every
// tile input brought in by TMA bulk copies (cp.async.bulk + mbarrier) into a
// per-warp double buffer. While a warp computes tile i, the index blob, point
// window and H~_pp^-1 of its next tile are in flight (level A); the next
// tile's camera records and direction vectors (level C, addressed by the
// blob's camera ids) are issued right after phase 1. A tile's memory latency
// is thus overlapped with the previous tile's arithmetic.
// ---------------------------------------------------------------------------
__device__ __forceinline__ void pipe_issue_a(const Dev& d, int t, char* buf, unsigned long long* bar) {
  fence_proxy_async();
  __syncwarp();
  if (lane_id() == 0) {
    const int4 ds = d.tile_desc[t];  // blob/16, blob bytes, first point, points
    const long long pb = ds.z;
    const int npts = ds.w;
    const char* ps = reinterpret_cast<const char*>(d.pts + pb * 3);
    const unsigned long long a0 = reinterpret_cast<unsigned long long>(ps) & ~15ull;
    const unsigned long long a1 = (reinterpret_cast<unsigned long long>(ps + npts * 24) + 15) & ~15ull;
    const unsigned pbytes = static_cast<unsigned>(a1 - a0);
    const unsigned hbytes = static_cast<unsigned>(npts) * 48u;
    mbar_expect_tx(bar, static_cast<unsigned>(ds.y) + pbytes + hbytes);
    bulk_g2s(buf + kBufBlob, d.tile_blob + static_cast<long long>(ds.x) * 16, static_cast<unsigned>(ds.y), bar);
    bulk_g2s(buf + kBufPts, reinterpret_cast<const void*>(a0), pbytes, bar);
    bulk_g2s(buf + kBufHinv, d.hinv + pb * 6, hbytes, bar);
  }
}

__device__ __forceinline__ void pipe_issue_c(const Dev& d, const PcgDev& st, char* buf, unsigned long long* bar) {
  const int* hdr = reinterpret_cast<const int*>(buf + kBufBlob);
  const int ncam = hdr[5];
  const bool two = st.dir == kDirZBetaP;
  const double* va = st.dir == kDirX ? d.x : d.z;
  fence_proxy_async();
  __syncwarp();
  const int lane = lane_id();
  if (lane == 0) mbar_expect_tx(bar, static_cast<unsigned>(ncam) * (two ? 224u : 176u));
  __syncwarp();
  if (lane < ncam) {
    const long long c = hdr[8 + lane];
    bulk_g2s(buf + kBufCam + lane * 128, d.camrec + c * kCamRec, 128u, bar);
    bulk_g2s(buf + kBufVz + lane * 48, va + c * 6, 48u, bar);
    if (two) bulk_g2s(buf + kBufVp + lane * 48, d.p + c * 6, 48u, bar);
  }
}

// Computes one small tile whose level-A and level-C data have landed in
// `buf`; `next` (optional) issues the next tile's level C after phase 1.
template <class Next>
__device__ __forceinline__ void sx_pipe_tile(const Dev& d, const PcgDev& st, char* buf, char* wsm, Next next) {
  const int lane = lane_id();
  const int* hdr = reinterpret_cast<const int*>(buf + kBufBlob);
  const int nobs = hdr[1], pb = hdr[2], npts = hdr[3], eb = hdr[4], ncam = hdr[5];
  const int* ent = hdr + 8 + ncam;
  const int* pptr = ent + ncam + 1;
  const std::uint32_t* lcpt = reinterpret_cast<const std::uint32_t*>(pptr + npts + 1);
  const std::uint16_t* ptl = reinterpret_cast<const std::uint16_t*>(lcpt + nobs);
  const double* pts = reinterpret_cast<const double*>(buf + kBufPts + ((pb * 24) & 15));
  const double* hinv = reinterpret_cast<const double*>(buf + kBufHinv);
  const double* cams = reinterpret_cast<const double*>(buf + kBufCam);
  double* vz = reinterpret_cast<double*>(buf + kBufVz);
  double* stage = reinterpret_cast<double*>(wsm + kScrStage);
  double* tp = reinterpret_cast<double*>(wsm + kScrTp);
  if (st.dir == kDirZBetaP) {  // v = z + beta p, the same fused expression as the camera part
    const double* vp = reinterpret_cast<const double*>(buf + kBufVp);
    for (int i = lane; i < ncam * 6; i += 32) vz[i] = fma(st.beta, vp[i], vz[i]);
    __syncwarp();
  }
  // phase 1: s_k = J_p^T J_c v
  constexpr int kRounds = (kPipeObs + 31) / 32;  // observations per lane
  double cD[kRounds][6];
  P3 cy[kRounds];
  std::uint32_t lc[kRounds];
#pragma unroll
  for (int r = 0; r < kRounds; ++r) {
    const int s = r * 32 + lane;
    lc[r] = lcpt[min(s, nobs - 1)];
    if (s < nobs) {
      const int l = lc[r] & 0xffff;
      const double* cam = cams + l * 16;
      obs_geometry(d.pinhole, cam, pts + (lc[r] >> 16) * 3, cy[r], cD[r]);
      double sv[3];
      jpt_jc_v(cD[r], cy[r], cam, vz + l * 6, sv);
      stage[s] = sv[0];
      stage[kPipeObs + s] = sv[1];
      stage[2 * kPipeObs + s] = sv[2];
    }
  }
  __syncwarp();
  next();  // the next tile's camera gathers fly during the rest of this tile
  // point phase: t_p = H~_pp^-1 sum_k s_k (observations in id order)
  if (lane < npts) {
    const double* hi = hinv + lane * 6;
    double w0 = 0.0, w1 = 0.0, w2 = 0.0;
    for (int q = pptr[lane]; q < pptr[lane + 1]; ++q) {
      const int s = ptl[q];
      w0 += stage[s];
      w1 += stage[kPipeObs + s];
      w2 += stage[2 * kPipeObs + s];
    }
    tp[lane * 3] = hi[0] * w0 + hi[1] * w1 + hi[2] * w2;
    tp[lane * 3 + 1] = hi[1] * w0 + hi[3] * w1 + hi[4] * w2;
    tp[lane * 3 + 2] = hi[2] * w0 + hi[4] * w1 + hi[5] * w2;
  }
  __syncwarp();
  // phase 3: z_k = J_c^T J_p t_p -> stage rows 0..5
#pragma unroll
  for (int r = 0; r < kRounds; ++r) {
    const int s = r * 32 + lane;
    if (s < nobs) {
      double z[6];
      jct_jp_t(cD[r], cy[r], cams + (lc[r] & 0xffff) * 16, tp + (lc[r] >> 16) * 3, z);
#pragma unroll
      for (int j = 0; j < 6; ++j) stage[j * kPipeObs + s] = z[j];
    }
  }
  __syncwarp();
  // one lane per tile camera: its 6-vector over its slot range, slot order
  if (lane < ncam) {
    double a[6] = {0, 0, 0, 0, 0, 0};
    for (int q = ent[lane]; q < ent[lane + 1]; ++q)
#pragma unroll
      for (int j = 0; j < 6; ++j) a[j] += stage[j * kPipeObs + q];
    double* out = d.partial + static_cast<long long>(eb + lane) * 6;
#pragma unroll
    for (int j = 0; j < 6; ++j) out[j] = a[j];
  }
  __syncwarp();
}

// Per-warp pipeline state: mbarriers A0 A1 C0 C1 live at wsm + kScrBar and
// are initialised once per kernel; their phase parities persist across calls.
struct PipeState {
  unsigned pa0 = 0, pa1 = 0, pc0 = 0, pc1 = 0;
};
__device__ __forceinline__ void pipe_init(char* wsm) {
  unsigned long long* bar = reinterpret_cast<unsigned long long*>(wsm + kScrBar);
  if (lane_id() == 0) {
#pragma unroll
    for (int k = 0; k < 4; ++k) mbar_init(bar + k, 1);
    mbar_fence_init();
  }
  __syncwarp();
}

// All small tiles of this warp (gwarp, gwarp + nwarps, ...), software
// pipelined through the two buffers of the warp's shared-memory slice.
__device__ __forceinline__ void sx_pipelined(const Dev& d, const PcgDev& st, char* wsm, int gwarp, int nwarps,
                                             PipeState& ps) {
  char* buf[2] = {wsm, wsm + kBufBytes};
  unsigned long long* bar = reinterpret_cast<unsigned long long*>(wsm + kScrBar);  // A0 A1 C0 C1
  unsigned& pa0 = ps.pa0;
  unsigned& pa1 = ps.pa1;
  unsigned& pc0 = ps.pc0;
  unsigned& pc1 = ps.pc1;
  int i = gwarp;
  if (i >= d.n_small) return;
  pipe_issue_a(d, d.small_tiles[i], buf[0], bar + 0);
  mbar_wait(bar + 0, pa0);
  pa0 ^= 1;
  pipe_issue_c(d, st, buf[0], bar + 2);
  int b = 0;
  for (; i < d.n_small; i += nwarps) {
    const int in = i + nwarps;
    const bool more = in < d.n_small;
    if (more) pipe_issue_a(d, d.small_tiles[in], buf[b ^ 1], bar + (b ^ 1));
    if (b == 0) {
      mbar_wait(bar + 2, pc0);
      pc0 ^= 1;
    } else {
      mbar_wait(bar + 3, pc1);
      pc1 ^= 1;
    }
    sx_pipe_tile(d, st, buf[b], wsm, [&] {
      if (!more) return;
      if (b == 0) {
        mbar_wait(bar + 1, pa1);
        pa1 ^= 1;
      } else {
        mbar_wait(bar + 0, pa0);
        pa0 ^= 1;
      }
      pipe_issue_c(d, st, buf[b ^ 1], bar + 2 + (b ^ 1));
    });
    b ^= 1;
  }
}

// K5 camera part for one camera (warp; persistent single-rank PCG):
// y_c = H~_cc v_c - sum partial, p <- v. Returns v.y (lane 0).
__device__ __forceinline__ double sx_camera(const Dev& d, const PcgDev& st, int c) {
  double acc[6];
  warp_entry_sum<6>(d, c, acc);
  double pap = 0.0;
  if (lane_id() == 0) {
    double v[6];
    dir_vector(st, d, c, v);
    const double* h = d.hccd + (long long)c * 21;
#pragma unroll
    for (int a = 0; a < 6; ++a) {
      double hv = 0.0;
#pragma unroll
      for (int b = 0; b < 6; ++b) hv += h[sym6(a, b)] * v[b];
      const double yy = hv - acc[a];
      d.y[(long long)c * 6 + a] = yy;
      if (st.dir != kDirX) d.p[(long long)c * 6 + a] = v[a];
      pap += v[a] * yy;
    }
  }
  return pap;
}

// PCG vector update for one camera (pcg.hpp:78-117): accumulates r.r, r.z.
__device__ __forceinline__ void pcg_camera_update(const Dev& d, const PcgDev& st, double alpha, int c, double& rr,
                                                  double& rz) {
  double rv[6];
#pragma unroll
  for (int a = 0; a < 6; ++a) {
    const long long o = (long long)c * 6 + a;
    if (st.state == kPcgIter) {
      d.x[o] += alpha * d.p[o];
      rv[a] = d.r[o] - alpha * d.y[o];
    } else {  // verify: true residual b - S x
      rv[a] = d.rhs[o] - d.y[o];
    }
    d.r[o] = rv[a];
    rr += rv[a] * rv[a];
  }
  const double* m = d.minv + (long long)c * 36;
#pragma unroll
  for (int a = 0; a < 6; ++a) {
    double zz = 0.0;
#pragma unroll
    for (int b = 0; b < 6; ++b) zz += m[a * 6 + b] * rv[b];
    d.z[(long long)c * 6 + a] = zz;
    rz += rv[a] * zz;
  }
}

// Recurrence / true-residual state machine (pcg.hpp:68-129) on the grid
// totals r.r and r.z; identical in every block that evaluates it.
__host__ __device__ __forceinline__ void pcg_decide(PcgDev& o, double rr, double rz_new) {
  const double rnorm = sqrt(rr);
  o.rnorm = rnorm;
  if (o.state == kPcgIter) {
    o.iters += 1;
    if (!isfinite(rnorm)) {
      o.state = kPcgBreakdown;
    } else if (rnorm <= o.tol * o.bnorm) {
      o.state = kPcgVerify;  // confirm with the true residual (pcg.hpp:86-109)
      o.dir = kDirX;
    } else {
      const double beta = rz_new / o.rz;
      if (!isfinite(beta)) {
        o.state = kPcgBreakdown;
      } else {
        o.beta = beta;
        o.rz = rz_new;
        o.dir = kDirZBetaP;
        if (o.iters >= o.budget) o.state = kPcgDone;
      }
    }
  } else {
    o.true_norm = rnorm;
    if (rnorm <= o.tol * o.bnorm) {
      o.state = kPcgDone;
      o.converged = 1;
    } else {  // restart from the true residual
      o.rz = rz_new;
      o.beta = 0.0;
      o.dir = kDirZ;
      o.state = (o.iters >= o.budget) ? kPcgDone : kPcgIter;
    }
  }
}

// Standalone S*v tile pass (graph-mode PCG and kernel timing): persistent
// grid, pipelined small tiles, then the rare big tiles from global scratch.
__device__ __forceinline__ void sx_all_tiles(const Dev& d, const PcgDev& st, char* smem, int gwarp, int nwarps,
                                             PipeState& ps) {
  sx_pipelined(d, st, smem + (threadIdx.x >> 5) * kPipeWarpBytes, gwarp, nwarps, ps);
  for (int i = gwarp; i < d.n_big_tiles; i += nwarps) sx_tile(d, st, d.big_tiles[i], smem, 0);
}

__global__ void __maxnreg__(kSchurMaxReg) k_schur_tiles(Dev d, int slice) {
  extern __shared__ __align__(128) char smem[];
  grid_dep_wait();
  const PcgDev st = *d.pcg;
  if (st.state >= kPcgDone) return;
  const int wpb = blockDim.x >> 5;
  pipe_init(smem + (threadIdx.x >> 5) * kPipeWarpBytes);
  PipeState ps;
  sx_all_tiles(d, st, smem, blockIdx.x * wpb + (threadIdx.x >> 5), gridDim.x * wpb, ps);
}

// K5 camera part (block per camera): y_c = H~_cc v_c - sum of the camera's
// entry partials (rank-summed on sharded runs), p <- v, and v.y per camera.
__global__ void __launch_bounds__(128) k_schur_cams(Dev d) {
  __shared__ double red[20 * 6];
  __shared__ double acc[6];
  grid_dep_wait();
  const PcgDev st = *d.pcg;
  if (st.state >= kPcgDone) return;
  const int c = blockIdx.x;
  cam_block_acc<6, 128>(d, c, red, acc);
  if (threadIdx.x != 0) return;
  double v[6];
  dir_vector(st, d, c, v);
  const double* h = d.hccd + (long long)c * 21;
  double pap = 0.0;
#pragma unroll
  for (int a = 0; a < 6; ++a) {
    double hv = 0.0;
#pragma unroll
    for (int b = 0; b < 6; ++b) hv += h[sym6(a, b)] * v[b];
    const double yy = hv - acc[a];
    d.y[(long long)c * 6 + a] = yy;
    if (st.dir != kDirX) d.p[(long long)c * 6 + a] = v[a];
    pap += v[a] * yy;
  }
  d.cam_dot[c] = pap;
}

// PCG step on the camera vectors (pcg.hpp:73-129), a thread per camera:
// every block forms p.Sp from the per-camera dots in the same fixed order
// (so all blocks hold the identical alpha), updates x, r, z of its cameras,
// and the last block to finish sums the blocks' r.r, r.z in block order and
// runs the recurrence / true-residual decision.
constexpr int kUpdNT = 256;
__global__ void __launch_bounds__(kUpdNT) k_pcg_update(Dev d) {
  __shared__ double red[32];
  __shared__ double s_pap;
  grid_dep_wait();
  const PcgDev st = *d.pcg;
  if (st.state >= kPcgDone) return;
  double alpha = 0.0;
  if (st.dir != kDirX) {
    double pap = 0.0;
    for (int c = threadIdx.x; c < d.C; c += blockDim.x) pap += d.cam_dot[c];
    pap = block_sum(pap, red);
    if (threadIdx.x == 0) s_pap = pap;
    __syncthreads();
    alpha = st.rz / s_pap;
    if (!isfinite(alpha)) {  // pcg.hpp:77 (every block sees it and stops)
      if (blockIdx.x == 0 && threadIdx.x == 0) d.pcg->state = kPcgBreakdown;
      return;
    }
  }
  double rr = 0.0, rz = 0.0;
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c < d.C) pcg_camera_update(d, st, alpha, c, rr, rz);
  __syncthreads();
  rr = block_sum(rr, red);
  __syncthreads();
  rz = block_sum(rz, red);
  const double part[2] = {rr, rz};
  double tot[2];
  if (grid_reduce<2>(part, d.block_red, d.tickets, tot) && threadIdx.x == 0) {
    PcgDev o = st;
    o.alpha = alpha;
    pcg_decide(o, tot[0], tot[1]);
    *d.pcg = o;
  }
}

// Sum of per-block partials in block order, identical in every block (one
// warp: lane-strided sums, fixed xor tree). Valid in all lanes.
template <int K>
__device__ __forceinline__ void sum_block_partials(const double* part, int nblocks, double (&tot)[K]) {
  const int lane = lane_id();
#pragma unroll
  for (int k = 0; k < K; ++k) tot[k] = 0.0;
  for (int b = lane; b < nblocks; b += 32)
#pragma unroll
    for (int k = 0; k < K; ++k) tot[k] += __ldcg(part + (long long)b * K + k);
#pragma unroll
  for (int k = 0; k < K; ++k) tot[k] = warp_sum(tot[k]);
}

// Whole PCG solve in one cooperative launch: warp-tiles, camera reduction and
// vector update separated by grid barriers; the scalar recurrence is
// evaluated redundantly (bit-identically) by every block, so no block waits
// on another for alpha / beta. Runs up to max_iters iterations per launch.
__global__ void __launch_bounds__(32 * kSchurWarps, 2) k_pcg_persistent(Dev d, int slice, long long max_iters) {
  namespace cg = cooperative_groups;
  cg::grid_group grid = cg::this_grid();
  extern __shared__ __align__(128) char smem[];
  __shared__ double red[32];
  __shared__ PcgDev st;
  __shared__ double s_tot[2];
  if (threadIdx.x == 0) st = *d.pcg;
  __syncthreads();
  double* partB = d.block_red;              // gridDim doubles
  double* partC = d.block_red + gridDim.x;  // 2 * gridDim doubles
  const int wpb = blockDim.x >> 5;
  const int gwarp = blockIdx.x * wpb + (threadIdx.x >> 5);
  const int nwarps = gridDim.x * wpb;
  const long long stop_at = st.iters + max_iters;
  pipe_init(smem + (threadIdx.x >> 5) * kPipeWarpBytes);
  PipeState ps;
  while (st.state < kPcgDone && st.iters < stop_at) {
    const PcgDev cur = st;
    // A: warp-tiles (pipelined small tiles, then big tiles)
    sx_all_tiles(d, cur, smem, gwarp, nwarps, ps);
    grid.sync();
    // B: cameras (warp per camera)
    double pap = 0.0;
    for (int c = gwarp; c < d.C; c += nwarps) pap += sx_camera(d, cur, c);
    pap = block_sum(pap, red);
    if (threadIdx.x == 0) partB[blockIdx.x] = pap;
    grid.sync();
    if (threadIdx.x < 32) {
      double tot[1];
      sum_block_partials<1>(partB, gridDim.x, tot);
      if (threadIdx.x == 0) s_tot[0] = tot[0];
    }
    __syncthreads();
    double alpha = 0.0;
    if (cur.state == kPcgIter) {
      alpha = cur.rz / s_tot[0];
      if (!isfinite(alpha)) {  // pcg.hpp:77: identical decision in every block
        if (threadIdx.x == 0) st.state = kPcgBreakdown;
        __syncthreads();
        break;
      }
    }
    // C: vector update (thread per camera)
    double rr = 0.0, rz = 0.0;
    for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < d.C; c += gridDim.x * blockDim.x)
      pcg_camera_update(d, cur, alpha, c, rr, rz);
    rr = block_sum(rr, red);
    __syncthreads();
    rz = block_sum(rz, red);
    if (threadIdx.x == 0) {
      partC[2 * blockIdx.x] = rr;
      partC[2 * blockIdx.x + 1] = rz;
    }
    grid.sync();
    if (threadIdx.x < 32) {
      double tot[2];
      sum_block_partials<2>(partC, gridDim.x, tot);
      if (threadIdx.x == 0) {
        PcgDev o = cur;
        o.alpha = alpha;
        pcg_decide(o, tot[0], tot[1]);
        st = o;
      }
    }
    __syncthreads();
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) *d.pcg = st;
}

// ---------------------------------------------------------------------------
// K7 + K8: camera retraction Exp(dc) o T (lm.hpp:157-167) into the trial
// buffers, then point back-substitution + trial cost in one tile pass.
// ---------------------------------------------------------------------------
__global__ void k_cam_retract(Dev d) {
  grid_dep_wait();
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= d.C) return;
  const double* s = d.pose + (long long)c * 7;
  double tau[6];
#pragma unroll
  for (int j = 0; j < 6; ++j) tau[j] = d.x[(long long)c * 6 + j];
  Q4 q;
  P3 t;
  if (!se3_retract({s[3], s[4], s[5], s[6]}, {s[0], s[1], s[2]}, tau, q, t)) {
    atomicExch(&d.lm->retract_bad, 1);
    q = {s[3], s[4], s[5], s[6]};
    t = {s[0], s[1], s[2]};
  }
  double* o = d.pose_t + (long long)c * 7;
  o[0] = t.x;
  o[1] = t.y;
  o[2] = t.z;
  o[3] = q.x;
  o[4] = q.y;
  o[5] = q.z;
  o[6] = q.w;
  double* rec = d.camrec_t + (long long)c * kCamRec;
  quat_to_R(q, rec);
  rec[9] = t.x;
  rec[10] = t.y;
  rec[11] = t.z;
  rec[12] = d.intr[c * 4];
  rec[13] = d.intr[c * 4 + 1];
  rec[14] = d.intr[c * 4 + 2];
  rec[15] = d.intr[c * 4 + 3];
}

// cam: R9 t3 k4 dc6 | trial t3 q4 (29), intrinsics at 12..15 ; pt: p3 ptrial3 ; stage 3

template <bool kShared>
__device__ __forceinline__ void trial_tile(const Dev& d, const TileGeom& g, char* smem, int slice, int t) {
  const Ws ws = ws_carve(ws_base<kShared>(d, g, smem, slice), kTrialWs, g.ncam, g.npts, g.nobs);
  const int lane = lane_id();
  load_point_fields<3>(ws, 6, 0, d.pts, g.pb, g.npts);
  load_tile_index(d, g, ws);
  __syncwarp();
  load_cam_fields<16>(ws, g.ncam, 29, 0, d.camrec, kCamRec);
  load_cam_fields<6>(ws, g.ncam, 29, 16, d.x, 6);
  load_cam_fields<7>(ws, g.ncam, 29, 22, d.pose_t, 7);
  __syncwarp();
  for (int s = lane; s < g.nobs; s += 32) {
    const std::uint32_t lcpt = ws.lcpt[s];
    const double* cam = ws.cam + (lcpt & 0xffff) * 29;
    P3 y;
    double D[6];
    obs_geometry(d.pinhole, cam, ws.pt + (lcpt >> 16) * 6, y, D);
    jpt_jc_v(D, y, cam, cam + 16, ws.stage + s * 3);
  }
  __syncwarp();
  // Delta p = H~_pp^-1 (-g_p - sum_k J_p^T J_c dc), p_trial = p + Delta p
  for (int lp = lane; lp < g.npts; lp += 32) {
    const long long ip = g.pb + lp;
    double w0 = 0.0, w1 = 0.0, w2 = 0.0;
    for (int q = ws.pptr[lp]; q < ws.pptr[lp + 1]; ++q) {
      const double* sv = ws.stage + ws.ptl[q] * 3;
      w0 += sv[0];
      w1 += sv[1];
      w2 += sv[2];
    }
    const double b0 = -d.gp[ip * 3] - w0, b1 = -d.gp[ip * 3 + 1] - w1, b2 = -d.gp[ip * 3 + 2] - w2;
    const double* hi = d.hinv + ip * 6;
    const double dp0 = hi[0] * b0 + hi[1] * b1 + hi[2] * b2;
    const double dp1 = hi[1] * b0 + hi[3] * b1 + hi[4] * b2;
    const double dp2 = hi[2] * b0 + hi[4] * b1 + hi[5] * b2;
    double* sp = ws.pt + lp * 6;
    const double n0 = sp[0] + dp0, n1 = sp[1] + dp1, n2 = sp[2] + dp2;  // lm.hpp:168-173
    sp[3] = n0;
    sp[4] = n1;
    sp[5] = n2;
    d.dp[ip * 3] = dp0;
    d.dp[ip * 3 + 1] = dp1;
    d.dp[ip * 3 + 2] = dp2;
    d.pts_t[ip * 3] = n0;
    d.pts_t[ip * 3 + 1] = n1;
    d.pts_t[ip * 3 + 2] = n2;
  }
  __syncwarp();
  SplitSum cost;
  int bad = 0;
  for (int s = lane; s < g.nobs; s += 32) {
    const std::uint32_t lcpt = ws.lcpt[s];
    const double* cam = ws.cam + (lcpt & 0xffff) * 29;
    const double* pt = ws.pt + (lcpt >> 16) * 6 + 3;
    // trial camera in the [t3 q4 k4] layout of residual()
    const double tc[11] = {cam[22], cam[23], cam[24], cam[25], cam[26], cam[27], cam[28],
                           cam[12], cam[13], cam[14], cam[15]};
    const double2 px = reinterpret_cast<const double2*>(d.obs_px)[g.ob + s];
    double r0, r1;
    P3 y;
    if (residual(d.pinhole, tc, pt, px, r0, r1, y))
      cost.add(s, r0 * r0 + r1 * r1);
    else
      bad = 1;  // CheiralityError in the trial evaluate -> cost = inf (lm.hpp:176-181)
  }
  if (bad) atomicExch(&d.lm->trial_bad, 1);
  const double ct = cost.warp_total();
  if (lane == 0) d.tile_red[t * 2] = ct;
  __syncwarp();
}

__global__ void __launch_bounds__(256) k_backsub_trial(Dev d, int slice, int pf) {
  grid_dep_wait();
  extern __shared__ __align__(16) char smem[];
  const int t = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (t >= d.T) return;
  const TileSpan nx = pf > 0 && lane_id() == 0 ? tile_span(d, t + pf) : TileSpan{0, 0, 0, 0, 0, 0};
  const TileGeom g = tile_geom(d, t);
  if (lane_id() == 0) prefetch_tile(d, nx, d.gp, 3, d.hinv, 6);  // one wave ahead
  BAE_TILE_DISPATCH(trial_tile, d, g, smem, slice, t);
}

// Accept: trial parameters become current (lm.hpp:183-189).
__global__ void k_commit(Dev d) {
  grid_dep_wait();
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < (long long)d.P * 3) d.pts[i] = d.pts_t[i];
  if (i < (long long)d.C * 7) d.pose[i] = d.pose_t[i];
  if (i < (long long)d.C * kCamRec) d.camrec[i] = d.camrec_t[i];
}

// ---------------------------------------------------------------------------
// launch wrappers
// ---------------------------------------------------------------------------
long long tile_ws_bytes(int kind, int ncam, int npts, int nobs) { return kind_ws_bytes(kind, ncam, npts, nobs); }

static int resident_grid(const void* fn, int threads, int smem);
// Tiles of one resident wave of a warp-tile kernel (its L2 prefetch
// distance); BAE_PREFETCH=<waves> (0 disables).
static int prefetch_distance(const void* fn, const TileLaunch& tl, int nt = 32) {
  static const int waves = [] {
    const char* e = std::getenv("BAE_PREFETCH");
    return e ? std::max(0, std::atoi(e)) : 1;
  }();
  if (!waves) return 0;
  return waves * resident_grid(fn, nt * tl.wpb, tl.wpb * tl.slice) * tl.wpb;
}


void set_smem_limits(int max_bytes) {
  cudaFuncSetAttribute(k_linearize, cudaFuncAttributeMaxDynamicSharedMemorySize, max_bytes);
  cudaFuncSetAttribute(k_lin_prep, cudaFuncAttributeMaxDynamicSharedMemorySize, max_bytes);
  cudaFuncSetAttribute(k_cost, cudaFuncAttributeMaxDynamicSharedMemorySize, max_bytes);
  cudaFuncSetAttribute(k_prep<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, max_bytes);
  cudaFuncSetAttribute(k_prep<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, max_bytes);
  cudaFuncSetAttribute(k_schur_tiles, cudaFuncAttributeMaxDynamicSharedMemorySize, max_bytes);
  cudaFuncSetAttribute(k_backsub_trial, cudaFuncAttributeMaxDynamicSharedMemorySize, max_bytes);
  cudaFuncSetAttribute(k_pcg_persistent, cudaFuncAttributeMaxDynamicSharedMemorySize, max_bytes);
}

static inline int cam_blocks(int C) { return (C + kWarpsPerCamBlock - 1) / kWarpsPerCamBlock; }
static inline int elt_blocks(long long n, int bs) { return (int)((n + bs - 1) / bs); }
static inline int tile_blocks(int T, const TileLaunch& tl) { return (T + tl.wpb - 1) / tl.wpb; }
static int schur_grid(const Dev& d, const SmemSizes& sm);

// Points between the caller's order and the internal (camera-sorted) order:
// internal point i is caller point src[i].
__global__ void k_points_permute(const double* __restrict__ in, const int* __restrict__ src, double* __restrict__ out,
                                 int P, int to_internal) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= P) return;
  const long long u = 3LL * src[i], v = 3LL * i;
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    if (to_internal)
      out[v + a] = in[u + a];
    else
      out[u + a] = in[v + a];
  }
}
int launch_points_permute(const double* in, const int* src, double* out, int P, bool to_internal, cudaStream_t s) {
  k_points_permute<<<elt_blocks(P, 256), 256, 0, s>>>(in, src, out, P, to_internal ? 1 : 0);
  return 1;
}

// Observation pixels from the caller's order into slot order.
__global__ void k_gather_pixels(const double2* __restrict__ raw, const int* __restrict__ orig, double2* __restrict__ px,
                                long long N) {
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i < N) px[i] = raw[orig[i]];
}
int launch_gather_pixels(const double* raw, const int* orig, double* px, long long N, cudaStream_t s) {
  k_gather_pixels<<<static_cast<unsigned>((N + 255) / 256), 256, 0, s>>>(reinterpret_cast<const double2*>(raw), orig,
                                                                      reinterpret_cast<double2*>(px), N);
  return 1;
}

// Programmatic dependent launch: the kernel may be scheduled while its
// predecessor in the stream drains (its blocks wait in griddepcontrol.wait,
// the first statement of every kernel launched this way), so kernel
// boundaries cost no launch gap; in a captured graph the edge becomes a
// programmatic one. BAE_PDL=0 turns it off. Sharded runs keep plain
// launches (their exchanges sit between the kernels).
static bool pdl_on() {
  static const bool on = [] {
    const char* e = std::getenv("BAE_PDL");
    return !(e && e[0] == '0');
  }();
  return on;
}
template <class... K, class... A>
static void launch_k(bool pdl, void (*k)(K...), dim3 grid, dim3 block, std::size_t smem, cudaStream_t s,
                     A&&... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = (pdl && pdl_on()) ? 1 : 0;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, k, std::forward<A>(args)...);
}

template <class... K, class... A>
static void launch_pdl(void (*k)(K...), dim3 grid, dim3 block, std::size_t smem, cudaStream_t s, A&&... args) {
  launch_k(true, k, grid, block, smem, s, std::forward<A>(args)...);
}

int launch_camrec(const Dev& d, bool trial, cudaStream_t s) {
  k_camrec<<<elt_blocks(d.C, 128), 128, 0, s>>>(trial ? d.pose_t : d.pose, d.intr, trial ? d.camrec_t : d.camrec, d.C);
  return 1;
}
// Sharded runs: this rank's camera partials -> cross-rank sum in d.cred.
// (the same block layout as the single-rank camera pass it stands in for:
// the linearisation's kCamNT, the PCG prep's 256)
static int reduce_cams27(const Dev& d, int extra, int nextra, Comm* comm, cudaStream_t s) {
  if (extra == 1)
    k_cam_entry_sums<27, kCamNT><<<d.C + 1, kCamNT, 0, s>>>(d, extra, 0);
  else
    k_cam_entry_sums<27, 256><<<d.C + 1, 256, 0, s>>>(d, extra, 0);
  comm->allreduce_sum(d.cred, 27 * static_cast<std::size_t>(d.C) + nextra, s);
  return 1;
}
int launch_linearize(const Dev& d, const SmemSizes& sm, bool write_jac, cudaStream_t s, Comm* comm) {
  int n = 3;
  launch_k(!comm, k_linearize, tile_blocks(d.T, sm.lin), 32 * sm.lin.wpb, sm.lin.wpb * sm.lin.slice, s, d,
           sm.lin.slice, write_jac ? 1 : 0, prefetch_distance((const void*)k_linearize, sm.lin));
  if (comm) {
    n += reduce_cams27(d, 1, 2, comm, s);
    comm->allreduce_min(&d.lm->err_obs, 1, s);
  }
  launch_k(!comm, k_cam_linearize, d.C, kCamNT, 0, s, d);
  launch_k(!comm, k_lin_totals, 1, 1024, 0, s, d);
  return n;
}
int launch_lin_prep_tiles(const Dev& d, const SmemSizes& sm, double clo, double chi, cudaStream_t s) {
  launch_k(true, k_lin_prep, tile_blocks(d.T, sm.linprep), kLinThreads * sm.linprep.wpb,
           sm.linprep.wpb * sm.linprep.slice, s, d, sm.linprep.slice, clo, chi,
           prefetch_distance((const void*)k_lin_prep, sm.linprep, kLinThreads));
  return 1;
}
int launch_lin_prep_cams(const Dev& d, double clo, double chi, cudaStream_t s) {
  launch_k(true, k_cam_lin_prep, d.C, kCamNT, 0, s, d, clo, chi);
  launch_k(true, k_lin_totals, 1, 1024, 0, s, d);
  return 2;
}
int launch_lin_prep(const Dev& d, const SmemSizes& sm, double clo, double chi, cudaStream_t s) {
  return launch_lin_prep_tiles(d, sm, clo, chi, s) + launch_lin_prep_cams(d, clo, chi, s);
}
int launch_cost(const Dev& d, const SmemSizes& sm, cudaStream_t s, Comm* comm) {
  launch_k(!comm, k_cost, tile_blocks(d.T, sm.cost), 32 * sm.cost.wpb, sm.cost.wpb * sm.cost.slice, s, d,
           sm.cost.slice);
  launch_k(!comm, k_sum_tiles, 1, 1024, 0, s, d, 0);
  if (!comm) return 2;
  comm->allreduce_sum(d.cred, 2, s);
  comm->allreduce_min(&d.lm->err_obs, 1, s);
  k_finish_cost<<<1, 1, 0, s>>>(d, 0);
  return 3;
}
int launch_prep(const Dev& d, const SmemSizes& sm, double lambda, double clo, double chi, double tol,
                long long budget, cudaStream_t s, Comm* comm, bool direct) {
  if (direct) {  // RHS, damped H_cc and the per-slot W / W H~^-1 only
    launch_k(!comm, (k_prep<true>), tile_blocks(d.T, sm.prepd), 32 * sm.prepd.wpb, sm.prepd.wpb * sm.prepd.slice, s,
             d, sm.prepd.slice, lambda, clo, chi, prefetch_distance((const void*)k_prep<true>, sm.prepd));
    int n = 2;
    if (comm) {
      k_cam_entry_sums<6, kCamNT><<<d.C + 1, kCamNT, 0, s>>>(d, 2, 0);
      comm->allreduce_sum(d.cred, 6 * static_cast<std::size_t>(d.C) + 1, s);
      ++n;
    }
    launch_k(!comm, k_cam_prep_direct, d.C, kCamNT, 0, s, d, lambda, clo, chi);
    return n;
  }
  int n = 3;
  launch_k(!comm, (k_prep<false>), tile_blocks(d.T, sm.prep), 32 * sm.prep.wpb, sm.prep.wpb * sm.prep.slice, s, d,
           sm.prep.slice, lambda, clo, chi, prefetch_distance((const void*)k_prep<false>, sm.prep));
  if (comm) n += reduce_cams27(d, 2, 1, comm, s);
  launch_k(!comm, k_cam_prep, d.C, 256, 0, s, d, lambda, clo, chi);
  launch_k(!comm, k_prep_totals, 1, 1024, 0, s, d, tol, budget);
  return n;
}
int launch_pcg_iteration(const Dev& d, const SmemSizes& sm, cudaStream_t s, Comm* comm) {
  int n = 3;
  if (comm) {  // the one exchange per PCG iteration: 6C doubles
    k_schur_tiles<<<schur_grid(d, sm), 32 * sm.schur.wpb, sm.schur.wpb * sm.schur.slice, s>>>(d, sm.schur.slice);
    k_cam_entry_sums<6, 128><<<d.C + 1, 128, 0, s>>>(d, 0, 1);
    comm->allreduce_sum(d.cred, 6 * static_cast<std::size_t>(d.C), s);
    k_schur_cams<<<d.C, 128, 0, s>>>(d);
    k_pcg_update<<<elt_blocks(d.C, kUpdNT), kUpdNT, 0, s>>>(d);
    return n + 1;
  }
  launch_pdl(k_schur_tiles, schur_grid(d, sm), 32 * sm.schur.wpb, sm.schur.wpb * sm.schur.slice, s, d,
             sm.schur.slice);
  launch_pdl(k_schur_cams, d.C, 128, 0, s, d);
  launch_pdl(k_pcg_update, elt_blocks(d.C, kUpdNT), kUpdNT, 0, s, d);
  return n;
}
static int resident_grid(const void* fn, int threads, int smem) {
  int per_sm = 0, dev = 0, nsm = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, threads, smem);
  return std::max(1, per_sm * nsm);
}
int pcg_persistent_grid(const Dev& d, const SmemSizes& sm) {
  const int cap = resident_grid((const void*)k_pcg_persistent, 32 * sm.schur.wpb, sm.schur.wpb * sm.schur.slice);
  const int want = std::max(std::max(tile_blocks(d.T, sm.schur), (d.C + sm.schur.wpb - 1) / sm.schur.wpb), 1);
  return std::max(1, std::min(cap, want));
}
static int schur_grid(const Dev& d, const SmemSizes& sm) {
  static int cap = 0;
  if (!cap) cap = resident_grid((const void*)k_schur_tiles, 32 * sm.schur.wpb, sm.schur.wpb * sm.schur.slice);
  return std::max(1, std::min(cap, tile_blocks(d.T, sm.schur)));
}
cudaError_t launch_pcg_persistent(const Dev& d, const SmemSizes& sm, int grid, long long max_iters, cudaStream_t s) {
  Dev dd = d;
  int slice = sm.schur.slice;
  void* args[] = {&dd, &slice, &max_iters};
  return cudaLaunchCooperativeKernel((void*)k_pcg_persistent, dim3(grid), dim3(32 * sm.schur.wpb), args,
                                     sm.schur.wpb * sm.schur.slice, s);
}
int launch_schur_only(const Dev& d, const SmemSizes& sm, cudaStream_t s) {
  k_schur_tiles<<<schur_grid(d, sm), 32 * sm.schur.wpb, sm.schur.wpb * sm.schur.slice, s>>>(d, sm.schur.slice);
  return 1;
}
int launch_trial(const Dev& d, const SmemSizes& sm, cudaStream_t s, Comm* comm) {
  launch_k(!comm, k_cam_retract, elt_blocks(d.C, 128), 128, 0, s, d);
  launch_k(!comm, k_backsub_trial, tile_blocks(d.T, sm.trial), 32 * sm.trial.wpb, sm.trial.wpb * sm.trial.slice, s,
           d, sm.trial.slice, prefetch_distance((const void*)k_backsub_trial, sm.trial));
  launch_k(!comm, k_sum_tiles, 1, 1024, 0, s, d, 1);
  if (!comm) return 3;
  comm->allreduce_sum(d.cred, 2, s);
  k_finish_cost<<<1, 1, 0, s>>>(d, 1);
  return 4;
}
int launch_schur_dense(const Dev& d, cudaStream_t s, Comm* comm, bool defer_hccd) {
  int n = 0;
  if (d.nblk > 0) {
    cudaMemsetAsync(d.blk_ticket, 0, sizeof(unsigned) * d.nblk, s);
    Dev dd = d;
    dd.defer_hccd = defer_hccd ? 1 : 0;
    k_schur_dense<<<(d.nchunk + kSchurDenseThreads / 32 - 1) / (kSchurDenseThreads / 32), kSchurDenseThreads, 0, s>>>(
        dd);
    ++n;
  }
  if (comm) {  // the direct solve's exchange: the reduced matrix, once per LM iteration
    const std::size_t nn = 6 * static_cast<std::size_t>(d.C);
    if (d.stiles) {  // summed onto rank 0, which factors it (solve_direct broadcasts the step)
      comm->reduce_sum(d.stiles, static_cast<std::size_t>(d.stile_count) * kSTileElems, 0, s);
      if (comm->rank() != 0) return n;
    } else {
      comm->allreduce_sum(d.schur, nn * nn, s);
    }
    k_add_hccd<<<elt_blocks(36LL * d.C, 256), 256, 0, s>>>(d);
    ++n;
  }
  return n;
}
int launch_add_hccd(const Dev& d, cudaStream_t s) {
  k_add_hccd<<<elt_blocks(36LL * d.C, 256), 256, 0, s>>>(d);
  return 1;
}
int launch_commit(const Dev& d, cudaStream_t s) {
  const long long n = std::max<long long>((long long)d.P * 3, (long long)d.C * kCamRec);
  launch_k(true, k_commit, elt_blocks(n, 256), 256, 0, s, d);
  return 1;
}

}  // namespace bae
