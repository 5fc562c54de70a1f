// sm_100a kernels of the BA hot path. FP64 throughout (the reference is FP64,
// SPEC.md:332). All camera-side sums are deterministic segmented reductions
// (no floating-point atomics); see device.cuh.
//
// Per-observation algebra (one observation k, camera c, point p, camera-frame
// point y = R p + t, D = d(pixel)/d(y) from camera.hpp:59-71):
//   J_c = D [I | -[y]x]   (2x6, trace.hpp:612-629: up * [I | -skew(y)])
//   J_p = D R             (2x3, trace.hpp:612-629: up * R)
//   J_c v   = D (v_rho + v_omega x y)         J_c^T e = [g ; y x g], g = D^T e
//   J_p t   = D (R t)                         J_p^T u = R^T (D^T u)
#include <cfloat>
#include <climits>

#include "device.cuh"
#include "kernels.cuh"

namespace bae {

// ---------------------------------------------------------------------------
// shared helpers
// ---------------------------------------------------------------------------

__device__ __forceinline__ char* tile_base(const Dev& d, const TileGeom& g, char* smem) {
  return g.big >= 0 ? d.bigws + (long long)g.big * d.big_stride : smem;
}

__device__ __forceinline__ void load_entries(const Dev& d, const TileGeom& g, const Ws& ws) {
  for (int l = threadIdx.x; l <= g.ncam; l += blockDim.x) ws.ent[l] = d.ent_obs_begin[g.eb + l] - g.ob;
}

// y = R p + t and D for one observation from a 15-double camera record
// (R[9] t[3] f k1 k2).
__device__ __forceinline__ void obs_geometry(const double* cam, const double* pt, P3& y, double* D) {
  const double* R = cam;
  y.x = R[0] * pt[0] + R[1] * pt[1] + R[2] * pt[2] + cam[9];
  y.y = R[3] * pt[0] + R[4] * pt[1] + R[5] * pt[2] + cam[10];
  y.z = R[6] * pt[0] + R[7] * pt[1] + R[8] * pt[2] + cam[11];
  bal_dproj(y, cam[12], cam[13], cam[14], D);
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
  // a = v_rho + v_omega x y
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

__device__ __forceinline__ void load_camrec(const Dev& d, const TileGeom& g, const Ws& ws, int camw, const double* rec) {
  for (int idx = threadIdx.x; idx < g.ncam * 15; idx += blockDim.x) {
    const int l = idx / 15, j = idx - l * 15;
    ws.cam[l * camw + j] = rec[(long long)d.ent_cam[g.eb + l] * kCamRec + j];
  }
}

__device__ __forceinline__ void load_points(const Ws& ws, int ptw, const double* src, int pb, int npts) {
  for (int idx = threadIdx.x; idx < npts * 3; idx += blockDim.x) {
    const int lp = idx / 3, j = idx - lp * 3;
    ws.pt[lp * ptw + j] = src[(long long)pb * 3 + idx];
  }
}

// ---------------------------------------------------------------------------
// K-rec: camera records (R from the quaternion, lie.hpp:68-70) after any
// pose update.
// ---------------------------------------------------------------------------
__global__ void k_camrec(const double* __restrict__ pose, const double* __restrict__ intr, double* __restrict__ rec,
                         int C) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= C) return;
  const double* s = pose + (long long)c * 7;
  double* o = rec + (long long)c * kCamRec;
  quat_to_R({s[3], s[4], s[5], s[6]}, o);
  o[9] = s[0];
  o[10] = s[1];
  o[11] = s[2];
  o[12] = intr[c * 3];
  o[13] = intr[c * 3 + 1];
  o[14] = intr[c * 3 + 2];
  o[15] = 0.0;
}

// ---------------------------------------------------------------------------
// K1: fused residual + Jacobian + block reductions (the linearisation).
// Replaces evaluate + sparse_jacobian + the CC/LL SpGEMM quadrants and the
// b = -J^T r SpMVs (trace.hpp:412-806, assemble.hpp:61-84).
//   per point : H_pp (6), g_p (3)          -> hpp, gp
//   per entry : H_cc (21), g_c (6) partial -> partial[e][27]
//   per tile  : sum r^2, sum |g_p|^2       -> tile_red
// The forward residual follows the reference (quaternion rotate, trace.hpp:
// 439-452; bal_cam, :464-474); its Jacobian uses that forward value y.
// ---------------------------------------------------------------------------
constexpr WsDims kLinWs{19, 3, 9, 27};

__global__ void __launch_bounds__(kTileThreads) k_linearize(Dev d, int write_jac) {
  extern __shared__ __align__(16) char smem[];
  __shared__ double red[32];
  const int t = blockIdx.x;
  const TileGeom g = tile_geom(d, t);
  const Ws ws = ws_carve(tile_base(d, g, smem), kLinWs, g.ncam, g.npts, g.nobs);
  // cameras: [t3 q4 f k1 k2 R9]
  for (int idx = threadIdx.x; idx < g.ncam * 19; idx += blockDim.x) {
    const int l = idx / 19, j = idx - l * 19;
    const long long c = d.ent_cam[g.eb + l];
    double v;
    if (j < 7)
      v = d.pose[c * 7 + j];
    else if (j < 10)
      v = d.intr[c * 3 + (j - 7)];
    else
      v = d.camrec[c * kCamRec + (j - 10)];
    ws.cam[idx] = v;
  }
  load_points(ws, 3, d.pts, g.pb, g.npts);
  load_entries(d, g, ws);
  __syncthreads();

  const int nchunk = (g.nobs + 31) / 32;
  double cost = 0.0;
  int bad = INT_MAX;
  for (int base = 0; base < g.nobs; base += blockDim.x) {
    const int s = base + threadIdx.x;
    double v27[27];
#pragma unroll
    for (int j = 0; j < 27; ++j) v27[j] = 0.0;
    int seg = -1;
    if (s < g.nobs) {
      const std::uint32_t lcpt = d.obs_lcpt[g.ob + s];
      const int lc = lcpt & 0xffff, lp = lcpt >> 16;
      seg = lc;
      const double* cam = ws.cam + lc * 19;
      const double* pt = ws.pt + lp * 3;
      const P3 yr = quat_rotate({cam[3], cam[4], cam[5], cam[6]}, {pt[0], pt[1], pt[2]});
      const P3 y{yr.x + cam[0], yr.y + cam[1], yr.z + cam[2]};
      double u = 0.0, w = 0.0;
      double r0 = 0.0, r1 = 0.0;
      double stg[9];
#pragma unroll
      for (int j = 0; j < 9; ++j) stg[j] = 0.0;
      if (bal_project(y, cam[7], cam[8], cam[9], u, w)) {
        const double2 px = reinterpret_cast<const double2*>(d.obs_px)[g.ob + s];
        r0 = u + -1.0 * px.x;
        r1 = w + -1.0 * px.y;
        double D[6], Jc[12], Jp[6];
        bal_dproj(y, cam[7], cam[8], cam[9], D);
        jac_cam(D, y, Jc);
        jac_pt(D, cam + 10, Jp);
        int q = 0;
#pragma unroll
        for (int a = 0; a < 6; ++a)
#pragma unroll
          for (int b = a; b < 6; ++b) v27[q++] = Jc[a] * Jc[b] + Jc[6 + a] * Jc[6 + b];
#pragma unroll
        for (int a = 0; a < 6; ++a) v27[21 + a] = Jc[a] * r0 + Jc[6 + a] * r1;
        q = 0;
#pragma unroll
        for (int a = 0; a < 3; ++a)
#pragma unroll
          for (int b = a; b < 3; ++b) stg[q++] = Jp[a] * Jp[b] + Jp[3 + a] * Jp[3 + b];
#pragma unroll
        for (int a = 0; a < 3; ++a) stg[6 + a] = Jp[a] * r0 + Jp[3 + a] * r1;
        if (write_jac && d.jstore) {
          const long long gs = g.ob + s;
#pragma unroll
          for (int j = 0; j < 12; ++j) d.jstore[(long long)j * d.N + gs] = Jc[j];
#pragma unroll
          for (int j = 0; j < 6; ++j) d.jstore[(long long)(12 + j) * d.N + gs] = Jp[j];
        }
        if (d.resid) {
          d.resid[g.ob + s] = r0;
          d.resid[(long long)d.N + g.ob + s] = r1;
        }
        cost += r0 * r0 + r1 * r1;
      } else {
        bad = min(bad, d.obs_orig[g.ob + s]);
      }
#pragma unroll
      for (int j = 0; j < 9; ++j) ws.stage[s * 9 + j] = stg[j];
    }
    seg_reduce_pieces<27>(v27, seg, s, nchunk, ws.piece);
  }
  if (bad != INT_MAX) atomicMin(&d.lm->err_obs, bad);
  __syncthreads();
  entries_from_pieces<27>(ws, g.ncam, g.nobs, g.eb, d.partial);
  double gsq = 0.0;
  for (int lp = threadIdx.x; lp < g.npts; lp += blockDim.x) {
    const int ip = g.pb + lp;
    double h[9];
#pragma unroll
    for (int j = 0; j < 9; ++j) h[j] = 0.0;
    for (int q = d.pt_ptr[ip]; q < d.pt_ptr[ip + 1]; ++q) {
      const double* st = ws.stage + d.ptobs[q] * 9;
#pragma unroll
      for (int j = 0; j < 9; ++j) h[j] += st[j];
    }
#pragma unroll
    for (int j = 0; j < 6; ++j) d.hpp[(long long)ip * 6 + j] = h[j];
#pragma unroll
    for (int j = 0; j < 3; ++j) d.gp[(long long)ip * 3 + j] = h[6 + j];
    gsq += h[6] * h[6] + h[7] * h[7] + h[8] * h[8];
  }
  const double cs = block_sum(cost, red);
  const double gs = block_sum(gsq, red);
  if (threadIdx.x == 0) {
    d.tile_red[t * 2] = cs;
    d.tile_red[t * 2 + 1] = gs;
  }
}

// Residual only (evaluate + squared_norm, problems.hpp:66, lm.hpp:81-85) at
// the current (trial = 0) or trial (trial = 1) parameters.
__global__ void __launch_bounds__(kTileThreads) k_cost(Dev d, int trial) {
  extern __shared__ __align__(16) char smem[];
  __shared__ double red[32];
  const int t = blockIdx.x;
  const TileGeom g = tile_geom(d, t);
  const WsDims wd{10, 3, 0, 0};
  const Ws ws = ws_carve(tile_base(d, g, smem), wd, g.ncam, g.npts, g.nobs);
  const double* pose = trial ? d.pose_t : d.pose;
  for (int idx = threadIdx.x; idx < g.ncam * 10; idx += blockDim.x) {
    const int l = idx / 10, j = idx - l * 10;
    const long long c = d.ent_cam[g.eb + l];
    ws.cam[idx] = j < 7 ? pose[c * 7 + j] : d.intr[c * 3 + (j - 7)];
  }
  load_points(ws, 3, trial ? d.pts_t : d.pts, g.pb, g.npts);
  __syncthreads();
  double cost = 0.0;
  int bad = INT_MAX;
  for (int s = threadIdx.x; s < g.nobs; s += blockDim.x) {
    const std::uint32_t lcpt = d.obs_lcpt[g.ob + s];
    const double* cam = ws.cam + (lcpt & 0xffff) * 10;
    const double* pt = ws.pt + (lcpt >> 16) * 3;
    const P3 yr = quat_rotate({cam[3], cam[4], cam[5], cam[6]}, {pt[0], pt[1], pt[2]});
    double u, w;
    if (bal_project({yr.x + cam[0], yr.y + cam[1], yr.z + cam[2]}, cam[7], cam[8], cam[9], u, w)) {
      const double2 px = reinterpret_cast<const double2*>(d.obs_px)[g.ob + s];
      const double r0 = u + -1.0 * px.x, r1 = w + -1.0 * px.y;
      if (d.resid && !trial) {
        d.resid[g.ob + s] = r0;
        d.resid[(long long)d.N + g.ob + s] = r1;
      }
      cost += r0 * r0 + r1 * r1;
    } else {
      bad = min(bad, d.obs_orig[g.ob + s]);
    }
  }
  if (bad != INT_MAX) {
    if (trial)
      atomicExch(&d.lm->trial_bad, 1);
    else
      atomicMin(&d.lm->err_obs, bad);
  }
  const double cs = block_sum(cost, red);
  if (threadIdx.x == 0) d.tile_red[t * 2] = cs;
}

// ---------------------------------------------------------------------------
// Camera-side reduction after K1: H_cc, g_c per camera (warp per camera,
// lane-strided over the camera's entries, fixed xor tree), then the grid
// totals cost / ||J^T r||^2 (last block).
// ---------------------------------------------------------------------------
template <int W>
__device__ __forceinline__ void warp_entry_sum(const Dev& d, int c, double (&acc)[W]) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int j = 0; j < W; ++j) acc[j] = 0.0;
  for (int q = d.cam_ent_ptr[c] + lane; q < d.cam_ent_ptr[c + 1]; q += 32) {
    const double* src = d.partial + (long long)d.cam_ent[q] * W;
#pragma unroll
    for (int j = 0; j < W; ++j) acc[j] += src[j];
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1)
#pragma unroll
    for (int j = 0; j < W; ++j) acc[j] += __shfl_xor_sync(0xffffffffu, acc[j], off);
}

__global__ void k_cam_linearize(Dev d) {
  __shared__ double red[32];
  const int c = blockIdx.x * kWarpsPerCamBlock + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  double gsq = 0.0;
  if (c < d.C) {
    double acc[27];
    warp_entry_sum<27>(d, c, acc);
    if (lane == 0) {
#pragma unroll
      for (int j = 0; j < 21; ++j) d.hcc[(long long)c * 21 + j] = acc[j];
#pragma unroll
      for (int j = 0; j < 6; ++j) {
        d.gc[(long long)c * 6 + j] = acc[21 + j];
        gsq += acc[21 + j] * acc[21 + j];
      }
    }
  }
  const double bs = block_sum(gsq, red);
  const double vals[1] = {bs};
  double tot[1];
  if (grid_reduce<1>(vals, d.block_red, d.tickets + 0, tot)) {
    // tile totals in tile order
    __shared__ double tcost, tg;
    double a = 0.0, b = 0.0;
    for (int tt = threadIdx.x; tt < d.T; tt += blockDim.x) {
      a += d.tile_red[tt * 2];
      b += d.tile_red[tt * 2 + 1];
    }
    a = block_sum(a, red);
    __syncthreads();
    b = block_sum(b, red);
    if (threadIdx.x == 0) {
      tcost = a;
      tg = b;
      d.lm->cost = tcost;
      d.lm->grad_sq = tg + tot[0];
    }
  }
}

// Total of the per-tile costs (after k_cost), fixed order, one block.
__global__ void k_sum_tiles(Dev d, int trial) {
  __shared__ double red[32];
  double a = 0.0;
  for (int tt = threadIdx.x; tt < d.T; tt += blockDim.x) a += d.tile_red[tt * 2];
  a = block_sum(a, red);
  if (threadIdx.x == 0) {
    if (trial)
      d.lm->new_cost = (d.lm->trial_bad || !isfinite(a)) ? INFINITY : a;
    else
      d.lm->cost = a;
  }
}

// ---------------------------------------------------------------------------
// K3/K4 prep for one damping value: per point H~_pp^-1 and v = H~_pp^-1 g_p;
// per entry the Schur right-hand side (J_c^T J_p v) and the block-Jacobi
// blocks (W H~_pp^-1 W^T, W = J_c^T J_p) of S's diagonal.
// ---------------------------------------------------------------------------
constexpr WsDims kPrepWs{15, 12, 0, 27};  // pt: p3 hinv6 v3

__global__ void __launch_bounds__(kTileThreads) k_prep(Dev d, double lambda, double clo, double chi) {
  extern __shared__ __align__(16) char smem[];
  const int t = blockIdx.x;
  const TileGeom g = tile_geom(d, t);
  const Ws ws = ws_carve(tile_base(d, g, smem), kPrepWs, g.ncam, g.npts, g.nobs);
  load_camrec(d, g, ws, 15, d.camrec);
  load_points(ws, 12, d.pts, g.pb, g.npts);
  load_entries(d, g, ws);
  int fail = 0;
  for (int lp = threadIdx.x; lp < g.npts; lp += blockDim.x) {
    const long long ip = g.pb + lp;
    double h[6], inv[9];
#pragma unroll
    for (int j = 0; j < 6; ++j) h[j] = d.hpp[ip * 6 + j];
    h[0] = damp_diag(h[0], lambda, clo, chi);
    h[3] = damp_diag(h[3], lambda, clo, chi);
    h[5] = damp_diag(h[5], lambda, clo, chi);
    if (!spd_inverse<3>(h, inv)) {
      fail = 1;
#pragma unroll
      for (int j = 0; j < 9; ++j) inv[j] = 0.0;
    }
    double* sp = ws.pt + lp * 12;
    const double hi[6] = {inv[0], inv[1], inv[2], inv[4], inv[5], inv[8]};
#pragma unroll
    for (int j = 0; j < 6; ++j) {
      sp[3 + j] = hi[j];
      d.hinv[ip * 6 + j] = hi[j];
    }
    const double g0 = d.gp[ip * 3], g1 = d.gp[ip * 3 + 1], g2 = d.gp[ip * 3 + 2];
    sp[9] = inv[0] * g0 + inv[1] * g1 + inv[2] * g2;
    sp[10] = inv[3] * g0 + inv[4] * g1 + inv[5] * g2;
    sp[11] = inv[6] * g0 + inv[7] * g1 + inv[8] * g2;
  }
  if (fail) atomicExch(&d.pcg->not_spd, 1);
  __syncthreads();
  const int nchunk = (g.nobs + 31) / 32;
  for (int base = 0; base < g.nobs; base += blockDim.x) {
    const int s = base + threadIdx.x;
    double v27[27];
#pragma unroll
    for (int j = 0; j < 27; ++j) v27[j] = 0.0;
    int seg = -1;
    if (s < g.nobs) {
      const std::uint32_t lcpt = d.obs_lcpt[g.ob + s];
      const int lc = lcpt & 0xffff, lp = lcpt >> 16;
      seg = lc;
      const double* cam = ws.cam + lc * 15;
      const double* sp = ws.pt + lp * 12;
      P3 y;
      double D[6], Jc[12], Jp[6];
      obs_geometry(cam, sp, y, D);
      jac_cam(D, y, Jc);
      jac_pt(D, cam, Jp);
      double W[18];  // 6x3
#pragma unroll
      for (int a = 0; a < 6; ++a)
#pragma unroll
        for (int j = 0; j < 3; ++j) W[a * 3 + j] = Jc[a] * Jp[j] + Jc[6 + a] * Jp[3 + j];
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
          v27[q++] = WH[a * 3] * W[b * 3] + WH[a * 3 + 1] * W[b * 3 + 1] + WH[a * 3 + 2] * W[b * 3 + 2];
      const double* vp = sp + 9;
#pragma unroll
      for (int a = 0; a < 6; ++a) v27[21 + a] = W[a * 3] * vp[0] + W[a * 3 + 1] * vp[1] + W[a * 3 + 2] * vp[2];
    }
    seg_reduce_pieces<27>(v27, seg, s, nchunk, ws.piece);
  }
  __syncthreads();
  entries_from_pieces<27>(ws, g.ncam, g.nobs, g.eb, d.partial);
}

// Camera side of the prep: damped H~_cc, block-Jacobi inverse of S_cc
// (falls back to H~_cc^-1 when the 6x6 Schur block is not numerically SPD),
// Schur RHS, and PCG initialisation x = 0, r = b, z = M^-1 r, p = z.
__global__ void k_cam_prep(Dev d, double lambda, double clo, double chi, double tol, long long budget) {
  __shared__ double red[32];
  const int c = blockIdx.x * kWarpsPerCamBlock + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  double rr = 0.0, rz = 0.0;
  int fail = 0;
  if (c < d.C) {
    double acc[27];
    warp_entry_sum<27>(d, c, acc);
    if (lane == 0) {
      double hd[21], s[21], m[36], b[6];
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
          fail = 1;
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
    }
  }
  if (fail) atomicExch(&d.pcg->not_spd, 1);
  const double v0 = block_sum(rr, red);
  __syncthreads();
  const double v1 = block_sum(rz, red);
  const double vals[2] = {v0, v1};
  double tot[2];
  if (grid_reduce<2>(vals, d.block_red, d.tickets + 1, tot) && threadIdx.x == 0) {
    PcgDev& s = *d.pcg;
    s.bnorm = sqrt(tot[0]);
    s.rz = tot[1];
    s.tol = tol;
    s.iters = 0;
    s.budget = budget;
    s.dir = kDirZ;
    s.beta = 0.0;
    s.converged = 0;
    s.true_norm = 0.0;
    if (s.not_spd) {
      s.state = kPcgBreakdown;
    } else if (s.bnorm == 0.0) {
      s.state = kPcgDone;
      s.converged = 1;
    } else {
      s.state = kPcgIter;
    }
  }
}

// ---------------------------------------------------------------------------
// K5: implicit Schur product, tile part. For v = current PCG direction
// (z, z + beta p, or x when verifying the true residual):
//   s_k = J_p^T J_c v_c(k);  w_p = sum_k s_k;  t_p = H~_pp^-1 w_p;
//   partial[e] = sum_{k in e} J_c^T J_p t_p(k)
// The camera kernel then forms y = H~_cc v - sum partial.
// D and y of the first kCacheRounds rounds stay in registers between the two
// observation phases; longer tiles recompute them.
// ---------------------------------------------------------------------------
constexpr WsDims kSxWs{21, 6, 3, 6};  // cam: R9 t3 f k1 k2 v6 ; pt: p3 t3
constexpr int kCacheRounds = 2;

// The PCG direction is formed lazily (p = z + beta p) by both the tile and
// the camera kernel with the same fused expression, so both see identical bits.
__device__ __forceinline__ double dir_component(const PcgDev& s, const Dev& d, long long o) {
  return s.dir == kDirX ? d.x[o] : (s.dir == kDirZ ? d.z[o] : fma(s.beta, d.p[o], d.z[o]));
}
__device__ __forceinline__ void dir_vector(const PcgDev& s, const Dev& d, long long c, double* v) {
#pragma unroll
  for (int j = 0; j < 6; ++j) v[j] = dir_component(s, d, c * 6 + j);
}

template <bool kVecIsDelta>
__device__ __forceinline__ void sx_tile_body(const Dev& d, const TileGeom& g, const Ws& ws) {
  const int nchunk = (g.nobs + 31) / 32;
  const int nrounds = (g.nobs + blockDim.x - 1) / blockDim.x;
  double cD[kCacheRounds][6];
  P3 cy[kCacheRounds];
  // phase 1
#pragma unroll
  for (int r = 0; r < kCacheRounds; ++r) {
    const int s = r * blockDim.x + threadIdx.x;
    if (r < nrounds && s < g.nobs) {
      const std::uint32_t lcpt = d.obs_lcpt[g.ob + s];
      const double* cam = ws.cam + (lcpt & 0xffff) * 21;
      obs_geometry(cam, ws.pt + (lcpt >> 16) * 6, cy[r], cD[r]);
      jpt_jc_v(cD[r], cy[r], cam, cam + 15, ws.stage + s * 3);
    }
  }
  for (int r = kCacheRounds; r < nrounds; ++r) {
    const int s = r * blockDim.x + threadIdx.x;
    if (s < g.nobs) {
      const std::uint32_t lcpt = d.obs_lcpt[g.ob + s];
      const double* cam = ws.cam + (lcpt & 0xffff) * 21;
      P3 y;
      double D[6];
      obs_geometry(cam, ws.pt + (lcpt >> 16) * 6, y, D);
      jpt_jc_v(D, y, cam, cam + 15, ws.stage + s * 3);
    }
  }
  __syncthreads();
  // point phase
  for (int lp = threadIdx.x; lp < g.npts; lp += blockDim.x) {
    const int ip = g.pb + lp;
    double w0 = 0.0, w1 = 0.0, w2 = 0.0;
    for (int q = d.pt_ptr[ip]; q < d.pt_ptr[ip + 1]; ++q) {
      const double* st = ws.stage + d.ptobs[q] * 3;
      w0 += st[0];
      w1 += st[1];
      w2 += st[2];
    }
    const double* hi = d.hinv + (long long)ip * 6;
    double* tp = ws.pt + lp * 6 + 3;
    tp[0] = hi[0] * w0 + hi[1] * w1 + hi[2] * w2;
    tp[1] = hi[1] * w0 + hi[3] * w1 + hi[4] * w2;
    tp[2] = hi[2] * w0 + hi[4] * w1 + hi[5] * w2;
  }
  __syncthreads();
  // phase 3
  for (int r = 0; r < nrounds; ++r) {
    const int s = r * blockDim.x + threadIdx.x;
    double z6[6] = {0, 0, 0, 0, 0, 0};
    int seg = -1;
    if (s < g.nobs) {
      const std::uint32_t lcpt = d.obs_lcpt[g.ob + s];
      const int lc = lcpt & 0xffff, lp = lcpt >> 16;
      seg = lc;
      const double* cam = ws.cam + lc * 21;
      const double* tp = ws.pt + lp * 6 + 3;
      if (r < kCacheRounds) {
        // select the cached round without dynamic register indexing
        double D[6];
        P3 y;
#pragma unroll
        for (int rr = 0; rr < kCacheRounds; ++rr)
          if (rr == r) {
#pragma unroll
            for (int j = 0; j < 6; ++j) D[j] = cD[rr][j];
            y = cy[rr];
          }
        jct_jp_t(D, y, cam, tp, z6);
      } else {
        P3 y;
        double D[6];
        obs_geometry(cam, ws.pt + lp * 6, y, D);
        jct_jp_t(D, y, cam, tp, z6);
      }
    }
    seg_reduce_pieces<6>(z6, seg, s, nchunk, ws.piece);
  }
  __syncthreads();
}

__global__ void __launch_bounds__(kTileThreads) k_schur_tiles(Dev d) {
  extern __shared__ __align__(16) char smem[];
  const PcgDev s = *d.pcg;
  if (s.state >= kPcgDone) return;
  const TileGeom g = tile_geom(d, blockIdx.x);
  const Ws ws = ws_carve(tile_base(d, g, smem), kSxWs, g.ncam, g.npts, g.nobs);
  for (int idx = threadIdx.x; idx < g.ncam * 21; idx += blockDim.x) {
    const int l = idx / 21, j = idx - l * 21;
    const long long c = d.ent_cam[g.eb + l];
    double v;
    if (j < 15) {
      v = d.camrec[c * kCamRec + j];
    } else {
      const long long o = c * 6 + (j - 15);
      v = dir_component(s, d, o);
    }
    ws.cam[idx] = v;
  }
  load_points(ws, 6, d.pts, g.pb, g.npts);
  load_entries(d, g, ws);
  __syncthreads();
  sx_tile_body<false>(d, g, ws);
  entries_from_pieces<6>(ws, g.ncam, g.nobs, g.eb, d.partial);
}

// K5 camera part: y_c = H~_cc v_c - sum partial; p <- v (direction update);
// dot(v, y) -> alpha = rz / pAp in the last block.
__global__ void k_schur_cams(Dev d) {
  __shared__ double red[32];
  const PcgDev s = *d.pcg;
  if (s.state >= kPcgDone) return;
  const int c = blockIdx.x * kWarpsPerCamBlock + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  double pap = 0.0;
  if (c < d.C) {
    double acc[6];
    warp_entry_sum<6>(d, c, acc);
    if (lane == 0) {
      double v[6];
      dir_vector(s, d, c, v);
      const double* h = d.hccd + (long long)c * 21;
#pragma unroll
      for (int a = 0; a < 6; ++a) {
        double hv = 0.0;
#pragma unroll
        for (int b = 0; b < 6; ++b) hv += h[sym6(a, b)] * v[b];
        const double yy = hv - acc[a];
        d.y[(long long)c * 6 + a] = yy;
        if (s.dir != kDirX) d.p[(long long)c * 6 + a] = v[a];
        pap += v[a] * yy;
      }
    }
  }
  const double bs = block_sum(pap, red);
  const double vals[1] = {bs};
  double tot[1];
  if (grid_reduce<1>(vals, d.block_red, d.tickets + 2, tot) && threadIdx.x == 0) {
    if (s.dir != kDirX) {
      const double alpha = s.rz / tot[0];
      d.pcg->alpha = alpha;
      if (!isfinite(alpha)) d.pcg->state = kPcgBreakdown;  // pcg.hpp:77
    }
  }
}

// PCG vector update (pcg.hpp:78-117) on the camera vectors, with the
// recurrence / true-residual state machine in the last block.
__global__ void k_pcg_update(Dev d) {
  __shared__ double red[32];
  const PcgDev s = *d.pcg;
  if (s.state >= kPcgDone) return;
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  double rr = 0.0, rz = 0.0;
  if (c < d.C) {
    double rv[6];
#pragma unroll
    for (int a = 0; a < 6; ++a) {
      const long long o = (long long)c * 6 + a;
      if (s.state == kPcgIter) {
        d.x[o] += s.alpha * d.p[o];
        rv[a] = d.r[o] - s.alpha * d.y[o];
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
  const double v0 = block_sum(rr, red);
  __syncthreads();
  const double v1 = block_sum(rz, red);
  const double vals[2] = {v0, v1};
  double tot[2];
  if (grid_reduce<2>(vals, d.block_red, d.tickets + 3, tot) && threadIdx.x == 0) {
    PcgDev& o = *d.pcg;
    const double rnorm = sqrt(tot[0]);
    o.rnorm = rnorm;
    if (s.state == kPcgIter) {
      o.iters = s.iters + 1;
      if (!isfinite(rnorm)) {
        o.state = kPcgBreakdown;
      } else if (rnorm <= s.tol * s.bnorm) {
        o.state = kPcgVerify;  // confirm with the true residual (pcg.hpp:86-109)
        o.dir = kDirX;
      } else {
        const double beta = tot[1] / s.rz;
        if (!isfinite(beta)) {
          o.state = kPcgBreakdown;
        } else {
          o.beta = beta;
          o.rz = tot[1];
          o.dir = kDirZBetaP;
          if (o.iters >= s.budget) o.state = kPcgDone;
        }
      }
    } else {
      o.true_norm = rnorm;
      if (rnorm <= s.tol * s.bnorm) {
        o.state = kPcgDone;
        o.converged = 1;
      } else {  // restart from the true residual
        o.rz = tot[1];
        o.beta = 0.0;
        o.dir = kDirZ;
        o.state = (s.iters >= s.budget) ? kPcgDone : kPcgIter;
      }
    }
  }
}

// ---------------------------------------------------------------------------
// K7 + K8: camera retraction Exp(dc) o T (lm.hpp:157-167) into the trial
// buffers, then point back-substitution + trial cost in one tile pass.
// ---------------------------------------------------------------------------
__global__ void k_cam_retract(Dev d) {
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
  rec[12] = d.intr[c * 3];
  rec[13] = d.intr[c * 3 + 1];
  rec[14] = d.intr[c * 3 + 2];
  rec[15] = 0.0;
}

// cam: R9 t3 f k1 k2 dc6 | trial t3 q4  (28) ; pt: p3 ptrial3
constexpr WsDims kTrialWs{28, 6, 3, 0};

__global__ void __launch_bounds__(kTileThreads) k_backsub_trial(Dev d) {
  extern __shared__ __align__(16) char smem[];
  __shared__ double red[32];
  const int t = blockIdx.x;
  const TileGeom g = tile_geom(d, t);
  const Ws ws = ws_carve(tile_base(d, g, smem), kTrialWs, g.ncam, g.npts, g.nobs);
  for (int idx = threadIdx.x; idx < g.ncam * 28; idx += blockDim.x) {
    const int l = idx / 28, j = idx - l * 28;
    const long long c = d.ent_cam[g.eb + l];
    double v;
    if (j < 15)
      v = d.camrec[c * kCamRec + j];
    else if (j < 21)
      v = d.x[c * 6 + (j - 15)];
    else
      v = d.pose_t[c * 7 + (j - 21)];
    ws.cam[idx] = v;
  }
  load_points(ws, 6, d.pts, g.pb, g.npts);
  __syncthreads();
  for (int s = threadIdx.x; s < g.nobs; s += blockDim.x) {
    const std::uint32_t lcpt = d.obs_lcpt[g.ob + s];
    const double* cam = ws.cam + (lcpt & 0xffff) * 28;
    P3 y;
    double D[6];
    obs_geometry(cam, ws.pt + (lcpt >> 16) * 6, y, D);
    jpt_jc_v(D, y, cam, cam + 15, ws.stage + s * 3);
  }
  __syncthreads();
  // Delta p = H~_pp^-1 (-g_p - sum_k J_p^T J_c dc), p_trial = p + Delta p
  for (int lp = threadIdx.x; lp < g.npts; lp += blockDim.x) {
    const long long ip = g.pb + lp;
    double w0 = 0.0, w1 = 0.0, w2 = 0.0;
    for (int q = d.pt_ptr[ip]; q < d.pt_ptr[ip + 1]; ++q) {
      const double* st = ws.stage + d.ptobs[q] * 3;
      w0 += st[0];
      w1 += st[1];
      w2 += st[2];
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
  __syncthreads();
  double cost = 0.0;
  int bad = 0;
  for (int s = threadIdx.x; s < g.nobs; s += blockDim.x) {
    const std::uint32_t lcpt = d.obs_lcpt[g.ob + s];
    const double* cam = ws.cam + (lcpt & 0xffff) * 28;
    const double* pt = ws.pt + (lcpt >> 16) * 6 + 3;
    const P3 yr = quat_rotate({cam[24], cam[25], cam[26], cam[27]}, {pt[0], pt[1], pt[2]});
    double u, w;
    if (bal_project({yr.x + cam[21], yr.y + cam[22], yr.z + cam[23]}, cam[12], cam[13], cam[14], u, w)) {
      const double2 px = reinterpret_cast<const double2*>(d.obs_px)[g.ob + s];
      const double r0 = u + -1.0 * px.x, r1 = w + -1.0 * px.y;
      cost += r0 * r0 + r1 * r1;
    } else {
      bad = 1;  // CheiralityError in the trial evaluate -> cost = inf (lm.hpp:176-181)
    }
  }
  if (bad) atomicExch(&d.lm->trial_bad, 1);
  const double cs = block_sum(cost, red);
  if (threadIdx.x == 0) d.tile_red[t * 2] = cs;
}

// Accept: trial parameters become current (lm.hpp:183-189).
__global__ void k_commit(Dev d) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < (long long)d.P * 3) d.pts[i] = d.pts_t[i];
  if (i < (long long)d.C * 7) d.pose[i] = d.pose_t[i];
  if (i < (long long)d.C * kCamRec) d.camrec[i] = d.camrec_t[i];
}

// ---------------------------------------------------------------------------
// launch wrappers
// ---------------------------------------------------------------------------
static inline long long lin_bytes(int ncam, int npts, int nobs) { return ws_bytes(kLinWs, ncam, npts, nobs); }

long long tile_ws_bytes(int kind, int ncam, int npts, int nobs) {
  switch (kind) {
    case kWsLin:
      return lin_bytes(ncam, npts, nobs);
    case kWsCost:
      return ws_bytes(WsDims{10, 3, 0, 0}, ncam, npts, nobs);
    case kWsPrep:
      return ws_bytes(kPrepWs, ncam, npts, nobs);
    case kWsSchur:
      return ws_bytes(kSxWs, ncam, npts, nobs);
    case kWsTrial:
      return ws_bytes(kTrialWs, ncam, npts, nobs);
  }
  return 0;
}

void set_smem_limits(int max_bytes) {
  cudaFuncSetAttribute(k_linearize, cudaFuncAttributeMaxDynamicSharedMemorySize, max_bytes);
  cudaFuncSetAttribute(k_cost, cudaFuncAttributeMaxDynamicSharedMemorySize, max_bytes);
  cudaFuncSetAttribute(k_prep, cudaFuncAttributeMaxDynamicSharedMemorySize, max_bytes);
  cudaFuncSetAttribute(k_schur_tiles, cudaFuncAttributeMaxDynamicSharedMemorySize, max_bytes);
  cudaFuncSetAttribute(k_backsub_trial, cudaFuncAttributeMaxDynamicSharedMemorySize, max_bytes);
}

static inline int cam_blocks(int C) { return (C + kWarpsPerCamBlock - 1) / kWarpsPerCamBlock; }
static inline int elt_blocks(long long n, int bs) { return (int)((n + bs - 1) / bs); }

void launch_camrec(const Dev& d, bool trial, cudaStream_t s) {
  k_camrec<<<elt_blocks(d.C, 128), 128, 0, s>>>(trial ? d.pose_t : d.pose, d.intr, trial ? d.camrec_t : d.camrec, d.C);
}
void launch_linearize(const Dev& d, const SmemSizes& sm, bool write_jac, cudaStream_t s) {
  k_linearize<<<d.T, kTileThreads, sm.lin, s>>>(d, write_jac ? 1 : 0);
  k_cam_linearize<<<cam_blocks(d.C), 32 * kWarpsPerCamBlock, 0, s>>>(d);
}
void launch_cost(const Dev& d, const SmemSizes& sm, bool trial, cudaStream_t s) {
  k_cost<<<d.T, kTileThreads, sm.cost, s>>>(d, trial ? 1 : 0);
  k_sum_tiles<<<1, 1024, 0, s>>>(d, trial ? 1 : 0);
}
void launch_prep(const Dev& d, const SmemSizes& sm, double lambda, double clo, double chi, double tol,
                 long long budget, cudaStream_t s) {
  k_prep<<<d.T, kTileThreads, sm.prep, s>>>(d, lambda, clo, chi);
  k_cam_prep<<<cam_blocks(d.C), 32 * kWarpsPerCamBlock, 0, s>>>(d, lambda, clo, chi, tol, budget);
}
void launch_pcg_iteration(const Dev& d, const SmemSizes& sm, cudaStream_t s) {
  k_schur_tiles<<<d.T, kTileThreads, sm.schur, s>>>(d);
  k_schur_cams<<<cam_blocks(d.C), 32 * kWarpsPerCamBlock, 0, s>>>(d);
  k_pcg_update<<<elt_blocks(d.C, 128), 128, 0, s>>>(d);
}
void launch_schur_only(const Dev& d, const SmemSizes& sm, cudaStream_t s) {
  k_schur_tiles<<<d.T, kTileThreads, sm.schur, s>>>(d);
}
void launch_trial(const Dev& d, const SmemSizes& sm, cudaStream_t s) {
  k_cam_retract<<<elt_blocks(d.C, 128), 128, 0, s>>>(d);
  k_backsub_trial<<<d.T, kTileThreads, sm.trial, s>>>(d);
  k_sum_tiles<<<1, 1024, 0, s>>>(d, 1);
}
void launch_commit(const Dev& d, cudaStream_t s) {
  const long long n = std::max<long long>((long long)d.P * 3, (long long)d.C * kCamRec);
  k_commit<<<elt_blocks(n, 256), 256, 0, s>>>(d);
}

}  // namespace bae
