// Pose-graph optimisation on the device (see pgo.hpp).
//
// Per edge (one thread): e = zi^-1 zj T^-1, r = Log(e) (trace.hpp:475-487),
// whitened r_w = W r with W = L^T of the edge information (problems.hpp:
// 169-184), the reverse-pass Jacobians J_j = W Jl^-1(r) Ad(zi^-1), J_i = -J_j
// (trace.hpp:657-671), and the edge's normal-equation pieces M = J_j^T J_j,
// v = J_j^T r_w: the normal matrix gets +M on both diagonal blocks and -M on
// the coupling block, the gradient -v / +v. Per unknown pose and per pose
// pair, a warp sums its edges' pieces in edge order (deterministic, no
// atomics) straight into the tile-sparse matrix of the Cholesky (chol.cuh).
#include <algorithm>
#include <chrono>
#include <climits>
#include <cmath>
#include <cstring>
#include <limits>
#include <string>

#include "device.cuh"
#include "pgo.hpp"

namespace bae {

namespace {

void ck(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw Error(BAE_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

// ---- SE(3) pieces the relative-pose residual needs (lie.hpp) ---------------
__device__ __forceinline__ void skew3(const P3& v, double* m) {  // lie.hpp:20-24
  m[0] = 0.0;
  m[1] = -v.z;
  m[2] = v.y;
  m[3] = v.z;
  m[4] = 0.0;
  m[5] = -v.x;
  m[6] = -v.y;
  m[7] = v.x;
  m[8] = 0.0;
}
__device__ __forceinline__ void mm3(const double* a, const double* b, double* c) {
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j) c[i * 3 + j] = a[i * 3] * b[j] + a[i * 3 + 1] * b[3 + j] + a[i * 3 + 2] * b[6 + j];
}
// se3_inverse (lie.hpp:209-212): conjugate, -R^T t
__device__ __forceinline__ void se3_inv(const Q4& q, const P3& t, Q4& qi, P3& ti) {
  qi = {-q.x, -q.y, -q.z, q.w};
  const P3 r = quat_rotate(qi, t);
  ti = {-r.x, -r.y, -r.z};
}
// se3_compose (lie.hpp:204-207)
__device__ __forceinline__ bool se3_comp(const Q4& qa, const P3& ta, const Q4& qb, const P3& tb, Q4& q, P3& t) {
  if (!quat_mul(qa, qb, q)) return false;
  const P3 r = quat_rotate(qa, tb);
  t = {r.x + ta.x, r.y + ta.y, r.z + ta.z};
  return true;
}
// log_translation_factor_inv (lie.hpp:158-168), row-major
__device__ __forceinline__ void log_tf_inv(const P3& om, double theta, double* m) {
  double o[9], oo[9];
  skew3(om, o);
  mm3(o, o, oo);
  double c;
  if (theta < 1e-8) {
    c = 1.0 / 12.0 + theta * theta / 720.0;
  } else {
    const double half = 0.5 * theta;
    c = (1.0 - half * cos(half) / sin(half)) / (theta * theta);
  }
#pragma unroll
  for (int i = 0; i < 9; ++i) m[i] = ((i % 4 == 0) ? 1.0 : 0.0) - 0.5 * o[i] + c * oo[i];
}
// se3_log (lie.hpp:189-202): [rho, omega]
__device__ __forceinline__ void se3_logm(const Q4& q, const P3& t, double* xi) {
  const P3 om = so3_log(q);
  const double s = sqrt(q.x * q.x + q.y * q.y + q.z * q.z);
  const double theta = 2.0 * atan2(s, q.w);
  double m[9];
  log_tf_inv(om, theta, m);
  xi[0] = m[0] * t.x + m[1] * t.y + m[2] * t.z;
  xi[1] = m[3] * t.x + m[4] * t.y + m[5] * t.z;
  xi[2] = m[6] * t.x + m[7] * t.y + m[8] * t.z;
  xi[3] = om.x;
  xi[4] = om.y;
  xi[5] = om.z;
}
// se3_left_jacobian_q (lie.hpp:251-285)
__device__ __forceinline__ void left_jac_q(const double* xi, double* q) {
  const P3 rho{xi[0], xi[1], xi[2]}, om{xi[3], xi[4], xi[5]};
  const double theta = sqrt(om.x * om.x + om.y * om.y + om.z * om.z);
  double rx[9], ox[9], oxrx[9], rxox[9], oxrxox[9], a[9], b[9];
  skew3(rho, rx);
  skew3(om, ox);
  mm3(ox, rx, oxrx);
  mm3(rx, ox, rxox);
  mm3(oxrx, ox, oxrxox);
  double c1, c2, c3;
  const double t2 = theta * theta;
  if (theta < 1e-4) {
    c1 = 1.0 / 6.0 - t2 / 120.0;
    c2 = 1.0 / 24.0 - t2 / 720.0;
    c3 = -1.0 / 120.0 + t2 / 5040.0;
  } else {
    const double t3 = t2 * theta, st = sin(theta), ct = cos(theta);
    c1 = (theta - st) / t3;
    c2 = (1.0 - 0.5 * t2 - ct) / (t2 * t2);
    c3 = (theta - st - t3 / 6.0) / (t3 * t2);
  }
#pragma unroll
  for (int i = 0; i < 9; ++i) q[i] = 0.5 * rx[i];
#pragma unroll
  for (int i = 0; i < 9; ++i) q[i] += c1 * (oxrx[i] + rxox[i] + oxrxox[i]);
  mm3(ox, oxrx, a);
  mm3(rxox, ox, b);
#pragma unroll
  for (int i = 0; i < 9; ++i) q[i] -= c2 * (a[i] + b[i] - 3.0 * oxrxox[i]);
  mm3(oxrxox, ox, a);
  mm3(ox, oxrxox, b);
  const double s = 0.5 * (c2 - 3.0 * c3);
#pragma unroll
  for (int i = 0; i < 9; ++i) q[i] -= s * (a[i] + b[i]);
}

// d_j = Jl^-1(r) Ad(zi^-1) (trace.hpp:665): Jl^-1 = [[J, -J Q J], [0, J]]
// (lie.hpp:291-299), Ad(T) = [[R, [t]x R], [0, R]] (lie.hpp:224-231).
__device__ __forceinline__ void pgo_dj(const double* r, const Q4& qi, const P3& ti, double* dj) {
  double j[9], qm[9], jq[9], jqj[9], rm[9], tx[9], txr[9];
  log_tf_inv({r[3], r[4], r[5]}, sqrt(r[3] * r[3] + r[4] * r[4] + r[5] * r[5]), j);
  left_jac_q(r, qm);
  mm3(j, qm, jq);
  mm3(jq, j, jqj);
  quat_to_R(qi, rm);
  skew3(ti, tx);
  mm3(tx, rm, txr);
  // [[J, -JQJ], [0, J]] * [[R, txR], [0, R]] = [[J R, J txR - JQJ R], [0, J R]]
  double jr[9], jt[9], jqjr[9];
  mm3(j, rm, jr);
  mm3(j, txr, jt);
  mm3(jqj, rm, jqjr);
#pragma unroll
  for (int a = 0; a < 3; ++a)
#pragma unroll
    for (int b = 0; b < 3; ++b) {
      dj[a * 6 + b] = jr[a * 3 + b];
      dj[a * 6 + b + 3] = jt[a * 3 + b] + -jqjr[a * 3 + b];
      dj[(a + 3) * 6 + b] = 0.0;
      dj[(a + 3) * 6 + b + 3] = jr[a * 3 + b];
    }
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
  return v;
}

__device__ __forceinline__ Q4 ld_q(const double* p) { return {p[3], p[4], p[5], p[6]}; }
__device__ __forceinline__ P3 ld_t(const double* p) { return {p[0], p[1], p[2]}; }

// Edge residuals (and, when linearising, the normal-equation pieces).
__global__ void k_pgo_edges(PgoDev d, const double* __restrict__ pose, int linearize, int trial) {
  const long long k = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= d.m) return;
  const double* zi = pose + 7LL * d.ei[k];
  const double* zj = pose + 7LL * d.ej[k];
  const double* tm = d.meas + 7 * k;
  Q4 qi, qa, qti, qe;
  P3 ti, ta, tti, te;
  se3_inv(ld_q(zi), ld_t(zi), qi, ti);
  se3_inv(ld_q(tm), ld_t(tm), qti, tti);
  bool ok = se3_comp(qi, ti, ld_q(zj), ld_t(zj), qa, ta);
  ok = ok && se3_comp(qa, ta, qti, tti, qe, te);
  double r[6], rw[6];
  if (ok) {
    se3_logm(qe, te, r);
  } else {
#pragma unroll
    for (int i = 0; i < 6; ++i) r[i] = NAN;
  }
  const double* w = d.white ? d.white + 36 * k : nullptr;
#pragma unroll
  for (int i = 0; i < 6; ++i) {
    if (w) {  // row_matmul forward (trace.hpp:508-520)
      double s = 0.0;
#pragma unroll
      for (int j = 0; j < 6; ++j) s += w[i * 6 + j] * r[j];
      rw[i] = s;
    } else {
      rw[i] = r[i];
    }
  }
  double cost = 0.0;
#pragma unroll
  for (int i = 0; i < 6; ++i) cost += rw[i] * rw[i];
  if (!ok || !isfinite(cost)) atomicExch(reinterpret_cast<unsigned long long*>(d.scal + (trial ? 4 : 3)),
                                         __double_as_longlong(1.0));
  double* eb = d.edge + 28 * k;
  eb[27] = cost;
  if (d.resid)
#pragma unroll
    for (int i = 0; i < 6; ++i) d.resid[6 * k + i] = rw[i];
  if (!linearize) return;
  double dj[36], jw[36];
  pgo_dj(r, qi, ti, dj);
#pragma unroll
  for (int i = 0; i < 6; ++i)
#pragma unroll
    for (int c = 0; c < 6; ++c) {
      if (w) {
        double s = 0.0;
#pragma unroll
        for (int j = 0; j < 6; ++j) s += w[i * 6 + j] * dj[j * 6 + c];
        jw[i * 6 + c] = s;
      } else {
        jw[i * 6 + c] = dj[i * 6 + c];
      }
    }
  if (d.jexp)
#pragma unroll
    for (int i = 0; i < 36; ++i) d.jexp[36 * k + i] = jw[i];
  int q = 0;
#pragma unroll
  for (int a = 0; a < 6; ++a)
#pragma unroll
    for (int b = a; b < 6; ++b) {
      double s = 0.0;
#pragma unroll
      for (int i = 0; i < 6; ++i) s += jw[i * 6 + a] * jw[i * 6 + b];
      eb[q++] = s;
    }
#pragma unroll
  for (int a = 0; a < 6; ++a) {
    double s = 0.0;
#pragma unroll
    for (int i = 0; i < 6; ++i) s += jw[i * 6 + a] * rw[i];
    eb[21 + a] = s;
  }
}

// Cost of all edges in edge order (one block): scal[0] (current) / scal[2] (trial).
__global__ void __launch_bounds__(1024) k_pgo_cost(PgoDev d, int trial) {
  __shared__ double red[32];
  double a = 0.0;
  for (long long k = threadIdx.x; k < d.m; k += blockDim.x) a += d.edge[28 * k + 27];
  a = block_sum(a, red);
  if (threadIdx.x == 0) {
    if (trial)
      d.scal[2] = (d.scal[4] != 0.0 || !isfinite(a)) ? INFINITY : a;
    else
      d.scal[0] = a;
  }
}

// Normal matrix into the tiles: warp per unknown pose (+M of its edges,
// damped diagonal, gradient -v / +v) then warp per pose pair (-M).
__global__ void k_pgo_assemble(PgoDev d, double lambda, double clo, double chi) {
  const int w = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (w < d.nsys) {
    double acc[27];
#pragma unroll
    for (int j = 0; j < 27; ++j) acc[j] = 0.0;
    for (int q = d.inc_ptr[w] + lane; q < d.inc_ptr[w + 1]; q += 32) {
      const int code = d.inc[q];
      const double* eb = d.edge + 28LL * (code >> 1);
      const double sg = (code & 1) ? 1.0 : -1.0;
#pragma unroll
      for (int j = 0; j < 21; ++j) acc[j] += eb[j];
#pragma unroll
      for (int j = 0; j < 6; ++j) acc[21 + j] += sg * eb[21 + j];
    }
#pragma unroll
    for (int j = 0; j < 27; ++j) acc[j] = warp_sum(acc[j]);
    if (lane == 0) {
      const int2 dt = d.diag_tile[w];
      double* base = d.tiles + (long long)dt.x * kSTileElems + dt.y * 48 + dt.y;
#pragma unroll
      for (int r = 0; r < 6; ++r)
#pragma unroll
        for (int c = 0; c < 6; ++c) {
          double v = acc[sym6(r, c)];
          if (r == c) v = damp_diag(v, lambda, clo, chi);
          base[c * 48 + r] = v;
        }
      double gsq = 0.0;
#pragma unroll
      for (int a = 0; a < 6; ++a) {
        d.rhs[6LL * w + a] = -acc[21 + a];
        gsq += acc[21 + a] * acc[21 + a];
      }
      d.pose_gsq[w] = gsq;
    }
    return;
  }
  const int pr = w - d.nsys;
  if (pr >= d.npair) return;
  double acc[21];
#pragma unroll
  for (int j = 0; j < 21; ++j) acc[j] = 0.0;
  for (int q = d.pair_ptr[pr] + lane; q < d.pair_ptr[pr + 1]; q += 32) {
    const double* eb = d.edge + 28LL * d.pair_edge[q];
#pragma unroll
    for (int j = 0; j < 21; ++j) acc[j] += eb[j];
  }
#pragma unroll
  for (int j = 0; j < 21; ++j) acc[j] = warp_sum(acc[j]);
  if (lane == 0) {
    const int2 bt = d.pair_tile[pr];
    const int ro = bt.y & 0xff, co = (bt.y >> 8) & 0xff;
    double* base = d.tiles + (long long)bt.x * kSTileElems + co * 48 + ro;
#pragma unroll
    for (int r = 0; r < 6; ++r)
#pragma unroll
      for (int c = 0; c < 6; ++c) base[c * 48 + r] = -acc[sym6(r, c)];  // -M is symmetric: no transpose needed
  }
}

// ||J^T r||^2 over the unknowns (one block, fixed order).
__global__ void __launch_bounds__(1024) k_pgo_grad(PgoDev d) {
  __shared__ double red[32];
  double a = 0.0;
  for (int c = threadIdx.x; c < d.nsys; c += blockDim.x) a += d.pose_gsq[c];
  a = block_sum(a, red);
  if (threadIdx.x == 0) d.scal[1] = a;
}

// Trial poses: Exp(delta) o T for the unknowns (lm.hpp:159-167).
__global__ void k_pgo_retract(PgoDev d) {
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= d.n) return;
  const double* s = d.pose + 7LL * p;
  double* o = d.pose_t + 7LL * p;
  if (p < d.anchor) {
#pragma unroll
    for (int i = 0; i < 7; ++i) o[i] = s[i];
    return;
  }
  const double* tau = d.x + 6LL * (p - d.anchor);
  Q4 q;
  P3 t;
  if (!se3_retract(ld_q(s), ld_t(s), tau, q, t)) {
    atomicExch(reinterpret_cast<unsigned long long*>(d.scal + 4), __double_as_longlong(1.0));
    q = ld_q(s);
    t = ld_t(s);
  }
  o[0] = t.x;
  o[1] = t.y;
  o[2] = t.z;
  o[3] = q.x;
  o[4] = q.y;
  o[5] = q.z;
  o[6] = q.w;
}

}  // namespace

template <class T>
T* PgoProblem::dalloc(std::size_t n) {
  void* p = nullptr;
  ck(cudaMalloc(&p, std::max<std::size_t>(n, 1) * sizeof(T)), "cudaMalloc");
  allocs_.push_back(p);
  return static_cast<T*>(p);
}
template <class T>
T* PgoProblem::upload(const std::vector<T>& v) {
  T* p = dalloc<T>(v.size());
  if (!v.empty()) ck(cudaMemcpyAsync(p, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice, stream_), "upload");
  return p;
}
void PgoProblem::sync() { ck(cudaStreamSynchronize(stream_), "kernel execution"); }

// 6x6 lower Cholesky (Eigen::LLT of the information matrix); false unless SPD.
static bool llt6(const double* a, double* l) {
  for (int i = 0; i < 36; ++i) l[i] = 0.0;
  for (int j = 0; j < 6; ++j) {
    double dsum = a[j * 6 + j];
    for (int k = 0; k < j; ++k) dsum -= l[j * 6 + k] * l[j * 6 + k];
    if (!(dsum > 0.0)) return false;
    const double ljj = std::sqrt(dsum);
    l[j * 6 + j] = ljj;
    for (int i = j + 1; i < 6; ++i) {
      double s = a[i * 6 + j];
      for (int k = 0; k < j; ++k) s -= l[i * 6 + k] * l[j * 6 + k];
      l[i * 6 + j] = s / ljj;
    }
  }
  return true;
}

PgoProblem::PgoProblem(const double* poses7, int n, const std::int32_t* ei, const std::int32_t* ej,
                       const double* meas7, const double* info36, const std::int32_t* has_info, std::int64_t m,
                       bool anchor_first, const bae_create_options& opt)
    : opt_(opt) {
  // make_pgo_problem validation (problems.hpp:143-157)
  if (n < 1) throw Error(BAE_ERR_INVALID_ARGUMENT, "make_pgo_problem: no poses");
  if (m < 1) throw Error(BAE_ERR_INVALID_ARGUMENT, "make_pgo_problem: no edges");
  if (m >= INT_MAX / 2) throw Error(BAE_ERR_UNSUPPORTED, "too many edges");
  for (std::int64_t k = 0; k < m; ++k) {
    if (ei[k] < 0 || ei[k] >= n) throw Error(BAE_ERR_INDEX, "make_pgo_problem: edge endpoint i out of range", k);
    if (ej[k] < 0 || ej[k] >= n) throw Error(BAE_ERR_INDEX, "make_pgo_problem: edge endpoint j out of range", k);
    if (ei[k] == ej[k]) throw Error(BAE_ERR_INVALID_ARGUMENT, "make_pgo_problem: self edge");
  }
  bool any_info = false;
  for (std::int64_t k = 0; info36 && k < m; ++k) any_info = any_info || (!has_info || has_info[k]);
  std::vector<double> white;
  if (any_info) {
    white.assign(36 * static_cast<std::size_t>(m), 0.0);
    for (std::int64_t k = 0; k < m; ++k) {
      double* w = &white[36 * k];
      if (!has_info || has_info[k]) {
        double l[36];
        if (!llt6(info36 + 36 * k, l))
          throw Error(BAE_ERR_INVALID_ARGUMENT, "make_pgo_problem: information matrix not SPD");
        for (int i = 0; i < 6; ++i)
          for (int j = 0; j < 6; ++j) w[i * 6 + j] = l[j * 6 + i];
      } else {
        for (int i = 0; i < 6; ++i) w[i * 6 + i] = 1.0;
      }
    }
  }
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
    throw Error(BAE_ERR_CUDA, "no CUDA device available (the B200 path has no CPU fallback)");
  if (opt.device < 0 || opt.device >= ndev) throw Error(BAE_ERR_INVALID_ARGUMENT, "bad device ordinal");
  ck(cudaSetDevice(opt.device), "cudaSetDevice");
  ck(cudaStreamCreateWithFlags(&stream_, cudaStreamNonBlocking), "stream");

  PgoDev& d = d_;
  d.n = n;
  d.m = m;
  d.anchor = anchor_first ? 1 : 0;
  d.nsys = n - d.anchor;
  // incidence of the unknown poses and the pose pairs, edge order
  std::vector<int> inc_ptr(static_cast<std::size_t>(std::max(d.nsys, 0)) + 1, 0), inc;
  std::vector<std::vector<int>> incl(static_cast<std::size_t>(std::max(d.nsys, 0)));
  std::vector<long long> keys;
  for (std::int64_t k = 0; k < m; ++k) {
    const int a = ei[k] - d.anchor, b = ej[k] - d.anchor;
    if (a >= 0) incl[a].push_back(static_cast<int>(k) << 1);
    if (b >= 0) incl[b].push_back(static_cast<int>(k) << 1 | 1);
    if (a >= 0 && b >= 0) keys.push_back(static_cast<long long>(std::max(a, b)) * d.nsys + std::min(a, b));
  }
  for (int c = 0; c < d.nsys; ++c) {
    inc.insert(inc.end(), incl[c].begin(), incl[c].end());
    inc_ptr[c + 1] = static_cast<int>(inc.size());
  }
  std::vector<long long> ukeys(keys);
  std::sort(ukeys.begin(), ukeys.end());
  ukeys.erase(std::unique(ukeys.begin(), ukeys.end()), ukeys.end());
  std::vector<std::vector<int>> pedges(ukeys.size());
  for (std::int64_t k = 0; k < m; ++k) {
    const int a = ei[k] - d.anchor, b = ej[k] - d.anchor;
    if (a < 0 || b < 0) continue;
    const long long key = static_cast<long long>(std::max(a, b)) * d.nsys + std::min(a, b);
    pedges[std::lower_bound(ukeys.begin(), ukeys.end(), key) - ukeys.begin()].push_back(static_cast<int>(k));
  }
  std::vector<int> pair_ptr{0}, pair_edge;
  for (const auto& pe : pedges) {
    pair_edge.insert(pair_edge.end(), pe.begin(), pe.end());
    pair_ptr.push_back(static_cast<int>(pair_edge.size()));
  }
  d.npair = static_cast<int>(ukeys.size());
  // tile structure: nested-dissection order of the unknown poses
  std::vector<std::pair<int, int>> gedges;
  for (long long key : ukeys) gedges.emplace_back(static_cast<int>(key / d.nsys), static_cast<int>(key % d.nsys));
  std::vector<int> pos(static_cast<std::size_t>(d.nsys), -1), pos_cam;
  for (const auto& g : nd_camera_groups(d.nsys, gedges, 24)) {
    for (int c : g) {
      pos[c] = static_cast<int>(pos_cam.size());
      pos_cam.push_back(c);
    }
    while (pos_cam.size() % 8) pos_cam.push_back(-1);
  }
  const int npos = static_cast<int>(pos_cam.size()), nt = npos / 8;
  std::vector<std::pair<int, int>> tp;
  for (const auto& e : gedges) {
    const int a = pos[e.first] / 8, b = pos[e.second] / 8;
    tp.emplace_back(std::max(a, b), std::min(a, b));
  }
  const TileCholPlan pl = plan_tile_chol(6 * npos, tp);
  auto slot_of = [&](int ti, int tj) {
    const auto first = pl.rowidx.begin() + pl.colptr[tj], last = pl.rowidx.begin() + pl.colptr[tj + 1];
    return static_cast<int>(std::lower_bound(first, last, ti) - pl.rowidx.begin());
  };
  std::vector<int2> diag_tile(static_cast<std::size_t>(d.nsys)), pair_tile;
  for (int c = 0; c < d.nsys; ++c) diag_tile[c] = int2{slot_of(pos[c] / 8, pos[c] / 8), 6 * (pos[c] % 8)};
  for (const auto& e : gedges) {
    int p1 = pos[e.first], p2 = pos[e.second];
    if (p1 < p2) std::swap(p1, p2);
    pair_tile.push_back(int2{slot_of(p1 / 8, p2 / 8), 6 * (p1 % 8) | (6 * (p2 % 8)) << 8});
  }
  std::vector<unsigned long long> padmask(static_cast<std::size_t>(nt), 0ull);
  for (int q = 0; q < npos; ++q)
    if (pos_cam[q] < 0) padmask[q / 8] |= 0x3full << (6 * (q % 8));

  std::vector<int> vei(ei, ei + m), vej(ej, ej + m);
  std::vector<double> vmeas(meas7, meas7 + 7 * m);
  d.ei = upload(vei);
  d.ej = upload(vej);
  d.meas = upload(vmeas);
  d.white = any_info ? upload(white) : nullptr;
  d.pose = dalloc<double>(7 * static_cast<std::size_t>(n));
  d.pose_t = dalloc<double>(7 * static_cast<std::size_t>(n));
  d.edge = dalloc<double>(28 * static_cast<std::size_t>(m));
  d.inc_ptr = upload(inc_ptr);
  d.inc = upload(inc);
  d.pair_ptr = upload(pair_ptr);
  d.pair_edge = upload(pair_edge);
  d.diag_tile = upload(diag_tile);
  d.pair_tile = upload(pair_tile);
  d.tiles = dalloc<double>(static_cast<std::size_t>(pl.nnz_tiles()) * kTT);
  d.rhs = dalloc<double>(6 * static_cast<std::size_t>(std::max(d.nsys, 1)));
  d.x = dalloc<double>(6 * static_cast<std::size_t>(std::max(d.nsys, 1)));
  d.pose_gsq = dalloc<double>(static_cast<std::size_t>(std::max(d.nsys, 1)));
  d.scal = dalloc<double>(8);
  TileChol& t = tchol_;
  t.nt = nt;
  t.n = 6 * npos;
  t.nnz = static_cast<int>(pl.nnz_tiles());
  t.colptr = upload(pl.colptr);
  t.rowidx = upload(pl.rowidx);
  t.rptr = upload(pl.rptr);
  t.rk = upload(pl.rk);
  t.rslot = upload(pl.rslot);
  t.uptr = upload(pl.uptr);
  t.usrc = upload(pl.usrc);
  t.udst = upload(pl.udst);
  t.bptr = upload(pl.bptr);
  t.bop = upload(pl.bop);
  t.tiles = d.tiles;
  t.rhs = d.rhs;
  t.y = dalloc<double>(static_cast<std::size_t>(std::max(nt, 1)) * kTB);
  t.x = d.x;
  t.pos_cam = upload(pos_cam);
  t.padmask = upload(padmask);
  t.flags = dalloc<unsigned>(static_cast<std::size_t>(t.nnz) + nt);
  ck(cudaMemsetAsync(t.flags, 0, sizeof(unsigned) * (static_cast<std::size_t>(t.nnz) + nt), stream_), "memset");
  t.fail = dalloc<int>(1);
  t.next = dalloc<unsigned>(3);
  ck(cudaMemsetAsync(t.next, 0, 3 * sizeof(unsigned), stream_), "memset counters");
  t.trace = nullptr;
  chol_grid_ = tile_chol_grid(std::max(nt, 1));
  ck(cudaMallocHost(&scal_host_, 8 * sizeof(double)), "cudaMallocHost");
  ck(cudaMallocHost(&fail_host_, sizeof(int)), "cudaMallocHost");
  set_parameters(poses7);
}

PgoProblem::~PgoProblem() {
  cudaSetDevice(opt_.device);
  for (void* p : allocs_) cudaFree(p);
  if (scal_host_) cudaFreeHost(scal_host_);
  if (fail_host_) cudaFreeHost(fail_host_);
  if (stream_) cudaStreamDestroy(stream_);
}

void PgoProblem::set_parameters(const double* poses7) {
  ck(cudaSetDevice(opt_.device), "cudaSetDevice");
  ck(cudaMemcpyAsync(d_.pose, poses7, 7 * sizeof(double) * d_.n, cudaMemcpyHostToDevice, stream_), "H2D poses");
  sync();
}

void PgoProblem::get_parameters(double* poses7) {
  ck(cudaSetDevice(opt_.device), "cudaSetDevice");
  ck(cudaMemcpy(poses7, d_.pose, 7 * sizeof(double) * d_.n, cudaMemcpyDeviceToHost), "D2H poses");
}

void PgoProblem::read_scal() {
  ck(cudaMemcpyAsync(scal_host_, d_.scal, 5 * sizeof(double), cudaMemcpyDeviceToHost, stream_), "D2H");
  sync();
}

static int blocks_of(long long n, int bs) { return static_cast<int>(std::max<long long>(1, (n + bs - 1) / bs)); }

double PgoProblem::evaluate(double* resid6) {
  ck(cudaSetDevice(opt_.device), "cudaSetDevice");
  double* buf = nullptr;
  if (resid6) {
    ck(cudaMalloc(&buf, 6 * sizeof(double) * d_.m), "cudaMalloc");
    d_.resid = buf;
  }
  ck(cudaMemsetAsync(d_.scal, 0, 8 * sizeof(double), stream_), "memset");
  k_pgo_edges<<<blocks_of(d_.m, 128), 128, 0, stream_>>>(d_, d_.pose, 0, 0);
  k_pgo_cost<<<1, 1024, 0, stream_>>>(d_, 0);
  launches_ += 2;
  d_.resid = nullptr;
  read_scal();
  if (buf) {
    ck(cudaMemcpy(resid6, buf, 6 * sizeof(double) * d_.m, cudaMemcpyDeviceToHost), "D2H");
    cudaFree(buf);
  }
  return scal_host_[0];
}

void PgoProblem::jacobian(double* ji36, double* jj36) {
  ck(cudaSetDevice(opt_.device), "cudaSetDevice");
  double* buf = nullptr;
  ck(cudaMalloc(&buf, 36 * sizeof(double) * d_.m), "cudaMalloc");
  d_.jexp = buf;
  ck(cudaMemsetAsync(d_.scal, 0, 8 * sizeof(double), stream_), "memset");
  k_pgo_edges<<<blocks_of(d_.m, 128), 128, 0, stream_>>>(d_, d_.pose, 1, 0);
  launches_ += 1;
  d_.jexp = nullptr;
  sync();
  std::vector<double> h(36 * static_cast<std::size_t>(d_.m));
  ck(cudaMemcpy(h.data(), buf, h.size() * sizeof(double), cudaMemcpyDeviceToHost), "D2H");
  cudaFree(buf);
  for (std::size_t i = 0; i < h.size(); ++i) {
    if (jj36) jj36[i] = h[i];
    if (ji36) ji36[i] = 0.0 - h[i];  // trace.hpp:668: a_i -= up * d_j
  }
}

void PgoProblem::linearize() {
  ck(cudaMemsetAsync(d_.scal, 0, 8 * sizeof(double), stream_), "memset");
  k_pgo_edges<<<blocks_of(d_.m, 128), 128, 0, stream_>>>(d_, d_.pose, 1, 0);
  k_pgo_cost<<<1, 1024, 0, stream_>>>(d_, 0);
  launches_ += 2;
}

// Damped normal matrix into the tiles, tile Cholesky solve of H dx = -g;
// false when a pivot is not positive (NotSpdError -> rejected step).
bool PgoProblem::solve(double lambda, const bae_lm_config& cfg) {
  if (d_.nsys == 0) return false;
  ck(cudaMemsetAsync(d_.tiles, 0, sizeof(double) * kTT * tchol_.nnz, stream_), "memset tiles");
  const int warps = d_.nsys + d_.npair;
  k_pgo_assemble<<<blocks_of(warps, 8), 256, 0, stream_>>>(d_, lambda, cfg.clamp_min, cfg.clamp_max);
  k_pgo_grad<<<1, 1024, 0, stream_>>>(d_);
  ck(cudaMemsetAsync(tchol_.fail, 0, sizeof(int), stream_), "memset fail");
  launches_ += 2 + launch_tile_chol(tchol_, chol_grid_, stream_);
  ck(cudaMemcpyAsync(fail_host_, tchol_.fail, sizeof(int), cudaMemcpyDeviceToHost, stream_), "D2H");
  read_scal();
  if (*fail_host_ == kCholTimeout) throw Error(BAE_ERR_CUDA, "tile Cholesky: dataflow flag wait timed out");
  return *fail_host_ == 0;
}

void PgoProblem::optimize(const double* poses7, const bae_lm_config& cfg, std::vector<bae_iter_record>& traj,
                          bae_lm_report& rep) {
  ck(cudaSetDevice(opt_.device), "cudaSetDevice");
  if (cfg.solver != BAE_SOLVER_CHOLESKY)
    throw Error(BAE_ERR_UNSUPPORTED, "pose graphs use the direct solver (solver = cholesky) on the B200 path");
  if (!(cfg.damping_min <= cfg.initial_damping && cfg.initial_damping <= cfg.damping_max))
    throw Error(BAE_ERR_INVALID_ARGUMENT, "LmConfig: damping out of bounds");
  if (!(cfg.damping_up > 0.0 && cfg.damping_down > 0.0))
    throw Error(BAE_ERR_INVALID_ARGUMENT, "LmConfig: damping factors must be positive");
  if (cfg.plateau_patience < 1) throw Error(BAE_ERR_INVALID_ARGUMENT, "LmConfig: patience must be >= 1");
  if (poses7) set_parameters(poses7);
  const double rows = static_cast<double>(d_.m);
  cudaEvent_t ev0, ev1;
  ck(cudaEventCreate(&ev0), "event");
  ck(cudaEventCreate(&ev1), "event");
  ck(cudaEventRecord(ev0, stream_), "event");
  const auto t0 = std::chrono::steady_clock::now();
  linearize();
  read_scal();
  double cost = scal_host_[0];
  std::vector<double> history{cost};
  double lambda = cfg.initial_damping;
  traj.clear();
  traj.push_back({0, 1, cost, cost / rows, lambda, 0.0, 0, 0.0, cost});
  int iterations = 0, accepted_steps = 0, rejected_steps = 0;
  bool need_lin = false;
  rep = bae_lm_report{};
  rep.reason = BAE_TERM_MAX_ITERS;
  while (iterations < cfg.max_iterations) {  // lm_step, lm.hpp:115-200
    const double lambda_used = lambda;
    const bool saturated = lambda >= cfg.damping_max;
    if (need_lin) {
      linearize();
      need_lin = false;
    }
    const bool ok = solve(lambda_used, cfg);
    const double grad = std::sqrt(scal_host_[1]);
    if (iterations == 0) traj[0].grad_norm = grad;
    bool accepted = false;
    double trial = std::numeric_limits<double>::quiet_NaN();
    if (ok) {
      k_pgo_retract<<<blocks_of(d_.n, 128), 128, 0, stream_>>>(d_);
      k_pgo_edges<<<blocks_of(d_.m, 128), 128, 0, stream_>>>(d_, d_.pose_t, 0, 1);
      k_pgo_cost<<<1, 1024, 0, stream_>>>(d_, 1);
      launches_ += 3;
      read_scal();
      trial = scal_host_[2];
      if (trial < cost) {
        ck(cudaMemcpyAsync(d_.pose, d_.pose_t, 7 * sizeof(double) * d_.n, cudaMemcpyDeviceToDevice, stream_),
           "commit");
        cost = trial;
        history.push_back(cost);
        ++accepted_steps;
        accepted = true;
        need_lin = true;
      }
    }
    if (accepted)
      lambda = std::max(lambda * cfg.damping_down, cfg.damping_min);
    else {
      ++rejected_steps;
      lambda = std::min(lambda * cfg.damping_up, cfg.damping_max);
    }
    ++iterations;
    const double el = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    traj.push_back({iterations, accepted ? 1 : 0, history.back(), history.back() / rows, lambda_used, el, 0, grad,
                    trial});
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
  ck(cudaEventRecord(ev1, stream_), "event");
  sync();
  float ms = 0.f;
  ck(cudaEventElapsedTime(&ms, ev0, ev1), "elapsed");
  cudaEventDestroy(ev0);
  cudaEventDestroy(ev1);
  rep.device_seconds = ms * 1e-3;
  rep.iterations = iterations;
  rep.final_cost = history.back();
  rep.final_mse = rep.final_cost / rows;
  rep.accepted_steps = accepted_steps;
  rep.rejected_steps = rejected_steps;
  rep.final_lambda = lambda;
  rep.solve_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
}

}  // namespace bae
