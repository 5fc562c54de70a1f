// Synthetic BAL-shaped scenes. The reference generator
// synth_ba (io/synthetic.hpp:46-91) gives every camera every point, so it
// cannot produce the BAL observation counts; this generator keeps its scene
// conventions -- unit-box points, a radius-4 ring of inward-looking cameras
// with the BAL -z convention (look_at_origin, io/synthetic.hpp:26-38),
// f = 500, exact projections plus pixel noise, poses perturbed in the tangent
// -- and adds banded sparse visibility with exactly the requested number of
// observations, none duplicated, ordered camera-major like BAL files.
//
// The BAL text round trip (serialize_bal at %.17g, parse_bal,
// io/bal.hpp:103-157) is the identity on doubles (%.17g round-trips), so it is
// skipped; the camera rotation still goes through Rodrigues and back exactly
// as BalCamera::pose does (io/bal.hpp:24-26).
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <stdexcept>
#include <vector>

#include "bae/rng.hpp"
#include "bae_internal.hpp"
#include "bal_io.hpp"
#include "lie.cuh"

namespace bae {

// look_at_origin (io/synthetic.hpp:26-38) including Eigen's matrix ->
// quaternion conversion.
void look_at_origin(const P3& pos, Q4& q, P3& t) {
  const double n = std::sqrt(pos.x * pos.x + pos.y * pos.y + pos.z * pos.z);
  const P3 zc{pos.x / n, pos.y / n, pos.z / n};
  P3 up{0, 0, 1};
  if (std::fabs(up.x * zc.x + up.y * zc.y + up.z * zc.z) > 0.95) up = {0, 1, 0};
  P3 xc = cross3(up, zc);
  const double xn = std::sqrt(xc.x * xc.x + xc.y * xc.y + xc.z * xc.z);
  xc = {xc.x / xn, xc.y / xn, xc.z / xn};
  const P3 yc = cross3(zc, xc);
  const double m[9] = {xc.x, xc.y, xc.z, yc.x, yc.y, yc.z, zc.x, zc.y, zc.z};
  double c[4];  // x y z w
  double tr = m[0] + m[4] + m[8];
  if (tr > 0.0) {
    tr = std::sqrt(tr + 1.0);
    c[3] = 0.5 * tr;
    tr = 0.5 / tr;
    c[0] = (m[7] - m[5]) * tr;
    c[1] = (m[2] - m[6]) * tr;
    c[2] = (m[3] - m[1]) * tr;
  } else {
    int i = 0;
    if (m[4] > m[0]) i = 1;
    if (m[8] > m[i * 4]) i = 2;
    const int j = (i + 1) % 3, k = (j + 1) % 3;
    tr = std::sqrt(m[i * 4] - m[j * 4] - m[k * 4] + 1.0);
    c[i] = 0.5 * tr;
    tr = 0.5 / tr;
    c[3] = (m[k * 3 + j] - m[j * 3 + k]) * tr;
    c[j] = (m[j * 3 + i] + m[i * 3 + j]) * tr;
    c[k] = (m[k * 3 + i] + m[i * 3 + k]) * tr;
  }
  if (!quat_normalize(c[0], c[1], c[2], c[3], q)) throw Error(BAE_ERR_INVALID_ARGUMENT, "look_at_origin");
  t = {-(m[0] * pos.x + m[1] * pos.y + m[2] * pos.z), -(m[3] * pos.x + m[4] * pos.y + m[5] * pos.z),
       -(m[6] * pos.x + m[7] * pos.y + m[8] * pos.z)};
}

void synth_bal_shaped(int C, int P, std::int64_t N, std::uint64_t seed, double pixel_sigma, double pose_sigma,
                      double point_sigma, double* poses7, double* points3, double* intr3, std::int32_t* cam_idx,
                      std::int32_t* pt_idx, double* px2, double* true_poses7, double* true_points3) {
  if (C < 1 || P < 1) throw Error(BAE_ERR_INVALID_ARGUMENT, "synth: counts must be positive");
  const int W = std::min(C, 16);
  if (N < 2 * std::int64_t{P} && C >= 2)
    throw Error(BAE_ERR_INVALID_ARGUMENT, "synth: need at least two observations per point");
  if (N > std::int64_t{P} * W) throw Error(BAE_ERR_INVALID_ARGUMENT, "synth: too many observations for window");
  Rng rng(seed);

  std::vector<P3> tp(static_cast<std::size_t>(P));
  for (int p = 0; p < P; ++p) {
    const double x = rng.uniform(-0.5, 0.5);
    const double y = rng.uniform(-0.5, 0.5);
    const double z = rng.uniform(-0.5, 0.5);
    tp[p] = {x, y, z};
  }
  std::vector<Q4> tq(static_cast<std::size_t>(C));
  std::vector<P3> tt(static_cast<std::size_t>(C));
  for (int c = 0; c < C; ++c) {
    const double ang = 2.0 * M_PI * c / C;
    const P3 pos{4.0 * std::cos(ang), 4.0 * std::sin(ang), 0.5 + 0.1 * rng.normal()};
    look_at_origin(pos, tq[c], tt[c]);
    intr3[c * 3] = 500.0;
    intr3[c * 3 + 1] = rng.uniform(-0.1, 0.1);
    intr3[c * 3 + 2] = rng.uniform(-0.01, 0.01);
  }

  // Banded visibility: point j sees m_j distinct cameras drawn by a partial
  // Fisher-Yates shuffle of the window {a, ..., a+W-1} mod C.
  const std::int64_t base = N / P, extra = N % P;
  std::vector<std::int64_t> cam_count(static_cast<std::size_t>(C) + 1, 0);
  std::vector<std::int32_t> vis_cam(static_cast<std::size_t>(N));
  std::vector<std::int64_t> pt_begin(static_cast<std::size_t>(P) + 1, 0);
  int window[16];
  std::int64_t w = 0;
  for (int j = 0; j < P; ++j) {
    const int m = static_cast<int>(base + (j < extra ? 1 : 0));
    const int a = static_cast<int>(rng.index(static_cast<std::uint64_t>(C)));
    for (int i = 0; i < W; ++i) window[i] = (a + i) % C;
    for (int i = 0; i < m; ++i) {
      const int r = i + static_cast<int>(rng.index(static_cast<std::uint64_t>(W - i)));
      std::swap(window[i], window[r]);
      vis_cam[w++] = window[i];
      ++cam_count[window[i] + 1];
    }
    pt_begin[j + 1] = w;
  }
  // Camera-major order (then point ascending), like BAL files.
  for (int c = 0; c < C; ++c) cam_count[c + 1] += cam_count[c];
  std::vector<std::int64_t> cursor(cam_count.begin(), cam_count.end() - 1);
  for (int j = 0; j < P; ++j)
    for (std::int64_t i = pt_begin[j]; i < pt_begin[j + 1]; ++i) {
      const std::int64_t k = cursor[vis_cam[i]]++;
      cam_idx[k] = vis_cam[i];
      pt_idx[k] = j;
    }
  for (std::int64_t k = 0; k < N; ++k) {
    const int c = cam_idx[k];
    const P3 y = quat_rotate(tq[c], tp[pt_idx[k]]);
    double u = 0, v = 0;
    if (!bal_project({y.x + tt[c].x, y.y + tt[c].y, y.z + tt[c].z}, intr3[c * 3], intr3[c * 3 + 1],
                     intr3[c * 3 + 2], u, v))
      throw Error(BAE_ERR_CHEIRALITY, "synth: point on camera plane", k);
    const double n0 = rng.normal(), n1 = rng.normal();
    px2[k * 2] = u + pixel_sigma * n0;
    px2[k * 2 + 1] = v + pixel_sigma * n1;
  }
  for (int c = 0; c < C; ++c) {
    double tau[6];
    for (int i = 0; i < 6; ++i) tau[i] = pose_sigma * rng.normal();
    Q4 q;
    P3 t;
    if (!se3_retract(tq[c], tt[c], tau, q, t)) throw Error(BAE_ERR_INVALID_ARGUMENT, "synth: retract");
    // BAL camera record: Rodrigues vector, then BalCamera::pose re-derives the
    // quaternion through se3_exp (io/bal.hpp:24-26).
    const P3 rod = so3_log(q);
    const double tau_rot[6] = {0, 0, 0, rod.x, rod.y, rod.z};
    Q4 qb;
    P3 unused;
    se3_exp(tau_rot, qb, unused);
    double* o = poses7 + c * 7;
    o[0] = t.x; o[1] = t.y; o[2] = t.z;
    o[3] = qb.x; o[4] = qb.y; o[5] = qb.z; o[6] = qb.w;
    if (true_poses7) {
      double* g = true_poses7 + c * 7;
      g[0] = tt[c].x; g[1] = tt[c].y; g[2] = tt[c].z;
      g[3] = tq[c].x; g[4] = tq[c].y; g[5] = tq[c].z; g[6] = tq[c].w;
    }
  }
  for (int p = 0; p < P; ++p) {
    const double a = rng.normal(), b = rng.normal(), c = rng.normal();
    points3[p * 3] = tp[p].x + point_sigma * a;
    points3[p * 3 + 1] = tp[p].y + point_sigma * b;
    points3[p * 3 + 2] = tp[p].z + point_sigma * c;
    if (true_points3) {
      true_points3[p * 3] = tp[p].x;
      true_points3[p * 3 + 1] = tp[p].y;
      true_points3[p * 3 + 2] = tp[p].z;
    }
  }
}

}  // namespace bae
