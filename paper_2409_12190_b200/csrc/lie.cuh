// SE(3) / BAL-camera arithmetic for the device kernels (and the host-side
// scene generator). Formulas follow the reference's lie.hpp and camera.hpp
// line for line (cited per function); storage is plain doubles so the same
// code runs in registers on sm_100a and on the host.
#pragma once

#include <cmath>

#if defined(__CUDACC__)
#define BAE_HD __host__ __device__ __forceinline__
#else
#define BAE_HD inline
#endif

namespace bae {

struct Q4 {
  double x, y, z, w;
};
struct P3 {
  double x, y, z;
};

BAE_HD P3 cross3(const P3& a, const P3& b) {
  return {a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x};
}

// QuatRotation ctor: normalise then canonicalise to w >= 0 (lie.hpp:33-45).
// Returns false for a zero / non-finite quaternion.
BAE_HD bool quat_normalize(double x, double y, double z, double w, Q4& out) {
  const double n = sqrt(x * x + y * y + z * z + w * w);
  if (!(n > 0.0) || !isfinite(n)) return false;
  double inv = 1.0 / n;
  if (w < 0.0) inv = -inv;
  out = {x * inv, y * inv, z * inv, w * inv};
  return true;
}

// Hamilton product then renormalise (lie.hpp:82-86).
BAE_HD bool quat_mul(const Q4& a, const Q4& b, Q4& out) {
  const double w = a.w * b.w - a.x * b.x - a.y * b.y - a.z * b.z;
  const double x = a.w * b.x + a.x * b.w + a.y * b.z - a.z * b.y;
  const double y = a.w * b.y + a.y * b.w + a.z * b.x - a.x * b.z;
  const double z = a.w * b.z + a.z * b.w + a.x * b.y - a.y * b.x;
  return quat_normalize(x, y, z, w, out);
}

// toRotationMatrix (lie.hpp:68-70), row-major.
BAE_HD void quat_to_R(const Q4& q, double* r) {
  const double tx = 2.0 * q.x, ty = 2.0 * q.y, tz = 2.0 * q.z;
  const double twx = tx * q.w, twy = ty * q.w, twz = tz * q.w;
  const double txx = tx * q.x, txy = ty * q.x, txz = tz * q.x;
  const double tyy = ty * q.y, tyz = tz * q.y, tzz = tz * q.z;
  r[0] = 1.0 - (tyy + tzz);
  r[1] = txy - twz;
  r[2] = txz + twy;
  r[3] = txy + twz;
  r[4] = 1.0 - (txx + tzz);
  r[5] = tyz - twx;
  r[6] = txz - twy;
  r[7] = tyz + twx;
  r[8] = 1.0 - (txx + tyy);
}

// q p q* through the double-cross identity (lie.hpp:88-93).
BAE_HD P3 quat_rotate(const Q4& q, const P3& p) {
  const P3 u{q.x, q.y, q.z};
  P3 t = cross3(u, p);
  t = {2.0 * t.x, 2.0 * t.y, 2.0 * t.z};
  const P3 c = cross3(u, t);
  return {p.x + q.w * t.x + c.x, p.y + q.w * t.y + c.y, p.z + q.w * t.z + c.z};
}

// se3_exp (lie.hpp:173-186): quaternion from sin(theta/2)/theta with the
// Taylor branch below 1e-8, translation V(omega) rho (lie.hpp:141-156).
BAE_HD bool se3_exp(const double* tau, Q4& q, P3& t) {
  const double ox = tau[3], oy = tau[4], oz = tau[5];
  const double theta = sqrt(ox * ox + oy * oy + oz * oz);
  const double sh = theta < 1e-8 ? 0.5 - theta * theta / 48.0 : sin(0.5 * theta) / theta;
  if (!quat_normalize(sh * ox, sh * oy, sh * oz, cos(0.5 * theta), q)) return false;
  const double a = theta < 1e-8 ? 0.5 - theta * theta / 24.0 : (1.0 - cos(theta)) / (theta * theta);
  const double b =
      theta < 1e-8 ? 1.0 / 6.0 - theta * theta / 120.0 : (theta - sin(theta)) / (theta * theta * theta);
  const double o[9] = {0.0, -oz, oy, oz, 0.0, -ox, -oy, ox, 0.0};
  double v[9];
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) {
      const double oo = o[i * 3] * o[j] + o[i * 3 + 1] * o[3 + j] + o[i * 3 + 2] * o[6 + j];
      v[i * 3 + j] = (i == j ? 1.0 : 0.0) + a * o[i * 3 + j] + b * oo;
    }
  t = {v[0] * tau[0] + v[1] * tau[1] + v[2] * tau[2], v[3] * tau[0] + v[4] * tau[1] + v[5] * tau[2],
       v[6] * tau[0] + v[7] * tau[1] + v[8] * tau[2]};
  return isfinite(t.x) && isfinite(t.y) && isfinite(t.z);
}

// Left retraction Exp(delta) o T (lie.hpp:204-207, 219-221).
BAE_HD bool se3_retract(const Q4& q0, const P3& t0, const double* tau, Q4& q1, P3& t1) {
  Q4 qe;
  P3 te;
  if (!se3_exp(tau, qe, te)) return false;
  if (!quat_mul(qe, q0, q1)) return false;
  const P3 r = quat_rotate(qe, t0);
  t1 = {r.x + te.x, r.y + te.y, r.z + te.z};
  return true;
}

// se3_log rotation part (lie.hpp:189-199): omega only.
BAE_HD P3 so3_log(const Q4& q) {
  const double s = sqrt(q.x * q.x + q.y * q.y + q.z * q.z);
  const double theta = 2.0 * atan2(s, q.w);
  const double k = s < 1e-8 ? 2.0 + theta * theta / 12.0 : theta / s;
  return {k * q.x, k * q.y, k * q.z};
}

constexpr double kBalDepthEps = 1e-12;  // camera.hpp:30

// bal_project_cam forward (camera.hpp:50-57). Returns false on the camera
// plane (CheiralityError in the reference).
BAE_HD bool bal_project(const P3& p, double f, double k1, double k2, double& u, double& v) {
  if (!(fabs(p.z) > kBalDepthEps)) return false;
  const double qx = -p.x / p.z, qy = -p.y / p.z;
  const double s = qx * qx + qy * qy;
  const double d = 1.0 + s * (k1 + s * k2);
  const double fd = f * d;
  u = fd * qx;
  v = fd * qy;
  return true;
}

// bal_project_cam_jacobian (camera.hpp:59-71): D (2x3, row-major) of the
// pixel w.r.t. the camera-frame point.
BAE_HD void bal_dproj(const P3& p, double f, double k1, double k2, double* D) {
  const double iz = 1.0 / p.z;
  const double qx = -p.x * iz, qy = -p.y * iz;
  const double s = qx * qx + qy * qy;
  const double d = 1.0 + s * (k1 + s * k2);
  const double dd = k1 + 2.0 * k2 * s;
  const double dq02 = p.x * iz * iz, dq12 = p.y * iz * iz;
  const double ds0 = (2.0 * qx) * (-iz);
  const double ds1 = (2.0 * qy) * (-iz);
  const double ds2 = (2.0 * qx) * dq02 + (2.0 * qy) * dq12;
  const double a0 = dd * ds0, a1 = dd * ds1, a2 = dd * ds2;
  D[0] = f * (d * (-iz) + qx * a0);
  D[1] = f * (qx * a1);
  D[2] = f * (d * dq02 + qx * a2);
  D[3] = f * (qy * a0);
  D[4] = f * (d * (-iz) + qy * a1);
  D[5] = f * (d * dq12 + qy * a2);
}

constexpr double kPinholeDepthEps = 1e-9;  // camera.hpp:30

// pinhole_project_cam forward (camera.hpp:33-38): false unless the point is
// in front of the camera (CheiralityError in the reference).
BAE_HD bool pinhole_project(const P3& p, double fx, double fy, double cx, double cy, double& u, double& v) {
  if (!(p.z > kPinholeDepthEps)) return false;
  u = fx * p.x / p.z + cx;
  v = fy * p.y / p.z + cy;
  return true;
}

// pinhole_project_cam_jacobian (camera.hpp:40-46).
BAE_HD void pinhole_dproj(const P3& p, double fx, double fy, double* D) {
  const double iz = 1.0 / p.z;
  D[0] = fx * iz;
  D[1] = 0.0;
  D[2] = -fx * p.x * iz * iz;
  D[3] = 0.0;
  D[4] = fy * iz;
  D[5] = -fy * p.y * iz * iz;
}

// The camera variant of a problem (make_ba_problem, problems.hpp:94-98: one
// variant per problem) on a 4-double intrinsics record: BAL [f k1 k2 0],
// pinhole [fx fy cx cy].
BAE_HD bool cam_project(bool pinhole, const P3& p, const double* k, double& u, double& v) {
  return pinhole ? pinhole_project(p, k[0], k[1], k[2], k[3], u, v) : bal_project(p, k[0], k[1], k[2], u, v);
}
BAE_HD void cam_dproj(bool pinhole, const P3& p, const double* k, double* D) {
  if (pinhole)
    pinhole_dproj(p, k[0], k[1], D);
  else
    bal_dproj(p, k[0], k[1], k[2], D);
}

}  // namespace bae
