// C++ mirror of the reference's BA / LM API (traceopt, header-only C++20)
// over the C ABI of libbae_b200.so. A caller of the reference's
//   make_ba_problem (problems.hpp:87-136), TracedProblem (problems.hpp:36-82),
//   optimize / LmConfig / LmReport (lm.hpp:23-77, 205-255)
// switches includes and namespace (traceopt:: -> bae::traceopt::) and keeps
// its call sites; the exception classes of errors.hpp are re-thrown from the
// ABI's return codes. Types are plain structs (no Eigen dependency):
// Vec3 {x, y, z}, QuatRotation {x, y, z, w}, PoseSE3 {rotation, translation}.
#pragma once

#include <cstdint>
#include <memory>
#include <span>
#include <stdexcept>
#include <string>
#include <variant>
#include <vector>

#include "bae_b200.h"

namespace bae::traceopt {

struct Vec3 {
  double x = 0, y = 0, z = 0;
};
struct Vec2 {
  double x = 0, y = 0;
};
struct QuatRotation {  // unit, w >= 0 (lie.hpp:26-45); taken as-is like read_pose
  double x = 0, y = 0, z = 0, w = 1;
};
struct PoseSE3 {  // world -> camera (lie.hpp:119-136)
  QuatRotation rotation;
  Vec3 translation;
};
struct PinholeIntrinsics {  // camera.hpp:17-19
  double fx = 0, fy = 0, cx = 0, cy = 0;
};
struct BalIntrinsics {  // camera.hpp:23-25
  double f = 0, k1 = 0, k2 = 0;
};
using CameraIntrinsics = std::variant<PinholeIntrinsics, BalIntrinsics>;  // camera.hpp:27
struct Observation {  // problems.hpp:19-23
  std::int32_t camera_index = 0;
  std::int32_t point_index = 0;
  Vec2 pixel;
};

// errors.hpp:10-69
class IndexError : public std::out_of_range {
 public:
  IndexError(const std::string& m, std::size_t pos) : std::out_of_range(m), position_(pos) {}
  std::size_t position() const { return position_; }

 private:
  std::size_t position_;
};
class UnsupportedOperationError : public std::logic_error {
 public:
  using std::logic_error::logic_error;
};
class CheiralityError : public std::runtime_error {
 public:
  CheiralityError(const std::string& m, std::size_t obs) : std::runtime_error(m), observation_(obs) {}
  std::size_t observation() const { return observation_; }

 private:
  std::size_t observation_;
};
class NotSpdError : public std::runtime_error {
 public:
  NotSpdError(const std::string& m, int pivot) : std::runtime_error(m), pivot_(pivot) {}
  int pivot() const { return pivot_; }

 private:
  int pivot_;
};
class NumericalBreakdownError : public std::runtime_error {
 public:
  using std::runtime_error::runtime_error;
};
class DeviceError : public std::runtime_error {
 public:
  using std::runtime_error::runtime_error;
};

namespace detail {
inline void check(int code) {
  if (code == BAE_OK) return;
  const std::string msg = bae_last_error();
  const std::int64_t idx = bae_last_error_index();
  switch (code) {
    case BAE_ERR_INVALID_ARGUMENT:
      throw std::invalid_argument(msg);
    case BAE_ERR_INDEX:
      throw IndexError(msg, static_cast<std::size_t>(idx));
    case BAE_ERR_CHEIRALITY:
      throw CheiralityError(msg, static_cast<std::size_t>(idx));
    case BAE_ERR_NOT_SPD:
      throw NotSpdError(msg, static_cast<int>(idx));
    case BAE_ERR_NUMERICAL_BREAKDOWN:
      throw NumericalBreakdownError(msg);
    case BAE_ERR_UNSUPPORTED:
      throw UnsupportedOperationError(msg);
    default:
      throw DeviceError(msg);
  }
}
inline void pack_poses(std::span<const PoseSE3> in, std::vector<double>& out) {
  out.resize(in.size() * 7);
  for (std::size_t i = 0; i < in.size(); ++i) {
    const PoseSE3& p = in[i];
    double* o = out.data() + i * 7;
    o[0] = p.translation.x;
    o[1] = p.translation.y;
    o[2] = p.translation.z;
    o[3] = p.rotation.x;
    o[4] = p.rotation.y;
    o[5] = p.rotation.z;
    o[6] = p.rotation.w;
  }
}
inline void pack_points(std::span<const Vec3> in, std::vector<double>& out) {
  out.resize(in.size() * 3);
  for (std::size_t i = 0; i < in.size(); ++i) {
    out[i * 3] = in[i].x;
    out[i * 3 + 1] = in[i].y;
    out[i * 3 + 2] = in[i].z;
  }
}
}  // namespace detail

enum class SolverChoice { cholesky = BAE_SOLVER_CHOLESKY, pcg = BAE_SOLVER_PCG };
enum class TerminationReason { plateau = BAE_TERM_PLATEAU, max_iters = BAE_TERM_MAX_ITERS,
                               solver_failure = BAE_TERM_SOLVER_FAILURE };

struct LmConfig {  // lm.hpp:23-38
  double initial_damping = 1e-6;
  double damping_min = 1e-16;
  double damping_max = 1e16;
  double damping_up = 2.0;
  double damping_down = 0.5;
  double clamp_min = 1e-6;
  double clamp_max = 1e32;
  int max_iterations = 10;
  int plateau_patience = 3;
  double plateau_rel_tol = 1e-6;
  SolverChoice solver = SolverChoice::cholesky;
  double pcg_tol = 1e-8;
  std::int64_t pcg_max_iters = 0;
  bool use_caches = true;

  bae_lm_config to_c() const {
    bae_lm_config c;
    bae_lm_config_default(&c);
    c.initial_damping = initial_damping;
    c.damping_min = damping_min;
    c.damping_max = damping_max;
    c.damping_up = damping_up;
    c.damping_down = damping_down;
    c.clamp_min = clamp_min;
    c.clamp_max = clamp_max;
    c.max_iterations = max_iterations;
    c.plateau_patience = plateau_patience;
    c.plateau_rel_tol = plateau_rel_tol;
    c.solver = static_cast<int32_t>(solver);
    c.pcg_tol = pcg_tol;
    c.pcg_max_iters = pcg_max_iters;
    c.use_caches = use_caches ? 1 : 0;
    return c;
  }
};

struct LmIterationRecord {  // lm.hpp:62-69
  int iteration = 0;
  double cost = 0.0;
  double mse = 0.0;
  double lambda = 0.0;
  bool accepted = true;
  double cum_time_s = 0.0;
};

struct LmReport {  // lm.hpp:71-77
  double final_cost = 0.0;
  double final_mse = 0.0;
  int iterations = 0;
  std::vector<LmIterationRecord> trajectory;
  TerminationReason reason = TerminationReason::max_iters;
};

// Device-resident problem (TracedProblem, problems.hpp:36-82).
class TracedProblem {
 public:
  explicit TracedProblem(bae_problem* h) : h_(h, &bae_destroy) {}
  int num_poses() const { return bae_num_poses(h_.get()); }
  int num_points() const { return bae_num_points(h_.get()); }
  int residual_rows() const { return static_cast<int>(bae_residual_rows(h_.get())); }
  int residual_width() const { return 2; }
  bool has_poses() const { return true; }
  bool has_points() const { return true; }

  void set_parameters(std::span<const PoseSE3> poses, std::span<const Vec3> points) {
    std::vector<double> p7, p3;
    detail::pack_poses(poses, p7);
    detail::pack_points(points, p3);
    detail::check(bae_set_parameters(h_.get(), p7.data(), p3.data()));
  }
  // residual vector r = projection - pixel, 2 per observation (problems.hpp:66)
  std::vector<double> evaluate() {
    std::vector<double> r(static_cast<std::size_t>(residual_rows()) * 2);
    double cost = 0.0;
    detail::check(bae_evaluate(h_.get(), r.data(), &cost));
    return r;
  }
  bae_problem* handle() { return h_.get(); }

 private:
  std::unique_ptr<bae_problem, void (*)(bae_problem*)> h_;
};

// make_ba_problem (problems.hpp:87-136): one camera variant per problem,
// mixed variants are rejected like the reference (problems.hpp:94-98).
inline TracedProblem make_ba_problem(std::span<const PoseSE3> poses, std::span<const Vec3> points,
                                     std::span<const CameraIntrinsics> intrinsics,
                                     std::span<const Observation> observations, int device = 0) {
  if (intrinsics.size() != poses.size())
    throw std::invalid_argument("make_ba_problem: one intrinsics entry per camera required");
  if (observations.empty()) throw std::invalid_argument("make_ba_problem: no observations");
  const bool pinhole = std::holds_alternative<PinholeIntrinsics>(intrinsics[0]);
  for (const auto& k : intrinsics)
    if (std::holds_alternative<PinholeIntrinsics>(k) != pinhole)
      throw std::invalid_argument("make_ba_problem: mixed camera variants are not supported");
  const std::size_t kw = pinhole ? 4 : 3;
  std::vector<double> p7, p3, kk(intrinsics.size() * kw), px(observations.size() * 2);
  std::vector<std::int32_t> ci(observations.size()), pi(observations.size());
  detail::pack_poses(poses, p7);
  detail::pack_points(points, p3);
  for (std::size_t i = 0; i < intrinsics.size(); ++i) {
    if (pinhole) {
      const auto& k = std::get<PinholeIntrinsics>(intrinsics[i]);
      kk[i * 4] = k.fx;
      kk[i * 4 + 1] = k.fy;
      kk[i * 4 + 2] = k.cx;
      kk[i * 4 + 3] = k.cy;
    } else {
      const auto& k = std::get<BalIntrinsics>(intrinsics[i]);
      kk[i * 3] = k.f;
      kk[i * 3 + 1] = k.k1;
      kk[i * 3 + 2] = k.k2;
    }
  }
  for (std::size_t k = 0; k < observations.size(); ++k) {
    ci[k] = observations[k].camera_index;
    pi[k] = observations[k].point_index;
    px[k * 2] = observations[k].pixel.x;
    px[k * 2 + 1] = observations[k].pixel.y;
  }
  bae_create_options opt;
  bae_create_options_default(&opt);
  opt.device = device;
  opt.camera_model = pinhole ? BAE_CAMERA_PINHOLE : BAE_CAMERA_BAL;
  bae_problem* h = nullptr;
  detail::check(bae_create_ba(p7.data(), static_cast<int32_t>(poses.size()), p3.data(),
                              static_cast<int32_t>(points.size()), kk.data(), ci.data(), pi.data(), px.data(),
                              static_cast<int64_t>(observations.size()), &opt, &h));
  return TracedProblem(h);
}

// BAL-only convenience overload (the BalProblem path, io/bal.hpp:159-161).
inline TracedProblem make_ba_problem(std::span<const PoseSE3> poses, std::span<const Vec3> points,
                                     std::span<const BalIntrinsics> intrinsics,
                                     std::span<const Observation> observations, int device = 0) {
  std::vector<CameraIntrinsics> v(intrinsics.begin(), intrinsics.end());
  return make_ba_problem(poses, points, std::span<const CameraIntrinsics>(v), observations, device);
}

// optimize (lm.hpp:205-255); the model keeps the optimised parameters.
inline LmReport optimize(TracedProblem& model, std::span<const PoseSE3> init_poses, std::span<const Vec3> init_points,
                         const LmConfig& config, std::vector<PoseSE3>* out_poses = nullptr,
                         std::vector<Vec3>* out_points = nullptr) {
  std::vector<double> p7, p3;
  detail::pack_poses(init_poses, p7);
  detail::pack_points(init_points, p3);
  const bae_lm_config c = config.to_c();
  std::vector<bae_iter_record> recs(static_cast<std::size_t>(config.max_iterations) + 1);
  bae_lm_report rep{};
  std::vector<double> o7(p7.size()), o3(p3.size());
  detail::check(bae_optimize(model.handle(), p7.data(), p3.data(), &c, recs.data(),
                             static_cast<int32_t>(recs.size()), &rep, o7.data(), o3.data()));
  LmReport out;
  out.final_cost = rep.final_cost;
  out.final_mse = rep.final_mse;
  out.iterations = rep.iterations;
  out.reason = static_cast<TerminationReason>(rep.reason);
  for (int i = 0; i <= rep.iterations && i < static_cast<int>(recs.size()); ++i)
    out.trajectory.push_back({recs[i].iteration, recs[i].cost, recs[i].mse, recs[i].lambda, recs[i].accepted != 0,
                              recs[i].cum_time_s});
  if (out_poses) {
    out_poses->resize(init_poses.size());
    for (std::size_t i = 0; i < out_poses->size(); ++i) {
      const double* s = o7.data() + i * 7;
      (*out_poses)[i] = {{s[3], s[4], s[5], s[6]}, {s[0], s[1], s[2]}};
    }
  }
  if (out_points) {
    out_points->resize(init_points.size());
    for (std::size_t i = 0; i < out_points->size(); ++i) (*out_points)[i] = {o3[i * 3], o3[i * 3 + 1], o3[i * 3 + 2]};
  }
  return out;
}

}  // namespace bae::traceopt
