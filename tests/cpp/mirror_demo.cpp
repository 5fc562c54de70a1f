// Drop-in usage of the C++ mirror (include/bae/traceopt.hpp): the call sites
// read like the reference's (make_ba_problem + optimize). On a machine
// without a GPU, validation errors still surface as the reference's
// exception types; the device step reports DeviceError.
#include <cstdio>
#include <vector>

#include "bae/traceopt.hpp"

using namespace bae::traceopt;

int main(int argc, char** argv) {
  const bool expect_gpu = argc > 1;
  std::vector<PoseSE3> poses(2);
  poses[1].translation = {0.3, 0.0, 0.0};
  std::vector<Vec3> points = {{0.1, 0.0, -3.0}, {-0.2, 0.1, -3.5}, {0.0, 0.2, -2.5}};
  std::vector<BalIntrinsics> intr(2, BalIntrinsics{500.0, 0.0, 0.0});
  std::vector<Observation> obs;
  for (int c = 0; c < 2; ++c)
    for (int p = 0; p < 3; ++p) obs.push_back({c, p, {1.0 * c, 2.0 * p}});
  // IndexError carries the offending position (problems.hpp:107-110)
  auto bad = obs;
  bad[4].point_index = 7;
  try {
    make_ba_problem(poses, points, intr, bad);
    std::printf("FAIL no IndexError\n");
    return 1;
  } catch (const IndexError& e) {
    if (e.position() != 4) return 2;
  }
  try {
    make_ba_problem(poses, points, std::vector<BalIntrinsics>(1), obs);
    return 3;
  } catch (const std::invalid_argument&) {
  }
  try {
    TracedProblem prob = make_ba_problem(poses, points, intr, obs);
    LmConfig cfg;
    cfg.max_iterations = 5;
    const LmReport rep = optimize(prob, poses, points, cfg);
    std::printf("optimize: %d iterations, final cost %.6g\n", rep.iterations, rep.final_cost);
    return rep.trajectory.size() == static_cast<std::size_t>(rep.iterations) + 1 ? 0 : 4;
  } catch (const DeviceError& e) {
    std::printf("device: %s\n", e.what());
    return expect_gpu ? 5 : 0;
  }
}
