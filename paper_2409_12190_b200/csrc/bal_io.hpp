// BAL files and the reference's dense synthetic scene (bal_io.cpp).
#pragma once

#include <cstdint>
#include <string>
#include <vector>

#include "lie.cuh"

namespace bae {

// BalProblem (io/bal.hpp:29-47): cameras as the 9 BAL scalars
// [rodrigues3, translation3, f, k1, k2], points, observations.
struct BalData {
  int C = 0, P = 0;
  std::int64_t N = 0;
  std::vector<double> cameras;  // 9 C
  std::vector<double> points;   // 3 P
  std::vector<std::int32_t> cam_idx, pt_idx;
  std::vector<double> px;       // 2 N
};

BalData parse_bal_text(const char* begin, const char* end);  // parse_bal, io/bal.hpp:103-142
BalData parse_bal_file(const char* path);
std::string serialize_bal_text(const BalData& d);             // serialize_bal, io/bal.hpp:145-157
void write_bal_file(const BalData& d, const char* path);
void write_bal_binary(const BalData& d, const char* path);  // binary cache (row f4); parse_bal_file reads both
void bal_poses(const BalData& d, double* poses7, double* intr3);  // BalCamera::pose, io/bal.hpp:24-26
BalData synth_ba_dense(int C, int P, double pixel_sigma, double pose_sigma, std::uint64_t seed);  // synth_ba
void look_at_origin(const P3& pos, Q4& q, P3& t);  // io/synthetic.hpp:26-38 (synth.cpp)

// PoseGraph (io/g2o.hpp:16-23): vertices as pose7 in file order (ids kept),
// edges with endpoints remapped to vertex positions, information matrices
// (36 row-major, has_info = not the identity), skipped-tag warnings.
struct G2oData {
  std::vector<std::int64_t> ids;
  std::vector<double> poses;  // 7 n
  std::vector<std::int32_t> ei, ej, has_info;
  std::vector<double> meas;   // 7 m
  std::vector<double> info;   // 36 m
  std::vector<std::string> warnings;
};
G2oData parse_g2o_text(const char* begin, const char* end);  // parse_g2o, io/g2o.hpp:30-80
G2oData parse_g2o_file(const char* path);

}  // namespace bae
