// BAL problem files and the reference's dense synthetic scene (SURVEY.md 8f,
// row f1): parse_bal / serialize_bal (io/bal.hpp:103-157), BalCamera::pose
// (io/bal.hpp:24-26) and synth_ba (io/synthetic.hpp:46-91).
//
// The parser reads the whole file and scans it with std::from_chars (the
// reference reads character by character through an istream), keeping the
// reference's token rules, messages and line numbers: whitespace-separated
// tokens, a number must span the whole token, the line of an error is the
// line the scanner stands on (io/bal.hpp:52-95).
#include <charconv>
#include <cmath>
#include <cstdio>
#include <cctype>
#include <cstring>
#include <string>
#include <unordered_map>
#include <vector>

#include "bae/rng.hpp"
#include "bae_internal.hpp"
#include "bal_io.hpp"
#include "lie.cuh"

namespace bae {

namespace {

class Scanner {
 public:
  Scanner(const char* b, const char* e) : p_(b), e_(e) {}
  std::size_t line() const { return line_; }

  // next whitespace-delimited token; false at end of input
  bool token(const char*& tb, const char*& te) {
    while (p_ < e_ && is_space(*p_)) {
      if (*p_ == '\n') ++line_;
      ++p_;
    }
    if (p_ >= e_) return false;
    tb = p_;
    while (p_ < e_ && !is_space(*p_)) ++p_;
    te = p_;
    if (p_ < e_ && *p_ == '\n') {  // the reference consumes the delimiter too
      ++line_;
      ++p_;
    } else if (p_ < e_) {
      ++p_;
    }
    return true;
  }

  double read_double(const char* what) {
    const char *b, *e;
    if (!token(b, e)) throw Error(BAE_ERR_PARSE, std::string("unexpected end of file reading ") + what, line_);
    double v = 0;
    const auto r = std::from_chars(b, e, v);
    if (r.ec != std::errc{} || r.ptr != e)
      throw Error(BAE_ERR_PARSE, "malformed number '" + std::string(b, e) + "' reading " + what, line_);
    return v;
  }

  std::int64_t read_int(const char* what) {
    const char *b, *e;
    if (!token(b, e)) throw Error(BAE_ERR_PARSE, std::string("unexpected end of file reading ") + what, line_);
    std::int64_t v = 0;
    const auto r = std::from_chars(b, e, v);
    if (r.ec != std::errc{} || r.ptr != e)
      throw Error(BAE_ERR_PARSE, "malformed integer '" + std::string(b, e) + "' reading " + what, line_);
    return v;
  }

 private:
  static bool is_space(char c) { return c == ' ' || c == '\n' || c == '\t' || c == '\r' || c == '\v' || c == '\f'; }
  const char* p_;
  const char* e_;
  std::size_t line_ = 1;
};

void put_double(std::string& out, double v) {  // ostream precision(17), default format == %.17g
  char buf[40];
  const auto r = std::to_chars(buf, buf + sizeof(buf), v, std::chars_format::general, 17);
  out.append(buf, r.ptr);
}

}  // namespace

BalData parse_bal_text(const char* b, const char* e) {
  Scanner r(b, e);
  const std::int64_t C = r.read_int("camera count");
  const std::int64_t P = r.read_int("point count");
  const std::int64_t N = r.read_int("observation count");
  if (C < 1 || P < 1 || N < 1) throw Error(BAE_ERR_PARSE, "non-positive counts in header", r.line());
  if (C > INT32_MAX || P > INT32_MAX || N >= (std::int64_t{1} << 31) - 1)
    throw Error(BAE_ERR_UNSUPPORTED, "BAL counts exceed the 32-bit index range", r.line());
  BalData d;
  d.C = static_cast<int>(C);
  d.P = static_cast<int>(P);
  d.N = N;
  d.cam_idx.resize(static_cast<std::size_t>(N));
  d.pt_idx.resize(static_cast<std::size_t>(N));
  d.px.resize(2 * static_cast<std::size_t>(N));
  for (std::int64_t i = 0; i < N; ++i) {
    const std::int64_t cam = r.read_int("camera index");
    const std::int64_t pt = r.read_int("point index");
    if (cam < 0 || cam >= C) throw Error(BAE_ERR_PARSE, "camera index out of range", r.line());
    if (pt < 0 || pt >= P) throw Error(BAE_ERR_PARSE, "point index out of range", r.line());
    d.cam_idx[i] = static_cast<std::int32_t>(cam);
    d.pt_idx[i] = static_cast<std::int32_t>(pt);
    d.px[2 * i] = r.read_double("pixel x");
    d.px[2 * i + 1] = r.read_double("pixel y");
  }
  d.cameras.resize(9 * static_cast<std::size_t>(C));
  for (std::int64_t c = 0; c < C; ++c) {
    double* o = &d.cameras[9 * c];
    for (int i = 0; i < 3; ++i) o[i] = r.read_double("camera rotation");
    for (int i = 0; i < 3; ++i) o[3 + i] = r.read_double("camera translation");
    o[6] = r.read_double("focal length");
    o[7] = r.read_double("k1");
    o[8] = r.read_double("k2");
  }
  d.points.resize(3 * static_cast<std::size_t>(P));
  for (std::size_t i = 0; i < d.points.size(); ++i) d.points[i] = r.read_double("point coordinate");
  const char *tb, *te;
  if (r.token(tb, te)) throw Error(BAE_ERR_PARSE, "trailing data after point list", r.line());
  return d;
}

// Binary problem cache: the parsed arrays as they
// are in memory, so a large synthetic or converted problem loads at disk
// speed instead of through the text scanner. Layout (little endian):
// "BAEBAL\0\1" | int32 C | int32 P | int64 N | cameras 9C f64 | points 3P f64 |
// cam_idx N i32 | pt_idx N i32 | pixels 2N f64. parse_bal_file recognises it
// by the magic; indices are validated like the text parser's.
namespace {
constexpr char kBinMagic[8] = {'B', 'A', 'E', 'B', 'A', 'L', '\0', '\1'};

BalData decode_bal_binary(const char* b, std::size_t len) {
  auto need = [&](std::size_t at, std::size_t n) {
    if (at + n > len) throw Error(BAE_ERR_PARSE, "binary BAL: truncated file", 0);
  };
  std::size_t at = 8;
  std::int32_t C = 0, P = 0;
  std::int64_t N = 0;
  need(at, 16);
  std::memcpy(&C, b + at, 4);
  std::memcpy(&P, b + at + 4, 4);
  std::memcpy(&N, b + at + 8, 8);
  at += 16;
  if (C < 1 || P < 1 || N < 1) throw Error(BAE_ERR_PARSE, "binary BAL: non-positive counts in header", 0);
  if (N >= (std::int64_t{1} << 31) - 1) throw Error(BAE_ERR_UNSUPPORTED, "binary BAL: counts exceed the 32-bit range", 0);
  const std::size_t total = 8 + 16 + 8 * (9 * static_cast<std::size_t>(C) + 3 * static_cast<std::size_t>(P)) +
                            static_cast<std::size_t>(N) * (4 + 4 + 16);
  if (len != total) throw Error(BAE_ERR_PARSE, "binary BAL: size does not match the header", 0);
  BalData d;
  d.C = C;
  d.P = P;
  d.N = N;
  auto take = [&](auto& v, std::size_t n) {
    v.resize(n);
    std::memcpy(v.data(), b + at, n * sizeof(v[0]));
    at += n * sizeof(v[0]);
  };
  take(d.cameras, 9 * static_cast<std::size_t>(C));
  take(d.points, 3 * static_cast<std::size_t>(P));
  take(d.cam_idx, static_cast<std::size_t>(N));
  take(d.pt_idx, static_cast<std::size_t>(N));
  take(d.px, 2 * static_cast<std::size_t>(N));
  for (std::int64_t k = 0; k < N; ++k) {
    if (d.cam_idx[k] < 0 || d.cam_idx[k] >= C) throw Error(BAE_ERR_PARSE, "camera index out of range", k);
    if (d.pt_idx[k] < 0 || d.pt_idx[k] >= P) throw Error(BAE_ERR_PARSE, "point index out of range", k);
  }
  return d;
}
}  // namespace

void write_bal_binary(const BalData& d, const char* path) {
  std::FILE* f = std::fopen(path, "wb");
  if (!f) throw Error(BAE_ERR_IO, std::string("cannot open '") + path + "' for writing");
  const std::int32_t C = d.C, P = d.P;
  const std::int64_t N = d.N;
  bool ok = std::fwrite(kBinMagic, 1, 8, f) == 8 && std::fwrite(&C, 4, 1, f) == 1 && std::fwrite(&P, 4, 1, f) == 1 &&
            std::fwrite(&N, 8, 1, f) == 1;
  auto put = [&](const auto& v) {
    if (ok && !v.empty()) ok = std::fwrite(v.data(), sizeof(v[0]), v.size(), f) == v.size();
  };
  put(d.cameras);
  put(d.points);
  put(d.cam_idx);
  put(d.pt_idx);
  put(d.px);
  if (std::fclose(f) != 0 || !ok) throw Error(BAE_ERR_IO, std::string("cannot write '") + path + "'");
}

BalData parse_bal_file(const char* path) {
  std::FILE* f = std::fopen(path, "rb");
  if (!f) throw Error(BAE_ERR_IO, std::string("cannot open '") + path + "'");
  std::string buf;
  char chunk[1 << 16];
  std::size_t n;
  while ((n = std::fread(chunk, 1, sizeof(chunk), f)) > 0) buf.append(chunk, n);
  std::fclose(f);
  if (buf.size() >= 8 && std::memcmp(buf.data(), kBinMagic, 8) == 0) return decode_bal_binary(buf.data(), buf.size());
  return parse_bal_text(buf.data(), buf.data() + buf.size());
}

std::string serialize_bal_text(const BalData& d) {
  std::string out;
  out.reserve(static_cast<std::size_t>(d.N) * 48 + static_cast<std::size_t>(d.C) * 200 + d.points.size() * 26);
  out += std::to_string(d.C) + " " + std::to_string(d.P) + " " + std::to_string(d.N) + "\n";
  for (std::int64_t i = 0; i < d.N; ++i) {
    out += std::to_string(d.cam_idx[i]);
    out += ' ';
    out += std::to_string(d.pt_idx[i]);
    out += ' ';
    put_double(out, d.px[2 * i]);
    out += ' ';
    put_double(out, d.px[2 * i + 1]);
    out += '\n';
  }
  for (double v : d.cameras) {
    put_double(out, v);
    out += '\n';
  }
  for (double v : d.points) {
    put_double(out, v);
    out += '\n';
  }
  return out;
}

void write_bal_file(const BalData& d, const char* path) {
  const std::string s = serialize_bal_text(d);
  std::FILE* f = std::fopen(path, "wb");
  if (!f) throw Error(BAE_ERR_IO, std::string("cannot open '") + path + "' for writing");
  const bool ok = std::fwrite(s.data(), 1, s.size(), f) == s.size();
  if (std::fclose(f) != 0 || !ok) throw Error(BAE_ERR_IO, std::string("cannot write '") + path + "'");
}

// BalCamera::pose (io/bal.hpp:24-26): rotation of se3_exp(0, rodrigues), the
// BAL translation; intrinsics [f, k1, k2].
void bal_poses(const BalData& d, double* poses7, double* intr3) {
  for (int c = 0; c < d.C; ++c) {
    const double* cam = &d.cameras[9 * static_cast<std::size_t>(c)];
    if (poses7) {
      const double tau[6] = {0, 0, 0, cam[0], cam[1], cam[2]};
      Q4 q;
      P3 unused;
      se3_exp(tau, q, unused);
      double* o = poses7 + 7 * static_cast<std::size_t>(c);
      o[0] = cam[3];
      o[1] = cam[4];
      o[2] = cam[5];
      o[3] = q.x;
      o[4] = q.y;
      o[5] = q.z;
      o[6] = q.w;
    }
    if (intr3) {
      intr3[3 * c] = cam[6];
      intr3[3 * c + 1] = cam[7];
      intr3[3 * c + 2] = cam[8];
    }
  }
}

namespace {
// QuatRotation(x, y, z, w) (lie.hpp:33-45): normalise, w >= 0; invalid_argument otherwise.
void quat_ctor(double x, double y, double z, double w, double* out4) {
  if (!std::isfinite(x) || !std::isfinite(y) || !std::isfinite(z) || !std::isfinite(w))
    throw Error(BAE_ERR_INVALID_ARGUMENT, "QuatRotation: non-finite component");
  Q4 q;
  if (!quat_normalize(x, y, z, w, q)) throw Error(BAE_ERR_INVALID_ARGUMENT, "QuatRotation: zero quaternion");
  out4[0] = q.x;
  out4[1] = q.y;
  out4[2] = q.z;
  out4[3] = q.w;
}
bool parse_num(const std::string& t, double& v) {
  const auto r = std::from_chars(t.data(), t.data() + t.size(), v);
  return r.ec == std::errc{} && r.ptr == t.data() + t.size();
}
bool parse_num(const std::string& t, std::int64_t& v) {
  const auto r = std::from_chars(t.data(), t.data() + t.size(), v);
  return r.ec == std::errc{} && r.ptr == t.data() + t.size();
}
}  // namespace

G2oData parse_g2o_text(const char* b, const char* e) {
  G2oData g;
  std::unordered_map<std::int64_t, std::int32_t> index;
  std::size_t line_no = 0;
  std::vector<std::string> tok;
  const char* p = b;
  while (p < e) {
    const char* le = p;
    while (le < e && *le != '\n') ++le;
    ++line_no;
    tok.clear();
    for (const char* q = p; q < le;) {  // whitespace tokens of the line
      while (q < le && std::isspace(static_cast<unsigned char>(*q))) ++q;
      const char* t0 = q;
      while (q < le && !std::isspace(static_cast<unsigned char>(*q))) ++q;
      if (q > t0) tok.emplace_back(t0, q);
    }
    p = le < e ? le + 1 : le;
    if (tok.empty() || tok[0][0] == '#') continue;
    const std::string& tag = tok[0];
    if (tag == "VERTEX_SE3:QUAT") {
      std::int64_t id = 0;
      double v[7];
      bool ok = tok.size() >= 9 && parse_num(tok[1], id);
      for (int i = 0; ok && i < 7; ++i) ok = parse_num(tok[2 + i], v[i]);
      if (!ok) throw Error(BAE_ERR_PARSE, "malformed VERTEX_SE3:QUAT line", static_cast<std::int64_t>(line_no));
      if (index.count(id)) throw Error(BAE_ERR_PARSE, "duplicate vertex id", static_cast<std::int64_t>(line_no));
      index[id] = static_cast<std::int32_t>(g.ids.size());
      g.ids.push_back(id);
      double q[4];
      quat_ctor(v[3], v[4], v[5], v[6], q);
      g.poses.insert(g.poses.end(), {v[0], v[1], v[2], q[0], q[1], q[2], q[3]});
    } else if (tag == "EDGE_SE3:QUAT") {
      std::int64_t i = 0, j = 0;
      double v[7];
      bool ok = tok.size() >= 10 && parse_num(tok[1], i) && parse_num(tok[2], j);
      for (int k = 0; ok && k < 7; ++k) ok = parse_num(tok[3 + k], v[k]);
      if (!ok) throw Error(BAE_ERR_PARSE, "malformed EDGE_SE3:QUAT line", static_cast<std::int64_t>(line_no));
      double info[36];
      std::size_t at = 10;
      for (int r = 0; r < 6; ++r)
        for (int c = r; c < 6; ++c) {
          double x = 0;
          if (at >= tok.size() || !parse_num(tok[at], x))
            throw Error(BAE_ERR_PARSE, "missing information entries on edge", static_cast<std::int64_t>(line_no));
          ++at;
          info[r * 6 + c] = x;
          info[c * 6 + r] = x;
        }
      const auto it_i = index.find(i), it_j = index.find(j);
      if (it_i == index.end() || it_j == index.end())
        throw Error(BAE_ERR_PARSE, "edge references undeclared vertex", static_cast<std::int64_t>(line_no));
      g.ei.push_back(it_i->second);
      g.ej.push_back(it_j->second);
      double q[4];
      quat_ctor(v[3], v[4], v[5], v[6], q);
      g.meas.insert(g.meas.end(), {v[0], v[1], v[2], q[0], q[1], q[2], q[3]});
      // Eigen isApprox(Identity): ||info - I||_F <= 1e-12 min(||info||_F, ||I||_F)
      double dn = 0.0, an = 0.0;
      for (int r = 0; r < 36; ++r) {
        const double id = (r % 7 == 0) ? 1.0 : 0.0;
        dn += (info[r] - id) * (info[r] - id);
        an += info[r] * info[r];
      }
      const bool identity = std::sqrt(dn) <= 1e-12 * std::min(std::sqrt(an), std::sqrt(6.0));
      g.has_info.push_back(identity ? 0 : 1);
      g.info.insert(g.info.end(), info, info + 36);
    } else {
      g.warnings.push_back("line " + std::to_string(line_no) + ": skipped unknown tag '" + tag + "'");
    }
  }
  return g;
}

G2oData parse_g2o_file(const char* path) {
  std::FILE* f = std::fopen(path, "rb");
  if (!f) throw Error(BAE_ERR_IO, std::string("cannot open '") + path + "'");
  std::string buf;
  char chunk[1 << 16];
  std::size_t n;
  while ((n = std::fread(chunk, 1, sizeof(chunk), f)) > 0) buf.append(chunk, n);
  std::fclose(f);
  return parse_g2o_text(buf.data(), buf.data() + buf.size());
}

BalData synth_ba_dense(int C, int P, double pixel_sigma, double pose_sigma, std::uint64_t seed) {
  if (C < 1 || P < 1) throw Error(BAE_ERR_INVALID_ARGUMENT, "synth_ba: counts must be positive");
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
  }
  BalData d;
  d.C = C;
  d.P = P;
  d.N = static_cast<std::int64_t>(C) * P;
  d.points.resize(3 * static_cast<std::size_t>(P));
  for (int p = 0; p < P; ++p) {
    d.points[3 * p] = tp[p].x;
    d.points[3 * p + 1] = tp[p].y;
    d.points[3 * p + 2] = tp[p].z;
  }
  d.cam_idx.resize(static_cast<std::size_t>(d.N));
  d.pt_idx.resize(static_cast<std::size_t>(d.N));
  d.px.resize(2 * static_cast<std::size_t>(d.N));
  d.cameras.resize(9 * static_cast<std::size_t>(C));
  std::int64_t k = 0;
  for (int c = 0; c < C; ++c) {
    for (int p = 0; p < P; ++p, ++k) {
      const P3 y = quat_rotate(tq[c], tp[p]);
      double u = 0, v = 0;
      if (!bal_project({y.x + tt[c].x, y.y + tt[c].y, y.z + tt[c].z}, 500.0, 0.0, 0.0, u, v))
        throw Error(BAE_ERR_CHEIRALITY, "bal projection: point on camera plane", k);
      d.cam_idx[k] = c;
      d.pt_idx[k] = p;
      const double n0 = rng.normal();
      const double n1 = rng.normal();
      d.px[2 * k] = u + pixel_sigma * n0;
      d.px[2 * k + 1] = v + pixel_sigma * n1;
    }
    double tau[6];  // Tangent6(sigma * (n, n, n), sigma * (n, n, n)): rho first, then omega
    for (int i = 0; i < 6; ++i) tau[i] = pose_sigma * rng.normal();
    Q4 q;
    P3 t;
    if (!se3_retract(tq[c], tt[c], tau, q, t)) throw Error(BAE_ERR_INVALID_ARGUMENT, "synth_ba: retract");
    const P3 rod = so3_log(q);  // se3_log(PoseSE3(init.rotation, 0)).omega
    double* o = &d.cameras[9 * static_cast<std::size_t>(c)];
    o[0] = rod.x;
    o[1] = rod.y;
    o[2] = rod.z;
    o[3] = t.x;
    o[4] = t.y;
    o[5] = t.z;
    o[6] = 500.0;
    o[7] = 0.0;
    o[8] = 0.0;
  }
  return d;
}

}  // namespace bae
