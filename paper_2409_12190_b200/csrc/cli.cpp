// The drop-in benchmark CLI: cli_main of the
// reference (cli.hpp:116-200) over the B200 path. Same subcommands, flags,
// defaults, summary line, CSV schema (cli.hpp:69-79) and exit codes: 0
// success, 1 usage error, 2 data error, 3 solver failure. The argument
// parser follows CLI11's conventions for what the reference uses
// (`--opt value` or `--opt=value`, `-h/--help`, one required subcommand).
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "bae_b200.h"
#include "bae_internal.hpp"
#include "bal_io.hpp"

namespace bae {
namespace {

struct CliOptions {  // detail::CliOptions (cli.hpp:22-34)
  std::string input, synthetic, solver = "cholesky", csv_path;
  int max_iters = 50;
  double damping = 1e-6, pcg_tol = 1e-8;
  std::uint64_t seed = 0;
  double pixel_noise = 0.0, pose_noise = 0.05;
  int threads = 1;
  int device = 0;  // extension: CUDA ordinal
};

struct Usage {
  std::string msg;
};

const char* kHelp =
    "Sparse Levenberg-Marquardt benchmark for bundle adjustment and pose graphs (B200 path)\n"
    "Usage: traceopt_bench SUBCOMMAND [OPTIONS]\n\n"
    "Subcommands:\n"
    "  ba     Bundle adjustment on a BAL file or synthetic scene\n"
    "  pgo    Pose graph optimization on a g2o file\n\n"
    "ba options:\n"
    "  --input FILE          BAL problem file\n"
    "  --synthetic CxP       Synthetic scene CxP, e.g. 3x50\n"
    "  --pixel-noise S       Synthetic pixel noise sigma (0)\n"
    "  --pose-noise S        Synthetic pose perturbation sigma (0.05)\n"
    "  --solver {cholesky,pcg}  Linear solver (cholesky)\n"
    "  --max-iters N         Iteration budget (50)\n"
    "  --damping L           Initial damping lambda (1e-06)\n"
    "  --pcg-tol T           PCG relative tolerance (1e-08)\n"
    "  --seed S              Seed for synthetic problems (0)\n"
    "  --csv FILE            Write per-iteration CSV to this path\n"
    "  --threads N           Worker threads for batched kernels (1; host setup passes)\n"
    "  --device N            CUDA device ordinal (0)\n";

template <class T>
T parse_num(const std::string& opt, const std::string& v) {
  char* end = nullptr;
  errno = 0;
  if constexpr (std::is_same_v<T, double>) {
    const double x = std::strtod(v.c_str(), &end);
    if (v.empty() || *end || errno) throw Usage{opt + ": Value " + v + " could not be converted"};
    return x;
  } else if constexpr (std::is_same_v<T, std::uint64_t>) {
    if (!v.empty() && v[0] == '-') throw Usage{opt + ": Value " + v + " could not be converted"};
    const unsigned long long x = std::strtoull(v.c_str(), &end, 10);
    if (v.empty() || *end || errno) throw Usage{opt + ": Value " + v + " could not be converted"};
    return static_cast<T>(x);
  } else {
    const long x = std::strtol(v.c_str(), &end, 10);
    if (v.empty() || *end || errno || x < INT32_MIN || x > INT32_MAX)
      throw Usage{opt + ": Value " + v + " could not be converted"};
    return static_cast<T>(x);
  }
}

// Returns false when --help was given.
bool parse_args(int argc, const char* const* argv, std::string& sub, CliOptions& o) {
  if (argc < 2) throw Usage{"A subcommand is required"};
  sub = argv[1];
  if (sub == "-h" || sub == "--help") return false;
  if (sub != "ba" && sub != "pgo") throw Usage{"The following argument was not expected: " + sub};
  for (int i = 2; i < argc; ++i) {
    std::string a = argv[i], v;
    if (a == "-h" || a == "--help") return false;
    const auto eq = a.find('=');
    bool has_v = false;
    if (a.rfind("--", 0) == 0 && eq != std::string::npos) {
      v = a.substr(eq + 1);
      a = a.substr(0, eq);
      has_v = true;
    }
    auto value = [&]() -> std::string {
      if (has_v) return v;
      if (i + 1 >= argc) throw Usage{a + ": 1 required argument missing"};
      return argv[++i];
    };
    const bool ba = sub == "ba";
    if (a == "--input") o.input = value();
    else if (ba && a == "--synthetic") o.synthetic = value();
    else if (ba && a == "--pixel-noise") o.pixel_noise = parse_num<double>(a, value());
    else if (ba && a == "--pose-noise") o.pose_noise = parse_num<double>(a, value());
    else if (a == "--solver") {
      o.solver = value();
      if (o.solver != "cholesky" && o.solver != "pcg")
        throw Usage{"--solver: " + o.solver + " not in {cholesky,pcg}"};
    } else if (a == "--max-iters") o.max_iters = parse_num<int>(a, value());
    else if (a == "--damping") o.damping = parse_num<double>(a, value());
    else if (a == "--pcg-tol") o.pcg_tol = parse_num<double>(a, value());
    else if (a == "--seed") o.seed = parse_num<std::uint64_t>(a, value());
    else if (a == "--csv") o.csv_path = value();
    else if (a == "--threads") o.threads = parse_num<int>(a, value());
    else if (a == "--device") o.device = parse_num<int>(a, value());
    else throw Usage{"The following argument was not expected: " + a};
  }
  if (sub == "pgo" && o.input.empty()) throw Usage{"--input is required"};
  return true;
}

bool parse_cxp(const std::string& s, int& c, int& p) {  // cli.hpp:56-66
  const auto x = s.find('x');
  if (x == std::string::npos) return false;
  try {
    c = std::stoi(s.substr(0, x));
    p = std::stoi(s.substr(x + 1));
  } catch (...) {
    return false;
  }
  return c > 0 && p > 0;
}

const char* reason_name(int r) {
  switch (r) {
    case BAE_TERM_PLATEAU:
      return "plateau";
    case BAE_TERM_MAX_ITERS:
      return "max_iters";
    case BAE_TERM_SOLVER_FAILURE:
      return "solver_failure";
  }
  return "unknown";
}

// The library's error for the last failed call, as the reference CLI prints
// each exception class (cli.hpp:187-199); returns the exit code.
int report_error(int code) {
  const char* msg = bae_last_error();
  const long long idx = static_cast<long long>(bae_last_error_index());
  switch (code) {
    case BAE_ERR_PARSE:
      std::fprintf(stderr, "parse error (line %lld): %s\n", idx, msg);
      return 2;
    case BAE_ERR_IO:
      std::fprintf(stderr, "%s\n", msg);
      return 2;
    case BAE_ERR_CHEIRALITY:
      std::fprintf(stderr, "data error: %s (observation %lld)\n", msg, idx);
      return 2;
    case BAE_ERR_INDEX:
    case BAE_ERR_INVALID_ARGUMENT:
      std::fprintf(stderr, "data error: %s\n", msg);
      return 2;
    default:
      std::fprintf(stderr, "error: %s\n", msg);
      return 3;
  }
}

// run_and_report (cli.hpp:89-106): optimise, print the summary line, write
// the CSV; exit 3 on solver failure. Destroys the problem.
int run_and_report(bae_problem* prob, const double* poses, const double* points, const CliOptions& o,
                   const std::string& dataset) {
  bae_lm_config cfg;  // config_from (cli.hpp:47-54)
  bae_lm_config_default(&cfg);
  cfg.initial_damping = o.damping;
  cfg.max_iterations = o.max_iters;
  cfg.solver = o.solver == "pcg" ? BAE_SOLVER_PCG : BAE_SOLVER_CHOLESKY;
  cfg.pcg_tol = o.pcg_tol;
  std::vector<bae_iter_record> traj(static_cast<std::size_t>(std::max(o.max_iters, 0)) + 1);
  bae_lm_report rep;
  const auto t0 = std::chrono::steady_clock::now();
  const int rc = bae_optimize(prob, poses, points, &cfg, traj.data(), static_cast<int32_t>(traj.size()),
                              &rep, nullptr, nullptr);
  const double wall = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  if (rc) {
    const int code = report_error(rc);
    bae_destroy(prob);
    return code;
  }
  bae_destroy(prob);
  std::printf("dataset=%s solver=%s iterations=%d final_cost=%.9g final_mse=%.9g termination=%s time_s=%.3f\n",
              dataset.c_str(), o.solver.c_str(), rep.iterations, rep.final_cost, rep.final_mse,
              reason_name(rep.reason), wall);
  std::fflush(stdout);
  if (!o.csv_path.empty()) {
    const int n = std::min(rep.iterations + 1, static_cast<int>(traj.size()));
    if (int wc = bae_write_csv(o.csv_path.c_str(), traj.data(), n)) {
      std::fprintf(stderr, "error: %s\n", bae_last_error());
      return wc == BAE_ERR_IO ? 3 : 3;
    }
  }
  return rep.reason == BAE_TERM_SOLVER_FAILURE ? 3 : 0;
}

}  // namespace
}  // namespace bae

extern "C" int bae_cli_main(int argc, const char* const* argv) {
  using namespace bae;
  std::string sub;
  CliOptions o;
  try {
    if (!parse_args(argc, argv, sub, o)) {
      std::fputs(kHelp, stdout);
      return 0;
    }
  } catch (const Usage& u) {
    std::fprintf(stderr, "%s\n", u.msg.c_str());
    return 1;
  }
  if (o.threads > 0) {
    const std::string t = std::to_string(o.threads);
    setenv("BAE_HOST_THREADS", t.c_str(), 1);  // set_num_threads (cli.hpp:174)
  }
  if (sub == "pgo") {  // cli.hpp:179-185
    bae_g2o* g = nullptr;
    if (int rc = bae_g2o_read(o.input.c_str(), &g)) return report_error(rc);
    int32_t nv = 0, nw = 0;
    int64_t ne = 0;
    bae_g2o_counts(g, &nv, &ne, &nw);
    for (int32_t k = 0; k < nw; ++k) std::fprintf(stderr, "warning: %s\n", bae_g2o_warning(g, k));
    std::vector<double> poses(7 * static_cast<std::size_t>(nv)), meas(7 * static_cast<std::size_t>(ne)),
        info(36 * static_cast<std::size_t>(ne));
    std::vector<int32_t> ei(static_cast<std::size_t>(ne)), ej(static_cast<std::size_t>(ne)),
        has(static_cast<std::size_t>(ne));
    bae_g2o_arrays(g, poses.data(), nullptr, ei.data(), ej.data(), meas.data(), info.data(), has.data());
    bae_g2o_free(g);
    bae_create_options opt;
    bae_create_options_default(&opt);
    opt.device = o.device;
    bae_problem* prob = nullptr;
    if (int rc = bae_create_pgo(poses.data(), nv, ei.data(), ej.data(), meas.data(), info.data(), has.data(), ne, 1,
                                &opt, &prob))
      return report_error(rc);
    return run_and_report(prob, poses.data(), nullptr, o, o.input);
  }
  bae_bal* bal = nullptr;
  std::string dataset;
  if (!o.synthetic.empty()) {
    int c = 0, p = 0;
    if (!parse_cxp(o.synthetic, c, p)) {
      std::fprintf(stderr, "bad --synthetic value '%s' (expected CxP)\n", o.synthetic.c_str());
      return 1;
    }
    if (int rc = bae_bal_synthetic(c, p, o.pixel_noise, o.pose_noise, o.seed, &bal)) return report_error(rc);
    dataset = "synthetic-" + o.synthetic;
  } else if (!o.input.empty()) {
    if (int rc = bae_bal_read(o.input.c_str(), &bal)) return report_error(rc);
    dataset = o.input;
  } else {
    std::fprintf(stderr, "ba: one of --input or --synthetic is required\n");
    return 1;
  }
  int32_t C = 0, P = 0;
  int64_t N = 0;
  bae_bal_counts(bal, &C, &P, &N);
  std::vector<double> poses(7 * static_cast<std::size_t>(C)), intr(3 * static_cast<std::size_t>(C)),
      pts(3 * static_cast<std::size_t>(P)), px(2 * static_cast<std::size_t>(N));
  std::vector<int32_t> ci(static_cast<std::size_t>(N)), pi(static_cast<std::size_t>(N));
  bae_bal_arrays(bal, poses.data(), intr.data(), pts.data(), ci.data(), pi.data(), px.data(), nullptr);
  bae_bal_free(bal);
  bae_create_options opt;
  bae_create_options_default(&opt);
  opt.device = o.device;
  bae_problem* prob = nullptr;
  if (int rc = bae_create_ba(poses.data(), C, pts.data(), P, intr.data(), ci.data(), pi.data(), px.data(), N, &opt,
                             &prob))
    return report_error(rc);
  return run_and_report(prob, poses.data(), pts.data(), o, dataset);
}
