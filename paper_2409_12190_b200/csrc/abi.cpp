// extern "C" boundary (include/bae_b200.h): no exceptions or C++ types cross
// it. Each entry point maps the reference exception classes (errors.hpp) to
// return codes and records the message / index for bae_last_error*().
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <exception>
#include <memory>
#include <new>
#include <string>

#include "bae_b200.h"
#include "bae_internal.hpp"
#include "bal_io.hpp"
#include "chol.cuh"
#include "pgo.hpp"
#include "problem.hpp"

struct bae_problem {
  std::unique_ptr<bae::Problem> impl;    // bundle adjustment
  std::unique_ptr<bae::PgoProblem> pgo;  // pose graph (make_pgo_problem)
};

namespace {
// The BA problem behind a handle (entry points that only BA supports).
bae::Problem* ba(const bae_problem* p) {
  if (!p) throw bae::Error(BAE_ERR_INVALID_ARGUMENT, "null problem handle");
  if (!p->impl) throw bae::Error(BAE_ERR_UNSUPPORTED, "not available on a pose-graph problem");
  return p->impl.get();
}
}  // namespace

struct bae_bal {
  bae::BalData d;
};

struct bae_g2o {
  bae::G2oData d;
};

namespace {
thread_local std::string g_msg;
thread_local std::int64_t g_index = -1;

template <class F>
int guarded(F&& f) {
  try {
    g_msg.clear();
    g_index = -1;
    f();
    return BAE_OK;
  } catch (const bae::Error& e) {
    g_msg = e.msg;
    g_index = e.index;
    return e.code;
  } catch (const std::bad_alloc&) {
    g_msg = "host allocation failed";
    return BAE_ERR_CUDA;
  } catch (const std::exception& e) {
    g_msg = e.what();
    return BAE_ERR_INVALID_ARGUMENT;
  }
}
}  // namespace

extern "C" {

const char* bae_version(void) { return "bae-b200 0.1 (sm_100a, fp64)"; }

void bae_lm_config_default(bae_lm_config* c) {  // LmConfig defaults, lm.hpp:24-37
  std::memset(c, 0, sizeof(*c));
  c->initial_damping = 1e-6;
  c->damping_min = 1e-16;
  c->damping_max = 1e16;
  c->damping_up = 2.0;
  c->damping_down = 0.5;
  c->clamp_min = 1e-6;
  c->clamp_max = 1e32;
  c->plateau_rel_tol = 1e-6;
  c->pcg_tol = 1e-8;
  c->pcg_max_iters = 0;
  c->max_iterations = 10;
  c->plateau_patience = 3;
  c->solver = BAE_SOLVER_CHOLESKY;
  c->use_caches = 1;
}

void bae_create_options_default(bae_create_options* o) {
  std::memset(o, 0, sizeof(*o));
  o->world = 1;
}

const char* bae_last_error(void) { return g_msg.c_str(); }
int64_t bae_last_error_index(void) { return g_index; }

int bae_nccl_unique_id(void* out128) {
  return guarded([&] {
    if (!out128) throw bae::Error(BAE_ERR_INVALID_ARGUMENT, "null output");
    bae::nccl_unique_id(out128);
  });
}

int bae_group_create(int32_t world, bae_group** out) {
  return guarded([&] {
    if (!out) throw bae::Error(BAE_ERR_INVALID_ARGUMENT, "null output handle");
    *out = bae::group_create(world);
  });
}

void bae_group_destroy(bae_group* g) { bae::group_destroy(g); }

int bae_create_ba(const double* poses7, int32_t C, const double* points3, int32_t P, const double* intr3,
                  const int32_t* cam_idx, const int32_t* pt_idx, const double* px2, int64_t N,
                  const bae_create_options* opts, bae_problem** out) {
  return guarded([&] {
    if (!out) throw bae::Error(BAE_ERR_INVALID_ARGUMENT, "null output handle");
    *out = nullptr;
    if (N > 0 && (!cam_idx || !pt_idx || !px2)) throw bae::Error(BAE_ERR_INVALID_ARGUMENT, "null observation arrays");
    if ((C > 0 && (!poses7 || !intr3)) || (P > 0 && !points3))
      throw bae::Error(BAE_ERR_INVALID_ARGUMENT, "null parameter arrays");
    if (C < 0 || P < 0) throw bae::Error(BAE_ERR_INVALID_ARGUMENT, "negative counts");
    bae_create_options o;
    bae_create_options_default(&o);
    if (opts) o = *opts;
    if (o.group && o.nccl_id) throw bae::Error(BAE_ERR_INVALID_ARGUMENT, "pass an NCCL id or a rank group, not both");
    auto h = std::make_unique<bae_problem>();
    h->impl = std::make_unique<bae::Problem>(poses7, C, points3, P, intr3, cam_idx, pt_idx, px2, N, o);
    *out = h.release();
  });
}

void bae_destroy(bae_problem* p) { delete p; }

int bae_create_pgo(const double* poses7, int32_t num_poses, const int32_t* edge_i, const int32_t* edge_j,
                   const double* measurements7, const double* information36, const int32_t* has_information,
                   int64_t num_edges, int32_t anchor_first, const bae_create_options* opts, bae_problem** out) {
  return guarded([&] {
    if (!out) throw bae::Error(BAE_ERR_INVALID_ARGUMENT, "null output handle");
    *out = nullptr;
    if ((num_poses > 0 && !poses7) || (num_edges > 0 && (!edge_i || !edge_j || !measurements7)))
      throw bae::Error(BAE_ERR_INVALID_ARGUMENT, "null pose-graph arrays");
    bae_create_options o;
    bae_create_options_default(&o);
    if (opts) o = *opts;
    if (o.world != 1 || o.group || o.nccl_id)
      throw bae::Error(BAE_ERR_UNSUPPORTED, "pose graphs run on a single rank");
    auto h = std::make_unique<bae_problem>();
    h->pgo = std::make_unique<bae::PgoProblem>(poses7, num_poses, edge_i, edge_j, measurements7, information36,
                                               has_information, num_edges, anchor_first != 0, o);
    *out = h.release();
  });
}

int bae_pgo_jacobian(bae_problem* p, double* ji36, double* jj36) {
  return guarded([&] {
    if (!p || !p->pgo) throw bae::Error(BAE_ERR_INVALID_ARGUMENT, "not a pose-graph problem");
    p->pgo->jacobian(ji36, jj36);
  });
}

int32_t bae_num_poses(const bae_problem* p) {
  return !p ? 0 : p->pgo ? p->pgo->num_poses() : p->impl->num_cameras();
}
int32_t bae_num_points(const bae_problem* p) { return !p || p->pgo ? 0 : p->impl->num_points(); }
int64_t bae_residual_rows(const bae_problem* p) {
  return !p ? 0 : p->pgo ? p->pgo->num_edges() : p->impl->num_obs();
}

int bae_set_parameters(bae_problem* p, const double* poses7, const double* points3) {
  return guarded([&] {
    if (p && p->pgo) {
      if (poses7) p->pgo->set_parameters(poses7);
      return;
    }
    ba(p)->set_parameters(poses7, points3);
  });
}
int bae_get_parameters(bae_problem* p, double* poses7, double* points3) {
  return guarded([&] {
    if (p && p->pgo) {
      if (poses7) p->pgo->get_parameters(poses7);
      return;
    }
    ba(p)->get_parameters(poses7, points3);
  });
}
int bae_evaluate(bae_problem* p, double* residuals2, double* cost) {
  return guarded([&] {
    const double c = (p && p->pgo) ? p->pgo->evaluate(residuals2) : ba(p)->evaluate(residuals2);
    if (cost) *cost = c;
  });
}
int bae_jacobian(bae_problem* p, double* jpose, double* jpoint, int64_t* prp, int32_t* pcol, int64_t* lrp,
                 int32_t* lcol) {
  return guarded([&] {
    if (ba(p)->distributed()) throw bae::Error(BAE_ERR_UNSUPPORTED, "the Jacobian export needs a single-rank problem");
    if (jpose || jpoint) ba(p)->jacobian(jpose, jpoint, nullptr);
    if (!(prp || pcol || lrp || lcol)) return;
    // The pattern as the device holds it: every slot of every tile is one
    // 2x6 / 2x3 block row; its columns are the slot's entry camera and tile
    // point. row_ptr counts the slots that carry each observation (one each
    // when the decomposition is a permutation of the rows, trace.hpp:728-790).
    const bae::DeviceStructure ds = ba(p)->download_structure();
    const std::int64_t N = ds.N;
    std::vector<std::int64_t> rows(static_cast<std::size_t>(N) + 1, 0);
    std::vector<std::int32_t> cam(static_cast<std::size_t>(N), -1), pt(static_cast<std::size_t>(N), -1);
    for (int t = 0; t < ds.T; ++t)
      for (int e = ds.tile_ent_begin[t]; e < ds.tile_ent_begin[t + 1]; ++e)
        for (int s = ds.ent_obs_begin[e]; s < ds.ent_obs_begin[e + 1]; ++s) {
          const std::int32_t k = ds.obs_orig[s];
          if (k < 0 || k >= N) throw bae::Error(BAE_ERR_CUDA, "device decomposition: observation id out of range");
          ++rows[k + 1];
          cam[k] = ds.ent_cam[e];
          pt[k] = ds.slot_pt(t, s);
        }
    for (std::int64_t k = 0; k < N; ++k) rows[k + 1] += rows[k];
    if (prp) std::memcpy(prp, rows.data(), rows.size() * 8);
    if (lrp) std::memcpy(lrp, rows.data(), rows.size() * 8);
    if (pcol) std::memcpy(pcol, cam.data(), cam.size() * 4);
    if (lcol) std::memcpy(lcol, pt.data(), pt.size() * 4);
  });
}

int bae_transpose_plan(bae_problem* p, int32_t which, int64_t* row_ptr, int32_t* col_idx, int64_t* src_block) {
  return guarded([&] {
    if (ba(p)->distributed())
      throw bae::Error(BAE_ERR_UNSUPPORTED, "the transpose plans need a single-rank problem");
    if (which != 0 && which != 1) throw bae::Error(BAE_ERR_INVALID_ARGUMENT, "which must be 0 (pose) or 1 (point)");
    const bae::DeviceStructure ds = ba(p)->download_structure();
    if (which == 0) {
      // camera segments from the device's per-camera entry lists (the camera
      // reductions' segments). The device sums a camera's observations in
      // tile order; the plan lists them in ascending id (bsr.hpp:140-160).
      std::vector<std::int64_t> rp(static_cast<std::size_t>(ds.C) + 1, 0);
      std::vector<std::int32_t> ids;
      ids.reserve(static_cast<std::size_t>(ds.N));
      for (int c = 0; c < ds.C; ++c) {
        const std::size_t start = ids.size();
        for (int q = ds.cam_ent_ptr[c]; q < ds.cam_ent_ptr[c + 1]; ++q) {
          const int e = ds.cam_ent[q];
          if (ds.ent_cam[e] != c) throw bae::Error(BAE_ERR_CUDA, "device decomposition: entry list of wrong camera");
          for (int s = ds.ent_obs_begin[e]; s < ds.ent_obs_begin[e + 1]; ++s) ids.push_back(ds.obs_orig[s]);
        }
        std::sort(ids.begin() + static_cast<std::ptrdiff_t>(start), ids.end());
        rp[c + 1] = static_cast<std::int64_t>(ids.size());
      }
      std::memcpy(row_ptr, rp.data(), rp.size() * 8);
      std::memcpy(col_idx, ids.data(), ids.size() * 4);
      for (std::size_t i = 0; i < ids.size(); ++i) src_block[i] = ids[i];
    } else {
      // point segments: the device's per-point slot lists (ascending id,
      // the order the point reductions sum in)
      std::vector<std::int64_t> rp(static_cast<std::size_t>(ds.P) + 1, 0);
      for (int i = 0; i < ds.P; ++i) rp[ds.pt_of_internal[i] + 1] = ds.pt_ptr[i + 1] - ds.pt_ptr[i];
      for (int p2 = 0; p2 < ds.P; ++p2) rp[p2 + 1] += rp[p2];
      for (int t = 0; t < ds.T; ++t)
        for (int i = ds.tile_pt_begin[t]; i < ds.tile_pt_begin[t + 1]; ++i) {
          std::int64_t o = rp[ds.pt_of_internal[i]];
          for (int q = ds.pt_ptr[i]; q < ds.pt_ptr[i + 1]; ++q, ++o) {
            const std::int32_t k = ds.obs_orig[ds.tile_obs_begin[t] + ds.ptobs[q]];
            col_idx[o] = k;
            src_block[o] = k;
          }
        }
      std::memcpy(row_ptr, rp.data(), rp.size() * 8);
    }
  });
}

int bae_normal_pattern(bae_problem* p, int32_t which, int64_t* rows, int64_t* nnz, int64_t* row_ptr,
                       int32_t* col_idx) {
  return guarded([&] {
    if (ba(p)->distributed())
      throw bae::Error(BAE_ERR_UNSUPPORTED, "the normal-matrix pattern needs a single-rank problem");
    if (which < 0 || which > 4) throw bae::Error(BAE_ERR_INVALID_ARGUMENT, "which must be 0..4");
    const bae::DeviceStructure ds = ba(p)->download_structure();
    const int C = ds.C, P = ds.P;
    // unique (camera, point) pairs of the device decomposition: the CL
    // quadrant's blocks (spgemm_symbolic, spgemm.hpp:33-81: duplicates merge)
    std::vector<std::vector<std::int32_t>> cl(static_cast<std::size_t>(C)), lc(static_cast<std::size_t>(P));
    for (int t = 0; t < ds.T; ++t)
      for (int e = ds.tile_ent_begin[t]; e < ds.tile_ent_begin[t + 1]; ++e)
        for (int s = ds.ent_obs_begin[e]; s < ds.ent_obs_begin[e + 1]; ++s) {
          cl[ds.ent_cam[e]].push_back(ds.slot_pt(t, s));
          lc[ds.slot_pt(t, s)].push_back(ds.ent_cam[e]);
        }
    for (auto* v : {&cl, &lc})
      for (auto& r : *v) {
        std::sort(r.begin(), r.end());
        r.erase(std::unique(r.begin(), r.end()), r.end());
      }
    std::vector<std::int64_t> rp;
    std::vector<std::int32_t> ci;
    auto block_rows = [&](const std::vector<std::vector<std::int32_t>>& rws) {
      rp.assign(1, 0);
      for (const auto& r : rws) {
        ci.insert(ci.end(), r.begin(), r.end());
        rp.push_back(static_cast<std::int64_t>(ci.size()));
      }
    };
    auto diag_rows = [&](int n, const std::vector<std::vector<std::int32_t>>& seen) {
      rp.assign(1, 0);
      for (int i = 0; i < n; ++i) {
        if (!seen[i].empty()) ci.push_back(i);
        rp.push_back(static_cast<std::int64_t>(ci.size()));
      }
    };
    if (which == 0) {
      diag_rows(C, cl);  // one camera per Jacobian row: CC is block diagonal
    } else if (which == 1) {
      block_rows(cl);
    } else if (which == 2) {
      block_rows(lc);
    } else if (which == 3) {
      diag_rows(P, lc);
    } else {
      // scalar CSR of A = [CC CL; LC LL] (build_csr_pattern, assemble.hpp:135-177):
      // columns ascending, pose scalars 0..6C-1 then point scalars
      const std::int64_t off = 6LL * C;
      rp.assign(1, 0);
      for (int c = 0; c < C; ++c)
        for (int i = 0; i < 6; ++i) {
          if (!cl[c].empty())
            for (int j = 0; j < 6; ++j) ci.push_back(6 * c + j);
          for (int pt : cl[c])
            for (int j = 0; j < 3; ++j) ci.push_back(static_cast<std::int32_t>(off + 3LL * pt + j));
          rp.push_back(static_cast<std::int64_t>(ci.size()));
        }
      for (int pt = 0; pt < P; ++pt)
        for (int i = 0; i < 3; ++i) {
          for (int c : lc[pt])
            for (int j = 0; j < 6; ++j) ci.push_back(6 * c + j);
          if (!lc[pt].empty())
            for (int j = 0; j < 3; ++j) ci.push_back(static_cast<std::int32_t>(off + 3LL * pt + j));
          rp.push_back(static_cast<std::int64_t>(ci.size()));
        }
    }
    *rows = static_cast<std::int64_t>(rp.size()) - 1;
    *nnz = static_cast<std::int64_t>(ci.size());
    if (row_ptr) std::memcpy(row_ptr, rp.data(), rp.size() * 8);
    if (col_idx) std::memcpy(col_idx, ci.data(), ci.size() * 4);
  });
}

int bae_block_diagonals(bae_problem* p, double* hcc36, double* gc6, double* hpp9, double* gp3) {
  return guarded([&] { ba(p)->block_diagonals(hcc36, gc6, hpp9, gp3); });
}

int bae_optimize(bae_problem* p, const double* init_poses7, const double* init_points3, const bae_lm_config* cfg,
                 bae_iter_record* traj, int32_t traj_cap, bae_lm_report* report, double* poses_out,
                 double* points_out) {
  return guarded([&] {
    bae_lm_config c;
    bae_lm_config_default(&c);
    if (cfg) c = *cfg;
    std::vector<bae_iter_record> t;
    bae_lm_report r{};
    if (p && p->pgo)
      p->pgo->optimize(init_poses7, c, t, r);
    else
      ba(p)->optimize(init_poses7, init_points3, c, t, r);
    if (traj)
      for (int i = 0; i < std::min<int>(traj_cap, static_cast<int>(t.size())); ++i) traj[i] = t[i];
    if (report) *report = r;
    if (p->pgo) {
      if (poses_out) p->pgo->get_parameters(poses_out);
    } else if (poses_out || points_out) {
      ba(p)->get_parameters(poses_out, points_out);
    }
  });
}

int bae_solve_step(bae_problem* p, double lambda, const bae_lm_config* cfg, double* delta, int64_t* iters,
                   double* relres) {
  return guarded([&] {
    bae_lm_config c;
    bae_lm_config_default(&c);
    if (cfg) c = *cfg;
    ba(p)->solve_step(lambda, c, delta, iters, relres);
  });
}

int bae_stop_on_plateau(const double* history, int64_t n, const bae_lm_config* cfg, int32_t* stop) {
  return guarded([&] {  // stop_on_plateau, lm.hpp:104-108
    if (n <= 0) throw bae::Error(BAE_ERR_INVALID_ARGUMENT, "stop_on_plateau: empty history");
    if (n >= cfg->max_iterations) {
      *stop = 1;
      return;
    }
    *stop = bae::plateau_stagnation(history, static_cast<std::size_t>(n), cfg->plateau_patience,
                                    cfg->plateau_rel_tol)
                ? 1
                : 0;
  });
}

int bae_synth_bal_shaped(int32_t C, int32_t P, int64_t N, uint64_t seed, double pixel_sigma, double pose_sigma,
                         double point_sigma, double* poses7, double* points3, double* intr3, int32_t* cam_idx,
                         int32_t* pt_idx, double* px2, double* true_poses7, double* true_points3) {
  return guarded([&] {
    bae::synth_bal_shaped(C, P, N, seed, pixel_sigma, pose_sigma, point_sigma, poses7, points3, intr3, cam_idx,
                          pt_idx, px2, true_poses7, true_points3);
  });
}

int bae_synth_bal_shaped_device(int32_t C, int32_t P, int64_t N, uint64_t seed, double pixel_sigma,
                                double pose_sigma, double point_sigma, int32_t device, double* poses7, double* points3,
                                double* intr3, int32_t* cam_idx, int32_t* pt_idx, double* px2, double* true_poses7,
                                double* true_points3) {
  return guarded([&] {
    bae::synth_bal_shaped_device(C, P, N, seed, pixel_sigma, pose_sigma, point_sigma, device, poses7, points3, intr3,
                                 cam_idx, pt_idx, px2, true_poses7, true_points3);
  });
}

int bae_partition_points(int32_t C, int32_t P, const int32_t* cam_idx, const int32_t* pt_idx, int64_t N,
                         int32_t world, int32_t* rank_of_point) {
  return guarded([&] { bae::partition_points(C, P, cam_idx, pt_idx, N, world, rank_of_point); });
}

int bae_time_kernel(bae_problem* p, int32_t kind, int32_t reps, double* ms) {
  return guarded([&] { *ms = ba(p)->time_kernel(kind, reps); });
}

int64_t bae_launch_count(const bae_problem* p) {
  return !p ? 0 : p->pgo ? p->pgo->launches() : p->impl->launches();
}

int bae_phase_times(bae_problem* p, double* ms7, int32_t reset) {
  return guarded([&] {
    if (ms7) ba(p)->phase_times(ms7);
    if (reset) ba(p)->phase_reset();
  });
}

int bae_plan_array(bae_problem* p, int32_t which, void* out, int64_t cap, int64_t* count, int32_t* elem_bytes) {
  return guarded([&] {
    int eb = 0;
    const int64_t n = ba(p)->plan_array(which, out, cap, &eb);
    if (count) *count = n;
    if (elem_bytes) *elem_bytes = eb;
  });
}

int bae_direct_stats(const bae_problem* p, int64_t* out5) {
  return guarded([&] {
    long long v[5];
    ba(p)->direct_stats(v);
    for (int i = 0; i < 5; ++i) out5[i] = v[i];
  });
}

int bae_direct_pairs(const bae_problem* p, int64_t* pairs, int64_t* blocks) {
  return guarded([&] {
    if (pairs) *pairs = ba(p)->direct_pairs();
    if (blocks) *blocks = ba(p)->direct_blocks();
  });
}

int bae_problem_stats(const bae_problem* p, int64_t* out6) {
  return guarded([&] {
    const bae::Plan& pl = ba(p)->plan();
    out6[0] = pl.N;
    out6[1] = pl.P;
    out6[2] = pl.C;
    out6[3] = pl.T;
    out6[4] = pl.E;
    out6[5] = pl.max_tile_obs;
  });
}

int bae_problem_shard(const bae_problem* p, int32_t* rank, int32_t* world, int32_t* local_points,
                      int64_t* local_observations) {
  return guarded([&] {
    if (rank) *rank = ba(p)->rank();
    if (world) *world = ba(p)->world();
    if (local_points) *local_points = ba(p)->local_points();
    if (local_observations) *local_observations = ba(p)->local_obs();
  });
}

// ---- host-logic hooks of the tile Cholesky (tests) ---------------------------
int bae_nd_order(int32_t C, int64_t nedges, const int32_t* edges2, int32_t leaf, int32_t* order, int32_t* group_ptr,
                 int32_t* ngroups) {
  return guarded([&] {
    std::vector<std::pair<int, int>> e(static_cast<std::size_t>(nedges));
    for (int64_t i = 0; i < nedges; ++i) {
      if (edges2[2 * i] < 0 || edges2[2 * i] >= C || edges2[2 * i + 1] < 0 || edges2[2 * i + 1] >= C)
        throw bae::Error(BAE_ERR_INDEX, "edge out of range", i);
      e[i] = {edges2[2 * i], edges2[2 * i + 1]};
    }
    const auto groups = bae::nd_camera_groups(C, e, leaf);
    int at = 0, g = 0;
    group_ptr[0] = 0;
    for (const auto& gr : groups) {
      for (int c : gr) order[at++] = c;
      group_ptr[++g] = at;
    }
    *ngroups = g;
  });
}

int bae_tile_symbolic(int32_t nt, int64_t npairs, const int32_t* pairs2, int32_t* colptr, int32_t* rowidx,
                      int64_t cap, int64_t* nnz) {
  return guarded([&] {
    std::vector<std::pair<int, int>> tp(static_cast<std::size_t>(npairs));
    for (int64_t i = 0; i < npairs; ++i) tp[i] = {pairs2[2 * i], pairs2[2 * i + 1]};
    const bae::TileCholPlan pl = bae::plan_tile_chol(nt * bae::kTB, tp);
    *nnz = pl.nnz_tiles();
    if (pl.nnz_tiles() > cap) throw bae::Error(BAE_ERR_INVALID_ARGUMENT, "rowidx capacity too small");
    std::memcpy(colptr, pl.colptr.data(), pl.colptr.size() * sizeof(int32_t));
    std::memcpy(rowidx, pl.rowidx.data(), pl.rowidx.size() * sizeof(int32_t));
  });
}

int bae_chol_tasks(int32_t nt, int64_t npairs, const int32_t* pairs2, int32_t min_ops, int32_t tail_tasks,
                   int64_t cap, int32_t* orig_bptr, int32_t* orig_ops, int32_t* bptr, int32_t* ops, int32_t* tasks,
                   int32_t* ntask, uint32_t* hmask) {
  return guarded([&] {
    std::vector<std::pair<int, int>> tp(static_cast<std::size_t>(npairs));
    for (int64_t i = 0; i < npairs; ++i) tp[i] = {pairs2[2 * i], pairs2[2 * i + 1]};
    const bae::TileCholPlan pl = bae::plan_tile_chol(nt * bae::kTB, tp);
    const bae::TileCholTasks tk = bae::plan_chol_tasks(pl, min_ops, tail_tasks);
    if (static_cast<int64_t>(pl.bop.size() / 4) > cap || static_cast<int64_t>(tk.bop.size() / 4) > cap ||
        static_cast<int64_t>(tk.tasks.size() / 4) > cap)
      throw bae::Error(BAE_ERR_INVALID_ARGUMENT, "capacity too small");
    std::memcpy(orig_bptr, pl.bptr.data(), pl.bptr.size() * sizeof(int32_t));
    std::memcpy(orig_ops, pl.bop.data(), pl.bop.size() * sizeof(int32_t));
    std::memcpy(bptr, tk.bptr.data(), tk.bptr.size() * sizeof(int32_t));
    std::memcpy(ops, tk.bop.data(), tk.bop.size() * sizeof(int32_t));
    std::memcpy(tasks, tk.tasks.data(), tk.tasks.size() * sizeof(int32_t));
    std::memcpy(hmask, tk.hmask.data(), tk.hmask.size() * sizeof(uint32_t));
    *ntask = static_cast<int32_t>(tk.tasks.size() / 4);
  });
}

// ---- BAL files, the reference's synthetic scene, the CSV trajectory ---------
int bae_bal_read(const char* path, bae_bal** out) {
  return guarded([&] {
    if (!path || !out) throw bae::Error(BAE_ERR_INVALID_ARGUMENT, "null argument");
    auto h = std::make_unique<bae_bal>();
    h->d = bae::parse_bal_file(path);
    *out = h.release();
  });
}

int bae_bal_parse(const char* text, int64_t len, bae_bal** out) {
  return guarded([&] {
    if (!text || !out || len < 0) throw bae::Error(BAE_ERR_INVALID_ARGUMENT, "null argument");
    auto h = std::make_unique<bae_bal>();
    h->d = bae::parse_bal_text(text, text + len);
    *out = h.release();
  });
}

int bae_bal_synthetic(int32_t C, int32_t P, double pixel_noise, double pose_noise, uint64_t seed, bae_bal** out) {
  return guarded([&] {
    if (!out) throw bae::Error(BAE_ERR_INVALID_ARGUMENT, "null argument");
    auto h = std::make_unique<bae_bal>();
    h->d = bae::synth_ba_dense(C, P, pixel_noise, pose_noise, seed);
    *out = h.release();
  });
}

int bae_bal_from_arrays(int32_t C, int32_t P, int64_t N, const double* cameras9, const double* points3,
                        const int32_t* cam_idx, const int32_t* pt_idx, const double* px2, bae_bal** out) {
  return guarded([&] {
    if (!out || C < 1 || P < 1 || N < 1 || !cameras9 || !points3 || !cam_idx || !pt_idx || !px2)
      throw bae::Error(BAE_ERR_INVALID_ARGUMENT, "bad BAL arrays");
    auto h = std::make_unique<bae_bal>();
    bae::BalData& d = h->d;
    d.C = C;
    d.P = P;
    d.N = N;
    d.cameras.assign(cameras9, cameras9 + 9 * static_cast<std::size_t>(C));
    d.points.assign(points3, points3 + 3 * static_cast<std::size_t>(P));
    d.cam_idx.assign(cam_idx, cam_idx + N);
    d.pt_idx.assign(pt_idx, pt_idx + N);
    d.px.assign(px2, px2 + 2 * N);
    *out = h.release();
  });
}

int bae_bal_counts(const bae_bal* b, int32_t* C, int32_t* P, int64_t* N) {
  return guarded([&] {
    if (C) *C = b->d.C;
    if (P) *P = b->d.P;
    if (N) *N = b->d.N;
  });
}

int bae_bal_arrays(const bae_bal* b, double* poses7, double* intr3, double* points3, int32_t* cam_idx,
                   int32_t* pt_idx, double* px2, double* cameras9) {
  return guarded([&] {
    const bae::BalData& d = b->d;
    bae::bal_poses(d, poses7, intr3);
    if (points3) std::memcpy(points3, d.points.data(), d.points.size() * sizeof(double));
    if (cam_idx) std::memcpy(cam_idx, d.cam_idx.data(), d.cam_idx.size() * sizeof(int32_t));
    if (pt_idx) std::memcpy(pt_idx, d.pt_idx.data(), d.pt_idx.size() * sizeof(int32_t));
    if (px2) std::memcpy(px2, d.px.data(), d.px.size() * sizeof(double));
    if (cameras9) std::memcpy(cameras9, d.cameras.data(), d.cameras.size() * sizeof(double));
  });
}

int bae_bal_write(const bae_bal* b, const char* path) {
  return guarded([&] { bae::write_bal_file(b->d, path); });
}

int bae_bal_write_binary(const bae_bal* b, const char* path) {
  return guarded([&] { bae::write_bal_binary(b->d, path); });
}

void bae_bal_free(bae_bal* b) { delete b; }

int bae_g2o_read(const char* path, bae_g2o** out) {
  return guarded([&] {
    if (!path || !out) throw bae::Error(BAE_ERR_INVALID_ARGUMENT, "null argument");
    auto h = std::make_unique<bae_g2o>();
    h->d = bae::parse_g2o_file(path);
    *out = h.release();
  });
}

int bae_g2o_parse(const char* text, int64_t len, bae_g2o** out) {
  return guarded([&] {
    if (!text || !out || len < 0) throw bae::Error(BAE_ERR_INVALID_ARGUMENT, "null argument");
    auto h = std::make_unique<bae_g2o>();
    h->d = bae::parse_g2o_text(text, text + len);
    *out = h.release();
  });
}

int bae_g2o_counts(const bae_g2o* g, int32_t* num_vertices, int64_t* num_edges, int32_t* num_warnings) {
  return guarded([&] {
    if (num_vertices) *num_vertices = static_cast<int32_t>(g->d.ids.size());
    if (num_edges) *num_edges = static_cast<int64_t>(g->d.ei.size());
    if (num_warnings) *num_warnings = static_cast<int32_t>(g->d.warnings.size());
  });
}

int bae_g2o_arrays(const bae_g2o* g, double* poses7, int64_t* vertex_ids, int32_t* edge_i, int32_t* edge_j,
                   double* measurements7, double* information36, int32_t* has_information) {
  return guarded([&] {
    const bae::G2oData& d = g->d;
    auto cp = [](auto* dst, const auto& v) {
      if (dst && !v.empty()) std::memcpy(dst, v.data(), v.size() * sizeof(v[0]));
    };
    cp(poses7, d.poses);
    cp(vertex_ids, d.ids);
    cp(edge_i, d.ei);
    cp(edge_j, d.ej);
    cp(measurements7, d.meas);
    cp(information36, d.info);
    cp(has_information, d.has_info);
  });
}

const char* bae_g2o_warning(const bae_g2o* g, int32_t k) {
  return (g && k >= 0 && k < static_cast<int32_t>(g->d.warnings.size())) ? g->d.warnings[k].c_str() : nullptr;
}

void bae_g2o_free(bae_g2o* g) { delete g; }

int bae_write_csv(const char* path, const bae_iter_record* traj, int32_t n) {  // cli.hpp:69-79
  return guarded([&] {
    std::FILE* f = std::fopen(path, "w");
    if (!f) throw bae::Error(BAE_ERR_IO, std::string("cannot open CSV output '") + path + "'");
    std::fputs("iter,cost,mse,lambda,accepted,cum_time_s\n", f);
    for (int32_t i = 0; i < n; ++i) {
      const bae_iter_record& r = traj[i];
      std::fprintf(f, "%d,%.17g,%.17g,%.17g,%d,%.6f\n", r.iteration, r.cost, r.mse, r.lambda, r.accepted ? 1 : 0,
                   r.cum_time_s);
    }
    if (std::fclose(f) != 0) throw bae::Error(BAE_ERR_IO, std::string("cannot write CSV output '") + path + "'");
  });
}

}  // extern "C"
