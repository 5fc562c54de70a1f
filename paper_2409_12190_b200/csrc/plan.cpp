// Host-side setup: the one-time symbolic phase of the B200 path.
//
// The reference derives its cached structure from the Jacobian pattern:
// transpose plans (bsr.hpp:140-160) give the observations of each camera and
// of each point in ascending observation order, the pair tables
// (spgemm.hpp:33-81) fix the accumulation order of J^T J, and
// build_csr_pattern (assemble.hpp:135-177) lays out the scalar normal matrix.
// The device path never forms J^T J's off-diagonal blocks, so its symbolic
// phase is a decomposition of the observations into CTA-sized tiles instead
// (see Plan in bae_internal.hpp). Everything here is O(N + P + C) counting
// sorts.
#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <numeric>

#include "bae_internal.hpp"

namespace bae {

namespace {
// BAE_HOST_TIMING=1: planner stage times on stderr.
struct StageTimer {
  bool on = std::getenv("BAE_HOST_TIMING") != nullptr;
  std::chrono::steady_clock::time_point t = std::chrono::steady_clock::now();
  void mark(const char* what) {
    if (!on) return;
    const auto n = std::chrono::steady_clock::now();
    std::fprintf(stderr, "[bae plan] %-22s %8.3f ms\n", what, std::chrono::duration<double, std::milli>(n - t).count());
    t = n;
  }
};
}  // namespace

void validate_inputs(int C, int P, const std::int32_t* cam_idx, const std::int32_t* pt_idx, std::int64_t N) {
  if (N <= 0) throw Error(BAE_ERR_INVALID_ARGUMENT, "make_ba_problem: no observations");
  if (N >= (std::int64_t{1} << 31) - 1) throw Error(BAE_ERR_UNSUPPORTED, "more than 2^31-2 observations");
  for (std::int64_t k = 0; k < N; ++k) {
    if (cam_idx[k] < 0 || cam_idx[k] >= C) throw Error(BAE_ERR_INDEX, "make_ba_problem: camera index out of range", k);
    if (pt_idx[k] < 0 || pt_idx[k] >= P) throw Error(BAE_ERR_INDEX, "make_ba_problem: point index out of range", k);
  }
  if (C < 1) throw Error(BAE_ERR_INVALID_ARGUMENT, "track_poses: empty group");
  if (P < 1) throw Error(BAE_ERR_INVALID_ARGUMENT, "track_points: empty group");
}

Plan build_plan(int C, int P, const std::int32_t* cam_idx, const std::int32_t* pt_idx, const double* px2,
                std::int64_t N, int tile_obs_target, int tile_cam_cap, int tile_pts_cap, int smem_tile_obs_cap) {
  StageTimer st;
  Plan pl;
  pl.C = C;
  pl.P = P;
  pl.N = N;
  pl.tile_obs_target = tile_obs_target;
  pl.tile_cam_cap = tile_cam_cap;

  // Observations of each original point, ascending id (point transpose plan).
  std::vector<std::int32_t> pcnt(static_cast<std::size_t>(P) + 1, 0);
  for (std::int64_t k = 0; k < N; ++k) ++pcnt[pt_idx[k] + 1];
  std::vector<std::int32_t> camcnt(static_cast<std::size_t>(C), 0);
  for (std::int64_t k = 0; k < N; ++k) ++camcnt[cam_idx[k]];
  for (int c = 0; c < C; ++c)
    if (camcnt[c] == 0) pl.has_empty_camera = true;
  for (int p = 0; p < P; ++p) {
    if (pcnt[p + 1] == 0) pl.has_empty_point = true;
    if (pcnt[p + 1] > 65535) throw Error(BAE_ERR_UNSUPPORTED, "a point has more than 65535 observations");
  }
  std::partial_sum(pcnt.begin(), pcnt.end(), pcnt.begin());
  std::vector<std::int32_t> pobs(static_cast<std::size_t>(N));
  {
    std::vector<std::int32_t> cur(pcnt.begin(), pcnt.end() - 1);
    for (std::int64_t k = 0; k < N; ++k) pobs[cur[pt_idx[k]]++] = static_cast<std::int32_t>(k);
  }
  const int nth = N >= (1 << 16) ? host_threads() : 1;
  // camera of each observation in point order (one gather instead of one per pass)
  std::vector<std::int32_t> pcam(static_cast<std::size_t>(N));
  parallel_chunks(N, nth, [&](int, std::int64_t b, std::int64_t e) {
    for (std::int64_t j = b; j < e; ++j) pcam[j] = cam_idx[pobs[j]];
  });

  st.mark("point lists");
  // Internal point order: stable counting sort by the lowest observing camera,
  // so consecutive points share cameras and a tile touches few of them.
  std::vector<std::int32_t> mincam(static_cast<std::size_t>(P), C);
  for (std::int64_t k = 0; k < N; ++k) mincam[pt_idx[k]] = std::min(mincam[pt_idx[k]], cam_idx[k]);
  {
    std::vector<std::int32_t> bucket(static_cast<std::size_t>(C) + 2, 0);
    for (int p = 0; p < P; ++p) ++bucket[mincam[p] + 1];
    std::partial_sum(bucket.begin(), bucket.end(), bucket.begin());
    pl.pt_of_internal.resize(static_cast<std::size_t>(P));
    pl.internal_of_pt.resize(static_cast<std::size_t>(P));
    for (int p = 0; p < P; ++p) {
      const std::int32_t i = bucket[mincam[p]]++;
      pl.pt_of_internal[i] = p;
      pl.internal_of_pt[p] = i;
    }
  }

  st.mark("internal order");
  // Greedy tile packing over internal points.
  std::vector<std::int32_t> stamp(static_cast<std::size_t>(C), -1), seen(static_cast<std::size_t>(C), -1);
  std::vector<std::vector<std::int32_t>> tile_cams;
  pl.tile_pt_begin.push_back(0);
  pl.tile_obs_begin.push_back(0);
  int t = 0, t_obs = 0, t_pts = 0;
  std::vector<std::int32_t> cur_cams;
  auto distinct_new = [&](int p, int tile) {
    int n = 0;
    for (std::int32_t j = pcnt[p]; j < pcnt[p + 1]; ++j) {
      const int c = pcam[j];
      if (stamp[c] != tile && seen[c] != p) {
        seen[c] = p;
        ++n;
      }
    }
    for (std::int32_t j = pcnt[p]; j < pcnt[p + 1]; ++j) seen[pcam[j]] = -1;
    return n;
  };
  for (int i = 0; i < P; ++i) {
    const int p = pl.pt_of_internal[i];
    const int m = pcnt[p + 1] - pcnt[p];
    int newc = distinct_new(p, t);
    if (t_pts > 0 && (t_obs + m > tile_obs_target || static_cast<int>(cur_cams.size()) + newc > tile_cam_cap ||
                      t_pts + 1 > tile_pts_cap)) {
      tile_cams.push_back(cur_cams);
      cur_cams.clear();
      pl.tile_pt_begin.push_back(i);
      pl.tile_obs_begin.push_back(pl.tile_obs_begin.back() + t_obs);
      ++t;
      t_obs = 0;
      t_pts = 0;
      newc = distinct_new(p, t);
    }
    for (std::int32_t j = pcnt[p]; j < pcnt[p + 1]; ++j) {
      const int c = pcam[j];
      if (stamp[c] != t) {
        stamp[c] = t;
        cur_cams.push_back(c);
      }
    }
    t_obs += m;
    ++t_pts;
  }
  tile_cams.push_back(cur_cams);
  pl.tile_pt_begin.push_back(P);
  pl.tile_obs_begin.push_back(pl.tile_obs_begin.back() + t_obs);
  pl.T = t + 1;

  st.mark("tile packing");
  // Per-tile slot order: (local camera, internal point, observation id).
  // Tiles are independent once their entry offsets are known: sort the
  // camera lists and fill the slots in parallel chunks of tiles.
  pl.obs_lcpt.resize(static_cast<std::size_t>(N));
  pl.obs_orig.resize(static_cast<std::size_t>(N));
  pl.obs_px.resize(static_cast<std::size_t>(N) * 2);
  pl.pt_ptr.assign(static_cast<std::size_t>(P) + 1, 0);
  pl.ptobs.resize(static_cast<std::size_t>(N));
  pl.tile_ws.assign(static_cast<std::size_t>(pl.T), -1);
  pl.tile_ent_begin.assign(static_cast<std::size_t>(pl.T) + 1, 0);
  for (int tt = 0; tt < pl.T; ++tt) {
    if (pl.tile_obs_begin[tt + 1] - pl.tile_obs_begin[tt] > 65536)
      throw Error(BAE_ERR_UNSUPPORTED, "tile exceeds 65536 observations");
    pl.tile_ent_begin[tt + 1] = pl.tile_ent_begin[tt] + static_cast<std::int32_t>(tile_cams[tt].size());
  }
  pl.E = pl.tile_ent_begin[pl.T];
  pl.ent_cam.resize(static_cast<std::size_t>(pl.E));
  pl.ent_obs_begin.resize(static_cast<std::size_t>(pl.E) + 1);
  parallel_chunks(pl.T, pl.T >= 256 ? nth : 1, [&](int, std::int64_t t0, std::int64_t t1) {
    std::vector<std::int32_t> lcam_of(static_cast<std::size_t>(C), -1);
    std::vector<std::int32_t> seg;
    for (std::int64_t tt = t0; tt < t1; ++tt) {
      auto& cams = tile_cams[tt];
      std::sort(cams.begin(), cams.end());
      const int nc = static_cast<int>(cams.size());
      for (int l = 0; l < nc; ++l) lcam_of[cams[l]] = l;
      const std::int32_t ob = pl.tile_obs_begin[tt];
      const std::int32_t pb = pl.tile_pt_begin[tt], pe = pl.tile_pt_begin[tt + 1];
      seg.assign(static_cast<std::size_t>(nc) + 1, 0);
      for (int i = pb; i < pe; ++i) {
        const int p = pl.pt_of_internal[i];
        for (std::int32_t j = pcnt[p]; j < pcnt[p + 1]; ++j) ++seg[lcam_of[pcam[j]] + 1];
      }
      std::partial_sum(seg.begin(), seg.end(), seg.begin());
      const std::int32_t eb = pl.tile_ent_begin[tt];
      for (int l = 0; l < nc; ++l) {
        pl.ent_cam[eb + l] = cams[l];
        pl.ent_obs_begin[eb + l] = ob + seg[l];
      }
      std::int32_t pcur = ob;
      for (int i = pb; i < pe; ++i) {
        const int p = pl.pt_of_internal[i];
        pl.pt_ptr[i] = pcur;
        for (std::int32_t j = pcnt[p]; j < pcnt[p + 1]; ++j) {
          const std::int32_t k = pobs[j];
          const int l = lcam_of[pcam[j]];
          const std::int32_t local = seg[l]++;
          const std::int32_t slot = ob + local;
          pl.obs_lcpt[slot] = static_cast<std::uint32_t>(l) | (static_cast<std::uint32_t>(i - pb) << 16);
          pl.obs_orig[slot] = k;
          pl.obs_px[2 * static_cast<std::size_t>(slot)] = px2[2 * k];
          pl.obs_px[2 * static_cast<std::size_t>(slot) + 1] = px2[2 * k + 1];
          pl.ptobs[pcur++] = static_cast<std::uint16_t>(local);
        }
      }
      for (int l = 0; l < nc; ++l) lcam_of[cams[l]] = -1;
    }
  });
  for (int tt = 0; tt < pl.T; ++tt) {
    const int nobs = pl.tile_obs_begin[tt + 1] - pl.tile_obs_begin[tt];
    const int npts = pl.tile_pt_begin[tt + 1] - pl.tile_pt_begin[tt];
    const int nc = pl.tile_ent_begin[tt + 1] - pl.tile_ent_begin[tt];
    pl.max_tile_obs = std::max(pl.max_tile_obs, nobs);
    pl.max_tile_cams = std::max(pl.max_tile_cams, nc);
    pl.max_tile_pts = std::max(pl.max_tile_pts, npts);
    if (nobs > smem_tile_obs_cap || nc > tile_cam_cap) {
      pl.tile_ws[tt] = pl.n_big++;
      pl.big_obs = std::max(pl.big_obs, nobs);
      pl.big_cams = std::max(pl.big_cams, nc);
      pl.big_pts = std::max(pl.big_pts, npts);
    }
  }
  pl.pt_ptr[P] = static_cast<std::int32_t>(N);
  pl.ent_obs_begin[pl.E] = static_cast<std::int32_t>(N);

  st.mark("slot order");
  // Entries of each camera in ascending entry (= tile) order.
  pl.cam_ent_ptr.assign(static_cast<std::size_t>(C) + 1, 0);
  for (int e = 0; e < pl.E; ++e) ++pl.cam_ent_ptr[pl.ent_cam[e] + 1];
  std::partial_sum(pl.cam_ent_ptr.begin(), pl.cam_ent_ptr.end(), pl.cam_ent_ptr.begin());
  pl.cam_ent.resize(static_cast<std::size_t>(pl.E));
  {
    std::vector<std::int32_t> cur(pl.cam_ent_ptr.begin(), pl.cam_ent_ptr.end() - 1);
    for (int e = 0; e < pl.E; ++e) pl.cam_ent[cur[pl.ent_cam[e]]++] = e;
  }
  st.mark("camera entries");
  return pl;
}

// Landmark partition for multi-GPU runs: contiguous ranges of
// the internal point order (the order tiles are cut from), balanced by
// observation count; cameras are replicated on every rank.
void partition_points(int C, int P, const std::int32_t* cam_idx, const std::int32_t* pt_idx, std::int64_t N,
                      int world, std::int32_t* rank_of_point) {
  if (world < 1) throw Error(BAE_ERR_INVALID_ARGUMENT, "partition: world must be >= 1");
  validate_inputs(C, P, cam_idx, pt_idx, N);
  std::vector<std::int32_t> cnt(static_cast<std::size_t>(P), 0), mincam(static_cast<std::size_t>(P), C);
  for (std::int64_t k = 0; k < N; ++k) {
    ++cnt[pt_idx[k]];
    mincam[pt_idx[k]] = std::min(mincam[pt_idx[k]], cam_idx[k]);
  }
  std::vector<std::int32_t> bucket(static_cast<std::size_t>(C) + 2, 0), order(static_cast<std::size_t>(P));
  for (int p = 0; p < P; ++p) ++bucket[mincam[p] + 1];
  std::partial_sum(bucket.begin(), bucket.end(), bucket.begin());
  for (int p = 0; p < P; ++p) order[bucket[mincam[p]]++] = p;
  std::int64_t acc = 0;
  for (int i = 0; i < P; ++i) {
    const int p = order[i];
    // rank r owns observations [r N / world, (r+1) N / world) of the prefix
    rank_of_point[p] = static_cast<std::int32_t>(std::min<std::int64_t>(world - 1, (acc * world) / N));
    acc += cnt[p];
  }
}

}  // namespace bae
