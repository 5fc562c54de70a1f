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

void validate_inputs(int C, int P, const std::int32_t* cam_idx, const std::int32_t* pt_idx, std::int64_t N,
                     bool indices) {
  if (N <= 0) throw Error(BAE_ERR_INVALID_ARGUMENT, "make_ba_problem: no observations");
  if (N >= (std::int64_t{1} << 31) - 1) throw Error(BAE_ERR_UNSUPPORTED, "more than 2^31-2 observations");
  if (!indices) return;  // with N > 0, empty groups mean an out-of-range index: the device plan reports it
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

  // Observations of each original point, ascending id (point transpose plan):
  // per-chunk histograms over contiguous observation ranges, chunk-ordered
  // offsets, a parallel scatter -- the order inside a point is ascending k
  // whatever the chunking.
  const int nth = N >= (1 << 16) ? host_threads() : 1;
  const int nch = std::min(nth, 8);
  std::vector<std::vector<std::int32_t>> ccnt(static_cast<std::size_t>(nch));
  std::vector<std::vector<std::int32_t>> ccam(static_cast<std::size_t>(nch));
  parallel_chunks(N, nch, [&](int c, std::int64_t b, std::int64_t e) {
    ccnt[c].assign(static_cast<std::size_t>(P), 0);
    ccam[c].assign(static_cast<std::size_t>(C), 0);
    auto& h = ccnt[c];
    auto& hc = ccam[c];
    for (std::int64_t k = b; k < e; ++k) {
      ++h[pt_idx[k]];
      ++hc[cam_idx[k]];
    }
  });
  for (int c = 0; c < C; ++c) {
    std::int32_t n = 0;
    for (int ch = 0; ch < nch; ++ch) n += ccam[ch][c];
    if (n == 0) pl.has_empty_camera = true;
  }
  std::vector<std::int32_t> pcnt(static_cast<std::size_t>(P) + 1, 0);
  parallel_chunks(P, nth, [&](int, std::int64_t b, std::int64_t e) {
    for (std::int64_t p = b; p < e; ++p) {
      std::int32_t n = 0;
      for (int ch = 0; ch < nch; ++ch) n += ccnt[ch][p];
      pcnt[p + 1] = n;
    }
  });
  for (int p = 0; p < P; ++p) {
    if (pcnt[p + 1] == 0) pl.has_empty_point = true;
    if (pcnt[p + 1] > 65535) throw Error(BAE_ERR_UNSUPPORTED, "a point has more than 65535 observations");
  }
  std::partial_sum(pcnt.begin(), pcnt.end(), pcnt.begin());
  parallel_chunks(P, nth, [&](int, std::int64_t b, std::int64_t e) {  // chunk write cursors
    for (std::int64_t p = b; p < e; ++p) {
      std::int32_t run = pcnt[p];
      for (int ch = 0; ch < nch; ++ch) {
        const std::int32_t m = ccnt[ch][p];
        ccnt[ch][p] = run;
        run += m;
      }
    }
  });
  std::vector<std::int32_t> pobs(static_cast<std::size_t>(N));
  parallel_chunks(N, nch, [&](int c, std::int64_t b, std::int64_t e) {
    auto& cur = ccnt[c];
    for (std::int64_t k = b; k < e; ++k) pobs[cur[pt_idx[k]]++] = static_cast<std::int32_t>(k);
  });
  ccnt.clear();
  ccnt.shrink_to_fit();
  // camera of each observation in point order (one gather instead of one per pass)
  std::vector<std::int32_t> pcam(static_cast<std::size_t>(N));
  parallel_chunks(N, nth, [&](int, std::int64_t b, std::int64_t e) {
    for (std::int64_t j = b; j < e; ++j) pcam[j] = cam_idx[pobs[j]];
  });

  st.mark("point lists");
  // Internal point order: stable counting sort by the lowest observing camera,
  // so consecutive points share cameras and a tile touches few of them.
  std::vector<std::int32_t> mincam(static_cast<std::size_t>(P), C);
  parallel_chunks(P, nth, [&](int, std::int64_t b, std::int64_t e) {
    for (std::int64_t p = b; p < e; ++p) {
      std::int32_t m = C;
      for (std::int32_t j = pcnt[p]; j < pcnt[p + 1]; ++j) m = std::min(m, pcam[j]);
      mincam[p] = m;
    }
  });
  {
    const int pch = P >= (1 << 16) ? nch : 1;
    std::vector<std::vector<std::int32_t>> bucket(static_cast<std::size_t>(pch));
    parallel_chunks(P, pch, [&](int c, std::int64_t b, std::int64_t e) {
      bucket[c].assign(static_cast<std::size_t>(C) + 1, 0);
      for (std::int64_t p = b; p < e; ++p) ++bucket[c][mincam[p]];
    });
    std::int32_t run = 0;  // bucket-major, chunk-minor offsets: stable in p
    for (int m = 0; m <= C; ++m)
      for (int c = 0; c < pch; ++c) {
        const std::int32_t n = bucket[c][m];
        bucket[c][m] = run;
        run += n;
      }
    pl.pt_of_internal.resize(static_cast<std::size_t>(P));
    pl.internal_of_pt.resize(static_cast<std::size_t>(P));
    parallel_chunks(P, pch, [&](int c, std::int64_t b, std::int64_t e) {
      auto& cur = bucket[c];
      for (std::int64_t p = b; p < e; ++p) {
        const std::int32_t i = cur[mincam[p]]++;
        pl.pt_of_internal[i] = static_cast<std::int32_t>(p);
        pl.internal_of_pt[p] = i;
      }
    });
  }

  st.mark("internal order");
  // Greedy tile packing over internal points, in a fixed number of segments
  // (a function of P only, so the tiling depends neither on the thread count
  // nor on which planner runs: plan_device.cu packs the same segments); each
  // segment starts a fresh tile and is packed independently.
  const int nseg = plan_segments(P);
  struct Seg {
    std::vector<std::int32_t> pt_begin, obs_count;  // per tile
    std::vector<std::vector<std::int32_t>> cams;
  };
  std::vector<Seg> segs(static_cast<std::size_t>(nseg));
  parallel_chunks(nseg, std::min(nth, nseg), [&](int, std::int64_t s0, std::int64_t s1) {
    std::vector<std::int32_t> stamp(static_cast<std::size_t>(C), -1), seen(static_cast<std::size_t>(C), -1);
    int t = 0;  // running stamp over this thread's segments
    for (std::int64_t sg = s0; sg < s1; ++sg) {
      Seg& S = segs[sg];
      const int i0 = static_cast<int>(static_cast<std::int64_t>(P) * sg / nseg);
      const int i1 = static_cast<int>(static_cast<std::int64_t>(P) * (sg + 1) / nseg);
      if (i1 <= i0) continue;
      ++t;
      int t_obs = 0, t_pts = 0;
      std::vector<std::int32_t> cur_cams;
      S.pt_begin.push_back(i0);
      auto distinct_new = [&](int p) {
        int n = 0;
        for (std::int32_t j = pcnt[p]; j < pcnt[p + 1]; ++j) {
          const int c = pcam[j];
          if (stamp[c] != t && seen[c] != p) {
            seen[c] = p;
            ++n;
          }
        }
        for (std::int32_t j = pcnt[p]; j < pcnt[p + 1]; ++j) seen[pcam[j]] = -1;
        return n;
      };
      for (int i = i0; i < i1; ++i) {
        const int p = pl.pt_of_internal[i];
        const int m = pcnt[p + 1] - pcnt[p];
        const int newc = distinct_new(p);
        if (t_pts > 0 && (t_obs + m > tile_obs_target || static_cast<int>(cur_cams.size()) + newc > tile_cam_cap ||
                          t_pts + 1 > tile_pts_cap)) {
          S.cams.push_back(std::move(cur_cams));
          cur_cams.clear();
          S.obs_count.push_back(t_obs);
          S.pt_begin.push_back(i);
          ++t;
          t_obs = 0;
          t_pts = 0;
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
      S.cams.push_back(std::move(cur_cams));
      S.obs_count.push_back(t_obs);
    }
  });
  std::vector<std::vector<std::int32_t>> tile_cams;
  pl.tile_pt_begin.clear();
  pl.tile_obs_begin.assign(1, 0);
  for (Seg& S : segs)
    for (std::size_t k = 0; k < S.pt_begin.size(); ++k) {
      pl.tile_pt_begin.push_back(S.pt_begin[k]);
      pl.tile_obs_begin.push_back(pl.tile_obs_begin.back() + S.obs_count[k]);
      tile_cams.push_back(std::move(S.cams[k]));
    }
  pl.tile_pt_begin.push_back(P);
  pl.T = static_cast<int>(tile_cams.size());

  st.mark("tile packing");
  // Per-tile slot order: (local camera, internal point, observation id).
  // Tiles are independent once their entry offsets are known: sort the
  // camera lists and fill the slots in parallel chunks of tiles.
  pl.obs_lcpt.resize(static_cast<std::size_t>(N));
  pl.obs_orig.resize(static_cast<std::size_t>(N));
  if (px2) pl.obs_px.resize(static_cast<std::size_t>(N) * 2);  // null: the caller gathers them on the device
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
          if (px2) {
            pl.obs_px[2 * static_cast<std::size_t>(slot)] = px2[2 * k];
            pl.obs_px[2 * static_cast<std::size_t>(slot) + 1] = px2[2 * k + 1];
          }
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
