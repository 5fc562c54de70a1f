"""GPU parity: the sm_100a path through the C ABI vs the CPU oracle
(restatement of the reference hot path). Tolerances are the north star's
(BASELINE.json): bit-exact index structure, per-iteration cost 1e-6 relative,
parameters 1e-5 relative; kernel values 1e-12 relative with a unit floor
(acceptance.cpp:51-62)."""
import numpy as np
import pytest

import paper_2409_12190_b200 as bae

pytestmark = pytest.mark.gpu


def _scene(C=12, P=300, N=1500, seed=3):
    return bae.synthetic.bal_shaped(C, P, N, seed=seed)


def _pair(s, oracle, **kw):
    gpu = bae.make_ba_problem(s.poses, s.points, s.intrinsics, s.observations, **kw)
    ref = oracle.Problem(s.poses, s.points, s.intrinsics, s.cam_idx, s.pt_idx, s.pixels)
    return gpu, ref


def _blocks_match(a, b, tol):
    # per-block comparison with a unit absolute floor (acceptance.cpp:51-62)
    scale = np.maximum(1.0, np.abs(b).reshape(b.shape[0], -1).max(axis=1))
    err = np.abs(a - b).reshape(a.shape[0], -1).max(axis=1)
    return bool(np.all(err <= tol * scale)), float((err / scale).max())


def test_residual_matches_oracle(oracle):
    s = _scene()
    gpu, ref = _pair(s, oracle)
    r_gpu = gpu.evaluate()
    r_ref, c_ref = ref.evaluate()
    assert np.allclose(r_gpu, r_ref, rtol=1e-12, atol=1e-10)
    assert abs(gpu.cost() - c_ref) <= 1e-12 * c_ref


def test_jacobian_values_and_pattern(oracle):
    s = _scene(seed=4)
    gpu, ref = _pair(s, oracle)
    jg = gpu.jacobian()
    jr = ref.jacobian()
    ok, worst = _blocks_match(jg.j_pose.values, jr["j_pose"], 1e-12)
    assert ok, worst
    ok, worst = _blocks_match(jg.j_point.values, jr["j_point"], 1e-12)
    assert ok, worst
    # bit-exact index structure (one block per row at the gather column)
    assert np.array_equal(jg.j_pose.row_ptr, jr["pose_row_ptr"])
    assert np.array_equal(jg.j_pose.col_idx, jr["pose_col"])
    assert np.array_equal(jg.j_point.row_ptr, jr["point_row_ptr"])
    assert np.array_equal(jg.j_point.col_idx, jr["point_col"])


@pytest.mark.parametrize("which", [0, 1])
def test_transpose_plans_bit_exact(oracle, which):
    s = _scene(C=20, P=500, N=2600, seed=5)
    gpu, ref = _pair(s, oracle, tile_obs=64)  # many tiles
    tg = gpu.transpose_plan(which)
    rp, ci, sb = ref.transpose_plan(which)
    assert np.array_equal(tg.row_ptr, rp)
    assert np.array_equal(tg.col_idx, ci)
    assert np.array_equal(tg.src_block, sb)


def test_block_diagonals_match_normal_matrix(oracle):
    s = _scene(C=6, P=60, N=240, seed=6)
    gpu, ref = _pair(s, oracle)
    hcc, gc, hpp, gp = gpu.block_diagonals()
    A, b = ref.normal_dense(0.0, cmin=-1e300, cmax=1e300)  # undamped
    C, P = s.poses.shape[0], s.points.shape[0]
    for c in range(C):
        blk = A[6 * c:6 * c + 6, 6 * c:6 * c + 6]
        assert np.allclose(hcc[c], blk, rtol=1e-11, atol=1e-9 * np.abs(blk).max())
        assert np.allclose(-gc[c], b[6 * c:6 * c + 6], rtol=1e-11, atol=1e-9 * np.abs(b).max())
    o = 6 * C
    for p in range(P):
        blk = A[o + 3 * p:o + 3 * p + 3, o + 3 * p:o + 3 * p + 3]
        assert np.allclose(hpp[p], blk, rtol=1e-11, atol=1e-12 * np.abs(blk).max())
        assert np.allclose(-gp[p], b[o + 3 * p:o + 3 * p + 3], rtol=1e-11, atol=1e-9 * np.abs(b).max())


@pytest.mark.parametrize("lmbda", [1e-4, 1e-1, 10.0])
def test_schur_pcg_step_matches_cholesky(oracle, lmbda):
    s = _scene(C=10, P=200, N=900, seed=7)
    gpu, ref = _pair(s, oracle)
    cfg = bae.LmConfig(solver=bae.SolverChoice.pcg, pcg_tol=1e-13, pcg_max_iters=2000)
    dg, iters, rel = gpu.solve_step(lmbda, cfg)
    dr, _ = ref.solve_step(lmbda, bae.LmConfig())
    assert iters > 0
    assert np.linalg.norm(dg - dr) <= 1e-8 * np.linalg.norm(dr), (np.linalg.norm(dg - dr) / np.linalg.norm(dr))


def test_lm_trajectory_matches_oracle_ladybug(oracle):
    s = bae.synthetic.config_scene("ladybug-49")
    gpu, ref = _pair(s, oracle)
    cfg_g = bae.LmConfig(max_iterations=15, solver=bae.SolverChoice.pcg, pcg_tol=1e-12)
    rep = bae.optimize(gpu, s.poses, s.points, cfg_g)
    oracle.set_threads(8)
    oref = ref.optimize(bae.LmConfig(max_iterations=15))  # reference default: Cholesky (exact)
    n = min(len(rep.trajectory), len(oref["trajectory"]))
    assert n >= 4
    for a, b in zip(rep.trajectory[:n], oref["trajectory"][:n]):
        assert a.accepted == b["accepted"]
        assert abs(a.cost - b["cost"]) <= 1e-6 * b["cost"], (a.iteration, a.cost, b["cost"])
        assert a.lmbda == b["lmbda"]
    assert abs(rep.final_cost - oref["final_cost"]) <= 1e-6 * oref["final_cost"]
    p7, p3 = gpu.get_parameters()
    assert np.abs(p3 - oref["points"]).max() <= 1e-5 * max(1.0, np.abs(oref["points"]).max())
    assert np.abs(p7 - oref["poses"]).max() <= 1e-5 * max(1.0, np.abs(oref["poses"]).max())


def test_cheirality_reports_lowest_observation(oracle):
    s = _scene(C=4, P=40, N=120, seed=8)
    pts = s.points.copy()
    # put point pt_idx[k] on camera cam_idx[k]'s plane for two observations
    ks = [57, 91]
    for k in ks:
        c, p = s.cam_idx[k], s.pt_idx[k]
        q = s.poses[c, 3:]
        x, y, z, w = q
        R = np.array([[1 - 2 * (y * y + z * z), 2 * (x * y - z * w), 2 * (x * z + y * w)],
                      [2 * (x * y + z * w), 1 - 2 * (x * x + z * z), 2 * (y * z - x * w)],
                      [2 * (x * z - y * w), 2 * (y * z + x * w), 1 - 2 * (x * x + y * y)]])
        pts[p] = R.T @ (np.array([0.3, 0.1, 0.0]) - s.poses[c, :3])
    moved = {int(s.pt_idx[k]) for k in ks}
    with pytest.raises(bae.CheiralityError) as e:
        bae.make_ba_problem(s.poses, pts, s.intrinsics, s.observations)
    with pytest.raises(oracle.OracleError) as eo:
        oracle.Problem(s.poses, pts, s.intrinsics, s.cam_idx, s.pt_idx, s.pixels)
    assert e.value.observation == eo.value.index
    assert int(s.pt_idx[e.value.observation]) in moved


def test_index_error_position():
    s = _scene(C=4, P=40, N=120, seed=9)
    ci = s.cam_idx.copy()
    pi = s.pt_idx.copy()
    pi[17] = 40
    with pytest.raises(bae.IndexError) as e:
        bae.make_ba_problem(s.poses, s.points, s.intrinsics, (ci, pi, s.pixels))
    assert e.value.position == 17
    ci[5] = -1
    with pytest.raises(bae.IndexError) as e:
        bae.make_ba_problem(s.poses, s.points, s.intrinsics, (ci, pi, s.pixels))
    assert e.value.position == 5


def test_launch_counter_moves():
    s = _scene()
    gpu = bae.make_ba_problem(s.poses, s.points, s.intrinsics, s.observations)
    n0 = gpu.launch_count()
    bae.optimize(gpu, s.poses, s.points, bae.LmConfig(max_iterations=2, solver=bae.SolverChoice.pcg))
    assert gpu.launch_count() > n0 + 10


@pytest.mark.parametrize("lmbda", [1e-6, 1e-2, 3.0])
def test_direct_step_matches_cholesky(oracle, lmbda):
    s = _scene(C=8, P=120, N=500, seed=11)
    gpu, ref = _pair(s, oracle)
    dg, iters, _ = gpu.solve_step(lmbda, bae.LmConfig())  # reference default: cholesky
    dr, _ = ref.solve_step(lmbda, bae.LmConfig())
    assert iters == 0
    # both are exact solves: the GPU step satisfies the oracle's damped full
    # system to rounding, and the two steps agree up to the conditioning
    A, b = ref.normal_dense(lmbda)
    assert np.linalg.norm(A @ dg - b) <= 1e-9 * np.linalg.norm(b)
    cond = np.linalg.cond(A)
    assert np.linalg.norm(dg - dr) <= max(1e-10, 1e-15 * cond) * np.linalg.norm(dr), (
        np.linalg.norm(dg - dr) / np.linalg.norm(dr), cond)


def test_default_config_trajectory_matches_oracle(oracle):
    """LmConfig defaults (solver = cholesky) end to end: every iteration's
    cost, decision and damping against the oracle's exact solve."""
    s = bae.synthetic.config_scene("ladybug-49")
    gpu, ref = _pair(s, oracle)
    cfg = bae.LmConfig(max_iterations=20)
    rep = bae.optimize(gpu, s.poses, s.points, cfg)
    oracle.set_threads(8)
    oref = ref.optimize(cfg)
    assert len(rep.trajectory) == len(oref["trajectory"])
    assert rep.reason == bae.TerminationReason(oref["reason"])
    for a, b in zip(rep.trajectory, oref["trajectory"]):
        assert a.accepted == b["accepted"] and a.lmbda == b["lmbda"]
        # exact solves in different elimination orders (the oracle eliminates
        # points first, the GPU camera tiles in nested-dissection order) agree
        # to rounding amplified by the damped system's conditioning
        assert abs(a.cost - b["cost"]) <= 1e-8 * b["cost"], (a.iteration, a.cost, b["cost"])
    p7, p3 = gpu.get_parameters()
    assert np.abs(p3 - oref["points"]).max() <= 1e-7
    assert np.abs(p7 - oref["poses"]).max() <= 1e-7


@pytest.mark.parametrize("lmbda", [1e-6, 1e-1])
def test_tile_cholesky_step_many_tiles(oracle, lmbda):
    """Tile-sparse Cholesky with a banded, ring-closed tile pattern (C = 64
    cameras -> 8 tile columns, fill in the closing corner) against the
    oracle's damped full system."""
    s = _scene(C=64, P=500, N=2500, seed=12)
    gpu, ref = _pair(s, oracle)
    dg, iters, _ = gpu.solve_step(lmbda, bae.LmConfig())
    assert iters == 0
    A, b = ref.normal_dense(lmbda)
    assert np.linalg.norm(A @ dg - b) <= 1e-9 * np.linalg.norm(b)


@pytest.mark.parametrize("C,P,N", [(100, 2000, 9000), (257, 3000, 15000)])
def test_tile_cholesky_matches_dense_cusolver(monkeypatch, C, P, N):
    """The tile-sparse factorisation (default) and the dense cuSOLVER
    factorisation (BAE_DIRECT=cusolver) of the same reduced system agree."""
    s = _scene(C=C, P=P, N=N, seed=C)
    tile = bae.make_ba_problem(s.poses, s.points, s.intrinsics, s.observations)
    d_tile, _, _ = tile.solve_step(1e-4, bae.LmConfig())
    monkeypatch.setenv("BAE_DIRECT", "cusolver")
    dense = bae.make_ba_problem(s.poses, s.points, s.intrinsics, s.observations)
    d_dense, _, _ = dense.solve_step(1e-4, bae.LmConfig())
    assert np.linalg.norm(d_tile - d_dense) <= 1e-8 * np.linalg.norm(d_dense)


def _with_duplicates_and_singles(s, rng, ndup=40, nsingle=15):
    """Edge cases of the reference tests: duplicated (camera, point)
    observations (test_trace.cpp:296-311: independent identical rows), and
    points seen once (a rank-2 H_pp that only the clamp makes invertible,
    SURVEY.md 8a)."""
    ci, pi, px = s.cam_idx.copy(), s.pt_idx.copy(), s.pixels.copy()
    dup = rng.choice(ci.size, ndup, replace=False)
    ci = np.concatenate([ci, ci[dup]])
    pi = np.concatenate([pi, pi[dup]])
    px = np.concatenate([px, px[dup] + rng.normal(0, 0.5, (ndup, 2))])
    P = s.points.shape[0]
    new_pts = s.points[:nsingle] + 0.01
    cams = rng.integers(0, s.poses.shape[0], nsingle)
    ci = np.concatenate([ci, cams]).astype(np.int32)
    pi = np.concatenate([pi, P + np.arange(nsingle)]).astype(np.int32)
    px = np.concatenate([px, px[:nsingle]])
    return ci, pi, px, np.concatenate([s.points, new_pts])


@pytest.mark.parametrize("solver,lmbda", [("cholesky", 1e-4), ("cholesky", 1.0), ("pcg", 1e-4)])
def test_duplicates_and_single_observation_points(oracle, solver, lmbda):
    s = _scene(C=16, P=400, N=2000, seed=21)
    ci, pi, px, pts = _with_duplicates_and_singles(s, np.random.default_rng(5))
    gpu = bae.make_ba_problem(s.poses, pts, s.intrinsics, (ci, pi, px))
    ref = oracle.Problem(s.poses, pts, s.intrinsics, ci, pi, px)
    cfg = bae.LmConfig(solver=bae.SolverChoice[solver], pcg_tol=1e-13)
    dg, _, _ = gpu.solve_step(lmbda, cfg)
    A, b = ref.normal_dense(lmbda)
    assert np.linalg.norm(A @ dg - b) <= (1e-9 if solver == "cholesky" else 1e-8) * np.linalg.norm(b)
    r_gpu = gpu.evaluate()
    r_ref, _ = ref.evaluate()
    assert np.allclose(r_gpu, r_ref, rtol=1e-12, atol=1e-10)


def test_duplicates_lm_trajectory(oracle):
    s = _scene(C=16, P=400, N=2000, seed=22)
    ci, pi, px, pts = _with_duplicates_and_singles(s, np.random.default_rng(6))
    gpu = bae.make_ba_problem(s.poses, pts, s.intrinsics, (ci, pi, px))
    ref = oracle.Problem(s.poses, pts, s.intrinsics, ci, pi, px)
    cfg = bae.LmConfig(max_iterations=15)
    rep = bae.optimize(gpu, s.poses, pts, cfg)
    oref = ref.optimize(cfg)
    # decisions agree until the first near-tie (the points seen once make the
    # damped system ill-conditioned, so elimination-order rounding decides
    # ties at the plateau); the final costs agree to the north-star tolerance
    for a, b in zip(rep.trajectory, oref["trajectory"]):
        assert abs(a.cost - b["cost"]) <= 1e-8 * b["cost"], (a.iteration, a.cost, b["cost"])
        if abs(b["trial_cost"] - b["cost"]) <= 1e-6 * b["cost"]:
            break
        assert a.accepted == b["accepted"]
    assert abs(rep.final_cost - oref["final_cost"]) <= 1e-6 * oref["final_cost"]


def test_graph_replayed_iterations_match_plain_launches(monkeypatch):
    """The direct path's LM iterations replayed from captured CUDA graphs
    (damping from pinned memory, tile-Cholesky epoch on the device) give the
    same trajectory, bit for bit, as plain launches (BAE_LM_GRAPH=0)."""
    s = _scene(C=40, P=800, N=4000, seed=31)
    cfg = bae.LmConfig(max_iterations=12)
    runs = []
    for graph in ("1", "0"):
        monkeypatch.setenv("BAE_LM_GRAPH", graph)
        gpu = bae.make_ba_problem(s.poses, s.points, s.intrinsics, s.observations)
        rep = bae.optimize(gpu, s.poses, s.points, cfg)
        rep2 = bae.optimize(gpu, s.poses, s.points, cfg)  # replays the same graphs again
        runs.append((rep, rep2, gpu.get_parameters()))
    (a, a2, pa), (b, b2, pb) = runs
    for x, y in ((a, b), (a2, b2), (a, a2)):
        assert [(r.cost, r.lmbda, r.accepted) for r in x.trajectory] == \
               [(r.cost, r.lmbda, r.accepted) for r in y.trajectory]
    assert np.array_equal(pa[0], pb[0]) and np.array_equal(pa[1], pb[1])


@pytest.mark.parametrize("graph", ["1", "0"])
def test_fused_linearize_prep_matches_separate_passes(monkeypatch, graph):
    """After an accepted step the linearisation and the direct prep run as one
    pass (k_lin_prep + k_cam_lin_prep); the trajectory and the parameters are
    bit for bit those of the separate k_linearize / k_prep passes
    (BAE_LIN_PREP=0), with and without the captured LM graphs."""
    s = _scene(C=40, P=800, N=4000, seed=32)
    cfg = bae.LmConfig(max_iterations=10)
    monkeypatch.setenv("BAE_LM_GRAPH", graph)
    runs = []
    for fuse in ("1", "0"):
        monkeypatch.setenv("BAE_LIN_PREP", fuse)
        gpu = bae.make_ba_problem(s.poses, s.points, s.intrinsics, s.observations)
        rep = bae.optimize(gpu, s.poses, s.points, cfg)
        runs.append((rep, gpu.get_parameters()))
    (a, pa), (b, pb) = runs
    assert sum(r.accepted for r in a.trajectory) >= 2
    assert [(r.cost, r.lmbda, r.accepted) for r in a.trajectory] == \
           [(r.cost, r.lmbda, r.accepted) for r in b.trajectory]
    assert np.array_equal(pa[0], pb[0]) and np.array_equal(pa[1], pb[1])


def test_time_kernel_fused_lin_prep():
    s = _scene(C=20, P=300, N=1500, seed=33)
    gpu = bae.make_ba_problem(s.poses, s.points, s.intrinsics, s.observations)
    assert gpu.time_kernel(7, 2) > 0.0


def test_chol_update_helpers_are_bitwise_neutral(monkeypatch):
    """Tile-Cholesky update helpers (other CTAs pre-apply a tile's updates
    from all but the last contributing column, same order) leave the
    trajectory and the parameters bit for bit unchanged (BAE_CHOL_HELP=0:
    every update on the column's own CTA)."""
    s = bae.synthetic.config_scene("trafalgar-257")
    cfg = bae.LmConfig(max_iterations=6)
    runs = []
    for h in ("1", "0"):  # 1: a helper for every tile with an early update
        monkeypatch.setenv("BAE_CHOL_HELP", h)
        gpu = bae.make_ba_problem(s.poses, s.points, s.intrinsics, s.observations)
        rep = bae.optimize(gpu, s.poses, s.points, cfg)
        runs.append((rep, gpu.get_parameters()))
    (a, pa), (b, pb) = runs
    assert [(r.cost, r.lmbda, r.accepted) for r in a.trajectory] == \
           [(r.cost, r.lmbda, r.accepted) for r in b.trajectory]
    assert np.array_equal(pa[0], pb[0]) and np.array_equal(pa[1], pb[1])


@pytest.mark.parametrize("dups", [False, True])
def test_normal_matrix_patterns_bit_exact(oracle, dups):
    """The normal matrix's index structure, bit-exact: the four quadrant
    block patterns of spgemm_symbolic (spgemm.hpp:33-81; CL = the unique
    (camera, point) pairs, duplicates merged) and the scalar CSR pattern of
    build_csr_pattern (assemble.hpp:135-177), against the device's
    observation decomposition (tile_obs=64: many tiles). With duplicated
    observations and points seen once (test_trace.cpp:296-311)."""
    s = _scene(C=20, P=500, N=2600, seed=41)
    if dups:
        ci, pi, px, pts = _with_duplicates_and_singles(s, np.random.default_rng(41))
        gpu = bae.make_ba_problem(s.poses, pts, s.intrinsics, (ci, pi, px), tile_obs=64)
        ref = oracle.Problem(s.poses, pts, s.intrinsics, ci, pi, px)
    else:
        gpu, ref = _pair(s, oracle, tile_obs=64)
    for which in range(5):
        rg, cg = gpu.normal_pattern(which)
        rr, cr = ref.normal_pattern(which)
        assert np.array_equal(rg, rr), which
        assert np.array_equal(cg, cr), which
    # the Jacobian's row pointers come from the device decomposition too
    jg = gpu.jacobian()
    assert np.array_equal(jg.j_pose.row_ptr, np.arange(gpu.residual_rows() + 1))


@pytest.mark.parametrize("graph", ["1", "0"])
@pytest.mark.parametrize("solver", ["cholesky", "pcg"])
def test_not_spd_rejections_end_in_solver_failure(oracle, monkeypatch, graph, solver):
    """lm.hpp:146-152 and :234-237. A clamp ceiling of 1e-12 (assemble.hpp:94-101)
    leaves every damped system indefinite: each solve fails (NotSpdError in the
    reference's Cholesky; the device's point-block or tile factorisation flags
    it), the step is rejected, lambda doubles, and the first rejection at
    lambda >= damping_max ends the run as solver_failure -- the oracle's exact
    trajectory, with plain launches and with the captured LM graphs."""
    monkeypatch.setenv("BAE_LM_GRAPH", graph)
    s = _scene(C=8, P=120, N=500, seed=51)
    gpu, ref = _pair(s, oracle)
    cfg = bae.LmConfig(max_iterations=40, damping_max=1e-3, clamp_min=1e-12, clamp_max=1e-12,
                       solver=bae.SolverChoice[solver])
    rep = bae.optimize(gpu, s.poses, s.points, cfg)
    oref = ref.optimize(bae.LmConfig(max_iterations=40, damping_max=1e-3, clamp_min=1e-12, clamp_max=1e-12))
    assert oref["reason"] == int(bae.TerminationReason.solver_failure)
    assert rep.reason == bae.TerminationReason.solver_failure
    assert rep.iterations == oref["iterations"] == 11  # 1e-6 * 2^10 >= 1e-3
    for a, b in zip(rep.trajectory, oref["trajectory"]):
        assert not a.accepted or a.iteration == 0
        assert a.lmbda == b["lmbda"] and a.cost == pytest.approx(b["cost"], rel=1e-12)
    p7, p3 = gpu.get_parameters()
    assert np.array_equal(p7, s.poses) and np.array_equal(p3, s.points)  # rejections restore (test_optim.cpp:110-125)


@pytest.mark.parametrize("solver", ["cholesky", "pcg"])
def test_not_spd_until_damping_recovers(oracle, solver):
    """Diagonal entries clamped to at most 1 (assemble.hpp:94-101): the damped
    system is indefinite until (1 + lambda) outgrows the off-diagonal blocks,
    so LM rejects (NotSpd) for dozens of iterations, accepts, halves lambda,
    and is rejected again -- the accept / lambda sequence equals the oracle's
    exact-solve trajectory step for step."""
    s = _scene(C=8, P=120, N=500, seed=52)
    gpu, ref = _pair(s, oracle)
    kw = dict(max_iterations=50, clamp_max=1.0)
    rep = bae.optimize(gpu, s.poses, s.points,
                       bae.LmConfig(solver=bae.SolverChoice[solver], pcg_tol=1e-12, **kw))
    oref = ref.optimize(bae.LmConfig(**kw))
    acc = [r.accepted for r in rep.trajectory[1:]]
    assert acc[:10] == [False] * 10 and any(acc)
    assert len(rep.trajectory) == len(oref["trajectory"])
    for a, b in zip(rep.trajectory, oref["trajectory"]):
        assert a.accepted == b["accepted"] and a.lmbda == b["lmbda"], a.iteration
        assert abs(a.cost - b["cost"]) <= 1e-6 * b["cost"]
