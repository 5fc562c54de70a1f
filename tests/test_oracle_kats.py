"""Pin the CPU oracle with the reference's own unit-test expectations
(SURVEY.md 8c): each test cites the reference test it restates. Inputs come
from the restated make_random_ba / synth_ba driven by the reference RNG."""
import math

import numpy as np
import pytest

from paper_2409_12190_b200.api import LmConfig, SolverChoice

IDENT = np.array([0, 0, 0, 0, 0, 0, 1.0])


# ---- projection KATs (test_problems.cpp:20-68) -----------------------------
def test_pinhole_project_kats(oracle):
    k = np.array([200, 200, 100, 100.0])
    assert np.array_equal(oracle.pinhole_project(IDENT, [0, 0, 1], k), [100.0, 100.0])
    assert np.array_equal(oracle.pinhole_project(IDENT, [0.5, 0, 1], k), [200.0, 100.0])
    with pytest.raises(oracle.OracleError) as e:
        oracle.pinhole_project(IDENT, [0, 0, -1], k)
    assert e.value.code == 3


def test_bal_project_kats(oracle):
    a = oracle.bal_project(IDENT, [0, 0, -1], [100, 0, 0])
    assert a[0] == 0.0 and a[1] == 0.0
    b = oracle.bal_project(IDENT, [0.1, 0, -1], [100, 0, 0])
    assert b[0] == 10.0 and b[1] == 0.0
    c = oracle.bal_project(IDENT, [0.1, 0, -1], [100, 0.1, 0])
    assert abs(c[0] - 10.01) <= 1e-12 and c[1] == 0.0
    with pytest.raises(oracle.OracleError) as e:
        oracle.bal_project(IDENT, [0.1, 0, 0], [100, 0, 0])
    assert e.value.code == 3


def test_bal_matches_pinhole_through_axis_flip(oracle):
    rng = oracle.Rng(41)
    for _ in range(50):
        x = rng.uniform(-1, 1)
        y = rng.uniform(-1, 1)
        z = rng.uniform(-4, -1)
        a = oracle.bal_project(IDENT, [x, y, z], [170.0, 0, 0])
        b = oracle.pinhole_project(IDENT, [x, y, -z], [170.0, 170.0, 0, 0])
        assert np.linalg.norm(a - b) < 1e-12


# ---- residuals (test_problems.cpp:70-110) ----------------------------------
def _scalar_residuals(oracle, d):
    r = []
    for c, pt, px in zip(d["cam_idx"], d["pt_idx"], d["pixels"]):
        if d["pinhole"]:
            pr = oracle.pinhole_project(d["poses"][c], d["points"][pt], d["intrinsics"][c])
        else:
            pr = oracle.bal_project(d["poses"][c], d["points"][pt], d["intrinsics"][c])
        r.extend([pr[0] - px[0], pr[1] - px[1]])
    return np.array(r)


def test_perfect_scene_is_zero(oracle):
    rng = oracle.Rng(42)
    d = oracle.make_random_ba(rng, 3, 12, True)
    for i, (c, pt) in enumerate(zip(d["cam_idx"], d["pt_idx"])):
        d["pixels"][i] = oracle.pinhole_project(d["poses"][c], d["points"][pt], d["intrinsics"][c])
    r, cost = oracle.Problem.from_dict(d).evaluate()
    assert np.all(r == 0.0) and cost == 0.0


def test_residual_matches_scalar_loop(oracle):
    rng = oracle.Rng(43)
    for trial in range(20):
        pin = trial % 2 == 0
        d = oracle.make_random_ba(rng, 1 + rng.index(4), 1 + rng.index(15), pin)
        r, _ = oracle.Problem.from_dict(d).evaluate()
        ref = _scalar_residuals(oracle, d)
        assert np.all(np.abs(r - ref) <= 1e-12 * np.maximum(1.0, np.abs(ref)))


def test_input_validation(oracle):
    rng = oracle.Rng(44)
    d = oracle.make_random_ba(rng, 2, 4, True)
    bad = dict(d)
    bad["pt_idx"] = d["pt_idx"].copy()
    bad["pt_idx"][0] = 99
    with pytest.raises(oracle.OracleError) as e:
        oracle.Problem.from_dict(bad)
    assert e.value.code == 2 and e.value.index == 0
    empty = dict(d, cam_idx=d["cam_idx"][:0], pt_idx=d["pt_idx"][:0], pixels=d["pixels"][:0])
    with pytest.raises(oracle.OracleError) as e:
        oracle.Problem.from_dict(empty)
    assert e.value.code == 1


# ---- Jacobian (test_trace.cpp:192-324; oracles.hpp:80-112) -----------------
def _fd_jacobians(oracle, d, h=1e-6):
    prob = oracle.Problem.from_dict(d)
    C, P = d["poses"].shape[0], d["points"].shape[0]
    N = len(d["cam_idx"])
    jp = np.zeros((2 * N, 6 * C))
    jl = np.zeros((2 * N, 3 * P))
    for c in range(C):
        for t in range(6):
            e = np.zeros(6)
            e[t] = h
            pp, pm = d["poses"].copy(), d["poses"].copy()
            pp[c] = oracle.se3_retract(d["poses"][c], e)
            pm[c] = oracle.se3_retract(d["poses"][c], -e)
            rp, _ = prob.evaluate(pp, d["points"])
            rm, _ = prob.evaluate(pm, d["points"])
            jp[:, 6 * c + t] = (rp - rm) / (2 * h)
    for p_ in range(P):
        for t in range(3):
            xp, xm = d["points"].copy(), d["points"].copy()
            xp[p_, t] += h
            xm[p_, t] -= h
            rp, _ = prob.evaluate(d["poses"], xp)
            rm, _ = prob.evaluate(d["poses"], xm)
            jl[:, 3 * p_ + t] = (rp - rm) / (2 * h)
    return jp, jl


def _dense(vals, cols, ncols, bc):
    N = vals.shape[0]
    m = np.zeros((2 * N, ncols * bc))
    for k in range(N):
        m[2 * k:2 * k + 2, bc * cols[k]:bc * cols[k] + bc] = vals[k]
    return m


def _rel_err(a, b):  # oracles.hpp:192-195
    scale = max(1e-12, np.abs(a).max(), np.abs(b).max())
    return np.abs(a - b).max() / scale


def test_gather_pattern_for_ba_toy(oracle):
    rng = oracle.Rng(8)
    d = oracle.make_random_ba(rng, 2, 3, True, 1.1)
    d["cam_idx"] = np.array([0, 0, 1], np.int32)
    d["pt_idx"] = np.array([0, 1, 2], np.int32)
    d["pixels"] = np.zeros((3, 2))
    j = oracle.Problem.from_dict(d).jacobian()
    assert list(j["pose_col"]) == [0, 0, 1]
    assert list(j["point_col"]) == [0, 1, 2]
    assert list(np.diff(j["pose_row_ptr"])) == [1, 1, 1]
    jp, jl = _fd_jacobians(oracle, d)
    assert _rel_err(_dense(j["j_pose"], j["pose_col"], 2, 6), jp) < 1e-6
    assert _rel_err(_dense(j["j_point"], j["point_col"], 3, 3), jl) < 1e-6


@pytest.mark.parametrize("seed", [10, 101])
def test_random_instances_both_models_fd(oracle, seed):
    rng = oracle.Rng(seed)
    for trial in range(10):
        pin = trial % 2 == 0
        C, P = 1 + rng.index(5), 1 + rng.index(20)
        d = oracle.make_random_ba(rng, C, P, pin)
        j = oracle.Problem.from_dict(d).jacobian()
        jp, jl = _fd_jacobians(oracle, d)
        assert _rel_err(_dense(j["j_pose"], j["pose_col"], C, 6), jp) < 1e-6
        assert _rel_err(_dense(j["j_point"], j["point_col"], P, 3), jl) < 1e-6


def test_duplicate_observations_give_independent_rows(oracle):
    rng = oracle.Rng(13)
    d = oracle.make_random_ba(rng, 1, 2, True, 1.1)
    for k in ("cam_idx", "pt_idx", "pixels"):
        d[k] = np.concatenate([d[k], d[k][:1]])
    j = oracle.Problem.from_dict(d).jacobian()
    N = len(d["cam_idx"])
    assert j["j_pose"].shape[0] == N
    assert np.array_equal(j["j_pose"][N - 1], j["j_pose"][0])


# ---- damped system (test_optim.cpp:155-191) ---------------------------------
def test_damped_system_equals_clamp_then_scale(oracle):
    rng = oracle.Rng(35)
    d = oracle.make_random_ba(rng, 1, 6, True)
    prob = oracle.Problem.from_dict(d)
    j = prob.jacobian()
    C, P = 1, 6
    J = np.hstack([_dense(j["j_pose"], j["pose_col"], C, 6), _dense(j["j_point"], j["point_col"], P, 3)])
    r, _ = prob.evaluate()
    lam = 0.37
    A = J.T @ J
    for i in range(A.shape[0]):
        A[i, i] = min(max(A[i, i], 1e-6), 1e32) * (1.0 + lam)
    Ad, bd = prob.normal_dense(lam)
    assert np.allclose(Ad, A, rtol=1e-13, atol=1e-12 * np.abs(A).max())
    assert np.allclose(bd, -J.T @ r, rtol=1e-12, atol=1e-12 * np.abs(bd).max())
    x, _ = prob.solve_step(lam, LmConfig())
    assert np.linalg.norm(Ad @ x - bd) / np.linalg.norm(bd) < 1e-10


# ---- LM semantics (test_optim.cpp:59-153, 263-323) --------------------------
def test_linear_residual_one_undamped_step(oracle):
    sp = oracle.ScalarProblem(0, [1.5, -2.0, 0.25])
    sp.begin([1.5, -2.0, 0.25], 0.0)
    assert sp.step(LmConfig(initial_damping=0.0, damping_min=0.0))
    st = sp.state()
    assert np.array_equal(st["points"][0], [0, 0, 0])
    assert st["history"][-1] == 0.0


def test_quadratic_matches_scalar_oracle(oracle):
    cfg = LmConfig(max_iterations=20)
    sp = oracle.ScalarProblem(1, [1, 1, 1])
    sp.begin([1, 1, 1], cfg.initial_damping)
    theta, lam, acc_steps = 1.0, cfg.initial_damping, 0
    for it in range(12):
        accepted = sp.step(cfg)
        r = theta * theta - 2.0
        jac = 2.0 * theta
        damped = min(max(jac * jac, 1e-6), 1e32) * (1.0 + lam)
        trial = theta + (-jac * r / damped)
        if 3.0 * (trial * trial - 2.0) ** 2 < 3.0 * r * r:
            theta, lam = trial, max(lam * 0.5, cfg.damping_min)
            assert accepted, it
            acc_steps += 1
        else:
            lam = min(lam * 2.0, cfg.damping_max)
            assert not accepted, it
        assert abs(sp.state()["points"][0, 0] - theta) <= 1e-10 * abs(theta)
        if acc_steps >= 8:
            break
    pts = sp.state()["points"][0]
    assert abs(pts[0] - math.sqrt(2)) <= 1e-8 and abs(pts[2] - math.sqrt(2)) <= 1e-8


def test_rejected_step_restores_state_bitwise(oracle):
    cfg = LmConfig()
    sp = oracle.ScalarProblem(1, [0.1, 0.1, 0.1])
    sp.begin([0.1, 0.1, 0.1], cfg.initial_damping)
    assert not sp.step(cfg)
    st = sp.state()
    assert np.array_equal(st["points"][0], [0.1, 0.1, 0.1])
    assert len(st["history"]) == 1 and st["rejected"] == 1
    assert st["lmbda"] == cfg.initial_damping * cfg.damping_up


def test_optimize_termination_rules(oracle):
    rep = oracle.ScalarProblem(0, [0, 0, 0]).optimize(LmConfig(), [0, 0, 0])
    assert rep["iterations"] == 1 and rep["final_cost"] == 0.0 and rep["reason"] == 0
    assert len(rep["trajectory"]) == 2
    rep = oracle.ScalarProblem(1, [1, 1, 1]).optimize(LmConfig(max_iterations=6), [1, 1, 1])
    assert len(rep["trajectory"]) == rep["iterations"] + 1 and rep["trajectory"][0]["cost"] == 3.0
    rep = oracle.ScalarProblem(1, [1, 1, 1]).optimize(LmConfig(max_iterations=3), [1, 1, 1])
    assert rep["reason"] == 1 and rep["iterations"] == 3
    rep = oracle.ScalarProblem(2, [0, 0, 0]).optimize(LmConfig(max_iterations=2000, damping_max=1e4), [0, 0, 0])
    assert rep["reason"] == 2


def test_stop_on_plateau_spec_and_scalar_reference(oracle):
    cfg = LmConfig(max_iterations=100)
    assert not oracle.stop_on_plateau([10, 9, 8], cfg)
    st = [10.0]
    for _ in range(3):
        st.append(st[-1] * (1.0 - 1e-9))
    assert oracle.stop_on_plateau(st, cfg)
    assert oracle.stop_on_plateau([10, 9, 8], LmConfig(max_iterations=3))
    with pytest.raises(oracle.OracleError):
        oracle.stop_on_plateau([], cfg)
    rng = oracle.Rng(34)
    cfg = LmConfig(max_iterations=1000)
    for _ in range(50):
        h = [100.0]
        for _ in range(2 + rng.index(12)):
            drop = rng.uniform(0.0, 0.3) if rng.uniform() < 0.5 else rng.uniform(0.0, 1e-7)
            h.append(h[-1] * (1.0 - drop))
        exp = len(h) > 3 and all((h[i - 1] - h[i]) / h[i - 1] < 1e-6 for i in range(len(h) - 3, len(h)))
        assert oracle.stop_on_plateau(h, cfg) == exp


# ---- end-to-end BA (test_optim.cpp:34-55, 193-261; acceptance.cpp:249-272) --
def _synthetic_pinhole(oracle, seed, cams, pts, pose_sigma, pixel_sigma):
    rng = oracle.Rng(seed)
    d = oracle.make_random_ba(rng, cams, pts, True, 1.1)
    for i, (c, p_) in enumerate(zip(d["cam_idx"], d["pt_idx"])):
        px = oracle.pinhole_project(d["poses"][c], d["points"][p_], d["intrinsics"][c])
        d["pixels"][i] = px + pixel_sigma * np.array([rng.normal(), rng.normal()])
    init = np.array([oracle.se3_retract(pp, pose_sigma * np.array([rng.normal() for _ in range(6)]))
                     for pp in d["poses"]])
    return d, init


def test_synthetic_ba_converges_to_machine_zero(oracle):
    d, init = _synthetic_pinhole(oracle, 31, 3, 50, 0.05, 0.0)
    prob = oracle.Problem(init, d["points"], d["intrinsics"], d["cam_idx"], d["pt_idx"], d["pixels"], pinhole=True)
    rep = prob.optimize(LmConfig(max_iterations=20))
    assert rep["final_mse"] < 1e-10
    acc = [t["cost"] for t in rep["trajectory"] if t["accepted"]]
    assert all(b < a for a, b in zip(acc, acc[1:]))


def test_cholesky_and_pcg_agree(oracle):
    d, init = _synthetic_pinhole(oracle, 33, 3, 30, 0.05, 0.5)
    out = []
    for solver in (SolverChoice.cholesky, SolverChoice.pcg):
        prob = oracle.Problem(init, d["points"], d["intrinsics"], d["cam_idx"], d["pt_idx"], d["pixels"], pinhole=True)
        out.append(prob.optimize(LmConfig(max_iterations=15, solver=solver, pcg_tol=1e-10))["final_cost"])
    assert abs(out[0] - out[1]) / out[0] <= 1e-6


def test_acceptance_synthetic_ba(oracle):
    d = oracle.synth_ba(3, 50, 0.0, 0.05, 7)
    rep = oracle.Problem.from_dict(d).optimize(LmConfig(max_iterations=20))
    assert rep["final_mse"] < 1e-10
    d = oracle.synth_ba(3, 50, 1.0, 0.05, 9)
    rep = oracle.Problem.from_dict(d).optimize(LmConfig(max_iterations=50))
    assert 0.5 <= rep["final_mse"] <= 2.0


# --- Philox4x32-10 (row f4's on-device generator) ------------------------------
# Known answers of the published algorithm (Random123 kat_vectors).
@pytest.mark.parametrize("ctr,key,want", [
    ([0, 0, 0, 0], [0, 0], [0x6627e8d5, 0xe169c58d, 0xbc57ac4c, 0x9b00dbd8]),
    ([0xffffffff] * 4, [0xffffffff] * 2, [0x408f276d, 0x41c83b0e, 0xa20bc7c6, 0x6d5451fd]),
    ([0x243f6a88, 0x85a308d3, 0x13198a2e, 0x03707344], [0xa4093822, 0x299f31d0],
     [0xd16cfe09, 0x94fdcceb, 0x5001e420, 0x24126ea1]),
])
def test_philox_known_answers(oracle, ctr, key, want):
    assert oracle.philox4x32_10(ctr, key) == want


def test_philox_scene_shape(oracle):
    """The restated device generator: exactly N observations, camera-major
    with points ascending, no duplicate (camera, point), every point's
    cameras inside a window of min(C, 16), BAL-shaped counts."""
    C, P, N = 40, 300, 1237
    s = oracle.synth_bal_shaped_philox(C, P, N, 40)
    ci, pi = s["cam_idx"], s["pt_idx"]
    key = ci.astype(np.int64) * P + pi
    assert np.all(np.diff(key) > 0)  # camera-major, points ascending, no duplicates
    counts = np.bincount(pi, minlength=P)
    assert counts.sum() == N and counts.min() == N // P and counts.max() == N // P + 1
    for j in range(P):
        cams = ci[pi == j]
        assert any(max((c - a) % C for c in cams) < 16 for a in cams)  # inside some window of 16
    assert np.all(np.abs(s["true_points"]) <= 0.5)
    assert np.all(np.abs(s["intrinsics"][:, 1]) <= 0.1) and np.all(np.abs(s["intrinsics"][:, 2]) <= 0.01)
    b = oracle.synth_bal_shaped_philox(C, P, N, 40)
    assert all(np.array_equal(s[k], b[k]) for k in s)  # deterministic


def test_oracle_normal_patterns_against_numpy(oracle):
    """The oracle's spgemm_symbolic quadrant patterns (spgemm.hpp:33-81) and
    scalar CSR pattern (assemble.hpp:135-177) against a numpy derivation from
    the observation list, duplicates included (test_trace.cpp:296-311)."""
    rng = oracle.Rng(17)
    d = oracle.make_random_ba(rng, 5, 30, False, keep=0.5)
    ci = np.concatenate([d["cam_idx"], d["cam_idx"][:7]])
    pi = np.concatenate([d["pt_idx"], d["pt_idx"][:7]])
    px = np.concatenate([d["pixels"], d["pixels"][:7]])
    prob = oracle.Problem(d["poses"], d["points"], d["intrinsics"], ci, pi, px)
    C, P = 5, 30
    pairs = sorted(set(zip(ci.tolist(), pi.tolist())))
    rp, col = prob.normal_pattern(1)
    assert [(c, int(col[k])) for c in range(C) for k in range(rp[c], rp[c + 1])] == pairs
    rp, col = prob.normal_pattern(2)
    assert sorted((int(col[k]), p) for p in range(P) for k in range(rp[p], rp[p + 1])) == pairs
    dense = np.zeros((6 * C + 3 * P, 6 * C + 3 * P), bool)
    for c, p in pairs:
        dense[6 * c:6 * c + 6, 6 * c:6 * c + 6] = True
        dense[6 * c:6 * c + 6, 6 * C + 3 * p:6 * C + 3 * p + 3] = True
        dense[6 * C + 3 * p:6 * C + 3 * p + 3, 6 * c:6 * c + 6] = True
        dense[6 * C + 3 * p:6 * C + 3 * p + 3, 6 * C + 3 * p:6 * C + 3 * p + 3] = True
    rp, col = prob.normal_pattern(4)
    got = np.zeros_like(dense)
    for r in range(dense.shape[0]):
        assert np.all(np.diff(col[rp[r]:rp[r + 1]]) > 0)
        got[r, col[rp[r]:rp[r + 1]]] = True
    assert np.array_equal(got, dense)
