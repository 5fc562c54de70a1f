"""Row f3: the pinhole camera variant of make_ba_problem
(PinholeIntrinsics, camera.hpp:17-46) on the B200 path, against the oracle on
the reference's own random instances (tests/oracles.hpp:26-61): residuals and
Jacobian blocks at 1e-12, LM trajectories with both solvers, cheirality."""
import numpy as np
import pytest

import paper_2409_12190_b200 as bae

pytestmark = pytest.mark.gpu


def _instance(oracle, seed, C=8, P=150):
    return oracle.make_random_ba(oracle.Rng(seed), C, P, True)


def _pair(inst, oracle):
    gpu = bae.make_ba_problem(inst["poses"], inst["points"], inst["intrinsics"],
                              (inst["cam_idx"], inst["pt_idx"], inst["pixels"]))
    ref = oracle.Problem(inst["poses"], inst["points"], inst["intrinsics"], inst["cam_idx"], inst["pt_idx"],
                         inst["pixels"], pinhole=True)
    return gpu, ref


def _blocks_match(a, b, tol):  # acceptance.cpp:51-62
    scale = np.maximum(1.0, np.abs(b).reshape(b.shape[0], -1).max(axis=1))
    err = np.abs(a - b).reshape(a.shape[0], -1).max(axis=1)
    return bool(np.all(err <= tol * scale)), float((err / scale).max())


@pytest.mark.parametrize("seed", [1, 2])
def test_pinhole_residual_and_jacobian(oracle, seed):
    inst = _instance(oracle, seed)
    assert inst["intrinsics"].shape[1] == 4
    gpu, ref = _pair(inst, oracle)
    r_ref, c_ref = ref.evaluate()
    assert np.allclose(gpu.evaluate(), r_ref, rtol=1e-12, atol=1e-10)
    jg, jr = gpu.jacobian(), ref.jacobian()
    ok, worst = _blocks_match(jg.j_pose.values, jr["j_pose"], 1e-12)
    assert ok, worst
    ok, worst = _blocks_match(jg.j_point.values, jr["j_point"], 1e-12)
    assert ok, worst
    assert np.array_equal(jg.j_point.col_idx, jr["point_col"])


@pytest.mark.parametrize("solver", ["cholesky", "pcg"])
def test_pinhole_lm_trajectory(oracle, solver):
    inst = _instance(oracle, 3)
    gpu, ref = _pair(inst, oracle)
    cfg = bae.LmConfig(max_iterations=12, solver=bae.SolverChoice[solver], pcg_tol=1e-12)
    rep = bae.optimize(gpu, inst["poses"], inst["points"], cfg)
    o = ref.optimize(bae.LmConfig(max_iterations=12))  # reference default: exact Cholesky
    n = min(len(rep.trajectory), len(o["trajectory"]))
    assert n >= 4
    tol = 1e-8 if solver == "cholesky" else 1e-6
    for a, b in zip(rep.trajectory[:n], o["trajectory"][:n]):
        assert a.accepted == b["accepted"] and a.lmbda == b["lmbda"]
        assert abs(a.cost - b["cost"]) <= tol * b["cost"], (a.iteration, a.cost, b["cost"])
    p7, p3 = gpu.get_parameters()
    assert np.abs(p3 - o["points"]).max() <= 1e-5 * max(1.0, np.abs(o["points"]).max())


def test_pinhole_cheirality(oracle):
    inst = _instance(oracle, 4, C=4, P=40)
    pts = inst["points"].copy()
    k = 17
    c, p = int(inst["cam_idx"][k]), int(inst["pt_idx"][k])
    R = oracle.quat_matrix(inst["poses"][c, 3:])
    pts[p] = R.T @ (np.array([0.1, 0.2, -1.0]) - inst["poses"][c, :3])  # behind camera c
    with pytest.raises(bae.CheiralityError) as e:
        bae.make_ba_problem(inst["poses"], pts, inst["intrinsics"], (inst["cam_idx"], inst["pt_idx"], inst["pixels"]))
    assert "behind camera" in str(e.value)
    with pytest.raises(oracle.OracleError) as eo:
        oracle.Problem(inst["poses"], pts, inst["intrinsics"], inst["cam_idx"], inst["pt_idx"], inst["pixels"],
                       pinhole=True)
    assert e.value.observation == eo.value.index
