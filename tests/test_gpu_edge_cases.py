"""Edge cases of make_ba_problem / optimize against the oracle on the same
inputs (problems.hpp:87-136, csr.hpp:41-53, lm.hpp:205-255):

* no observations: invalid_argument at construction;
* a camera or a point that no observation references: the normal matrix has
  no diagonal entry for it, optimize raises invalid_argument ("diagonal op:
  missing diagonal entry") on both solvers, while evaluate still works;
* a single camera and a single point with repeated observations (the
  smallest well-posed-in-damping problem) and max_iterations = 0 (the report
  is the initial cost, no step): the same trajectory as the oracle."""
import numpy as np
import pytest

import paper_2409_12190_b200 as bae


def _scene(C=6, P=60, N=300, seed=3):
    return bae.synthetic.bal_shaped(C, P, N, seed=seed)


def _both(s, cam, pt, px, oracle):
    gpu = bae.make_ba_problem(s.poses, s.points, s.intrinsics, (cam, pt, px), device=0)
    ref = oracle.Problem(s.poses, s.points, s.intrinsics, cam, pt, px)
    return gpu, ref


@pytest.mark.gpu
def test_no_observations_is_invalid(oracle):
    s = _scene()
    with pytest.raises(ValueError, match="no observations"):
        bae.make_ba_problem(s.poses, s.points, s.intrinsics,
                            (np.zeros(0, np.int32), np.zeros(0, np.int32), np.zeros((0, 2))), device=0)
    with pytest.raises(oracle.OracleError, match="no observations"):
        oracle.Problem(s.poses, s.points, s.intrinsics, np.zeros(0, np.int32), np.zeros(0, np.int32),
                       np.zeros((0, 2)))


@pytest.mark.gpu
@pytest.mark.parametrize("what", ["camera", "point"])
@pytest.mark.parametrize("solver", [bae.SolverChoice.cholesky, bae.SolverChoice.pcg])
def test_unobserved_camera_or_point_has_no_diagonal(oracle, what, solver):
    s = _scene()
    cam, pt, px = s.cam_idx.copy(), s.pt_idx.copy(), s.pixels.copy()
    keep = (cam != 2) if what == "camera" else (pt != 7)
    cam, pt, px = cam[keep], pt[keep], px[keep]
    gpu, ref = _both(s, cam, pt, px, oracle)
    r_gpu = gpu.evaluate()
    r_ref, _ = ref.evaluate()
    np.testing.assert_allclose(r_gpu, r_ref, rtol=1e-12, atol=1e-9)
    cfg = bae.LmConfig(max_iterations=3, solver=solver)
    with pytest.raises(ValueError, match="missing diagonal"):
        bae.optimize(gpu, s.poses, s.points, cfg)
    with pytest.raises(oracle.OracleError, match="missing diagonal"):
        ref.optimize(cfg)


@pytest.mark.gpu
@pytest.mark.parametrize("solver", [bae.SolverChoice.cholesky, bae.SolverChoice.pcg])
def test_single_camera_single_point(oracle, solver):
    s = _scene(C=1, P=1, N=1, seed=5)
    reps = 4  # the same observation four times: independent rows (test_problems duplicate rule)
    cam = np.repeat(s.cam_idx, reps)
    pt = np.repeat(s.pt_idx, reps)
    px = np.repeat(s.pixels, reps, axis=0) + 0.25 * np.arange(reps)[:, None]
    gpu, ref = _both(s, cam, pt, px, oracle)
    cfg = bae.LmConfig(max_iterations=6, solver=solver, pcg_tol=1e-12)
    rep = bae.optimize(gpu, s.poses, s.points, cfg)
    oref = ref.optimize(cfg)
    assert [r.accepted for r in rep.trajectory] == [r["accepted"] for r in oref["trajectory"]]
    for a, b in zip(rep.trajectory, oref["trajectory"]):
        assert abs(a.cost - b["cost"]) <= 1e-6 * abs(b["cost"]) + 1e-12


@pytest.mark.gpu
@pytest.mark.parametrize("solver", [bae.SolverChoice.cholesky, bae.SolverChoice.pcg])
def test_zero_iterations_reports_the_initial_cost(oracle, solver):
    s = _scene()
    gpu, ref = _both(s, s.cam_idx, s.pt_idx, s.pixels, oracle)
    cfg = bae.LmConfig(max_iterations=0, solver=solver)
    rep = bae.optimize(gpu, s.poses, s.points, cfg)
    oref = ref.optimize(cfg)
    assert rep.iterations == oref["iterations"] == 0
    assert rep.reason == bae.TerminationReason(oref["reason"])
    assert abs(rep.final_cost - oref["final_cost"]) <= 1e-10 * abs(oref["final_cost"])
