"""GPU-vs-oracle parity at the BASELINE.json configs the bench reports
(SURVEY.md 8c parity protocol, steps 3-4).

The scenes are the bench's own: the host generator with seed = camera count
(checked bit for bit against the oracle's restatement in
tests/test_generator_oracle.py). The comparator is the oracle's exact solve
(LmConfig defaults: Cholesky, lm.hpp:34), the precedent being the
reference's acceptance run of Trafalgar / Dubrovnik with 50 Cholesky
iterations (acceptance.cpp:276-329) and its Cholesky-vs-PCG agreement test
(test_optim.cpp:245-261). Per LM iteration, up to the first near-tie of the
accept test `new_cost < cost` (lm.hpp:183; a trial within 1e-6 relative of
the current cost, where the two elimination orders may decide differently):

* cost within 1e-6 relative (north star);
* gradient norm ||J^T r|| (b of assemble.hpp:75-83) within 1e-6 relative
  (up to the first near-tie; costs and decisions are compared past it for as
  long as the decisions agree);
* accept / reject and lambda identical.

Then the final cost within 1e-6 and the final parameters within 1e-5
(relative to max(1, |x|)), raw and after a 7-dof similarity alignment of
points and camera centres (gauge freedom, SURVEY.md 7 hard part 3).

The GPU runs both of its solvers: the reference default (tile-sparse
Cholesky of the reduced camera system) and the north-star implicit-Schur PCG
at a tight tolerance (1e-12)."""
import numpy as np
import pytest

import paper_2409_12190_b200 as bae

pytestmark = pytest.mark.gpu

COST_RTOL = 1e-6
GRAD_RTOL = 1e-6
PARAM_TOL = 1e-5
TIE_RTOL = 1e-6

_SCENES = {}
_ORACLE = {}


def _avail_gb():
    try:
        import psutil
        return psutil.virtual_memory().available / 1e9
    except Exception:
        return 0.0


def _scene(name):
    if name not in _SCENES:
        C, P, N = bae.synthetic.CONFIGS[name]
        _SCENES[name] = bae.synthetic.bal_shaped(C, P, N, seed=C)
    return _SCENES[name]


def _oracle_run(oracle, name, max_iterations):
    key = (name, max_iterations)
    if key not in _ORACLE:
        import os
        s = _scene(name)
        oracle.set_threads(os.cpu_count() or 1)
        ref = oracle.Problem(s.poses, s.points, s.intrinsics, s.cam_idx, s.pt_idx, s.pixels)
        _ORACLE[key] = ref.optimize(bae.LmConfig(max_iterations=max_iterations))
        del ref
    return _ORACLE[key]


def _centres(p7):
    """Camera centres -R^T t of [t q] poses (world -> camera)."""
    t, q = p7[:, :3], p7[:, 3:]
    x, y, z, w = q[:, 0], q[:, 1], q[:, 2], q[:, 3]
    R = np.stack([np.stack([1 - 2 * (y * y + z * z), 2 * (x * y - z * w), 2 * (x * z + y * w)], -1),
                  np.stack([2 * (x * y + z * w), 1 - 2 * (x * x + z * z), 2 * (y * z - x * w)], -1),
                  np.stack([2 * (x * z - y * w), 2 * (y * z + x * w), 1 - 2 * (x * x + y * y)], -1)], -2)
    return -np.einsum("nji,nj->ni", R, t)


def _similarity_aligned_error(src, dst):
    """Umeyama: the 7-dof similarity s R x + t that best maps src onto dst;
    returns max |aligned - dst| / max(1, |dst|)."""
    mu_s, mu_d = src.mean(0), dst.mean(0)
    a, b = src - mu_s, dst - mu_d
    U, S, Vt = np.linalg.svd(b.T @ a / len(src))
    D = np.eye(3)
    if np.linalg.det(U) * np.linalg.det(Vt) < 0:
        D[2, 2] = -1
    R = U @ D @ Vt
    s = np.trace(np.diag(S) @ D) / a.var(0).sum()
    aligned = s * a @ R.T + mu_d
    return float((np.abs(aligned - dst) / np.maximum(1.0, np.abs(dst))).max())


def check_trajectory(rep, oref, p7, p3, min_iters=3):
    """Every iteration while the accept decisions agree: cost 1e-6, lambda
    equal; the gradient norm 1e-6 up to the first near-tie (past it the two
    runs' parameters may differ by one near-neutral step, which moves a
    nearly-zero gradient by more than 1e-6 of itself). A decision may only
    differ at or after a near-tie; the comparison ends there."""
    traj_g, traj_o = rep.trajectory, oref["trajectory"]
    assert len(traj_g) > min_iters and len(traj_o) > min_iters
    tie, diverged = None, None
    worst = dict(cost=0.0, grad=0.0)
    for a, b in zip(traj_g[1:], traj_o[1:]):
        before = traj_o[b["iteration"] - 1]["cost"]  # the cost the trial is compared with (lm.hpp:183)
        near = abs(b["trial_cost"] - before) <= TIE_RTOL * before
        if a.accepted != b["accepted"]:
            assert near or tie is not None, (a.iteration, a.accepted, b["accepted"])
            diverged = a.iteration
            break
        assert a.lmbda == b["lmbda"], (a.iteration, a.lmbda, b["lmbda"])
        worst["cost"] = max(worst["cost"], abs(a.cost - b["cost"]) / b["cost"])
        assert abs(a.cost - b["cost"]) <= COST_RTOL * b["cost"], (a.iteration, a.cost, b["cost"])
        if tie is None:
            worst["grad"] = max(worst["grad"], abs(a.grad_norm - b["grad_norm"]) / b["grad_norm"])
            assert abs(a.grad_norm - b["grad_norm"]) <= GRAD_RTOL * b["grad_norm"], \
                (a.iteration, a.grad_norm, b["grad_norm"])
        if near and tie is None:
            tie = b["iteration"]
    if diverged is None:
        assert len(traj_g) == len(traj_o)
        assert rep.reason == bae.TerminationReason(oref["reason"])
    assert abs(rep.final_cost - oref["final_cost"]) <= COST_RTOL * oref["final_cost"]
    e3 = np.abs(p3 - oref["points"]) / np.maximum(1.0, np.abs(oref["points"]))
    e7 = np.abs(p7 - oref["poses"]) / np.maximum(1.0, np.abs(oref["poses"]))
    assert e3.max() <= PARAM_TOL, e3.max()
    assert e7.max() <= PARAM_TOL, e7.max()
    al = _similarity_aligned_error(np.concatenate([_centres(p7), p3]),
                                   np.concatenate([_centres(oref["poses"]), oref["points"]]))
    assert al <= PARAM_TOL, al
    print(f"parity: {len(traj_g) - 1} LM iterations (oracle {len(traj_o) - 1}), first near-tie {tie}, "
          f"decisions diverged at {diverged}, max rel err cost {worst['cost']:.2e} grad {worst['grad']:.2e} "
          f"points {e3.max():.2e} poses {e7.max():.2e} aligned {al:.2e}")
    return tie


@pytest.mark.parametrize("name", ["trafalgar-257", "dubrovnik-356"])
@pytest.mark.parametrize("solver", ["cholesky", "pcg"])
def test_full_solve_matches_oracle(oracle, name, solver):
    """LmConfig defaults with the reference CLI's max_iterations = 50
    (cli.hpp:25), the bench's exact scene, to plateau."""
    s = _scene(name)
    oref = _oracle_run(oracle, name, 50)
    gpu = bae.make_ba_problem(s.poses, s.points, s.intrinsics, s.observations)
    cfg = bae.LmConfig(max_iterations=50)
    if solver == "pcg":
        cfg = bae.LmConfig(max_iterations=50, solver=bae.SolverChoice.pcg, pcg_tol=1e-12)
    rep = bae.optimize(gpu, s.poses, s.points, cfg)
    p7, p3 = gpu.get_parameters()
    check_trajectory(rep, oref, p7, p3)


@pytest.mark.parametrize("name,need_gb", [("venice-1778", 24.0), ("final-13682", 140.0)])
def test_first_lm_iterations_large_configs(oracle, name, need_gb):
    """The two largest configs: the first two LM iterations (the oracle needs
    about 2.1 KB of host memory per observation)."""
    if _avail_gb() < need_gb:
        pytest.skip(f"host RAM: {_avail_gb():.0f} GB available, the oracle needs ~{need_gb:.0f} GB at {name}")
    s = _scene(name)
    oref = _oracle_run(oracle, name, 2)
    gpu = bae.make_ba_problem(s.poses, s.points, s.intrinsics, s.observations)
    rep = bae.optimize(gpu, s.poses, s.points, bae.LmConfig(max_iterations=2))
    assert len(rep.trajectory) == len(oref["trajectory"]) == 3
    for a, b in zip(rep.trajectory[1:], oref["trajectory"][1:]):
        assert a.accepted == b["accepted"] and a.lmbda == b["lmbda"]
        assert abs(a.cost - b["cost"]) <= COST_RTOL * b["cost"], (a.iteration, a.cost, b["cost"])
        assert abs(a.grad_norm - b["grad_norm"]) <= GRAD_RTOL * b["grad_norm"]
    p7, p3 = gpu.get_parameters()
    e3 = (np.abs(p3 - oref["points"]) / np.maximum(1.0, np.abs(oref["points"]))).max()
    e7 = (np.abs(p7 - oref["poses"]) / np.maximum(1.0, np.abs(oref["poses"]))).max()
    assert e3 <= PARAM_TOL and e7 <= PARAM_TOL, (e3, e7)
    ce = max(abs(a.cost - b["cost"]) / b["cost"] for a, b in zip(rep.trajectory[1:], oref["trajectory"][1:]))
    ge = max(abs(a.grad_norm - b["grad_norm"]) / b["grad_norm"]
             for a, b in zip(rep.trajectory[1:], oref["trajectory"][1:]))
    ct = [r["cum_time_s"] for r in oref["trajectory"]]
    print(f"parity {name}: 2 LM iterations, max rel err cost {ce:.2e} grad {ge:.2e} points {e3:.2e} poses {e7:.2e}; "
          f"oracle wall s per iteration {ct[1] - ct[0]:.1f} (first, with the symbolic phase), {ct[2] - ct[1]:.1f}")
