"""GPU parity of the landmark-sharded path on one device.

The ranks of an in-process rank group (one host thread per rank, all on
cuda:0) run exactly the sharded code path the NCCL build runs on 8 GPUs: each
rank keeps its point partition, and the camera-sized partial sums are summed
over ranks once per LM phase and once per PCG iteration. The sharded solve
must reproduce the single-rank solve (and through it the oracle) within the
north star's tolerances: cost 1e-6 relative per iteration (here much tighter,
since only summation order differs), parameters 1e-5 relative; every rank must
hold bit-identical results. The NCCL backend itself is exercised at world = 1
(the communicator, graph capture of ncclAllReduce, the sharded kernels)."""
import threading

import numpy as np
import pytest

import paper_2409_12190_b200 as bae

pytestmark = pytest.mark.gpu


def _scene(C=16, P=600, N=3000, seed=21):
    return bae.synthetic.bal_shaped(C, P, N, seed=seed)


def _run_ranks(world, fn):
    """fn(rank, group) in `world` threads; returns the per-rank results."""
    g = bae.RankGroup(world)
    out, err = [None] * world, [None] * world

    def body(r):
        try:
            out[r] = fn(r, g)
        except BaseException as e:  # noqa: BLE001 - re-raised below
            err[r] = e

    ts = [threading.Thread(target=body, args=(r,)) for r in range(world)]
    for t in ts:
        t.start()
    for t in ts:
        t.join(timeout=600)
    assert not any(t.is_alive() for t in ts), "a rank hung"
    for e in err:
        if e is not None:
            raise e
    del g
    return out


def _solve(s, cfg, **kw):
    p = bae.make_ba_problem(s.poses, s.points, s.intrinsics, s.observations, device=0, **kw)
    st = {}
    rep = bae.optimize(p, s.poses, s.points, cfg, final_state=st)
    return rep, st, p.shard()


def _close_traj(a, b, rtol, tie=1e-10):
    """Same accept / lambda sequence and costs within rtol, up to the first
    near-tie (a trial cost within `tie` of the current cost, where rounding
    of a different summation order may flip accept/reject)."""
    prev = None
    for x, y in zip(a.trajectory, b.trajectory):
        if prev is not None and (abs(x.trial_cost - prev) <= tie * prev or abs(y.trial_cost - prev) <= tie * prev):
            return
        assert x.accepted == y.accepted, x.iteration
        assert abs(x.cost - y.cost) <= rtol * abs(y.cost), (x.iteration, x.cost, y.cost)
        assert x.lmbda == y.lmbda
        prev = y.cost
    assert len(a.trajectory) == len(b.trajectory)


def _rel(a, b):
    return float(np.abs(a - b).max() / max(1.0, np.abs(b).max()))


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("solver", ["pcg", "cholesky"])
def test_sharded_matches_single_rank(world, solver):
    s = _scene()
    cfg = bae.LmConfig(max_iterations=8, solver=bae.SolverChoice[solver], pcg_tol=1e-12)
    ref, st_ref, _ = _solve(s, cfg)
    res = _run_ranks(world, lambda r, g: _solve(s, cfg, rank=r, world=world, group=g))
    owned = bae.partition_points(16, 600, s.observations, world)
    for r, (rep, st, shard) in enumerate(res):
        assert shard[:2] == (r, world)
        assert shard[2] == int((owned == r).sum())
        # direct: only the summation order differs; PCG: a different rounding
        # path through an inexact solve (tolerance relative to ||J^T r||), so
        # the north star's tolerances (cost 1e-6, parameters 1e-5) apply
        tol_c, tol_p = (1e-9, 1e-7) if solver == "cholesky" else (1e-6, 1e-5)
        _close_traj(rep, ref, tol_c)
        assert abs(rep.final_cost - ref.final_cost) <= tol_c * ref.final_cost
        assert _rel(st["poses"], st_ref["poses"]) <= tol_p
        assert _rel(st["points"], st_ref["points"]) <= tol_p
    # every rank holds bit-identical results (identical decisions, no divergence)
    for rep, st, _ in res[1:]:
        assert [t.cost for t in rep.trajectory] == [t.cost for t in res[0][0].trajectory]
        assert np.array_equal(st["poses"], res[0][1]["poses"])
        assert np.array_equal(st["points"], res[0][1]["points"])


def test_sharded_matches_oracle_ladybug(oracle):
    # the same protocol as the single-rank Ladybug parity test (test_gpu_parity.py)
    s = bae.synthetic.config_scene("ladybug-49")
    cfg = bae.LmConfig(max_iterations=15, solver=bae.SolverChoice.pcg, pcg_tol=1e-12)
    res = _run_ranks(2, lambda r, g: _solve(s, cfg, rank=r, world=2, group=g))
    ref = oracle.Problem(s.poses, s.points, s.intrinsics, s.cam_idx, s.pt_idx, s.pixels)
    oracle.set_threads(8)
    o = ref.optimize(bae.LmConfig(max_iterations=15))  # reference default: Cholesky (exact)
    rep, st, _ = res[0]
    n = min(len(rep.trajectory), len(o["trajectory"]))
    assert n >= 4
    for a, b in zip(rep.trajectory[:n], o["trajectory"][:n]):
        assert a.accepted == b["accepted"]
        assert abs(a.cost - b["cost"]) <= 1e-6 * b["cost"], (a.iteration, a.cost, b["cost"])
        assert a.lmbda == b["lmbda"]
    assert abs(rep.final_cost - o["final_cost"]) <= 1e-6 * o["final_cost"]
    assert _rel(st["points"], o["points"]) <= 1e-5
    assert _rel(st["poses"], o["poses"]) <= 1e-5


def test_sharded_cost_and_parameters_roundtrip():
    s = _scene(seed=22)
    single = bae.make_ba_problem(s.poses, s.points, s.intrinsics, s.observations)
    c1 = single.cost()

    def fn(r, g):
        p = bae.make_ba_problem(s.poses, s.points, s.intrinsics, s.observations, rank=r, world=4, group=g)
        poses, points = p.get_parameters()
        return p.cost(), poses, points

    for cost, poses, points in _run_ranks(4, fn):
        assert abs(cost - c1) <= 1e-12 * c1
        assert np.array_equal(poses, s.poses)
        assert np.array_equal(points, s.points)


def test_sharded_cheirality_reports_global_observation(oracle):
    s = _scene(C=8, P=200, N=900, seed=23)
    owner = bae.partition_points(8, 200, s.observations, 2)
    pts = s.points.copy()
    # one point of each rank on a camera plane: the lowest observation id over
    # both ranks must be reported by every rank (make_ba_problem's eager forward)
    ks = [int(np.flatnonzero(owner[s.pt_idx] == 1)[5]), int(np.flatnonzero(owner[s.pt_idx] == 0)[-3])]
    for k in ks:
        c, p = s.cam_idx[k], s.pt_idx[k]
        R = oracle.quat_matrix(s.poses[c, 3:])
        pts[p] = R.T @ (np.array([0.3, 0.1, 0.0]) - s.poses[c, :3])
    with pytest.raises(bae.CheiralityError) as e:
        bae.make_ba_problem(s.poses, pts, s.intrinsics, s.observations)
    single_idx = e.value.observation

    def fn(r, g):
        try:
            bae.make_ba_problem(s.poses, pts, s.intrinsics, s.observations, rank=r, world=2, group=g)
        except bae.CheiralityError as err:
            return err.observation
        return None

    assert _run_ranks(2, fn) == [single_idx, single_idx]


def test_sharded_refuses_per_observation_exports():
    s = _scene(C=8, P=200, N=900, seed=24)

    def fn(r, g):
        p = bae.make_ba_problem(s.poses, s.points, s.intrinsics, s.observations, rank=r, world=2, group=g)
        with pytest.raises(bae.UnsupportedOperationError):
            p.jacobian()
        with pytest.raises(bae.UnsupportedOperationError):
            p.evaluate()
        return True

    assert _run_ranks(2, fn) == [True, True]


@pytest.mark.parametrize("solver", ["pcg", "cholesky"])
def test_nccl_backend_single_rank(solver):
    s = _scene(seed=25)
    cfg = bae.LmConfig(max_iterations=6, solver=bae.SolverChoice[solver], pcg_tol=1e-12)
    ref, st_ref, _ = _solve(s, cfg)
    uid = bae.nccl_unique_id()
    rep, st, shard = _solve(s, cfg, rank=0, world=1, nccl_id=uid)
    assert shard == (0, 1, 600, 3000)
    _close_traj(rep, ref, 1e-12)
    assert _rel(st["points"], st_ref["points"]) <= 1e-9
