"""The symbolic phase on the device (plan_device.cu) against the host planner
(plan.cpp + problem.cu's tile classes and blobs): for the same inputs every
plan array must be identical element for element -- the transpose plans
(bsr.hpp:140-160) and the slot, entry, tile and blob layout all derive from
them -- so the two planners give bitwise-identical solves.

Scenes cover several packing segments (P > 2 x 8192), long tracks (warp
tiles over the kPipe* caps that run from global scratch), duplicated
observations and single-observation points (the reference's edge cases,
test_trace.cpp:296-311), and IndexError positions (problems.hpp:105-110)."""
import numpy as np
import pytest

import paper_2409_12190_b200 as bae

pytestmark = pytest.mark.gpu

N_ARRAYS = 19


def _make(monkeypatch, mode, poses, points, intr, obs):
    monkeypatch.setenv("BAE_PLAN", mode)
    return bae.make_ba_problem(poses, points, intr, obs)


def _edge_scene(rng):
    """Synthetic scene + 12 points seen by 40 cameras (long tracks), 30
    duplicated observations and 10 points seen once."""
    s = bae.synthetic.bal_shaped(48, 20000, 90000, seed=48)
    ci, pi, px = [s.cam_idx], [s.pt_idx], [s.pixels]
    P = s.points.shape[0]
    for j in range(12):
        cams = rng.choice(48, 40, replace=False).astype(np.int32)
        ci.append(cams)
        pi.append(np.full(40, P + j, np.int32))
        px.append(rng.normal(0.0, 50.0, (40, 2)))
    dup = rng.choice(s.cam_idx.size, 30, replace=False)
    ci.append(s.cam_idx[dup])
    pi.append(s.pt_idx[dup])
    px.append(s.pixels[dup] + 0.25)
    ci.append(rng.integers(0, 48, 10).astype(np.int32))
    pi.append((P + 12 + np.arange(10)).astype(np.int32))
    px.append(rng.normal(0.0, 50.0, (10, 2)))
    pts = np.concatenate([s.points, s.points[:12] * 0.5, s.points[12:22] + 0.01])
    obs = (np.concatenate(ci).astype(np.int32), np.concatenate(pi).astype(np.int32), np.concatenate(px))
    return s.poses, pts, s.intrinsics, obs


def _scenes():
    rng = np.random.default_rng(7)
    out = []
    for C, P, N in [(12, 300, 1500), (257, 20000, 70000), (356, 40000, 220000)]:
        s = bae.synthetic.bal_shaped(C, P, N, seed=C)
        out.append((f"bal-{C}", (s.poses, s.points, s.intrinsics, s.observations)))
    out.append(("edge", _edge_scene(rng)))
    return out


@pytest.mark.parametrize("name,scene", _scenes(), ids=lambda v: v if isinstance(v, str) else "")
def test_device_plan_equals_host_plan(monkeypatch, name, scene):
    host = _make(monkeypatch, "host", *scene)
    dev = _make(monkeypatch, "device", *scene)
    for which in range(N_ARRAYS):
        a, b = host.plan_array(which), dev.plan_array(which)
        assert a.dtype == b.dtype and a.shape == b.shape, (name, which, a.shape, b.shape)
        assert np.array_equal(a, b), (name, which, int(np.flatnonzero(a != b)[0]))
    if name == "edge":  # the long tracks run from global scratch
        assert host.plan_array(15).size > 0


def test_device_and_host_plans_solve_bitwise_alike(monkeypatch):
    s = bae.synthetic.bal_shaped(257, 20000, 70000, seed=257)
    reps = []
    for mode in ("host", "device"):
        g = _make(monkeypatch, mode, s.poses, s.points, s.intrinsics, s.observations)
        reps.append((bae.optimize(g, s.poses, s.points, bae.LmConfig(max_iterations=6)), g.get_parameters()))
    (ra, pa), (rb, pb) = reps
    assert [t.cost for t in ra.trajectory] == [t.cost for t in rb.trajectory]
    assert np.array_equal(pa[0], pb[0]) and np.array_equal(pa[1], pb[1])


@pytest.mark.parametrize("what", ["camera", "point"])
def test_device_plan_index_error_position(monkeypatch, what):
    s = bae.synthetic.bal_shaped(64, 30000, 140000, seed=3)
    ci, pi, px = s.cam_idx.copy(), s.pt_idx.copy(), s.pixels
    at = [77_777, 131_000]
    if what == "camera":
        ci[at[0]] = 64
        ci[at[1]] = -1
    else:
        pi[at[0]] = -5
        pi[at[1]] = 30000
    for mode in ("host", "device"):
        monkeypatch.setenv("BAE_PLAN", mode)
        with pytest.raises(bae.IndexError) as ei:
            bae.make_ba_problem(s.poses, s.points, s.intrinsics, (ci, pi, px))
        assert ei.value.position == at[0], (mode, str(ei.value))
        assert what in str(ei.value)
