"""The direct solver's Schur assembly: the supertile path (k_schur_super +
k_schur_reduce, the default) against the pair-chunk kernel (BAE_SCHUR=pairs)
and against the oracle's damped full system (assemble.hpp:61-101, the
reference's normal equations + clamp-then-scale damping).

Both assemblies sum the same V_k V_l^T products (V = W L^-T)
in different fixed orders, so their steps agree to rounding; each is
deterministic, so a repeated solve is bit-identical."""
import numpy as np
import pytest

import paper_2409_12190_b200 as bae

pytestmark = pytest.mark.gpu


def _problem(s, monkeypatch, mode):
    if mode == "pairs":
        monkeypatch.setenv("BAE_SCHUR", "pairs")
    else:
        monkeypatch.delenv("BAE_SCHUR", raising=False)
    return bae.make_ba_problem(s.poses, s.points, s.intrinsics, s.observations)


def _long_tracks(s, rng, npts=6, ncams=None):
    """Points seen by (nearly) every camera: their warp-tiles exceed the
    supertile caps (more than 16 cameras, or more than 384 observations)
    and run as single supertiles (V read from global memory)."""
    C = s.poses.shape[0]
    ncams = C if ncams is None else ncams
    ci, pi, px = [s.cam_idx], [s.pt_idx], [s.pixels]
    P = s.points.shape[0]
    for j in range(npts):
        cams = rng.choice(C, ncams, replace=False).astype(np.int32)
        ci.append(cams)
        pi.append(np.full(ncams, P + j, np.int32))
        px.append(rng.normal(0.0, 50.0, (ncams, 2)))
    pts = np.concatenate([s.points, s.points[:npts] * 0.5])
    return (np.concatenate(ci).astype(np.int32), np.concatenate(pi).astype(np.int32), np.concatenate(px), pts)


def _scene_obj(s, ci, pi, px, pts):
    return s.poses, pts, s.intrinsics, (ci, pi, px), ci, pi


@pytest.mark.parametrize("C,P,N", [(12, 300, 1500), (64, 500, 2500), (257, 3000, 15000)])
@pytest.mark.parametrize("lmbda", [1e-6, 1e-2])
def test_supertile_matches_pair_chunks(oracle, monkeypatch, C, P, N, lmbda):
    s = bae.synthetic.bal_shaped(C, P, N, seed=C)
    sup = _problem(s, monkeypatch, "super")
    d_sup, _, _ = sup.solve_step(lmbda, bae.LmConfig())
    st = sup.schur_stats()
    assert st["supertiles"] > 0 and st["units"] > 0
    ref = _problem(s, monkeypatch, "pairs")
    d_ref, _, _ = ref.solve_step(lmbda, bae.LmConfig())
    assert ref.schur_stats()["supertiles"] == 0
    # two exact solves of the same system, summed in different orders: equal
    # up to rounding amplified by the damped system's conditioning
    tol = 1e-8  # no dense oracle at this size: conditioning not computed
    if C <= 64:
        o = oracle.Problem(s.poses, s.points, s.intrinsics, s.cam_idx, s.pt_idx, s.pixels)
        A, b = o.normal_dense(lmbda)
        assert np.linalg.norm(A @ d_sup - b) <= 1e-9 * np.linalg.norm(b)
        tol = max(1e-10, 1e-15 * np.linalg.cond(A))
    assert np.linalg.norm(d_sup - d_ref) <= tol * np.linalg.norm(d_ref)
    d_again, _, _ = sup.solve_step(lmbda, bae.LmConfig())
    assert np.array_equal(d_sup, d_again)  # deterministic


@pytest.mark.parametrize("ncams", [None, 20])
def test_single_supertiles_long_tracks(oracle, monkeypatch, ncams):
    """Long tracks (every camera, or 20 of 40) go through k_schur_single; the
    step still satisfies the oracle's damped full system."""
    rng = np.random.default_rng(5)
    s = bae.synthetic.bal_shaped(40, 400, 2400, seed=40)
    ci, pi, px, pts = _long_tracks(s, rng, npts=8, ncams=ncams)
    poses, pts, intr, obs, ci, pi = _scene_obj(s, ci, pi, px, pts)
    monkeypatch.delenv("BAE_SCHUR", raising=False)
    gpu = bae.make_ba_problem(poses, pts, intr, obs)
    dg, iters, _ = gpu.solve_step(1e-3, bae.LmConfig())
    assert iters == 0
    assert gpu.schur_stats()["single_supertiles"] > 0
    ref = oracle.Problem(poses, pts, intr, ci, pi, px)
    A, b = ref.normal_dense(1e-3)
    assert np.linalg.norm(A @ dg - b) <= 1e-9 * np.linalg.norm(b)
    monkeypatch.setenv("BAE_SCHUR", "pairs")
    pairs = bae.make_ba_problem(poses, pts, intr, obs)
    dp, _, _ = pairs.solve_step(1e-3, bae.LmConfig())
    assert np.linalg.norm(dg - dp) <= 1e-10 * np.linalg.norm(dp)


def test_supertile_trajectory_matches_pair_chunks(monkeypatch):
    """Trafalgar-shaped LM solve with LmConfig defaults through both
    assemblies: identical decisions, costs to rounding."""
    s = bae.synthetic.config_scene("trafalgar-257")
    cfg = bae.LmConfig(max_iterations=10)
    reps = []
    for mode in ("super", "pairs"):
        p = _problem(s, monkeypatch, mode)
        reps.append(bae.optimize(p, s.poses, s.points, cfg))
    a, b = reps
    assert len(a.trajectory) == len(b.trajectory)
    for x, y in zip(a.trajectory, b.trajectory):
        assert x.accepted == y.accepted and x.lmbda == y.lmbda
        assert abs(x.cost - y.cost) <= 1e-9 * y.cost
