"""Multi-rank decomposition of the reduced camera system on CPU:
world_size 2 over gloo. Each rank owns the points bae_partition_points gives
it (cameras replicated) and computes its partial camera-side sums from the
oracle's per-observation Jacobian blocks; one allreduce per quantity must
reproduce the single-rank H_cc, g_c, Schur RHS and S*x (the exchanges the
multi-GPU path makes once per LM iteration and once per PCG iteration)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _blocks(seed):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import paper_2409_12190_b200 as bae
    from oracle import oracle as O
    sc = bae.synthetic.bal_shaped(10, 160, 700, seed=seed)
    prob = O.Problem(sc.poses, sc.points, sc.intrinsics, sc.cam_idx, sc.pt_idx, sc.pixels)
    r, _ = prob.evaluate()
    jac = prob.jacobian()
    return bae, sc, r.reshape(-1, 2), jac["j_pose"], jac["j_point"]


def _camera_sums(sc, r, jc, jp, mask, lam, x):
    C, P = sc.poses.shape[0], sc.points.shape[0]
    hcc = np.zeros((C, 6, 6))
    gc = np.zeros((C, 6))
    hpp = np.zeros((P, 3, 3))
    gp = np.zeros((P, 3))
    for k in np.nonzero(mask)[0]:
        c, p = sc.cam_idx[k], sc.pt_idx[k]
        hcc[c] += jc[k].T @ jc[k]
        gc[c] += jc[k].T @ r[k]
        hpp[p] += jp[k].T @ jp[k]
        gp[p] += jp[k].T @ r[k]
    hinv = np.zeros_like(hpp)
    for p in range(P):
        if mask[sc.pt_idx == p].any():
            h = hpp[p].copy()
            h[np.diag_indices(3)] = np.clip(np.diag(h), 1e-6, 1e32) * (1 + lam)
            hinv[p] = np.linalg.inv(h)
    # point-local Schur pieces: rhs partial and S*x partial (without H~cc x)
    rhs_part = np.zeros((C, 6))
    sx_part = np.zeros((C, 6))
    for p in range(P):
        ks = np.nonzero(mask & (sc.pt_idx == p))[0]
        if ks.size == 0:
            continue
        v = hinv[p] @ gp[p]
        w = sum(jp[k].T @ (jc[k] @ x[sc.cam_idx[k]]) for k in ks)
        t = hinv[p] @ w
        for k in ks:
            rhs_part[sc.cam_idx[k]] += jc[k].T @ (jp[k] @ v)
            sx_part[sc.cam_idx[k]] += jc[k].T @ (jp[k] @ t)
    return hcc, gc, rhs_part, sx_part


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        bae, sc, r, jc, jp = _blocks(seed=21)
        C, P = sc.poses.shape[0], sc.points.shape[0]
        owner = bae.api.partition_points(C, P, sc.observations, world)
        mask = owner[sc.pt_idx] == rank
        lam = 1e-3
        x = np.random.default_rng(5).normal(size=(C, 6))
        parts = _camera_sums(sc, r, jc, jp, mask, lam, x)
        red = []
        for a in parts:
            t = torch.from_numpy(np.ascontiguousarray(a))
            dist.all_reduce(t)  # sum over ranks
            red.append(t.numpy())
        full = _camera_sums(sc, r, jc, jp, np.ones_like(mask), lam, x)
        ok = all(np.allclose(a, b, rtol=1e-12, atol=1e-9 * max(1.0, np.abs(b).max())) for a, b in zip(red, full))
        q.put((rank, bool(ok), int(mask.sum()), int(np.unique(owner).size)))
    finally:
        dist.destroy_process_group()


def test_two_rank_partition_reproduces_single_rank_sums():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=240)
    res = sorted(q.get(timeout=10) for _ in procs)
    assert all(p.exitcode == 0 for p in procs)
    assert all(ok for _, ok, _, _ in res), res
    assert res[0][2] + res[1][2] == 700 and min(res[0][2], res[1][2]) > 250  # balanced by observations
    assert res[0][3] == 2


@pytest.mark.parametrize("world", [1, 2, 3, 8])
def test_partition_is_contiguous_and_balanced(world):
    import paper_2409_12190_b200 as bae
    sc = bae.synthetic.config_scene("ladybug-49")
    C, P = sc.poses.shape[0], sc.points.shape[0]
    owner = bae.api.partition_points(C, P, sc.observations, world)
    assert owner.min() == 0 and owner.max() == world - 1
    per_rank = np.bincount(owner[sc.pt_idx], minlength=world)
    assert per_rank.max() - per_rank.min() <= 2 * 16  # within one point's observations of even
