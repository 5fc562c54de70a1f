"""Row f3: pose-graph optimisation on the B200 path against
the oracle's restatement of make_pgo_problem (problems.hpp:141-188) on the
reference's random instances (tests/oracles.hpp:120-152): residuals,
Jacobian blocks (and the oracle's against finite differences, as
test_problems.cpp:138-151 does), LM trajectories, the recovered chain."""
import numpy as np
import pytest

import paper_2409_12190_b200 as bae

pytestmark = pytest.mark.gpu


def _pair(oracle, d, anchor=True):
    gpu = bae.make_pgo_problem(d["poses"], d["edge_i"], d["edge_j"], d["measurements"], d["information"],
                               d["has_information"], anchor)
    ref = oracle.PgoProblem.from_dict(d, anchor)
    return gpu, ref


@pytest.mark.parametrize("seed", [46, 47, 48])
def test_pgo_residuals_and_jacobian(oracle, seed):
    rng = oracle.Rng(seed)
    d = oracle.make_random_pgo(rng, 3 + seed % 7 + 4, True)
    gpu, ref = _pair(oracle, d)
    r_ref, c_ref = ref.evaluate()
    assert np.allclose(gpu.evaluate(), r_ref, rtol=1e-11, atol=1e-11)  # test_problems.cpp:126-136
    ji, jj = gpu.edge_jacobians()
    J = ref.jacobian_dense()
    m = len(d["edge_i"])
    scale = max(1.0, np.abs(J).max())
    for k in range(m):
        for pose, blk in ((d["edge_i"][k], ji[k]), (d["edge_j"][k], jj[k])):
            if pose == 0:  # anchored
                continue
            ref_blk = J[6 * k:6 * k + 6, 6 * (pose - 1):6 * pose]
            assert np.abs(blk - ref_blk).max() <= 1e-11 * scale, (k, pose)


def test_oracle_pgo_jacobian_matches_finite_differences(oracle):
    rng = oracle.Rng(47)
    for _ in range(3):
        d = oracle.make_random_pgo(rng, 6, True)
        ref = oracle.PgoProblem.from_dict(d)
        J = ref.jacobian_dense()
        h, poses = 1e-6, d["poses"]
        fd = np.zeros_like(J)
        for c in range(1, poses.shape[0]):
            for t in range(6):
                e = np.zeros(6)
                e[t] = h
                pp, pm = poses.copy(), poses.copy()
                pp[c] = oracle.se3_retract(poses[c], e)
                pm[c] = oracle.se3_retract(poses[c], -e)
                fd[:, 6 * (c - 1) + t] = (ref.evaluate(pp)[0] - ref.evaluate(pm)[0]) / (2 * h)
        assert np.abs(J - fd).max() <= 1e-6 * max(np.abs(J).max(), np.abs(fd).max())


def test_pgo_consistent_measurements_are_zero(oracle):  # test_problems.cpp:111-124
    d = oracle.make_random_pgo(oracle.Rng(45), 5, False, 0.0)
    gpu, _ = _pair(oracle, d)
    assert np.abs(gpu.evaluate()).max() <= 1e-12


@pytest.mark.parametrize("with_info", [False, True])
def test_pgo_lm_trajectory_matches_oracle(oracle, with_info):
    d = oracle.make_random_pgo(oracle.Rng(51 + with_info), 40, with_info)
    init = d["poses"].copy()
    rng = np.random.default_rng(3)
    for c in range(1, init.shape[0]):  # perturb every free pose
        init[c] = oracle.se3_retract(init[c], 0.05 * rng.standard_normal(6))
    gpu, ref = _pair(oracle, d)
    cfg = bae.LmConfig(max_iterations=15)
    rep = bae.optimize(gpu, init, None, cfg)
    o = ref.optimize(cfg, poses=init)
    n = min(len(rep.trajectory), len(o["trajectory"]))
    assert n >= 3
    for a, b in zip(rep.trajectory[:n], o["trajectory"][:n]):
        assert a.accepted == b["accepted"] and a.lmbda == b["lmbda"]
        assert abs(a.cost - b["cost"]) <= 1e-8 * b["cost"], (a.iteration, a.cost, b["cost"])
    p7, _ = gpu.get_parameters()
    assert np.abs(p7 - o["poses"]).max() <= 1e-7


def test_pgo_perturbed_chain_recovered(oracle):  # test_problems.cpp:163-176
    d = oracle.make_random_pgo(oracle.Rng(49), 3, False, 0.0)
    init = d["poses"].copy()
    init[1] = oracle.se3_retract(init[1], np.array([0.05, -0.02, 0.03, 0.02, 0.04, -0.01]))
    gpu, _ = _pair(oracle, d)
    rep = bae.optimize(gpu, init, None, bae.LmConfig(max_iterations=25, plateau_rel_tol=1e-14))
    assert rep.final_cost < 1e-10


def test_pgo_validation():
    poses = np.tile([0, 0, 0, 0, 0, 0, 1.0], (3, 1))
    meas = np.tile([0, 0, 0, 0, 0, 0, 1.0], (1, 1))
    with pytest.raises(bae.IndexError) as e:
        bae.make_pgo_problem(poses, [0], [5], meas)
    assert e.value.position == 0
    with pytest.raises(ValueError):
        bae.make_pgo_problem(poses, [1], [1], meas)  # self edge
