"""The product's host scene generator (csrc/synth.cpp, bae_synth_bal_shaped)
against the oracle's independent restatement of SURVEY.md 8d on the
reference Rng (oracle/bae_oracle.cpp or_synth_bal_shaped). Both bench arms
and every config-scale parity test consume these scenes, so they must agree
bit for bit. CPU only (no kernel launches)."""
import numpy as np
import pytest

import paper_2409_12190_b200 as bae

FIELDS = ("poses", "points", "intrinsics", "cam_idx", "pt_idx", "pixels", "true_poses", "true_points")


@pytest.mark.parametrize("name", ["ladybug-49", "trafalgar-257", "dubrovnik-356"])
def test_host_generator_matches_oracle_restatement(oracle, name):
    C, P, N = bae.synthetic.CONFIGS[name]
    ref = oracle.synth_bal_shaped(C, P, N)
    got = bae.synthetic.bal_shaped(C, P, N, seed=C)
    for f in FIELDS:
        assert np.array_equal(ref[f], getattr(got, f)), f


def test_generator_shape_rules(oracle):
    """exactly N observations, m_j = floor(N/P) + [j < N mod P]
    per point, no duplicate (camera, point) pair, camera-major order, every
    camera of a point inside a window of min(C, 16) ring neighbours."""
    C, P, N = 40, 900, 4123
    s = oracle.synth_bal_shaped(C, P, N, seed=5)
    ci, pi = s["cam_idx"].astype(np.int64), s["pt_idx"].astype(np.int64)
    assert ci.size == N
    m = np.bincount(pi, minlength=P)
    assert np.array_equal(m, N // P + (np.arange(P) < N % P))
    key = ci * P + pi
    assert np.all(np.diff(key) > 0)  # camera-major, points ascending, no duplicates
    for j in range(P):
        cams = np.sort(ci[pi == j])
        gaps = np.diff(np.concatenate([cams, cams[:1] + C]))
        assert C - gaps.max() < 16  # all within one cyclic window of 16


def test_generator_rejects_bad_counts(oracle):
    with pytest.raises(oracle.OracleError):
        oracle.synth_bal_shaped(4, 10, 15, seed=1)  # fewer than two observations per point
    with pytest.raises(oracle.OracleError):
        oracle.synth_bal_shaped(4, 10, 41, seed=1)  # more than P * min(C, 16)
