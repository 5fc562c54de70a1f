"""Row f4: the on-device BAL-shaped generator against the
oracle's sequential restatement of the same Philox streams: the observation
structure bit-exact, values to rounding (device and host transcendentals
differ in the last place), deterministic, and a scene the solver converges
on."""
import numpy as np
import pytest

import paper_2409_12190_b200 as bae

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("C,P,N,seed", [(12, 500, 2400, 3), (40, 2000, 11000, 40), (257, 6000, 21000, 257)])
def test_device_scene_matches_oracle(oracle, C, P, N, seed):
    d = bae.synthetic.bal_shaped_device(C, P, N, seed=seed)
    o = oracle.synth_bal_shaped_philox(C, P, N, seed)
    assert np.array_equal(d.cam_idx, o["cam_idx"]) and np.array_equal(d.pt_idx, o["pt_idx"])
    assert np.array_equal(d.true_points, o["true_points"])  # uniforms only: exact
    assert np.allclose(d.intrinsics, o["intrinsics"], rtol=0, atol=1e-17)
    assert np.allclose(d.points, o["points"], rtol=0, atol=1e-15)
    assert np.allclose(d.true_poses, o["true_poses"], rtol=0, atol=1e-13)
    assert np.allclose(d.poses, o["poses"], rtol=0, atol=1e-13)
    assert np.allclose(d.pixels, o["pixels"], rtol=1e-12, atol=1e-9)


def test_device_scene_deterministic():
    a = bae.synthetic.bal_shaped_device(30, 800, 4000, seed=9)
    b = bae.synthetic.bal_shaped_device(30, 800, 4000, seed=9)
    for f in ("poses", "points", "intrinsics", "cam_idx", "pt_idx", "pixels"):
        assert np.array_equal(getattr(a, f), getattr(b, f)), f
    c = bae.synthetic.bal_shaped_device(30, 800, 4000, seed=10)
    assert not np.array_equal(a.pixels, c.pixels)


def test_device_scene_solves():
    s = bae.synthetic.bal_shaped_device(49, 7776, 31843, seed=49)
    p = bae.make_ba_problem(s.poses, s.points, s.intrinsics, s.observations)
    rep = bae.optimize(p, s.poses, s.points, bae.LmConfig(max_iterations=30))
    assert 0.5 <= rep.final_mse <= 2.0  # pixel sigma 1: the noise floor


def test_device_scene_validation():
    with pytest.raises(ValueError):
        bae.synthetic.bal_shaped_device(10, 100, 150)  # fewer than two observations per point
    with pytest.raises(ValueError):
        bae.synthetic.bal_shaped_device(40, 100, 100 * 17)  # more than the window allows
