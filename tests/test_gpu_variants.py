"""Launch / scheduling variants of the direct path must not change the
results they claim not to change:

* BAE_FORK=0 (the fused linearise + prep's camera pass on the solver stream
  instead of beside the Schur assembly, H~_cc added in the assembly's epilogue
  instead of by k_add_hccd) and BAE_PDL=0 (plain launches instead of
  programmatic dependent launches): bitwise the same LM trajectory and
  parameters;
* BAE_CHOL_TAIL=0 (no update helpers): bitwise the same (a helper applies its
  tile's updates in the owner's order);
* BAE_CHOL_ORDER=natural (the tile Cholesky's work queue and every column's
  update order in column order instead of elimination-tree level order): the
  same solve up to the rounding of the reordered sums.

The switches are read once per process, so every variant runs in its own
interpreter on the same scene (the bench's Trafalgar-257)."""
import json
import os
import subprocess
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SOLVE = r"""
import json, sys
import numpy as np
sys.path.insert(0, {root!r})
import paper_2409_12190_b200 as bae
s = bae.synthetic.config_scene("trafalgar-257")
g = bae.make_ba_problem(s.poses, s.points, s.intrinsics, s.observations, device=0)
st = {{}}
rep = bae.optimize(g, s.poses, s.points, bae.LmConfig(), final_state=st)
np.savez({out!r}, poses=st["poses"], points=st["points"],
         costs=np.array([r.cost for r in rep.trajectory]), lams=np.array([r.lmbda for r in rep.trajectory]),
         acc=np.array([r.accepted for r in rep.trajectory]))
"""


def _solve(tmp_path, name, env):
    out = str(tmp_path / f"{name}.npz")
    e = dict(os.environ)
    e.update(env)
    subprocess.run([sys.executable, "-c", SOLVE.format(root=ROOT, out=out)], check=True, env=e, timeout=600)
    return np.load(out)


@pytest.mark.gpu
def test_launch_variants_are_bitwise_neutral(tmp_path):
    base = _solve(tmp_path, "base", {})
    for name, env in (("nofork", {"BAE_FORK": "0"}), ("nopdl", {"BAE_PDL": "0"}), ("nohelp", {"BAE_CHOL_TAIL": "0"})):
        v = _solve(tmp_path, name, env)
        for k in ("poses", "points", "costs", "lams", "acc"):
            assert np.array_equal(base[k], v[k]), (name, k)


@pytest.mark.gpu
def test_natural_chol_order_matches_level_order(tmp_path):
    base = _solve(tmp_path, "base", {})
    nat = _solve(tmp_path, "natural", {"BAE_CHOL_ORDER": "natural"})
    assert np.array_equal(base["acc"], nat["acc"])
    np.testing.assert_allclose(nat["costs"], base["costs"], rtol=1e-9)
    np.testing.assert_allclose(nat["points"], base["points"], rtol=1e-7, atol=1e-9)
    np.testing.assert_allclose(nat["poses"], base["poses"], rtol=1e-7, atol=1e-9)
