"""CPU-side checks of the product library: it loads, exports every symbol the
C header declares, its struct layouts match the ctypes mirror, and the
host-only entry points (scene generator, plateau rule, defaults) behave like
the reference."""
import ctypes
import os
import re
import subprocess

import numpy as np
import pytest

import paper_2409_12190_b200 as bae
from paper_2409_12190_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "bae_b200.h")


def _declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(bae_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    lib = _lib.load()
    names = _declared_functions()
    assert len(names) >= 24
    for n in names:
        assert hasattr(lib, n), n
        assert n in _lib.SIGNATURES, f"{n} missing from the ctypes mirror"


def test_struct_layouts_match_header(tmp_path):
    structs = {"bae_lm_config": _lib.LmConfigC, "bae_iter_record": _lib.IterRecordC,
               "bae_lm_report": _lib.LmReportC, "bae_create_options": _lib.CreateOptionsC}
    prog = ['#include <stdio.h>', '#include <stddef.h>', '#include "bae_b200.h"', 'int main(void){']
    for cname, cls in structs.items():
        prog.append(f'printf("{cname} %zu\\n", sizeof({cname}));')
        for fname, _ in cls._fields_:
            cf = "lambda" if fname == "lmbda" else fname
            prog.append(f'printf("{cname}.{fname} %zu\\n", offsetof({cname}, {cf}));')
    prog.append("return 0;}")
    c = tmp_path / "layout.c"
    c.write_text("\n".join(prog))
    exe = tmp_path / "layout"
    subprocess.run(["gcc", "-I", os.path.join(ROOT, "include"), str(c), "-o", str(exe)], check=True)
    out = dict(line.split() for line in subprocess.run([str(exe)], capture_output=True, text=True).stdout.split("\n")
               if line)
    for cname, cls in structs.items():
        assert int(out[cname]) == ctypes.sizeof(cls), cname
        for fname, _ in cls._fields_:
            assert int(out[f"{cname}.{fname}"]) == getattr(cls, fname).offset, (cname, fname)


def test_default_config_mirrors_lmconfig():
    lib = _lib.load()
    c = _lib.LmConfigC()
    lib.bae_lm_config_default(ctypes.byref(c))
    py = bae.LmConfig()
    for f in ("initial_damping", "damping_min", "damping_max", "damping_up", "damping_down", "clamp_min", "clamp_max",
              "plateau_rel_tol", "pcg_tol", "pcg_max_iters", "max_iterations", "plateau_patience"):
        assert getattr(c, f) == getattr(py, f), f
    assert c.solver == int(bae.SolverChoice.cholesky)  # lm.hpp:34


def test_plateau_rule_matches_oracle(oracle):
    rng = oracle.Rng(34)
    for patience in (1, 3, 5):
        cfg = bae.LmConfig(max_iterations=1000, plateau_patience=patience)
        for _ in range(60):
            h = [100.0]
            for _ in range(rng.index(12)):
                drop = rng.uniform(0.0, 0.3) if rng.uniform() < 0.5 else rng.uniform(0.0, 1e-7)
                h.append(h[-1] * (1.0 - drop))
            assert bae.stop_on_plateau(h, cfg) == oracle.stop_on_plateau(h, cfg)
    assert bae.stop_on_plateau([10, 9, 8], bae.LmConfig(max_iterations=3))
    with pytest.raises(ValueError):
        bae.stop_on_plateau([], bae.LmConfig())


@pytest.mark.parametrize("name", ["ladybug-49", "trafalgar-257"])
def test_generator_shapes_and_determinism(name):
    C, P, N = bae.synthetic.CONFIGS[name]
    a = bae.synthetic.config_scene(name)
    b = bae.synthetic.config_scene(name)
    for k in ("poses", "points", "intrinsics", "cam_idx", "pt_idx", "pixels"):
        assert np.array_equal(getattr(a, k), getattr(b, k)), k
    assert a.cam_idx.shape == (N,) and a.poses.shape == (C, 7) and a.points.shape == (P, 3)
    counts = np.bincount(a.pt_idx, minlength=P)
    assert counts.min() >= 2 and counts.max() - counts.min() <= 1 and counts.sum() == N
    assert np.all(np.diff(a.cam_idx) >= 0)  # camera-major like BAL files
    pairs = a.cam_idx.astype(np.int64) * P + a.pt_idx
    assert np.unique(pairs).size == N  # no duplicated (camera, point)
    assert np.allclose(np.linalg.norm(a.poses[:, 3:], axis=1), 1.0, atol=1e-15)
    assert np.all(a.poses[:, 6] >= 0.0)  # canonical w >= 0 (lie.hpp:40)


def test_generator_pixels_are_projections_plus_noise(oracle):
    s = bae.synthetic.bal_shaped(8, 100, 400, seed=3, pixel_sigma=0.0)
    for k in range(0, 400, 37):
        c, p = s.cam_idx[k], s.pt_idx[k]
        px = oracle.bal_project(s.true_poses[c], s.true_points[p], s.intrinsics[c])
        assert np.allclose(px, s.pixels[k], rtol=1e-13, atol=1e-11)


def test_generator_rejects_impossible_counts():
    with pytest.raises(ValueError):
        bae.synthetic.bal_shaped(4, 10, 10)  # fewer than 2 observations per point
    with pytest.raises(ValueError):
        bae.synthetic.bal_shaped(20, 10, 200)  # more than the 16-camera window allows
