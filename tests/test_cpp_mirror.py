"""The C++ mirror header compiles against the C ABI and reproduces the
reference's exception behaviour at the call site (CPU: validation; GPU: a
full optimize)."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIBDIR = os.path.join(ROOT, "paper_2409_12190_b200")


def _build(tmp_path):
    exe = tmp_path / "mirror_demo"
    subprocess.run(["g++", "-std=c++20", "-O1", "-I", os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "tests", "cpp", "mirror_demo.cpp"), "-L", LIBDIR, "-lbae_b200",
                    f"-Wl,-rpath,{LIBDIR}", "-o", str(exe)], check=True)
    return exe


def test_mirror_compiles_and_validates(tmp_path):
    exe = _build(tmp_path)
    r = subprocess.run([str(exe)], capture_output=True, text=True)
    assert r.returncode == 0, r.stdout + r.stderr


@pytest.mark.gpu
def test_mirror_optimizes_on_gpu(tmp_path):
    exe = _build(tmp_path)
    r = subprocess.run([str(exe), "gpu"], capture_output=True, text=True)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "optimize:" in r.stdout
