"""Row f1: BAL files, the reference's synthetic scene and the
drop-in CLI, following the reference's own tests (test_io.cpp): parse /
serialise round trip, parse errors with line numbers, synth_ba determinism
and ground truth, the CLI's CSV schema and exit codes."""
import os
import subprocess

import numpy as np
import pytest

import paper_2409_12190_b200 as bae

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BENCH = os.path.join(ROOT, "paper_2409_12190_b200", "traceopt_bench")

MINIMAL_BAL = ("1 1 1\n"
               "0 0 0.0 0.0\n"
               "0\n0\n0\n"  # rotation
               "0\n0\n0\n"  # translation
               "1\n0\n0\n"  # f k1 k2
               "0\n0\n0\n")  # point


def _cli(*args):
    r = subprocess.run([BENCH, *args], capture_output=True, text=True)
    return r.returncode, r.stdout, r.stderr


def test_minimal_file():  # test_io.cpp:57-65
    p = bae.parse_bal(MINIMAL_BAL)
    assert p.cameras.shape == (1, 9) and p.points.shape == (1, 3) and p.cam_idx.size == 1
    assert p.poses[0, 6] == 1.0  # rotation w of BalCamera::pose
    assert p.intrinsics[0, 0] == 1.0


def test_round_trip_through_serializer(tmp_path):  # test_io.cpp:67-86
    s = bae.synth_ba(3, 7, 0.5, 0.05, 11)
    a, b = tmp_path / "a.bal", tmp_path / "b.bal"
    bae.write_bal(a, s)
    p1 = bae.read_bal(a)
    bae.write_bal(b, p1)
    assert a.read_bytes() == b.read_bytes()  # %.17g round-trips doubles exactly
    p2 = bae.read_bal(b)
    for f in ("cameras", "points", "cam_idx", "pt_idx", "pixels", "poses", "intrinsics"):
        assert np.array_equal(getattr(s, f), getattr(p1, f)), f
        assert np.array_equal(getattr(p1, f), getattr(p2, f)), f


def test_serializer_layout(tmp_path):
    s = bae.parse_bal(MINIMAL_BAL)
    out = tmp_path / "m.bal"
    bae.write_bal(out, s)
    # header, one observation line, then one scalar per line (io/bal.hpp:145-157)
    assert out.read_text() == "1 1 1\n0 0 0 0\n" + "0\n" * 6 + "1\n0\n0\n" + "0\n" * 3


@pytest.mark.parametrize("text,line", [
    ("1 1 1\n0 0 zero 0\n", 2),            # malformed number (test_io.cpp:92-98)
    ("1 1 1\n0 5 0.0 0.0\n", 2),           # point index out of range
    ("2 2 2\n0 0 1.0 1.0\n", None),        # truncated
    (MINIMAL_BAL + "42\n", None),           # trailing data
    # the reference's TokenReader consumes the newline ending a token, so an
    # error on the last header token reports line 2 (io/bal.hpp:58-71)
    ("0 1 1\n", 2),                         # non-positive counts
    ("1 1 x\n", 2),                         # malformed integer
    ("1 1 x", 1),
])
def test_parse_errors_carry_line_numbers(text, line):
    with pytest.raises(bae.ParseError) as e:
        bae.parse_bal(text)
    if line is not None:
        assert e.value.line == line


def test_synth_ba_matches_oracle(oracle):
    """The library's synth_ba (used by the CLI) and the oracle's restatement
    of io/synthetic.hpp:46-91 give the same scene."""
    s = bae.synth_ba(4, 20, 1.0, 0.05, 3)
    o = oracle.synth_ba(4, 20, 1.0, 0.05, 3)
    assert np.array_equal(s.cam_idx, o["cam_idx"]) and np.array_equal(s.pt_idx, o["pt_idx"])
    assert np.array_equal(s.points, o["points"])
    assert np.allclose(s.pixels, o["pixels"], rtol=0, atol=1e-12)
    assert np.allclose(s.poses, o["poses"], rtol=0, atol=1e-14)
    assert np.array_equal(s.intrinsics, o["intrinsics"])


def test_synth_ba_same_seed_bitwise_identical():  # test_io.cpp:188-200
    a, b = bae.synth_ba(3, 10, 1.0, 0.05, 42), bae.synth_ba(3, 10, 1.0, 0.05, 42)
    assert np.array_equal(a.pixels, b.pixels) and np.array_equal(a.cameras, b.cameras)
    c = bae.synth_ba(3, 10, 1.0, 0.05, 43)
    assert not np.array_equal(a.pixels[0], c.pixels[0])


def test_cli_exit_codes(tmp_path):  # test_io.cpp:313-325 (the paths that need no device)
    assert _cli("ba")[0] == 1                                       # missing input
    assert _cli("ba", "--synthetic", "nonsense")[0] == 1            # bad CxP
    assert _cli("ba", "--input", "/nonexistent/file.txt")[0] == 2   # data error
    assert _cli("pgo", "--input", "/nonexistent/file.g2o")[0] == 2
    bad = tmp_path / "bad.bal"
    bad.write_text("1 1 1\n0 0 not_a_number 0\n")
    code, _, err = _cli("ba", "--input", str(bad))
    assert code == 2 and "parse error (line 2)" in err
    assert _cli()[0] == 1                                           # a subcommand is required
    assert _cli("ba", "--solver", "lu", "--synthetic", "3x5")[0] == 1
    assert _cli("ba", "--bogus", "1")[0] == 1
    code, out, _ = _cli("--help")
    assert code == 0 and "ba" in out
    assert bae.cli_main(["ba"]) == 1  # the same entry point in-process


def test_write_csv_schema(tmp_path):
    recs = [bae.LmIterationRecord(0, 12.5, 0.25, 1e-6, True, 0.0, 0, 1.0, 12.5),
            bae.LmIterationRecord(1, 1.0 / 3.0, 1.0 / 150.0, 5e-7, False, 0.0012345678, 3, 1.0, 2.0)]
    rep = bae.LmReport(1.0 / 3.0, 1.0 / 150.0, 1, recs, bae.TerminationReason.max_iters, 1, 1, 5e-7, 0.1, 3, 0.1)
    path = tmp_path / "t.csv"
    bae.write_csv(str(path), rep)
    lines = path.read_text().splitlines()
    assert lines[0] == "iter,cost,mse,lambda,accepted,cum_time_s"
    assert lines[1] == "0,12.5,0.25,9.9999999999999995e-07,1,0.000000"
    assert lines[2] == "1,%.17g,%.17g,%.17g,0,0.001235" % (1.0 / 3.0, 1.0 / 150.0, 5e-7)


def _strip_time(csv_text):
    return "\n".join(line.rsplit(",", 1)[0] for line in csv_text.splitlines())


@pytest.mark.gpu
def test_cli_synthetic_run_writes_bounded_csv(tmp_path):  # test_io.cpp:222-251
    csv = tmp_path / "rows.csv"
    code, out, err = _cli("ba", "--synthetic", "3x20", "--seed", "1", "--max-iters", "50", "--solver", "pcg",
                          "--csv", str(csv))
    assert code == 0, err
    assert "final_mse" in out and out.startswith("dataset=synthetic-3x20 solver=pcg iterations=")
    lines = csv.read_text().splitlines()
    assert lines[0] == "iter,cost,mse,lambda,accepted,cum_time_s"
    assert len(lines) - 1 <= 51
    acc = [float(r.split(",")[1]) for r in lines[1:] if r.split(",")[4] == "1"]
    assert all(b <= a for a, b in zip(acc, acc[1:]))


@pytest.mark.gpu
def test_cli_identical_seeds_identical_csvs(tmp_path):  # test_io.cpp:253-262
    a, b = tmp_path / "d1.csv", tmp_path / "d2.csv"
    assert _cli("ba", "--synthetic", "3x50", "--seed", "7", "--csv", str(a))[0] == 0
    assert _cli("ba", "--synthetic", "3x50", "--seed", "7", "--csv", str(b))[0] == 0
    assert _strip_time(a.read_text()) == _strip_time(b.read_text())


@pytest.mark.gpu
def test_cli_bal_file_matches_oracle(tmp_path, oracle):
    """A BAL file through the CLI: the same final cost as the oracle's LM
    (reference defaults) on the parsed problem."""
    s = bae.synthetic.bal_shaped(10, 200, 900, seed=5)
    cams = np.zeros((10, 9))
    for c in range(10):  # BAL camera records from the scene's poses
        q = s.poses[c, 3:]
        ang = 2.0 * np.arctan2(np.linalg.norm(q[:3]), q[3])
        n = np.linalg.norm(q[:3])
        cams[c, :3] = q[:3] / n * ang if n > 0 else 0.0
        cams[c, 3:6] = s.poses[c, :3]
        cams[c, 6:] = s.intrinsics[c]
    prob = bae.BalProblem(cams, s.points, s.cam_idx, s.pt_idx, s.pixels, None, None)
    path = tmp_path / "scene.bal"
    bae.write_bal(path, prob)
    parsed = bae.read_bal(path)
    code, out, err = _cli("ba", "--input", str(path), "--max-iters", "20")
    assert code == 0, err
    final = float(out.split("final_cost=")[1].split()[0])
    ref = oracle.Problem(parsed.poses, parsed.points, parsed.intrinsics, parsed.cam_idx, parsed.pt_idx,
                         parsed.pixels).optimize(bae.LmConfig(max_iterations=20))
    assert abs(final - ref["final_cost"]) <= 1e-6 * ref["final_cost"], (final, ref["final_cost"])


@pytest.mark.gpu
def test_synth_ba_zero_noise_recovers_ground_truth():  # test_io.cpp:202-209, acceptance.cpp:249-272
    s = bae.synth_ba(3, 50, 0.0, 0.05, 7)
    p = bae.make_ba_problem(s.poses, s.points, s.intrinsics, s.observations)
    rep = bae.optimize(p, s.poses, s.points, bae.LmConfig(max_iterations=20))
    assert rep.final_mse < 1e-10


@pytest.mark.gpu
def test_synth_ba_noise_floor():  # test_io.cpp:211-220
    s = bae.synth_ba(3, 50, 1.0, 0.05, 5)
    p = bae.make_ba_problem(s.poses, s.points, s.intrinsics, s.observations)
    rep = bae.optimize(p, s.poses, s.points, bae.LmConfig(max_iterations=50))
    assert 0.5 <= rep.final_mse <= 2.0


def test_binary_cache_round_trip(tmp_path):
    """Row f4: the binary problem cache holds exactly the parsed arrays and
    read_bal / the CLI recognise it."""
    s = bae.synth_ba(4, 25, 0.5, 0.05, 13)
    txt, binf = tmp_path / "s.bal", tmp_path / "s.baeb"
    bae.write_bal(txt, s)
    p = bae.read_bal(txt)
    bae.write_bal(binf, p, binary=True)
    q = bae.read_bal(binf)
    for f in ("cameras", "points", "cam_idx", "pt_idx", "pixels", "poses", "intrinsics"):
        assert np.array_equal(getattr(p, f), getattr(q, f)), f
    assert binf.stat().st_size == 24 + 8 * (9 * 4 + 3 * 25) + 24 * p.cam_idx.size


@pytest.mark.parametrize("mutate,err", [
    (lambda b: b[:-8], "truncated|size"),                      # short file
    (lambda b: b[:8] + (0).to_bytes(4, "little") + b[12:], "non-positive"),
])
def test_binary_cache_errors(tmp_path, mutate, err):
    s = bae.synth_ba(2, 5, 0.0, 0.0, 1)
    f = tmp_path / "s.baeb"
    bae.write_bal(f, s, binary=True)
    f.write_bytes(mutate(f.read_bytes()))
    with pytest.raises(bae.ParseError, match=err):
        bae.read_bal(f)


def test_binary_cache_index_validation(tmp_path):
    s = bae.synth_ba(2, 5, 0.0, 0.0, 1)
    f = tmp_path / "s.baeb"
    bae.write_bal(f, s, binary=True)
    raw = bytearray(f.read_bytes())
    off = 24 + 8 * (9 * 2 + 3 * 5)  # first camera index
    raw[off:off + 4] = (7).to_bytes(4, "little")
    f.write_bytes(bytes(raw))
    with pytest.raises(bae.ParseError, match="camera index out of range"):
        bae.read_bal(f)


@pytest.mark.gpu
def test_cli_binary_cache_same_solve(tmp_path):
    s = bae.synth_ba(3, 30, 1.0, 0.05, 21)
    txt, binf = tmp_path / "s.bal", tmp_path / "s.baeb"
    bae.write_bal(txt, s)
    bae.write_bal(binf, bae.read_bal(txt), binary=True)
    a, b = _cli("ba", "--input", str(txt), "--max-iters", "10"), _cli("ba", "--input", str(binf), "--max-iters", "10")
    assert a[0] == 0 and b[0] == 0, (a[2], b[2])
    strip = lambda out: out.split("final_cost=")[1].split(" time_s=")[0]  # noqa: E731
    assert strip(a[1]) == strip(b[1])
