"""Row f3: g2o pose graphs and the CLI's `pgo` subcommand,
following the reference's own tests (test_io.cpp:126-186 ParseG2o,
test_io.cpp:265-300 Cli.PgoSummaryLine)."""
import os
import subprocess

import numpy as np
import pytest

import paper_2409_12190_b200 as bae

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BENCH = os.path.join(ROOT, "paper_2409_12190_b200", "traceopt_bench")

IDENT21 = " ".join("1" if r == c else "0" for r in range(6) for c in range(r, 6))
FOURS21 = " ".join("4" if r == c else "0" for r in range(6) for c in range(r, 6))
TWO_VERTEX = ("VERTEX_SE3:QUAT 0 0 0 0 0 0 0 1\n"
              "VERTEX_SE3:QUAT 1 1 0 0 0 0 0 1\n"
              "EDGE_SE3:QUAT 0 1 1 0 0 0 0 0 1 %s\n")


def _cli(*args):
    r = subprocess.run([BENCH, *args], capture_output=True, text=True)
    return r.returncode, r.stdout, r.stderr


def test_single_vertex():  # test_io.cpp:126-132
    g = bae.parse_g2o("VERTEX_SE3:QUAT 0 0 0 0 0 0 0 1\n")
    assert g.vertices.shape == (1, 7) and g.vertices[0, 6] == 1.0
    assert g.edge_i.size == 0 and g.warnings == []


def test_consistent_two_vertex_graph_identity_elided():  # test_io.cpp:134-149 (parse half)
    g = bae.parse_g2o(TWO_VERTEX % IDENT21)
    assert g.vertices.shape == (2, 7) and g.edge_i.tolist() == [0] and g.edge_j.tolist() == [1]
    assert g.has_information.tolist() == [0]


def test_non_identity_information_is_kept():  # test_io.cpp:151-163
    g = bae.parse_g2o(TWO_VERTEX % FOURS21)
    assert g.has_information.tolist() == [1]
    assert g.information[0, 0, 0] == 4.0
    assert np.array_equal(g.information[0], 4.0 * np.eye(6))


def test_information_upper_triangle_is_symmetrised():
    vals = np.arange(1, 22, dtype=float)
    g = bae.parse_g2o(TWO_VERTEX % " ".join("%g" % v for v in vals))
    m = g.information[0]
    assert np.array_equal(m, m.T)
    k = 0
    for r in range(6):
        for c in range(r, 6):
            assert m[r, c] == vals[k]
            k += 1


def test_unknown_tag_skipped_with_warning():  # test_io.cpp:165-173
    g = bae.parse_g2o("VERTEX_SE2 0 0 0 0\nVERTEX_SE3:QUAT 0 0 0 0 0 0 0 1\n")
    assert g.vertices.shape[0] == 1
    assert len(g.warnings) == 1 and "VERTEX_SE2" in g.warnings[0] and g.warnings[0].startswith("line 1:")


def test_comments_blank_lines_and_ids_remapped():
    g = bae.parse_g2o("# header\n\nVERTEX_SE3:QUAT 17 0 0 0 0 0 0 1\n   \nVERTEX_SE3:QUAT 5 1 0 0 0 0 0 1\n"
                      "EDGE_SE3:QUAT 5 17 -1 0 0 0 0 0 1 %s\n" % IDENT21)
    assert g.vertex_ids.tolist() == [17, 5]
    assert g.edge_i.tolist() == [1] and g.edge_j.tolist() == [0]


def test_quaternions_normalised_and_canonical():  # QuatRotation ctor (lie.hpp:33-45)
    g = bae.parse_g2o("VERTEX_SE3:QUAT 0 0 0 0 0 0 0 -2\n")
    assert g.vertices[0, 3:].tolist() == [0.0, 0.0, 0.0, 1.0]
    with pytest.raises(ValueError):
        bae.parse_g2o("VERTEX_SE3:QUAT 0 0 0 0 0 0 0 0\n")  # zero quaternion: invalid_argument


@pytest.mark.parametrize("text,line", [
    ("VERTEX_SE3:QUAT 0 0 0\n", 1),  # test_io.cpp:175-182
    ("VERTEX_SE3:QUAT 0 0 0 0 0 0 0 1\nEDGE_SE3:QUAT 0 9 0 0 0 0 0 0 1 " + IDENT21 + "\n", 2),  # dangling
    ("VERTEX_SE3:QUAT 0 0 0 0 0 0 0 1\nVERTEX_SE3:QUAT 0 0 0 0 0 0 0 1\n", 2),  # duplicate id
    (TWO_VERTEX % "1 0 0", 3),  # missing information entries
    ("VERTEX_SE3:QUAT 0 0 0 x 0 0 0 1\n", 1),
])
def test_errors_carry_line_numbers(text, line):
    with pytest.raises(bae.ParseError) as e:
        bae.parse_g2o(text)
    assert e.value.line == line


def test_cli_pgo_data_errors(tmp_path):
    assert _cli("pgo")[0] == 1  # --input is required
    assert _cli("pgo", "--input", str(tmp_path / "missing.g2o"))[0] == 2
    bad = tmp_path / "bad.g2o"
    bad.write_text("VERTEX_SE3:QUAT 0 0 0\n")
    code, _, err = _cli("pgo", "--input", str(bad))
    assert code == 2 and "parse error (line 1)" in err


def _chain_g2o(oracle, path):
    """Cli.PgoSummaryLine's scene (test_io.cpp:265-290): a 5-pose chain with
    exact measurements, perturbed vertices, identity information."""
    step = oracle.se3_exp([1.0, 0.0, 0.0, 0.0, 0.0, 0.3])
    truth = [np.array([0, 0, 0, 0, 0, 0, 1.0])]
    for _ in range(4):
        truth.append(oracle.se3_compose(truth[-1], step))
    rng = np.random.default_rng(8)
    lines = []
    for i, t in enumerate(truth):
        v = t if i == 0 else oracle.se3_retract(t, np.concatenate([0.1 * rng.standard_normal(3),
                                                                   0.05 * rng.standard_normal(3)]))
        lines.append("VERTEX_SE3:QUAT %d " % i + " ".join("%.17g" % x for x in v))
    for i in range(4):
        lines.append("EDGE_SE3:QUAT %d %d " % (i, i + 1) + " ".join("%.17g" % x for x in step) + " " + IDENT21)
    path.write_text("\n".join(lines) + "\n")


@pytest.mark.gpu
def test_two_vertex_graph_residual_is_zero():  # test_io.cpp:147-148
    g = bae.parse_g2o(TWO_VERTEX % IDENT21)
    p = bae.make_pgo_problem(g)
    r = p.evaluate()
    assert r.shape == (6,) and np.all(r == 0.0)


@pytest.mark.gpu
def test_cli_pgo_summary_line(tmp_path, oracle):  # test_io.cpp:265-300
    path = tmp_path / "traceopt_cli_chain.g2o"
    _chain_g2o(oracle, path)
    code, out, err = _cli("pgo", "--input", str(path))
    assert code == 0, err
    assert out.startswith("dataset=%s solver=cholesky iterations=" % path)
    assert float(out.split("final_cost=")[1].split()[0]) < 1e-12
    assert "termination=" in out


@pytest.mark.gpu
def test_read_g2o_problem_matches_oracle(tmp_path, oracle):
    """A g2o file with information matrices through read_g2o → make_pgo_problem
    optimises to the oracle's final cost on the same graph."""
    rng = oracle.Rng(21)
    inst = oracle.make_random_pgo(rng, 12, True)
    lines = ["VERTEX_SE3:QUAT %d " % (100 + i) + " ".join("%.17g" % x for x in v)
             for i, v in enumerate(inst["poses"])]
    for k in range(len(inst["edge_i"])):
        info = inst["information"][k].reshape(6, 6) if inst["has_information"][k] else np.eye(6)
        up = " ".join("%.17g" % info[r, c] for r in range(6) for c in range(r, 6))
        lines.append("EDGE_SE3:QUAT %d %d " % (100 + inst["edge_i"][k], 100 + inst["edge_j"][k]) +
                     " ".join("%.17g" % x for x in inst["measurements"][k]) + " " + up)
    path = tmp_path / "g.g2o"
    path.write_text("\n".join(lines) + "\n")
    g = bae.read_g2o(path)
    assert g.vertex_ids.tolist() == [100 + i for i in range(12)]
    p = bae.make_pgo_problem(g)
    cfg = bae.LmConfig(max_iterations=30)
    rep = bae.optimize(p, g.vertices, None, cfg)
    ref = oracle.PgoProblem(g.vertices, g.edge_i, g.edge_j, g.measurements, g.information,
                            g.has_information).optimize(cfg)
    assert abs(rep.final_cost - ref["final_cost"]) <= 1e-9 * max(1.0, ref["final_cost"])
