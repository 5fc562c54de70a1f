"""Dev tool for ncu: one LM solve with the implicit-Schur PCG (north-star
solver) on a config; prints iterations and PCG iterations."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2409_12190_b200 as bae  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "trafalgar-257"
tol = float(sys.argv[2]) if len(sys.argv) > 2 else 1e-8
s = bae.synthetic.config_scene(name)
g = bae.make_ba_problem(s.poses, s.points, s.intrinsics, s.observations)
cfg = bae.LmConfig(solver=bae.SolverChoice.pcg, pcg_tol=tol)
rep = bae.optimize(g, s.poses, s.points, cfg)
print(name, rep.iterations, rep.total_pcg_iters, rep.final_mse, rep.reason, rep.device_seconds)
