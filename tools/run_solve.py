"""Dev tool: one full solve of a config with a given solver (for ncu launch lists)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2409_12190_b200 as bae  # noqa: E402

name = sys.argv[1]
solver = bae.SolverChoice[sys.argv[2]]
iters = int(sys.argv[3])
s = bae.synthetic.config_scene(name)
g = bae.make_ba_problem(s.poses, s.points, s.intrinsics, s.observations)
rep = bae.optimize(g, s.poses, s.points, bae.LmConfig(max_iterations=iters, solver=solver))
print(name, solver.name, rep.iterations, rep.final_mse, rep.device_seconds)
