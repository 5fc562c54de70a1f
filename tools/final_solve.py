"""Dev tool for ncu: one LmConfig-default solve of a config (host generator, as the bench)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2409_12190_b200 as bae  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "final-13682"
s = bae.synthetic.config_scene(name)
g = bae.make_ba_problem(s.poses, s.points, s.intrinsics, s.observations)
rep = bae.optimize(g, s.poses, s.points, bae.LmConfig())
print(name, rep.iterations, rep.final_mse, rep.reason)
