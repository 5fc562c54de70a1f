"""Dev tool: one direct LM iteration pair on a config (for ncu captures of the per-observation kernels)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2409_12190_b200 as bae  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "final-13682"
s = bae.synthetic.config_scene(name)
g = bae.make_ba_problem(s.poses, s.points, s.intrinsics, s.observations)
bae.optimize(g, s.poses, s.points, bae.LmConfig(max_iterations=2))
print("ok")
