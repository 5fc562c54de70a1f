"""Dev tool: one damped direct solve (solve_step) of a config, for ncu captures."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2409_12190_b200 as bae  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "trafalgar-257"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 1
s = bae.synthetic.config_scene(name)
g = bae.make_ba_problem(s.poses, s.points, s.intrinsics, s.observations)
for _ in range(reps):
    g.solve_step(1e-4, bae.LmConfig())
print("ok")
