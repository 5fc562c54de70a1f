"""Dev tool for ncu: run one kernel kind repeatedly in a live state.
usage: profile_kernel.py <config> <kind> <reps>   (kind: 0 lin, 1 schur tiles, 2 pcg iter, 3 jac store)"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2409_12190_b200 as bae  # noqa: E402

name, kind, reps = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
s = bae.synthetic.config_scene(name)
g = bae.make_ba_problem(s.poses, s.points, s.intrinsics, s.observations)
print(name, kind, g.time_kernel(kind, reps) * 1e3, "us")
