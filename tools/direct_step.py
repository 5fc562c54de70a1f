"""Dev tool: one damped direct solve (solve_step) of a config, for ncu captures;
prints the Schur assembly structure. usage: direct_step.py [config] [reps] [device-gen 0/1]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2409_12190_b200 as bae  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "trafalgar-257"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 1
devgen = len(sys.argv) > 3 and sys.argv[3] == "1"
C, P, N = bae.synthetic.CONFIGS[name]
s = bae.synthetic.bal_shaped_device(C, P, N) if devgen else bae.synthetic.config_scene(name)
g = bae.make_ba_problem(s.poses, s.points, s.intrinsics, s.observations)
for _ in range(reps):
    t = time.perf_counter()
    g.solve_step(1e-4, bae.LmConfig())
    print(f"solve_step {1e3 * (time.perf_counter() - t):.2f} ms")
print(g.direct_stats())
