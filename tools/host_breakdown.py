"""Dev tool: where the end-to-end time of create + optimize goes on the host."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2409_12190_b200 as bae  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "trafalgar-257"
solver = bae.SolverChoice[sys.argv[2] if len(sys.argv) > 2 else "cholesky"]
s = bae.synthetic.config_scene(name)
cfg = bae.LmConfig(max_iterations=50, solver=solver)
for rep_i in range(5):
    t0 = time.perf_counter()
    g = bae.make_ba_problem(s.poses, s.points, s.intrinsics, s.observations)
    t1 = time.perf_counter()
    r = bae.optimize(g, s.poses, s.points, cfg)
    t2 = time.perf_counter()
    r2 = bae.optimize(g, s.poses, s.points, cfg)
    t3 = time.perf_counter()
    del g
    t4 = time.perf_counter()
    print(f"{name} {solver.name}: create {1e3 * (t1 - t0):.1f} ms, optimize#1 {1e3 * (t2 - t1):.1f} ms "
          f"(device {1e3 * r.device_seconds:.1f}, loop wall {1e3 * r.solve_seconds:.1f}), optimize#2 "
          f"{1e3 * (t3 - t2):.1f} ms (device {1e3 * r2.device_seconds:.1f}), destroy {1e3 * (t4 - t3):.1f} ms, "
          f"iters {r.iterations}")
