"""Dev tool: wall-clock breakdown of one end-to-end solve (make_ba_problem +
optimize + read-back) with BAE_HOST_TIMING stage times on stderr."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2409_12190_b200 as bae  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "final-13682"
C, P, N = bae.synthetic.CONFIGS[name]
s = bae.synthetic.bal_shaped(C, P, N, seed=C)
for rep in range(int(os.environ.get("E2E_REPS", "3"))):
    print(f"--- rep {rep}", file=sys.stderr, flush=True)
    t0 = time.perf_counter()
    g = bae.make_ba_problem(s.poses, s.points, s.intrinsics, s.observations)
    t1 = time.perf_counter()
    r = bae.optimize(g, s.poses, s.points, bae.LmConfig(), final_state={})
    t2 = time.perf_counter()
    r2 = bae.optimize(g, s.poses, s.points, bae.LmConfig(), final_state={})
    t3 = time.perf_counter()
    print(f"rep {rep}: create {1e3*(t1-t0):.1f} ms, first optimize {1e3*(t2-t1):.1f} ms "
          f"({r.iterations} its), warm optimize {1e3*(t3-t2):.1f} ms", flush=True)
    del g
