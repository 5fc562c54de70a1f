"""Quick perf probe (dev tool): per-kernel device times and an LM run."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2409_12190_b200 as bae  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "trafalgar-257"
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 10
t = time.time()
s = bae.synthetic.config_scene(name)
print(f"gen {time.time() - t:.2f}s")
t = time.time()
g = bae.make_ba_problem(s.poses, s.points, s.intrinsics, s.observations)
print(f"create {time.time() - t:.2f}s stats {g.stats()}")
for kind, label in [(0, "linearize"), (1, "schur_tiles"), (2, "pcg_iter"), (3, "jac_store")]:
    ms = g.time_kernel(kind, 20)
    print(f"{label}: {ms * 1e3:.1f} us")
if iters == 0:
    sys.exit(0)
t = time.time()
rep = bae.optimize(g, s.poses, s.points, bae.LmConfig(max_iterations=iters, solver=bae.SolverChoice.pcg))
el = time.time() - t
for r in rep.trajectory:
    print(r.iteration, f"{r.cost:.9g}", r.accepted, r.lmbda, r.pcg_iters, f"{r.cum_time_s:.4f}")
print(f"optimize {el:.3f}s, {rep.iterations / rep.solve_seconds:.1f} LM it/s, pcg total {rep.total_pcg_iters}")
