"""Dev tool: LM solve time per solver / PCG mode on one config (device time)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2409_12190_b200 as bae  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "trafalgar-257"
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 50
solvers = sys.argv[3].split(",") if len(sys.argv) > 3 else ["cholesky", "pcg"]
t = time.time()
s = bae.synthetic.config_scene(name)
print(f"{name}: gen {time.time() - t:.2f}s", flush=True)
g = bae.make_ba_problem(s.poses, s.points, s.intrinsics, s.observations)
print("stats", g.stats(), flush=True)
for kind, label in [(0, "linearize"), (1, "schur_tiles"), (2, "pcg_iter")]:
    print(f"  {label}: {g.time_kernel(kind, 20) * 1e3:.1f} us", flush=True)
for sv in solvers:
    cfg = bae.LmConfig(max_iterations=iters, solver=bae.SolverChoice[sv])
    for rep_i in range(2):
        g.phase_times(reset=True)
        rep = bae.optimize(g, s.poses, s.points, cfg)
        ph = g.phase_times(reset=True)
    print(f"  {sv} mode={os.environ.get('BAE_PCG_MODE', 'graph')}: {rep.iterations} LM its, "
          f"device {rep.device_seconds * 1e3:.1f} ms, pcg its {rep.total_pcg_iters}, mse {rep.final_mse:.6f}, "
          f"{rep.reason.name}; phases " + ", ".join(f"{k} {v:.2f}" for k, v in ph.items() if v), flush=True)
