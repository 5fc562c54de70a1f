"""Dev tool: tile-Cholesky time per solve for one config under the current
BAE_* environment (ordering / helper knobs)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2409_12190_b200 as bae  # noqa: E402

name = sys.argv[1]
C, P, N = bae.synthetic.CONFIGS[name]
s = bae.synthetic.bal_shaped_device(C, P, N) if C > 1000 else bae.synthetic.config_scene(name)
g = bae.make_ba_problem(s.poses, s.points, s.intrinsics, s.observations)
rep = bae.optimize(g, s.poses, s.points, bae.LmConfig())
chol = g.time_kernel(4, 10) * 1e3
g.phase_times(reset=True) if hasattr(g, "phase_times") else None
import time
t = time.perf_counter()
rep = bae.optimize(g, s.poses, s.points, bae.LmConfig())
wall = time.perf_counter() - t
ds = g.direct_stats()
print(f"{name} leaf={os.environ.get('BAE_ND_LEAF', '24')} help={os.environ.get('BAE_CHOL_HELP', '2')}: "
      f"chol {chol:.1f} us, solve {1e3 * rep.device_seconds:.2f} ms dev / {1e3 * wall:.2f} ms wall, "
      f"{rep.iterations} its, tiles {ds['tiles']} updates {ds['tile_updates']} cols {ds['tile_columns']}", flush=True)
