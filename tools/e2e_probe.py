import time, sys
sys.path.insert(0, '.')
import numpy as np
import paper_2409_12190_b200 as bae
s = bae.synthetic.config_scene("trafalgar-257")
cfg = bae.LmConfig(max_iterations=50)
for i in range(12):
    t0 = time.perf_counter()
    p = bae.make_ba_problem(s.poses, s.points, s.intrinsics, s.observations)
    t1 = time.perf_counter()
    r = bae.optimize(p, s.poses, s.points, cfg, final_state={})
    t2 = time.perf_counter()
    del p
    t3 = time.perf_counter()
    print(f"create {1e3*(t1-t0):7.1f} optimize {1e3*(t2-t1):7.1f} destroy {1e3*(t3-t2):7.1f} iters {r.iterations}")
