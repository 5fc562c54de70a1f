import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2409_12190_b200 as bae
s = bae.synthetic.bal_shaped(12, 300, 1500, seed=7)
g = bae.make_ba_problem(s.poses, s.points, s.intrinsics, s.observations)
print("created", g.stats(), flush=True)
print("schur kernel", g.time_kernel(1, 2), flush=True)
d, it, rel = g.solve_step(1e-2, bae.LmConfig(solver=bae.SolverChoice.pcg, pcg_tol=1e-12, pcg_max_iters=200))
print("solve", it, rel, np.linalg.norm(d), flush=True)
