"""Dev tool for ncu: run one kernel kind repeatedly in a live state (bae_time_kernel).
usage: profile_kernel.py <config> <kind> <reps> [device-gen 0/1]
kinds: 0 linearise, 1 Schur tile pass, 2 PCG iteration, 3 linearise + Jacobian store,
       4 tile Cholesky, 5 direct prep, 6 Schur assembly, 7 fused linearise + prep, 8 trial"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2409_12190_b200 as bae  # noqa: E402

name, kind, reps = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
devgen = len(sys.argv) > 4 and sys.argv[4] == "1"
C, P, N = bae.synthetic.CONFIGS[name]
s = bae.synthetic.bal_shaped_device(C, P, N) if devgen else bae.synthetic.config_scene(name)
g = bae.make_ba_problem(s.poses, s.points, s.intrinsics, s.observations)
print(name, kind, g.time_kernel(kind, reps) * 1e3, "us")
