"""Host probe for the GPU box: cores, RAM, and the oracle's (CPU reference
restatement) cost per LM iteration at the BASELINE configs. Dev tool."""
import os
import resource
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2409_12190_b200 as bae  # noqa: E402
from oracle import oracle as O  # noqa: E402


def rss_gb():
    return resource.getrusage(resource.RUSAGE_SELF).ru_maxrss / 1e6


def main():
    print("nproc", os.cpu_count())
    print(open("/proc/meminfo").read().splitlines()[:3])
    try:
        print([ln for ln in open("/proc/cpuinfo").read().splitlines() if ln.startswith("model name")][0])
    except Exception:
        pass
    O.set_threads(os.cpu_count() or 1)
    for name, iters in [(a.split(":")[0], int(a.split(":")[1])) for a in sys.argv[1:]]:
        t0 = time.perf_counter()
        s = bae.synthetic.config_scene(name)
        t1 = time.perf_counter()
        ref = O.Problem(s.poses, s.points, s.intrinsics, s.cam_idx, s.pt_idx, s.pixels)
        t2 = time.perf_counter()
        rep = ref.optimize(bae.LmConfig(max_iterations=iters))
        t3 = time.perf_counter()
        print(f"{name}: gen {t1 - t0:.1f}s build {t2 - t1:.1f}s optimize {t3 - t2:.1f}s its {rep['iterations']} "
              f"reason {rep['reason']} mse {rep['final_mse']:.6f} maxrss {rss_gb():.1f} GB", flush=True)
        for r in rep["trajectory"]:
            print("   ", r["iteration"], r["accepted"], f"{r['cost']:.12e}", r["lmbda"], f"{r['cum_time_s']:.2f}",
                  f"{r['grad_norm']:.6e}")
        del ref


if __name__ == "__main__":
    main()
