"""Summarise gpurun_out ncu artefacts into profiles/ (text, committed)."""
import collections
import csv
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def launch_summary(csv_path, out_path, title):
    rows = list(csv.reader(open(csv_path)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hi]
    ki, vi = h.index("Kernel Name"), h.index("Metric Value")
    agg = collections.defaultdict(list)
    for r in rows[hi + 1:]:
        if len(r) > vi:
            agg[r[ki].split("(")[0][:70]].append(float(r[vi].replace(",", "")))
    tot = sum(sum(v) for v in agg.values())
    with open(out_path, "w") as f:
        f.write(f"# {title}\n# ncu --metrics gpu__time_duration.sum --clock-control none (cold-cache, serialised)\n")
        f.write(f"# total device time of listed launches: {tot / 1e6:.3f} ms\n")
        f.write(f"{'kernel':70s} {'launches':>8s} {'mean_us':>9s} {'share':>6s}\n")
        for k, v in sorted(agg.items(), key=lambda x: -sum(x[1])):
            f.write(f"{k:70s} {len(v):8d} {sum(v) / len(v) / 1e3:9.2f} {100 * sum(v) / tot:5.1f}%\n")


def ncu_summary(rep, out_path, title):
    a = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "ncu_summary.py"), rep], capture_output=True,
                       text=True).stdout
    b = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "ncu_lines.py"), rep, "25", "--inst"],
                       capture_output=True, text=True).stdout
    with open(out_path, "w") as f:
        f.write(f"# {title}\n# ncu --set full --clock-control none --import-source on (one launch)\n\n")
        f.write(a + "\n# per source line: warp-stall samples and executed-instruction share\n" + b)


if __name__ == "__main__":
    os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
    for spec in sys.argv[1:]:
        kind, src, dst, title = spec.split("::")
        src = os.path.join(ROOT, src)
        dst = os.path.join(ROOT, "profiles", dst)
        if kind == "launches":
            launch_summary(src, dst, title)
        else:
            ncu_summary(src, dst, title)
        print("wrote", dst)
