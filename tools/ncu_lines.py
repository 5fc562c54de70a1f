"""Aggregate ncu warp-stall samples per CUDA source line (needs -lineinfo)."""
import collections
import csv
import subprocess
import sys

rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 30
kf = [a for a in sys.argv[3:] if a.startswith("-k=")]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"] +
                     (["-k", kf[0][3:]] if kf else []),
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
agg = collections.Counter()
inst = collections.Counter()
srcs = {}
fname = "?"
cur = None
for r in rows:
    if r and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if len(r) > 4 and r[0] != "Line No":
        if r[0]:
            cur = (fname, r[0])
            srcs[cur] = r[1]
        try:
            agg[cur] += float(r[4] or 0)
            inst[cur] += float(r[7] or 0)
        except ValueError:
            pass
tot = sum(agg.values())
itot = sum(inst.values())
key = inst if "--inst" in sys.argv else agg
print("total samples", tot, "warp instructions", itot)
for k, _ in key.most_common(n):
    v = agg[k]
    print(f"{v:7.0f} {100 * v / max(tot, 1):5.1f}%  inst {100 * inst[k] / max(itot, 1):5.1f}%  {k[0]}:{k[1]}  {srcs.get(k, '')[:80]}")
