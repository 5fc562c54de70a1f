"""Dev tool: summarise a BAE_CHOL_TRACE=2 log (per-column timeline of the tile
Cholesky): where the factor span goes, by start-time window."""
import re
import statistics as st
import sys

txt = open(sys.argv[1]).read()
part = txt.split('[bae chol]')[1]
rows = []
for line in part.splitlines()[1:]:
    m = re.match(r'\s+col\s+(\d+): start\s+(\S+) last-k seen\s+(\S+) potrf\s+(\S+)\.\.\s*(\S+) first pub\s+(\S+) '
                 r'done\s+(\S+) bwd\s+(\S+)\.\.\s*(\S+)', line)
    if m:
        rows.append([int(m.group(1))] + [float(x) for x in m.groups()[1:]])
print(part.splitlines()[0])
span = max(r[6] for r in rows)
step = max(100.0, span / 10)
lo = 0.0
while lo < span:
    sel = [r for r in rows if lo <= r[1] < lo + step]
    if sel:
        w = [r[2] - r[1] for r in sel if r[2] >= 0]
        print(f"start in [{lo:6.0f},{lo + step:6.0f}): n={len(sel):4d} start->lastk {st.mean(w) if w else 0:6.1f} "
              f"potrf {st.mean(r[4] - r[3] for r in sel):5.1f} potrf->done {st.mean(r[6] - r[4] for r in sel):5.1f} "
              f"total {st.mean(r[6] - r[1] for r in sel):6.1f}")
    lo += step
busy = sorted(rows, key=lambda r: r[6])
print("last 12 columns to finish:")
for r in busy[-12:]:
    print("  col %4d start %7.1f lastk %7.1f potrf %7.1f..%7.1f pub %7.1f done %7.1f" % tuple(r[:7]))
