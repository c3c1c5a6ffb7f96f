"""Top SASS instructions by warp-stall samples (with their reasons) from an .ncu-rep."""
import csv
import io
import subprocess
import sys
from collections import Counter

rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 40
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(io.StringIO(src)))
h = rows[1]
ai, si, ei, wi = h.index("Address"), h.index("Source"), h.index("Instructions Executed"), h.index("Warp Stall Sampling (All Samples)")
sc = [i for i, x in enumerate(h) if x.startswith("stall_") and "Not Issued" not in x]
lines = []
for x in rows[2:]:
    if len(x) < len(h):
        continue
    try:
        w = int(x[wi] or 0)
    except ValueError:
        continue
    reasons = Counter({h[i][6:]: int(x[i] or 0) for i in sc if (x[i] or "0") != "0"})
    lines.append((x[ai][-5:], x[si].strip()[:60], int(x[ei] or 0), w, reasons))
tot = sum(l[3] for l in lines) or 1
agg = Counter()
for l in lines:
    agg.update(l[4])
print("all:", ", ".join(f"{k}={v/tot:.0%}" for k, v in agg.most_common(8)))
lo, hi = (int(sys.argv[3], 16), int(sys.argv[4], 16)) if len(sys.argv) > 4 else (None, None)
sel = [l for l in lines if lo is None or lo <= int(l[0], 16) <= hi]
for a, s, e, w, r in sel[:n] if lo is not None else sorted(lines, key=lambda l: -l[3])[:n]:
    print(f"{a} {e:8d} {w:5d} {s:60s} {dict(r.most_common(3))}")
