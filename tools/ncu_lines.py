"""Per-source-line executed warp instructions and stall samples from an .ncu-rep
(needs -lineinfo):  python tools/ncu_lines.py rep [top]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(src)))
data, fname = [], ""
hdr = None
for r in rows:
    if r and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) < len(hdr) or not r[0].isdigit():
        continue
    ie, ws = hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)")
    try:
        e, w = int(r[ie] or 0), int(r[ws] or 0)
    except ValueError:
        continue
    if e or w:
        data.append((e, w, f"{fname}:{r[0]}", r[1].strip()[:80]))
te = sum(x[0] for x in data) or 1
tw = sum(x[1] for x in data) or 1
for e, w, loc, s in sorted(data, reverse=True)[:top]:
    print(f"inst {e / te * 100:5.1f}%  stall {w / tw * 100:5.1f}%  {loc:24s} {s}")
