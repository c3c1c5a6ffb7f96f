"""Instruction mix of the hot loops (backward-branch bodies) of every function in a cubin/.so/.o:
    python tools/sass_loops.py <file> [min_ffma]"""
import re
import subprocess
import sys
from collections import Counter

txt = subprocess.run(["cuobjdump", "-sass", sys.argv[1]], capture_output=True, text=True).stdout
minf = int(sys.argv[2]) if len(sys.argv) > 2 else 20
for f in re.split(r"\n\s+Function : ", txt)[1:]:
    name = f.split("\n")[0].strip()
    ops = []
    for l in f.split("\n"):
        m = re.match(r"\s+/\*([0-9a-f]{4,5})\*/\s+(@!?U?P\w+\s+)?([A-Z0-9_.]+)(.*)", l)
        if m:
            ops.append((int(m.group(1), 16), m.group(3), m.group(4)))
    for addr, op, rest in ops:
        if op.startswith("BRA"):
            t = re.search(r"(0x[0-9a-f]+)", rest)
            if t and int(t.group(1), 16) < addr:
                body = [o.split(".")[0] for a, o, _ in ops if int(t.group(1), 16) <= a <= addr]
                c = Counter(body)
                if c["FFMA2"] + c["FFMA"] >= minf:
                    print(f"{name[:70]:70s} loop@{t.group(1)} n={len(body)}", dict(c.most_common(12)))
