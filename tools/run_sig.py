"""Run one config's signature call a few times (for ncu captures):
    python tools/run_sig.py c2 [reps] [U=..] [G=..] [Q=..] [family=pair]"""
import sys

import torch

sys.path.insert(0, ".")
import paper_2501_08455_b200 as sk  # noqa: E402

CFG = {"c1": (32, 100, 2, 4), "c2": (128, 1000, 5, 4), "c3": (128, 10000, 5, 4), "c4": (64, 500, 10, 5),
       "c5": (8192, 1000, 8, 4), "c2x": (592, 1000, 5, 4)}
name = sys.argv[1]
if name.count(",") == 3:  # explicit B,L,d,N
    CFG[name] = tuple(int(v) for v in name.split(","))
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
kw = {}
for a in sys.argv[3:]:
    k, v = a.split("=")
    if k == "family":
        kw["family"] = {"path": 1, "flat": 2, "pair": 3, "generic": 4, "pflat": 5}[v]
    else:
        kw[{"U": "chunks", "G": "segments", "Q": "prefix_len"}[k]] = int(v)
B, L, d, N = CFG[name]
X = torch.empty((B, L, d), device="cuda")
sk.brownian(X)
out = torch.empty((B, sk.sig_dim(d, N)), device="cuda")
st = sk.KernelStats()
for _ in range(reps):
    sk.signature(X, N, out=out, stats=st, **kw)
torch.cuda.synchronize()
print(st)
