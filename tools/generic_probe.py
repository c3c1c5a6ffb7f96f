"""Timing of shapes that fall to the shape-generic fold (no register-sliced instantiation):
    python tools/generic_probe.py   (device buffers, CUDA events)"""
import json
import sys

import torch

sys.path.insert(0, ".")
import paper_2501_08455_b200 as sk  # noqa: E402

for (B, L, d, N, dt) in ((128, 1000, 9, 3, torch.float32), (128, 1000, 9, 3, torch.float64),
                         (64, 1000, 3, 7, torch.float32), (64, 1000, 3, 7, torch.float64),
                         (128, 1000, 12, 2, torch.float64), (32, 2000, 2, 9, torch.float64)):
    X = torch.empty((B, L, d), device="cuda", dtype=torch.float64)
    sk.brownian(X)
    X = X.to(dt)
    st = sk.KernelStats()
    out = sk.signature(X, N, stats=st)
    torch.cuda.synchronize()
    for _ in range(2):
        sk.signature(X, N, out=out)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        sk.signature(X, N, out=out)
    e1.record()
    e1.synchronize()
    print(json.dumps({"B": B, "L": L, "d": d, "N": N, "dtype": str(dt), "family": sk.FAMILY_NAMES[st.family],
                      "ms": round(e0.elapsed_time(e1) / 5, 3)}), flush=True)
