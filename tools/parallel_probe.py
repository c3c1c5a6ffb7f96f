"""Timing of the paper's parallel formulation on the GPU (KernelKind::Parallel):
forward (sigk_signature_parallel_*) and reverse (sigk_signature_vjp_parallel_*),
device buffers, CUDA events; with the workspace bytes each materialises.
    python tools/parallel_probe.py [B L d N] [reps]"""
import json
import sys

import torch

sys.path.insert(0, ".")
import paper_2501_08455_b200 as sk  # noqa: E402

B, L, d, N = (int(x) for x in sys.argv[1:5]) if len(sys.argv) >= 5 else (128, 1000, 5, 4)
reps = int(sys.argv[5]) if len(sys.argv) > 5 else 5
D = sk.sig_dim(d, N)
for dt in (torch.float32, torch.float64):
    X = torch.empty((B, L, d), device="cuda", dtype=torch.float32)
    sk.brownian(X)
    X = X.to(dt)
    cot = torch.randn(B, D, device="cuda", dtype=dt)
    for name, fn in (("forward", lambda: sk.signature_parallel(X, N)),
                     ("vjp", lambda: sk.signature_vjp(X, N, cot, kernel=sk.KernelKind.Parallel))):
        fn()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(reps):
            fn()
        b.record()
        b.synchronize()
        ms = a.elapsed_time(b) / reps
        ws = (1 if name == "forward" else 3) * B * (L - 1) * D * X.element_size()
        print(json.dumps({"route": name, "dtype": str(dt).split(".")[-1], "B": B, "L": L, "d": d, "N": N,
                          "ms_per_call": round(ms, 3), "workspace_MB": round(ws / 2**20),
                          "workspace_GBs": round(ws / (ms * 1e-3) / 1e9)}))
