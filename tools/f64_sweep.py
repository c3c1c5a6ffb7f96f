"""fp64 fold: back-to-back time per call by chunk count (sigk_tuning.chunks) for the
five configs:  python tools/f64_sweep.py [c2 ...]"""
import ctypes as C
import json
import sys

import torch

sys.path.insert(0, ".")
import paper_2501_08455_b200 as sk  # noqa: E402

CFG = {"c1": (32, 100, 2, 4), "c2": (128, 1000, 5, 4), "c3": (128, 10000, 5, 4), "c4": (64, 500, 10, 5),
       "c5": (8192, 1000, 8, 4)}
for name in sys.argv[1:] or ["c2"]:
    B, L, d, N = CFG[name]
    X = torch.empty((B, L, d), device="cuda", dtype=torch.float64)
    sk.brownian(X)
    out = torch.empty((B, sk.sig_dim(d, N)), device="cuda", dtype=torch.float64)
    W = sum((N - k + 1) * d ** k for k in range(1, N + 1))
    for U in (0, 1, 2, 4, 6, 8, 10, 12, 16, 20, 24, 32):
        st = sk.KernelStats()
        try:
            sk.signature(X, N, out=out, chunks=U, stats=st)
        except Exception as e:  # noqa: BLE001
            print(name, U, "error", e)
            continue
        torch.cuda.synchronize()
        reps = 20 if B * L < 10**7 else 3
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            sk.signature(X, N, out=out, chunks=U)
        e1.record()
        e1.synchronize()
        ms = e0.elapsed_time(e1) / reps
        tf = B * 2 * W * (L - 1) / ms / 1e9
        print(json.dumps({"cfg": name, "U_req": U, "family": sk.FAMILY_NAMES[st.family], "U": st.chunks, "Q": st.prefix_len,
                          "us": round(ms * 1e3, 1), "TFLOPs": round(tf, 2), "frac_fp64_nominal": round(tf / 37.2, 3)}),
              flush=True)
