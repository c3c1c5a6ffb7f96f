"""Prefix-stream timing for shapes without the pair-family stream (fp64, large d^N):
    python tools/stream64_probe.py  (device buffers, CUDA events, 5 calls)"""
import sys, time, json, torch, numpy as np
sys.path.insert(0, ".")
import paper_2501_08455_b200 as sk
for (B, L, d, N, dt) in ((128, 1000, 5, 4, torch.float64), (128, 1000, 3, 5, torch.float32), (32, 1000, 10, 3, torch.float64), (128, 1000, 3, 5, torch.float64)):
    X = torch.empty((B, L, d), device="cuda", dtype=torch.float64); sk.brownian(X); X = X.to(dt)
    st = sk.KernelStats()
    out = sk.signature_stream(X, N, stats=st); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5): sk.signature_stream(X, N, out=out)
    e1.record(); e1.synchronize()
    ms = e0.elapsed_time(e1) / 5
    print(json.dumps({"B": B, "L": L, "d": d, "N": N, "dtype": str(dt), "family": sk.FAMILY_NAMES[st.family], "ms": round(ms, 3), "GBps": round(out.numel() * out.element_size() / ms / 1e6)}))
