"""Interleaved A/B of host-call (e2e) settings at one shape; per-call wall
times, so PCIe interference from other tenants shows up as spread:
    python tools/e2e_ab.py B,L,d,N "pieces:plan" ...   (plan: lat|thr; pieces: 0 = auto)"""
import ctypes as C
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2501_08455_b200 as sk  # noqa: E402

B, L, d, N = (int(v) for v in sys.argv[1].split(","))
cfgs = sys.argv[2:] or ["0:lat", "1:lat", "0:thr", "2:lat", "4:lat"]
D = sk.sig_dim(d, N)
X = torch.empty((B, L, d), device="cuda")
sk.brownian(X)
Xh = X.cpu().pin_memory()
outh = torch.empty((B, D)).pin_memory()
s = torch.cuda.Stream()
lib = sk.lib()
times = {c: [] for c in cfgs}


def setcfg(c):
    p, plan = c.split(":")
    os.environ.pop("SIGK_HOST_PIECES", None)
    os.environ.pop("SIGK_HOST_THROUGHPUT_PLAN", None)
    if int(p) > 0:
        os.environ["SIGK_HOST_PIECES"] = p
    if plan == "thr":
        os.environ["SIGK_HOST_THROUGHPUT_PLAN"] = "1"


for c in cfgs:  # warm every plan
    setcfg(c)
    for _ in range(5):
        sk._check(lib.sigk_signature_f32(Xh.data_ptr(), B, L, d, N, outh.data_ptr(), 0, C.c_void_p(s.cuda_stream),
                                         None, None))
for rnd in range(20):
    for c in cfgs:
        setcfg(c)
        for _ in range(10):
            t = time.perf_counter()
            sk._check(lib.sigk_signature_f32(Xh.data_ptr(), B, L, d, N, outh.data_ptr(), 0,
                                             C.c_void_p(s.cuda_stream), None, None))
            times[c].append(time.perf_counter() - t)
print(f"B={B} L={L} d={d} N={N}  per-call us: min / p25 / median / mean   (M paths/s at median)")
for c in cfgs:
    a = np.array(times[c]) * 1e6
    print(f"{c:8s} {a.min():8.1f} {np.percentile(a, 25):8.1f} {np.median(a):8.1f} {a.mean():8.1f}   {B / np.median(a):.3f}")
