"""Reverse-mode throughput (sigk_signature_vjp_f32, device buffers, CUDA
events) and the reference CPU adjoint on a row sample.
    python tools/vjp_bench.py [B L d N] [reps]"""
import ctypes as C
import json
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2501_08455_b200 as sk  # noqa: E402

B, L, d, N = (int(x) for x in sys.argv[1:5]) if len(sys.argv) >= 5 else (128, 1000, 5, 4)
reps = int(sys.argv[5]) if len(sys.argv) > 5 else 10
D = sk.sig_dim(d, N)
X = torch.empty((B, L, d), device="cuda")
sk.brownian(X)
cot = torch.randn(B, D, device="cuda")
g = torch.empty_like(X)
s = torch.cuda.current_stream()


import os  # noqa: E402

TUN = sk._Tuning(chunks=int(os.environ.get("VJP_CHUNKS", "0")))


def call():
    sk._check(sk.lib().sigk_signature_vjp_f32(X.data_ptr(), B, L, d, N, cot.data_ptr(), g.data_ptr(), 1,
                                              C.c_void_p(s.cuda_stream), C.byref(TUN), None))


for _ in range(2):
    call()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(reps):
    call()
e1.record()
e1.synchronize()
ms = e0.elapsed_time(e1) / reps
rec = {"B": B, "L": L, "d": d, "N": N, "ms_per_call": ms, "paths_per_s": B / ms * 1e3}
try:
    from oracle import oracle as O

    if O.ref() is not None:
        rows = 4
        Xh = X[:rows].double().cpu().numpy()
        ch = cot[:rows].double().cpu().numpy()
        t0 = time.perf_counter()
        O.ref_vjp(Xh, N, ch)
        dt = time.perf_counter() - t0
        rec["reference_cpu_paths_per_s_1thread"] = rows / dt
except Exception as e:  # noqa: BLE001
    rec["reference_cpu"] = str(e)
print(json.dumps(rec))
