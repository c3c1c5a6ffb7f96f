"""Where the host-buffer (e2e) call's time goes at one shape:
    python tools/e2e_probe.py [B,L,d,N] [reps]"""
import ctypes as C
import sys
import time

import torch

sys.path.insert(0, ".")
import paper_2501_08455_b200 as sk  # noqa: E402

B, L, d, N = (int(v) for v in (sys.argv[1] if len(sys.argv) > 1 else "128,1000,5,4").split(","))
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 200
D = sk.sig_dim(d, N)
X = torch.empty((B, L, d), device="cuda")
sk.brownian(X)
Xh = X.cpu().pin_memory()
outh = torch.empty((B, D)).pin_memory()
outd = torch.empty((B, D), device="cuda")
s = torch.cuda.Stream()
lib = sk.lib()


def wall(fn, n=reps):
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(n):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t) / n * 1e6


def h2d():
    with torch.cuda.stream(s):
        X.copy_(Xh, non_blocking=True)
    s.synchronize()


def d2h():
    with torch.cuda.stream(s):
        outh.copy_(outd, non_blocking=True)
    s.synchronize()


def dev_call():
    sk._check(lib.sigk_signature_f32(X.data_ptr(), B, L, d, N, outd.data_ptr(), 3, C.c_void_p(s.cuda_stream), None,
                                     None))
    s.synchronize()


ST = sk._Stats()


def host_call():
    sk._check(lib.sigk_signature_f32(Xh.data_ptr(), B, L, d, N, outh.data_ptr(), 0, C.c_void_p(s.cuda_stream), None,
                                     C.byref(ST)))


def empty_sync():
    s.synchronize()


print(f"shape B={B} L={L} d={d} N={N}: H2D {Xh.numel()*4/1e6:.2f} MB, D2H {outh.numel()*4/1e6:.2f} MB")
for name, fn in [("sync only", empty_sync), ("H2D+sync", h2d), ("D2H+sync", d2h), ("device call+sync", dev_call),
                 ("host call (e2e)", host_call), ("device call+sync", dev_call), ("host call (e2e)", host_call)]:
    us = wall(fn)
    print(f"{name:20s} {us:8.1f} us   {B / us * 1e6 / 1e6:8.3f} M paths/s")
print("host plan: family", ST.family, "chunks", ST.chunks, "segments", ST.segments, "launches", ST.launches)
