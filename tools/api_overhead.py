"""Host-side cost of a device-buffer call (no CUDA graph): back-to-back
sigk_signature_f32 calls on device tensors; wall time per call vs GPU time.
    python tools/api_overhead.py [B,L,d,N] [calls]"""
import ctypes as C
import sys
import time

import torch

sys.path.insert(0, ".")
import paper_2501_08455_b200 as sk  # noqa: E402

B, L, d, N = (int(v) for v in (sys.argv[1] if len(sys.argv) > 1 else "128,1000,5,4").split(","))
calls = int(sys.argv[2]) if len(sys.argv) > 2 else 2000
X = torch.empty((B, L, d), device="cuda")
sk.brownian(X)
out = torch.empty((B, sk.sig_dim(d, N)), device="cuda")
s = torch.cuda.current_stream()
lib = sk.lib()
fn = lib.sigk_signature_f32
args = (X.data_ptr(), B, L, d, N, out.data_ptr(), 3, C.c_void_p(s.cuda_stream), None, None)
for _ in range(20):
    fn(*args)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
t = time.perf_counter()
e0.record()
for _ in range(calls):
    fn(*args)
t_host = time.perf_counter() - t
e1.record()
e1.synchronize()
t_all = time.perf_counter() - t
print(f"B={B} L={L} d={d} N={N}: host {t_host / calls * 1e6:.2f} us/call to enqueue, "
      f"wall {t_all / calls * 1e6:.2f} us/call, GPU {e0.elapsed_time(e1) / calls * 1e3:.2f} us/call")
