"""Prefix-stream throughput (sigk_signature_stream_f32, device buffers,
back-to-back launches, CUDA events): output GB/s against the HBM peak.
    python tools/stream_bench.py [B L d N] [reps] [family]"""
import ctypes as C
import json
import os
import sys

import torch

sys.path.insert(0, ".")
import paper_2501_08455_b200 as sk  # noqa: E402

B, L, d, N = (int(x) for x in sys.argv[1:5]) if len(sys.argv) >= 5 else (128, 1000, 5, 4)
reps = int(sys.argv[5]) if len(sys.argv) > 5 else 50
fam = int(sys.argv[6]) if len(sys.argv) > 6 else 0
D = sk.sig_dim(d, N)
X = torch.empty((B, L, d), device="cuda")
sk.brownian(X)
out = torch.empty((B, L - 1, D), device="cuda")
s = torch.cuda.current_stream()
tun = sk._Tuning(family=fam, chunks=int(os.environ.get("STREAM_CHUNKS", "0")), segments=int(os.environ.get("STREAM_SEGMENTS", "0")))
st = sk._Stats()


def call():
    sk._check(sk.lib().sigk_signature_stream_f32(X.data_ptr(), B, L, d, N, out.data_ptr(), 3, C.c_void_p(s.cuda_stream),
                                                 C.byref(tun), C.byref(st)))


for _ in range(3):
    call()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(reps):
    call()
e1.record()
e1.synchronize()
ms = e0.elapsed_time(e1) / reps
wbytes = B * (L - 1) * D * 4
peak = json.load(open("MEASURED_PEAKS.json")).get("hbm_gbs") if os.path.exists("MEASURED_PEAKS.json") else None
print(json.dumps({"B": B, "L": L, "d": d, "N": N, "family": sk.FAMILY_NAMES.get(st.family), "chunks": st.chunks,
                  "ms_per_call": ms, "out_GBps": wbytes / ms / 1e6, "hbm_peak_GBps": peak,
                  "frac_of_hbm": (wbytes / ms / 1e6 / peak) if peak else None,
                  "prefix_rows_per_s": B * (L - 1) / ms * 1e3}))
