"""Quick device-side probes: fold/merge event timings for a config across chunk counts."""
import ctypes as C
import json
import sys

import torch

sys.path.insert(0, ".")
import paper_2501_08455_b200 as sk

cfg = {"c1": (32, 100, 2, 4), "c2": (128, 1000, 5, 4), "c3": (128, 10000, 5, 4), "c4": (64, 500, 10, 5),
       "c5": (8192, 1000, 8, 4)}
name = sys.argv[1] if len(sys.argv) > 1 else "c2"
Ks = sys.argv[2].split(",") if len(sys.argv) > 2 else ["0"]  # "K" or "K:Q"
B, L, d, N = cfg[name]
for a in sys.argv[3:]:
    if a.startswith("B="):
        B = int(a[2:])
    if a.startswith("L="):
        L = int(a[2:])
X = torch.empty((B, L, d), device="cuda")
sk.brownian(X)
D = sk.sig_dim(d, N)
out = torch.empty((B, D), device="cuda")
s = torch.cuda.current_stream()
for KQ in Ks:
    K, Qp = (int(x) for x in (KQ.split(":") + ["0"])[:2])
    res = []
    for it in range(6):
        e0, e1, e2, e3 = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
        e0.record(); e1.record(); e3.record()
        torch.cuda.synchronize()
        tun = sk._Tuning(chunks=K, prefix_len=Qp)
        tun.fold_event_start = C.c_void_p(e0.cuda_event)
        tun.fold_event_stop = C.c_void_p(e1.cuda_event)
        st = sk._Stats()
        e2.record()
        sk._check(sk.lib().sigk_signature_f32(X.data_ptr(), B, L, d, N, out.data_ptr(), 3, C.c_void_p(s.cuda_stream),
                                              C.byref(tun), C.byref(st)))
        e3.record()
        torch.cuda.synchronize()
        res.append((e0.elapsed_time(e1) * 1e3, e2.elapsed_time(e3) * 1e3))
    fold = min(r[0] for r in res)
    tot = min(r[1] for r in res)
    print(json.dumps({"cfg": name, "K": st.chunks, "Q": st.prefix_len, "CL": st.fold_steps, "fold_us": round(fold, 2),
                      "total_us": round(tot, 2), "merge_us": round(tot - fold, 2)}))
