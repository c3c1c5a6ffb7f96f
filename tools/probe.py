"""Device-side probes: kernel event timings (and per-CTA phase clocks) for a
config across (chunks, prefix length) choices.

    python tools/probe.py c2 16:2,51:1 [B=1] [L=2] [phases]
"""
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
want_phases = False
for a in sys.argv[3:]:
    if a.startswith("B="):
        B = int(a[2:])
    elif a.startswith("L="):
        L = int(a[2:])
    elif a == "phases":
        want_phases = True
X = torch.empty((B, L, d), device="cuda")
sk.brownian(X)
D = sk.sig_dim(d, N)
out = torch.empty((B, D), device="cuda")
ph = torch.zeros((B, 8), dtype=torch.int64, device="cuda")
s = torch.cuda.current_stream()
for KQ in Ks:
    K, Qp = (int(x) for x in (KQ.split(":") + ["0"])[:2])
    res = []
    for it in range(6):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        e1.record()
        torch.cuda.synchronize()
        tun = sk._Tuning(chunks=K, prefix_len=Qp)
        tun.fold_event_start = C.c_void_p(e0.cuda_event)
        tun.fold_event_stop = C.c_void_p(e1.cuda_event)
        if want_phases:
            tun.phase_buf = C.c_void_p(ph.data_ptr())
        st = sk._Stats()
        sk._check(sk.lib().sigk_signature_f32(X.data_ptr(), B, L, d, N, out.data_ptr(), 3, C.c_void_p(s.cuda_stream),
                                              C.byref(tun), C.byref(st)))
        torch.cuda.synchronize()
        res.append(e0.elapsed_time(e1) * 1e3)
    rec = {"cfg": name, "B": B, "L": L, "K": st.chunks, "Q": st.prefix_len, "CL": st.fold_steps,
           "kernel_us": round(min(res), 2)}
    if want_phases:
        p = ph.cpu()
        names = ["first_tile", "fold", "sync", "store_lower", "scan_lower", "top_cross", "top_sum"]
        if st.chunks == 1:  # U == 1 skips the scan phases
            p[:, 6] = p[:, 3]
            p[:, 4] = p[:, 3]
            p[:, 5] = p[:, 3]
        dlt = (p[:, 1:8] - p[:, 0:7]).double().median(dim=0).values.tolist()
        rec["phase_cycles"] = dict(zip(names, [int(x) for x in dlt]))
        rec["total_cycles"] = int((p[:, 7] - p[:, 0]).double().median().item())
    print(json.dumps(rec), flush=True)
