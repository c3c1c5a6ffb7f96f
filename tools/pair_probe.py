"""Pair-kernel phase clocks (SM cycles of thread 0 per CTA, median over CTAs)
and event-timed kernel duration, for a config and plan overrides.
    python tools/pair_probe.py c2 "U=20,G=1 U=10,G=1" [B=..] [L=..]"""
import ctypes as C
import json
import sys

import torch

sys.path.insert(0, ".")
import paper_2501_08455_b200 as sk  # noqa: E402

CFG = {"c1": (32, 100, 2, 4), "c2": (128, 1000, 5, 4), "c3": (128, 10000, 5, 4), "c4": (64, 500, 10, 5),
       "c5": (8192, 1000, 8, 4)}
name = sys.argv[1]
combos = sys.argv[2].split() if len(sys.argv) > 2 else ["U=0"]
B, L, d, N = CFG[name]
pipelined = "pipe" in sys.argv[3:]  # 40 back-to-back launches (PDL overlap), stamps of the last ones
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
names = ["stage", "table", "fold", "pdl_wait", "scan", "top_cross", "out", "seg_fence", "seg_combine"]
for combo in combos:
    kw = {}
    for kv in combo.split(","):
        k, v = kv.split("=")
        kw[{"U": "chunks", "G": "segments", "Q": "prefix_len", "M": "mode", "V": "fold_variant"}[k]] = int(v)
    plan = sk.plan(B, L, d, N, family=3, **kw)
    ph = torch.zeros((B * plan.segments, 12), dtype=torch.int64, device="cuda")
    res = []
    for it in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        e1.record()
        torch.cuda.synchronize()
        tun = sk._Tuning(family=3, **kw)
        if not pipelined:
            tun.fold_event_start = C.c_void_p(e0.cuda_event)
            tun.fold_event_stop = C.c_void_p(e1.cuda_event)
        tun.phase_buf = C.c_void_p(ph.data_ptr())
        st = sk._Stats()
        if pipelined:
            e0.record()
        for rep in range(40 if pipelined else 1):
            sk._check(sk.lib().sigk_signature_f32(X.data_ptr(), B, L, d, N, out.data_ptr(), 3,
                                                  C.c_void_p(s.cuda_stream), C.byref(tun), C.byref(st)))
        if pipelined:
            e1.record()
        torch.cuda.synchronize()
        res.append(e0.elapsed_time(e1) * 1e3 / (40 if pipelined else 1))
    p = ph.cpu()
    wall = p[:, 10:12].double()  # globaltimer ns at entry / exit
    cyc = (p[:, 9] - p[:, 0]).double()
    mhz = float((cyc / (wall[:, 1] - wall[:, 0]).clamp(min=1)).median().item() * 1e3)
    staged = None
    if plan.segments == 1:  # slot 8 holds the end of staging (inside the stage phase)
        staged = int((p[:, 8] - p[:, 0]).double().median().item())
        p[:, 8] = p[:, 7]
    if kw.get("fold_variant") == 2:  # ppair: 1 = first tile ready, 2 = producer done (its own clock), 3 = fold done
        names2 = {"first_tile": p[:, 1] - p[:, 0], "producer_done": p[:, 2] - p[:, 0], "fold_done": p[:, 3] - p[:, 0]}
        print(json.dumps({k: int(v.double().median().item()) for k, v in names2.items()}), flush=True)
        p[:, 2] = p[:, 1]
    dlt = (p[:, 1:10] - p[:, 0:9]).double().median(dim=0).values.tolist()
    t0 = wall[:, 0].min()
    rec = {"cfg": name, "B": B, "L": L, "G": st.segments, "U": st.chunks, "CL": st.fold_steps,
           "kernel_us": round(min(res), 2), "phase_cycles": dict(zip(names, [int(x) for x in dlt])),
           "total_cycles": int(cyc.median().item()), "sm_mhz": round(mhz),
           "cta_us_median": round(float((wall[:, 1] - wall[:, 0]).median().item()) / 1e3, 2),
           "first_to_last_exit_us": round(float((wall[:, 1].max() - t0).item()) / 1e3, 2),
           "start_spread_us": round(float((wall[:, 0].max() - t0).item()) / 1e3, 2),
           "staging_done_at": staged}
    print(json.dumps(rec), flush=True)
