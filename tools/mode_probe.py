"""Single-call vs back-to-back timing of the throughput and latency plans
(sigk_tuning.mode) on one config:  python tools/mode_probe.py c2 [reps]
single: CUDA events around the replay of a one-launch graph (after an L2
flush; includes the graph launch), median of reps; b2b: a graph of 200 back-to-back launches / 200;
sync_host: synchronous numpy calls (host buffers, H2D + kernel + D2H)."""
import json
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2501_08455_b200 as sk  # noqa: E402

CFG = {"c1": (32, 100, 2, 4), "c2": (128, 1000, 5, 4), "c3": (128, 10000, 5, 4), "c4": (64, 500, 10, 5),
       "c5": (8192, 1000, 8, 4)}
B, L, d, N = CFG[sys.argv[1]]
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 20
X = torch.empty((B, L, d), device="cuda")
sk.brownian(X)
out = torch.empty((B, sk.sig_dim(d, N)), device="cuda")
flush = torch.empty(256 * 2**20 // 4, device="cuda")
s = torch.cuda.Stream()
Xh = X.cpu().numpy()
import ctypes as C  # noqa: E402


def call(mode, ev=None):
    tun = sk._Tuning(mode=mode)
    if ev is not None:  # events recorded around the fold kernel by the library (graph-capturable)
        tun.fold_event_start = C.c_void_p(ev[0].cuda_event)
        tun.fold_event_stop = C.c_void_p(ev[1].cuda_event)
    st = torch.cuda.current_stream()
    sk._check(sk.lib().sigk_signature_f32(X.data_ptr(), B, L, d, N, out.data_ptr(), sk.SIGK_X_ON_DEVICE | sk.SIGK_OUT_ON_DEVICE,
                                          C.c_void_p(st.cuda_stream), C.byref(tun), None))


for mode in (sk.MODE_THROUGHPUT, sk.MODE_LATENCY):
    p = sk.plan(B, L, d, N, mode=mode)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    e1.record(s)
    s.synchronize()
    with torch.cuda.stream(s):
        call(mode)
        g1 = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g1, stream=s):
            call(mode)
        g2 = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g2, stream=s):
            for _ in range(200):
                call(mode)
    single = []
    for _ in range(reps):  # one launch alone: L2 flushed, events around a 1-launch graph replay
        with torch.cuda.stream(s):
            flush.fill_(1.0)
            e0.record(s)
            g1.replay()
            e1.record(s)
        s.synchronize()
        single.append(e0.elapsed_time(e1) * 1e3)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(s):
        g2.replay()
        a.record(s)
        g2.replay()
        b.record(s)
    s.synchronize()
    sk.signature(Xh, N, mode=mode)
    t0 = time.perf_counter()
    for _ in range(reps):
        sk.signature(Xh, N, mode=mode)
    sync = (time.perf_counter() - t0) / reps * 1e6
    print(json.dumps({"cfg": sys.argv[1], "mode": {1: "throughput", 2: "latency"}[mode],
                      "plan": {"family": sk.FAMILY_NAMES[p.family], "U": p.chunks, "G": p.segments,
                               "steps_per_chunk": p.fold_steps},
                      "single_us_median": round(float(np.median(single)), 2), "single_us_min": round(min(single), 2),
                      "b2b_us": round(a.elapsed_time(b) * 1e3 / 200, 3), "sync_host_us": round(sync, 1)}), flush=True)
