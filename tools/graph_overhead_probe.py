"""Fixed cost of a timed graph region (bench.py's timing at small --steps):
per-step time of R back-to-back replays of an S-step C2 graph after an L2
flush, for several S and R; and the same with a tiny warm-up kernel between
the flush and the first replay.  python tools/graph_overhead_probe.py"""
import json
import sys

import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
import paper_2501_08455_b200 as sk  # noqa: E402

B, L, d, N = 128, 1000, 5, 4
D = sk.sig_dim(d, N)
s = torch.cuda.Stream()
pool = torch.empty((104, B, L, d), device="cuda")
with torch.cuda.stream(s):
    for i in range(104):
        sk.brownian(pool[i], seed=42 + i)
out = torch.empty((B, D), device="cuda")
flush = torch.empty(512 * 2**20 // 4, device="cuda")
tiny = torch.empty(1, device="cuda")
with torch.cuda.stream(s):
    for j in range(8):
        bench._step(sk, pool[j], N, out, None)
s.synchronize()


def cap(S):
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        for j in range(S):
            bench._step(sk, pool[j % 104], N, out, None)
    return g


for S in (20, 64, 256):
    g = cap(S)
    with torch.cuda.stream(s):
        g.replay()
    s.synchronize()
    for R in (1, 2, 4):
        for pre in (0, 1):
            ts = []
            for rep in range(5):
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                with torch.cuda.stream(s):
                    flush.fill_(1.0)
                    if pre:
                        tiny.fill_(0.0)
                    a.record(s)
                    for _ in range(R):
                        g.replay()
                    b.record(s)
                b.synchronize()
                ts.append(a.elapsed_time(b) * 1e3 / (R * S))
            print(json.dumps({"S": S, "R": R, "pre_kernel": pre, "us_per_step_median": sorted(ts)[2]}))
    ts = []
    for rep in range(5):  # the same S steps launched eagerly (PDL chain, no graph)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(s):
            flush.fill_(1.0)
            a.record(s)
            for j in range(S):
                bench._step(sk, pool[j % 104], N, out, None)
            b.record(s)
        b.synchronize()
        ts.append(a.elapsed_time(b) * 1e3 / S)
    print(json.dumps({"S": S, "eager": True, "us_per_step_median": sorted(ts)[2], "all": [round(t, 3) for t in ts]}))
