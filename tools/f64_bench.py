import sys, torch
sys.path.insert(0, ".")
import paper_2501_08455_b200 as sk
for (B, L, d, N) in [(128, 1000, 5, 4), (64, 500, 10, 5), (8192, 1000, 8, 4)]:
    X = torch.empty((B, L, d), device="cuda", dtype=torch.float64)
    sk.brownian(X)
    out = torch.empty((B, sk.sig_dim(d, N)), device="cuda", dtype=torch.float64)
    st = sk.KernelStats()
    for _ in range(3): sk.signature(X, N, out=out, stats=st)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 20 if B < 1000 else 3
    e0.record()
    for _ in range(reps): sk.signature(X, N, out=out)
    e1.record(); e1.synchronize()
    ms = e0.elapsed_time(e1) / reps
    W = sum((N - k + 1) * d ** k for k in range(1, N + 1))
    tf = 2 * W * (L - 1) * B / (ms * 1e-3) / 1e12
    print(f"fp64 B={B} L={L} d={d} N={N}: {ms*1e3:.1f} us/call, {B/ms*1e3:.0f} paths/s, {tf:.1f} TFLOP/s credited, family {st.family} chunks {st.chunks}")
