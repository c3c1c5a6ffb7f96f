"""Host-to-device copy bandwidth from pinned memory vs the number of concurrent streams (tools for the e2e leg)."""
import torch, time
n = 2560000 // 4
for size_mb in (2.56, 10.24):
    n = int(size_mb * 1e6 / 4)
    hs = [torch.empty(n, dtype=torch.float32).pin_memory() for _ in range(8)]
    ds = [torch.empty(n, dtype=torch.float32, device="cuda") for _ in range(8)]
    for nstreams in (1, 2, 3, 4):
        ss = [torch.cuda.Stream() for _ in range(nstreams)]
        torch.cuda.synchronize()
        reps = 400
        t0 = time.perf_counter()
        for i in range(reps):
            s = ss[i % nstreams]
            with torch.cuda.stream(s):
                ds[i % 8].copy_(hs[i % 8], non_blocking=True)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        print(f"{size_mb} MB x {reps}, {nstreams} streams: {reps * n * 4 / dt / 1e9:.1f} GB/s")
    # split each copy in halves on 2 streams
