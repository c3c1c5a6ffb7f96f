"""Host threads calling the library at once, each on its own CUDA stream (the C ABI
releases the GIL through ctypes): forward, prefix stream and reverse mode match
the same calls made one at a time (per-(device, stream) scratch, plan cache and
host staging are shared state inside libsigk.so)."""
import threading

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def test_threads_on_separate_streams_match_serial(sk):
    torch = pytest.importorskip("torch")
    rng = np.random.default_rng(5)
    jobs = []
    for t in range(6):
        B, L, d = [(16, 1000, 5), (8, 2000, 5), (32, 300, 3), (4, 800, 4), (64, 100, 2), (16, 1000, 5)][t]
        X = np.cumsum(rng.standard_normal((B, L, d)) * 0.03, axis=1).astype(np.float32)
        cot = rng.standard_normal((B, sk.sig_dim(d, 4))).astype(np.float32)
        jobs.append((torch.from_numpy(X).cuda(), torch.from_numpy(cot).cuda()))
    torch.cuda.synchronize()

    def run(X, cot):
        return (sk.signature(X, 4).cpu(), sk.signature_stream(X, 3).cpu(), sk.signature_vjp(X, 4, cot).cpu(),
                sk.signature(X.cpu().numpy(), 4))  # host buffers too (staging per stream)

    serial = [run(X, c) for X, c in jobs]
    results = [None] * len(jobs)
    errors = []

    def worker(i):
        try:
            s = torch.cuda.Stream()
            with torch.cuda.stream(s):
                for _ in range(3):
                    out = run(*jobs[i])
                s.synchronize()
            results[i] = out
        except Exception as e:  # noqa: BLE001
            errors.append(e)

    threads = [threading.Thread(target=worker, args=(i,)) for i in range(len(jobs))]
    for th in threads:
        th.start()
    for th in threads:
        th.join()
    assert not errors, errors
    for i, (a, b) in enumerate(zip(serial, results)):
        for x, y in zip(a, b):
            x = x.numpy() if hasattr(x, "numpy") else x
            y = y.numpy() if hasattr(y, "numpy") else y
            assert np.array_equal(x, y), i
