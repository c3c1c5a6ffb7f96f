"""Asynchronous host-buffer mode (SIGK_ASYNC_HOST): pinned host X/out, ring of
staging slots, copies overlapped across consecutive calls. Results must be
bitwise those of the device-buffer path (same plan), for several calls in
flight at once."""
import ctypes as C

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


def brownian(B, L, d, seed):
    rng = np.random.default_rng(seed)
    X = np.zeros((B, L, d), np.float32)
    X[:, 1:] = np.cumsum(rng.standard_normal((B, L - 1, d)) / np.sqrt(L - 1), axis=1)
    return X


@pytest.mark.parametrize("B,L,d,N", [(128, 1000, 5, 4), (32, 100, 2, 4), (16, 300, 3, 3)])
def test_async_host_matches_device_path(sk, B, L, d, N):
    calls = 7  # more calls in flight than staging slots
    Xs = [torch.from_numpy(brownian(B, L, d, seed=i)).pin_memory() for i in range(calls)]
    outs = [torch.empty((B, sk.sig_dim(d, N)), pin_memory=True) for _ in range(calls)]
    for X, o in zip(Xs, outs):
        sk.signature(X, N, out=o)
    torch.cuda.current_stream().synchronize()
    for X, o in zip(Xs, outs):
        ref = sk.signature(X.cuda(), N)
        torch.cuda.synchronize()
        assert torch.equal(o, ref.cpu())


def test_async_host_f64_and_stream(sk):
    s = torch.cuda.Stream()
    X = torch.from_numpy(brownian(8, 64, 4, seed=3).astype(np.float64)).pin_memory()
    with torch.cuda.stream(s):
        o = sk.signature(X, 3)
    s.synchronize()
    assert torch.equal(o, sk.signature(X.cuda(), 3).cpu())


def test_async_host_needs_pinned(sk):
    X = torch.from_numpy(brownian(2, 10, 2, seed=1))
    with pytest.raises(sk.DomainError):
        sk.signature(X, 2)
    lib = sk.lib()
    Xn = brownian(2, 10, 2, seed=1)
    out = np.empty((2, 6), np.float32)
    rc = lib.sigk_signature_f32(Xn.ctypes.data, 2, 10, 2, 2, out.ctypes.data, sk.SIGK_ASYNC_HOST, None, None, None)
    assert rc == 1  # SIGK_EDOMAIN: pageable numpy memory
