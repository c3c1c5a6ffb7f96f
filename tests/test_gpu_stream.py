"""GPU parity of the prefix stream (reference signature_stream,
/root/reference/proj/src/kernels.cpp:156-198; rows = the stream_out of
detail::sequential_forward, sig_core.hpp:140-143) against the CPU oracle and
the reference's own golden stream vectors (tests/golden, generated from the
reference). fp32 bar: per-level relative error <= 1e-5 over all rows; fp64
<= 1e-12."""
import os

import numpy as np
import pytest

from oracle import oracle as O
from tests.helpers import level_errors

pytestmark = pytest.mark.gpu

F32_TOL = 1e-5
F64_TOL = 1e-12
THREADS = os.cpu_count() or 1


def brownian(B, L, d, seed=42, dtype=np.float32):
    rng = np.random.default_rng(seed)
    X = np.zeros((B, L, d), np.float64)
    if L > 1:
        X[:, 1:] = np.cumsum(rng.standard_normal((B, L - 1, d)) / np.sqrt(L - 1), axis=1)
    return X.astype(dtype)


def oracle_stream(X, N):
    _, so = O.signature(np.ascontiguousarray(X, np.float64), N, threads=THREADS, stream=True)
    return so


def errs(got, ref, d, N):
    D = got.shape[-1]
    return level_errors(got.reshape(-1, D), ref.reshape(-1, D), d, N)


def test_golden_stream(sk, golden):
    X = golden["stream/X"]
    ref = golden["stream/N3"]
    got = sk.signature_stream(X, 3)
    assert got.shape == ref.shape
    assert max(errs(got, ref, X.shape[2], 3)) <= F64_TOL
    got32 = sk.signature_stream(X.astype(np.float32), 3)
    ref32 = oracle_stream(X.astype(np.float32), 3)
    assert max(errs(got32, ref32, X.shape[2], 3)) <= F32_TOL


def test_headline_shape_pair_stream(sk):
    X = brownian(16, 1000, 5, seed=5)
    st = sk.KernelStats()
    got = sk.signature_stream(X, 4, stats=st)
    assert st.family == sk.FAMILY_PAIR, st
    e = errs(got, oracle_stream(X, 4), 5, 4)
    print("stream C2 rows", st, e)
    assert max(e) <= F32_TOL
    # the last prefix is the signature
    sig = sk.signature(X, 4)
    assert max(level_errors(got[:, -1], sig, 5, 4)) <= 2 * F32_TOL


@pytest.mark.parametrize("d,N", [(1, 3), (2, 1), (2, 4), (3, 3), (4, 4), (5, 2), (5, 4), (6, 3), (8, 4), (10, 3)])
@pytest.mark.parametrize("L", [2, 3, 37, 300])
def test_stream_shapes_f32(sk, d, N, L):
    X = brownian(3, L, d, seed=d * 100 + N * 10 + L)
    got = sk.signature_stream(X, N)
    ref = oracle_stream(X, N)
    own = max(errs(O.signature(X, N, stream=True)[1], ref, d, N))  # the reference's own float error
    assert max(errs(got, ref, d, N)) <= max(F32_TOL, 4 * own), (d, N, L)


@pytest.mark.parametrize("d,N", [(2, 4), (5, 4), (8, 3)])
def test_stream_f64(sk, d, N):
    X = brownian(4, 123, d, seed=9, dtype=np.float64)
    got = sk.signature_stream(X, N)
    assert max(errs(got, oracle_stream(X, N), d, N)) <= F64_TOL


def test_stream_generic_matches_pair(sk):
    X = brownian(8, 500, 5, seed=11)
    a = sk.signature_stream(X, 4)
    b = sk.signature_stream(X, 4, family=sk.FAMILY_GENERIC)
    assert max(errs(a, b, 5, 4)) <= 2 * F32_TOL


def test_stream_domain_errors(sk):
    with pytest.raises(sk.DomainError):
        sk.signature_stream(np.zeros((2, 1, 3), np.float32), 2)
    with pytest.raises(sk.DomainError):
        sk.signature_stream(np.zeros((2, 5, 3), np.float32), 0)


def test_stream_device_tensors(sk):
    torch = pytest.importorskip("torch")
    X = torch.from_numpy(brownian(32, 400, 5, seed=3)).cuda()
    out = sk.signature_stream(X, 4)
    torch.cuda.synchronize()
    assert tuple(out.shape) == (32, 399, 780)
    assert max(errs(out.cpu().numpy(), oracle_stream(X.cpu().numpy(), 4), 5, 4)) <= F32_TOL


@pytest.mark.parametrize("chunks", [2, 6, 20])
def test_stream_chunk_counts(sk, chunks):
    X = brownian(4, 257, 5, seed=31)
    st = sk.KernelStats()
    got = sk.signature_stream(X, 4, stats=st, chunks=chunks)
    assert st.chunks == chunks, st
    assert max(errs(got, oracle_stream(X, 4), 5, 4)) <= F32_TOL


@pytest.mark.parametrize("G", [2, 3, 5])
def test_stream_segments(sk, G):
    # segmented prefix stream: pieces started from the pair kernel's segment prefixes
    X = brownian(3, 700, 5, seed=41)
    st = sk.KernelStats()
    got = sk.signature_stream(X, 4, stats=st, segments=G)
    assert st.segments == G, st
    assert max(errs(got, oracle_stream(X, 4), 5, 4)) <= F32_TOL


@pytest.mark.parametrize("B,L,d,N", [(16, 1000, 5, 4), (8, 500, 10, 3), (8, 300, 3, 6)])
def test_stream_f64_full_length(sk, B, L, d, N):
    # fp64 prefix rows at full sequence length (the chunk-parallel generic stream since
    # round 2: chunk signatures, prefix products, per-chunk walks) <= 1e-12 against the oracle
    rng = np.random.default_rng(B * L + d)
    X = np.zeros((B, L, d))
    X[:, 1:] = np.cumsum(rng.standard_normal((B, L - 1, d)) / np.sqrt(L - 1), axis=1)
    got = sk.signature_stream(X, N)
    _, ref = O.signature(X, N, threads=os.cpu_count() or 1, stream=True)
    assert got.shape == ref.shape
    assert max(errs(got, ref, d, N)) <= F64_TOL


def test_stream_very_long_paths(sk):
    # 100K-step prefix streams (segments chained by in-launch look-back), fp64 and fp32
    rng = np.random.default_rng(101)
    X = np.zeros((2, 100001, 3))
    X[:, 1:] = np.cumsum(rng.standard_normal((2, 100000, 3)) / np.sqrt(100000), axis=1)
    _, ref = O.signature(X, 4, threads=os.cpu_count() or 1, stream=True)
    assert max(errs(sk.signature_stream(X, 4), ref, 3, 4)) <= F64_TOL
    X32 = X.astype(np.float32)
    _, ref32 = O.signature(X32.astype(np.float64), 4, threads=os.cpu_count() or 1, stream=True)
    _, own = O.signature(X32, 4, stream=True)  # the reference's own float error
    bar = max(F32_TOL, 4 * max(errs(own, ref32, 3, 4)))
    assert max(errs(sk.signature_stream(X32, 4), ref32, 3, 4)) <= bar
