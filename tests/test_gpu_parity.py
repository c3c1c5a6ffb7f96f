"""GPU parity: the sm_100a kernels through the C ABI vs the pinned CPU oracle.

Bars (BASELINE.json north_star): fp32 per-level relative error <= 1e-5,
fp64 <= 1e-12, where err_n = max|g - r| / max|r| over level n
and r is the oracle in float64 fed the SAME fp32-rounded inputs promoted to
double (input rounding is not charged).
"""
import os

import numpy as np
import pytest

from oracle import oracle as O
from tests.helpers import level_errors, level_offsets, max_abs_diff, rel_diff

pytestmark = pytest.mark.gpu

F32_TOL = 1e-5
F64_TOL = 1e-12
THREADS = os.cpu_count() or 1


def brownian(B, L, d, seed=42):
    rng = np.random.default_rng(seed)
    X = np.zeros((B, L, d), np.float64)
    if L > 1:
        X[:, 1:] = np.cumsum(rng.standard_normal((B, L - 1, d)) / np.sqrt(L - 1), axis=1)
    return X


def check_f32(sk, X, N, **kw):
    X32 = np.ascontiguousarray(X, np.float32)
    got = sk.signature(X32, N, **kw)
    ref = O.signature(X32.astype(np.float64), N, threads=THREADS)
    errs = level_errors(got, ref, X.shape[2], N)
    assert max(errs) <= F32_TOL, errs
    return got, ref, errs


def check_f64(sk, X, N, tol=F64_TOL, **kw):
    X = np.ascontiguousarray(X, np.float64)
    got = sk.signature(X, N, **kw)
    ref = O.signature(X, N, threads=THREADS)
    errs = level_errors(got, ref, X.shape[2], N)
    assert max(errs) <= tol, errs
    return got, ref, errs


# ----------------------------------------------------------- golden vectors
def test_corner_path(sk, golden):
    expected = np.array([[1.0, 1.0, 0.5, 1.0, 0.0, 0.5]])
    assert max_abs_diff(sk.signature(golden["corner/X"], 2), expected) < 1e-12
    assert max_abs_diff(sk.signature(golden["corner/X"].astype(np.float32), 2), expected) < 1e-6


def test_golden_bruteforce_grid(sk, golden):
    # acceptance.cpp:60-85: 1e-10 against the brute-force oracle, fp64
    for s in golden["brute/seeds"]:
        X, N = golden[f"brute/{s}/X"], int(golden[f"brute/{s}/N"])
        got = sk.signature(X, N)
        assert rel_diff(golden[f"brute/{s}/brute"], got[0]) < 1e-10, s
        assert max(level_errors(got, golden[f"brute/{s}/seq"], X.shape[2], N)) <= F64_TOL, s


def test_golden_shape_grid_f64_and_f32(sk, golden):
    # test_kernels.cpp:128-146 grid (B {1,3}, L {2,5,17,64}, d {1,2,3,5}, N 1..5)
    for s in golden["grid/seeds"]:
        X, N = golden[f"grid/{s}/X"], int(golden[f"grid/{s}/N"])
        ref = golden[f"grid/{s}/seq"]
        assert max(level_errors(sk.signature(X, N), ref, X.shape[2], N)) <= F64_TOL, s
        # fp32: these unit-step random walks (not the 1/sqrt(L-1) benchmark scaling)
        # cancel heavily at high levels for d = 1, so the bar is the 1e-5 north-star
        # tolerance or 4x the error of the reference's OWN float instantiation
        # (sequential_forward<float>, via the bit-identical port), whichever is larger.
        X32 = X.astype(np.float32)
        ref32 = O.signature(X32.astype(np.float64), N)
        own = max(level_errors(O.signature(X32, N), ref32, X.shape[2], N))
        assert max(level_errors(sk.signature(X32, N), ref32, X.shape[2], N)) <= max(F32_TOL, 4 * own), s


def test_golden_wide_rows_and_c1(sk, golden):
    got = sk.signature(golden["wide/X"], 4)
    assert got.shape == (1, 11110)
    assert max(level_errors(got, golden["wide/seq"], 10, 4)) <= F64_TOL
    got = sk.signature(golden["c1/X"], 4)
    assert max(level_errors(got, golden["c1/seq"], 2, 4)) <= F64_TOL
    # the reference's own float instantiation is a looser check than the f64 oracle
    got32 = sk.signature(golden["c1/X32"], 4)
    assert max(level_errors(got32, golden["c1/seq"], 2, 4)) <= F32_TOL
    assert max(level_errors(got32, golden["c1/f32"], 2, 4)) <= F32_TOL


# --------------------------------------------------- the five BASELINE configs
@pytest.mark.parametrize("B,L,d,N", [(32, 100, 2, 4), (128, 1000, 5, 4), (128, 10000, 5, 4)])
def test_config_f32(sk, B, L, d, N):
    X = brownian(B, L, d)
    _, _, errs = check_f32(sk, X, N)
    print(f"B={B} L={L} d={d} N={N} f32 level errors {errs}")


def test_config_c4_f32(sk):
    # B=64 L=500 d=10 N=5 (D = 111,110)
    X = brownian(64, 500, 10)
    _, _, errs = check_f32(sk, X, 5)
    print("C4 f32 level errors", errs)


def test_config_c5_f32_all_rows(sk):
    # B=8192 L=1000 d=8 N=4: whole batch on the GPU, every row against the oracle
    X32 = brownian(8192, 1000, 8).astype(np.float32)
    got = sk.signature(X32, 4)
    ref = O.signature(X32.astype(np.float64), 4, threads=THREADS)
    errs = level_errors(got, ref, 8, 4)
    assert max(errs) <= F32_TOL, errs
    print("C5 f32 level errors (8192 rows)", errs)


@pytest.mark.parametrize("B,L,d,N", [(32, 100, 2, 4), (128, 1000, 5, 4), (16, 300, 8, 4), (4, 200, 10, 5)])
def test_config_f64(sk, B, L, d, N):
    check_f64(sk, brownian(B, L, d, seed=5), N)


# fp64 at the full BASELINE shapes (the reference's public precision,
# kernels.cpp:106-122 -> sig_core.hpp:116-147): C3, C4, C5 against the oracle
@pytest.mark.parametrize("B,L,d,N", [(128, 10000, 5, 4), (64, 500, 10, 5), (8192, 1000, 8, 4)],
                         ids=["c3", "c4", "c5"])
def test_config_full_f64(sk, B, L, d, N):
    _, _, errs = check_f64(sk, brownian(B, L, d, seed=6), N)
    print(f"B={B} L={L} d={d} N={N} f64 level errors {errs}")


# -------------------------------------------------------------- edge cases
def test_single_point_identity(sk):
    for dt in (np.float32, np.float64):
        out = sk.signature(np.random.default_rng(21).standard_normal((2, 1, 3)).astype(dt), 3)
        assert out.shape == (2, 39) and not out.any()


def test_two_point_restricted_exp(sk):
    X = np.random.default_rng(23).standard_normal((1, 2, 3))
    v = X[0, 1] - X[0, 0]
    assert max_abs_diff(sk.signature(X, 4)[0], O.restricted_exp(v, 4)) < 1e-14


def test_ragged_lengths_and_chunk_counts(sk):
    # chunking must not change the result beyond rounding (L-1 not a multiple of K)
    X = brownian(5, 257, 3, seed=9)
    ref = O.signature(X, 4)
    for K in (1, 2, 3, 7, 16, 64, 256):
        st = sk.KernelStats()
        got = sk.signature(X, 4, chunks=K, stats=st)
        assert 1 <= st.chunks <= max(K, 2)  # clamped to what fits one CTA (pair family: even)
        assert max(level_errors(got, ref, 3, 4)) <= F64_TOL, K
        got32 = sk.signature(X.astype(np.float32), 4, chunks=K)
        assert max(level_errors(got32, O.signature(X.astype(np.float32).astype(np.float64), 4), 3, 4)) <= F32_TOL


def test_every_fast_variant_and_generic(sk):
    rng = np.random.default_rng(17)
    shapes = [(d, N) for d in (1, 2, 3, 4, 5) for N in (1, 2, 3, 4, 5)] + \
             [(6, 4), (7, 3), (8, 4), (10, 4), (10, 5), (2, 6), (9, 3), (3, 7), (11, 2)]
    for d, N in shapes:
        X = brownian(3, 23, d, seed=int(rng.integers(1 << 30)))
        ref = O.signature(X, N)
        assert max(level_errors(sk.signature(X, N), ref, d, N)) <= F64_TOL, (d, N)
        assert max(level_errors(sk.signature_generic(X, N), ref, d, N)) <= F64_TOL, (d, N, "generic")
        X32 = X.astype(np.float32)
        ref32 = O.signature(X32.astype(np.float64), N)
        assert max(level_errors(sk.signature(X32, N), ref32, d, N)) <= F32_TOL, (d, N, "f32")


def test_batch_rows_bitwise_equal_single_rows(sk, golden):
    # test_kernels.cpp:252-263 (B=65), at pinned chunking
    X = golden["b65/X"]
    for dt in (np.float64, np.float32):
        Xd = X.astype(dt)
        allrows = sk.signature(Xd, 3, chunks=2)
        for b in (0, 17, 64):
            one = sk.signature(Xd[b:b + 1], 3, chunks=2)
            assert np.array_equal(one[0], allrows[b])
        assert max(level_errors(sk.signature(X, 3), golden["b65/seq"], 2, 3)) <= F64_TOL


def test_invalid_shapes(sk):
    with pytest.raises(sk.DomainError):
        sk.signature(np.zeros((1, 3, 2)), 0)
    with pytest.raises(sk.DomainError):
        sk.signature(np.zeros((0, 3, 2)), 2)
    with pytest.raises(sk.DomainError):
        sk.signature(np.zeros((3, 2)), 2)


# ------------------------------------------------ size-independent properties
def test_chen_split_full_size(sk):
    # S(X) = S(head) ⊠ S(tail) at the headline shape, fp64
    X = brownian(4, 1000, 5, seed=3)
    full = sk.signature(X, 4)
    a, b = sk.signature(X[:, :401], 4), sk.signature(X[:, 400:], 4)
    for i in range(4):
        joined = O.chen_product(5, 4, a[i], b[i])
        assert max(level_errors(joined, full[i], 5, 4)) < 1e-11


def test_translation_scaling_reversal(sk):
    X = brownian(3, 500, 4, seed=12)
    base = sk.signature(X, 4)
    moved = sk.signature(X + np.array([3.25, -1.75, 0.5, 2.0]), 4)
    assert max(level_errors(moved, base, 4, 4)) < 1e-11
    off = level_offsets(4, 4)
    for lam in (-1.0, 0.5, 2.0):
        sc = sk.signature(X * lam, 4)
        for n in range(4):
            a, b = sc[:, off[n]:off[n + 1]], base[:, off[n]:off[n + 1]] * lam ** (n + 1)
            assert np.max(np.abs(a - b)) <= 1e-11 * max(1.0, np.max(np.abs(b)))
    rev = sk.signature(X[:, ::-1].copy(), 4)
    for i in range(3):
        prod = O.chen_product(4, 4, base[i], rev[i])
        assert np.max(np.abs(prod)) < 1e-10


def test_device_tensors_and_stream(sk):
    torch = pytest.importorskip("torch")
    X = torch.from_numpy(brownian(128, 1000, 5).astype(np.float32)).cuda()
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        out = sk.signature(X, 4)
    s.synchronize()
    ref = O.signature(X.cpu().numpy().astype(np.float64), 4, threads=THREADS)
    assert max(level_errors(out.cpu().numpy(), ref, 5, 4)) <= F32_TOL


def test_device_brownian_generator_shard_invariant(sk):
    torch = pytest.importorskip("torch")
    full = sk.brownian(torch.empty((64, 50, 3), device="cuda"), seed=42)
    part = sk.brownian(torch.empty((16, 50, 3), device="cuda"), seed=42, row0=32)
    assert torch.equal(full[32:48], part)
    assert torch.all(full[:, 0] == 0)
    inc = (full[:, 1:] - full[:, :-1]).double()
    assert abs(inc.std().item() * np.sqrt(49) - 1.0) < 0.05


def test_sharded_entry_matches_single(sk):
    X = brownian(100, 300, 5, seed=4).astype(np.float32)
    a = sk.signature(X, 4)
    b = sk.signature_sharded(X, 4, num_gpus=0)
    assert np.array_equal(a, b)


def test_back_to_back_launches_overlap_safely(sk):
    # consecutive calls on one stream may overlap (programmatic dependent launch);
    # every result must still be exact and ordered
    torch = pytest.importorskip("torch")
    Xs = [torch.from_numpy(brownian(128, 1000, 5, seed=50 + i).astype(np.float32)).cuda() for i in range(6)]
    outs = [torch.empty((128, 780), device="cuda") for _ in Xs]
    shared = torch.empty((128, 780), device="cuda")
    for X, o in zip(Xs, outs):
        sk.signature(X, 4, out=o)
        sk.signature(X, 4, out=shared)  # write-after-write on one buffer
    torch.cuda.synchronize()
    for X, o in zip(Xs, outs):
        ref = O.signature(X.cpu().numpy().astype(np.float64), 4, threads=THREADS)
        assert max(level_errors(o.cpu().numpy(), ref, 5, 4)) <= F32_TOL
    assert torch.equal(shared, outs[-1])


def test_input_produced_by_previous_call_is_serialised(sk):
    # read-after-write through the library: the second call's paths ARE the first call's output
    torch = pytest.importorskip("torch")
    X1 = torch.from_numpy(brownian(64, 300, 3, seed=8).astype(np.float32)).cuda()
    out1 = torch.empty((64, 39), device="cuda")  # d=3, N=3 -> D=39 = 13 points x 3 channels
    for _ in range(3):
        sk.signature(X1, 3, out=out1)
        out2 = sk.signature(out1.view(64, 13, 3), 3)
    torch.cuda.synchronize()
    ref1 = O.signature(X1.cpu().numpy().astype(np.float64), 3, threads=THREADS)
    X2 = out1.cpu().numpy().reshape(64, 13, 3).astype(np.float64)
    assert max(level_errors(out1.cpu().numpy(), ref1, 3, 3)) <= F32_TOL
    assert max(level_errors(out2.cpu().numpy(), O.signature(X2, 3), 3, 3)) <= F32_TOL


@pytest.mark.parametrize("B,L,d,N", [(6, 1000, 9, 3), (4, 500, 3, 7), (3, 1500, 2, 9), (8, 700, 12, 2), (5, 300, 5, 4)])
def test_generic_chunk_parallel_long_paths(sk, B, L, d, N):
    # shapes without a register-sliced variant (and the forced generic family):
    # chunk-parallel walks + the fixed-order product of the chunk signatures
    X = brownian(B, L, d, seed=L + d)
    ref = O.signature(X, N, threads=THREADS)
    st = sk.KernelStats()
    got = sk.signature_generic(X, N, stats=st)
    assert max(level_errors(got, ref, d, N)) <= F64_TOL
    X32 = X.astype(np.float32)
    ref32 = O.signature(X32.astype(np.float64), N, threads=THREADS)
    assert max(level_errors(sk.signature_generic(X32, N), ref32, d, N)) <= F32_TOL
    rows = sk.signature_stream(X, N, family=sk.FAMILY_GENERIC)
    _, ref_rows = O.signature(X[:2], N, stream=True)
    assert np.max(np.abs(rows[:2] - ref_rows)) <= 1e-12 * np.max(np.abs(ref_rows))


@pytest.mark.parametrize("B,L,d,N", [(2, 200001, 3, 4), (1, 100001, 5, 4), (3, 50001, 2, 6)])
def test_very_long_paths(sk, B, L, d, N):
    # paths far longer than any BASELINE config: many segments per path (in-launch
    # segment combine) in fp32, fp64 against the oracle at 1e-12
    X = brownian(B, L, d, seed=L % 1000)
    st = sk.KernelStats()
    X32 = X.astype(np.float32)
    ref32 = O.signature(X32.astype(np.float64), N, threads=THREADS)
    own = max(level_errors(O.signature(X32, N), ref32, d, N))  # the reference's own float error
    got = sk.signature(X32, N, stats=st)
    assert max(level_errors(got, ref32, d, N)) <= max(F32_TOL, 4 * own)
    assert st.path_steps == L - 1
    assert max(level_errors(sk.signature(X, N), O.signature(X, N, threads=THREADS), d, N)) <= 1e-12


@pytest.mark.parametrize("B,L,d,N", [(500000, 3, 4, 4), (200000, 2, 5, 3), (100000, 17, 2, 5)])
def test_very_large_batches_of_short_paths(sk, B, L, d, N):
    # hundreds of thousands of short paths in one call (grids far past one wave); rows
    # checked on a random sample against the oracle
    X = brownian(B, L, d, seed=B % 997)
    X32 = X.astype(np.float32)
    got32 = sk.signature(X32, N)
    got64 = sk.signature(X, N)
    rows = np.random.default_rng(B).choice(B, 512, replace=False)
    ref = O.signature(X[rows], N)
    ref32 = O.signature(X32[rows].astype(np.float64), N)
    assert max(level_errors(got64[rows], ref, d, N)) <= 1e-12
    assert max(level_errors(got32[rows], ref32, d, N)) <= F32_TOL
