"""GPU parity of the packed-FP32x2 pair family (pair_kernel.cuh) against the
CPU oracle, across its plan space: chunk counts (even, with empty chunks),
segment counts (the two-kernel segment combine), every registered (d, N),
and the determinism / batch-invariance properties the reference pins
(test_kernels.cpp:252-263). fp32 bar: per-level relative error <= 1e-5
(BASELINE.json north_star) against the oracle in float64 on the same
fp32-rounded inputs."""
import os

import numpy as np
import pytest

from oracle import oracle as O
from tests.helpers import level_errors

pytestmark = pytest.mark.gpu

F32_TOL = 1e-5
THREADS = os.cpu_count() or 1


def brownian(B, L, d, seed=42):
    rng = np.random.default_rng(seed)
    X = np.zeros((B, L, d), np.float64)
    if L > 1:
        X[:, 1:] = np.cumsum(rng.standard_normal((B, L - 1, d)) / np.sqrt(L - 1), axis=1)
    return X.astype(np.float32)


def oracle32(X, N):
    return O.signature(X.astype(np.float64), N, threads=THREADS)


def pair(sk, X, N, **kw):
    st = sk.KernelStats()
    got = sk.signature(X, N, stats=st, family=sk.FAMILY_PAIR, **kw)
    assert st.family == sk.FAMILY_PAIR, st
    return got, st


def test_plan_headline_uses_pair_family(sk):
    p = sk.plan(128, 1000, 5, 4)
    assert p.family == sk.FAMILY_PAIR and p.prefix_len == 2 and p.chunks % 2 == 0, p
    assert sk.plan(128, 1000, 5, 4, f64=True).family != sk.FAMILY_PAIR  # fp64 stays scalar


@pytest.mark.parametrize("U", [2, 4, 6, 10, 16, 20])
def test_headline_chunk_counts(sk, U):
    X = brownian(24, 1000, 5, seed=U)
    ref = oracle32(X, 4)
    got, st = pair(sk, X, 4, chunks=U, segments=1)
    assert st.chunks == U and st.segments == 1
    assert max(level_errors(got, ref, 5, 4)) <= F32_TOL


@pytest.mark.parametrize("G", [2, 3, 5, 8, 13])
def test_segments(sk, G):
    X = brownian(12, 1001, 5, seed=100 + G)
    ref = oracle32(X, 4)
    got, st = pair(sk, X, 4, segments=G)
    assert st.segments == G and st.launches == 1
    errs = level_errors(got, ref, 5, 4)
    assert max(errs) <= F32_TOL, errs


def test_long_path_segmented(sk):
    # C3 shape family: L = 10000 through the planned segment split
    X = brownian(16, 10000, 5, seed=7)
    ref = oracle32(X, 4)
    st = sk.KernelStats()
    got = sk.signature(X, 4, stats=st)
    errs = level_errors(got, ref, 5, 4)
    print("L=10000 plan", st, "errors", errs)
    assert max(errs) <= F32_TOL


def test_more_chunks_than_steps(sk):
    # empty chunks (start = end = M) must be exact identities
    for L in (2, 3, 5, 9):
        X = brownian(3, L, 5, seed=L)
        ref = oracle32(X, 4)
        for U in (2, 4, 8, 20):
            got, _ = pair(sk, X, 4, chunks=U)
            assert max(level_errors(got, ref, 5, 4)) <= F32_TOL, (L, U)


@pytest.mark.parametrize("d,N", [(1, 3), (1, 6), (2, 1), (2, 2), (2, 4), (2, 6), (3, 3), (3, 4), (4, 3), (4, 4),
                                 (5, 1), (5, 2), (5, 3), (5, 4), (6, 3), (7, 3), (8, 3), (10, 2), (10, 3)])
def test_every_pair_variant(sk, d, N):
    rng = np.random.default_rng(d * 31 + N)
    for L, G in ((2, 1), (37, 1), (301, 1), (301, 3)):
        X = brownian(3, L, d, seed=int(rng.integers(1 << 30)))
        ref = oracle32(X, N)
        if N == 1 and G > 1:
            continue
        got, _ = pair(sk, X, N, segments=G)
        # d = 1 levels are (X_T - X_0)^n / n! reached through heavy cancellation: the
        # bar is 1e-5 or 4x the error of the reference's own float instantiation
        own = max(level_errors(O.signature(X, N), ref, d, N))
        assert max(level_errors(got, ref, d, N)) <= max(F32_TOL, 4 * own), (d, N, L, G)


def test_pair_matches_path_family(sk):
    X = brownian(32, 700, 5, seed=11)
    a, _ = pair(sk, X, 4)
    st = sk.KernelStats()
    b = sk.signature(X, 4, stats=st, family=sk.FAMILY_PATH)
    assert st.family == sk.FAMILY_PATH
    assert max(level_errors(a, b, 5, 4)) <= 2 * F32_TOL


def test_deterministic_and_batch_invariant(sk):
    X = brownian(65, 513, 5, seed=3)
    a, _ = pair(sk, X, 4, chunks=8, segments=2)
    b, _ = pair(sk, X, 4, chunks=8, segments=2)
    assert np.array_equal(a, b)
    for r in (0, 31, 64):
        one, _ = pair(sk, X[r:r + 1], 4, chunks=8, segments=2)
        assert np.array_equal(one[0], a[r])


def test_headline_full_batch(sk):
    X = brownian(128, 1000, 5, seed=42)
    got, st = pair(sk, X, 4)
    errs = level_errors(got, oracle32(X, 4), 5, 4)
    print("C2 pair plan", st, "errors", errs)
    assert max(errs) <= F32_TOL


# ------------------------------------------------ inner-pair flat family (even d)
def pflat(sk, X, N):
    st = sk.KernelStats()
    got = sk.signature(X, N, stats=st, family=sk.FAMILY_PFLAT)
    assert st.family == sk.FAMILY_PFLAT, st
    return got, st


@pytest.mark.parametrize("d,N", [(2, 2), (2, 4), (2, 5), (4, 3), (4, 4), (4, 5), (6, 3), (6, 4), (8, 2), (8, 3),
                                 (8, 4), (10, 2), (10, 3), (10, 4), (10, 5)])
def test_pflat_every_variant(sk, d, N):
    rng = np.random.default_rng(d * 17 + N)
    for B, L in ((1, 2), (3, 37), (5, 301)):
        X = brownian(B, L, d, seed=int(rng.integers(1 << 30)))
        ref = oracle32(X, N)
        got, _ = pflat(sk, X, N)
        assert max(level_errors(got, ref, d, N)) <= F32_TOL, (d, N, B, L)


def test_pflat_plans_for_c4_c5(sk):
    assert sk.plan(64, 500, 10, 5).family == sk.FAMILY_PFLAT
    assert sk.plan(8192, 1000, 8, 4).family == sk.FAMILY_PATH  # measured faster for d = 8
    assert sk.plan(4, 500, 10, 5).family != sk.FAMILY_PFLAT  # too few lanes


def test_pflat_c4_shape(sk):
    X = brownian(64, 500, 10, seed=21)
    got, st = pflat(sk, X, 5)
    errs = level_errors(got, oracle32(X, 5), 10, 5)
    print("C4 pflat", st, errs)
    assert max(errs) <= F32_TOL


def test_pflat_c5_rows(sk):
    X = brownian(1000, 1000, 8, seed=22)  # 64000 lanes: ragged last CTA
    got, _ = pflat(sk, X, 4)
    for lo in (0, 500, 1000 - 40):
        errs = level_errors(got[lo:lo + 40], oracle32(X[lo:lo + 40], 4), 8, 4)
        assert max(errs) <= F32_TOL, (lo, errs)


# ---- the position-table fold with a producer warp (ppair_kernel.cuh)
@pytest.mark.parametrize("d,N", [(3, 4), (4, 4), (5, 3), (5, 4), (6, 3), (8, 3)])
def test_position_table_fold_shapes(sk, d, N):
    X = brownian(9, 301, d, seed=d * 10 + N)
    ref = oracle32(X, N)
    try:
        got, st = pair(sk, X, N, fold_variant=2)
    except sk.DeviceError:
        pytest.skip("no position-table instantiation for this shape")
    assert max(level_errors(got, ref, d, N)) <= F32_TOL, (d, N)


@pytest.mark.parametrize("U,G,L", [(2, 1, 1000), (4, 1, 997), (10, 1, 1000), (6, 1, 37), (10, 2, 1000),
                                   (8, 4, 2001), (10, 12, 10000), (10, 1, 2)])
def test_position_table_fold_plans(sk, U, G, L):
    # ragged chunk ends (empty / partial tiles), cluster and global segment combines
    X = brownian(7, L, 5, seed=U * 100 + G)
    ref = oracle32(X, 4)
    got, st = pair(sk, X, 4, fold_variant=2, chunks=U, segments=G)
    assert max(level_errors(got, ref, 5, 4)) <= F32_TOL, (U, G, L)


def test_position_table_fold_headline_and_batch_invariance(sk):
    X = brownian(128, 1000, 5, seed=77)
    ref = oracle32(X, 4)
    got, _ = pair(sk, X, 4, fold_variant=2, chunks=10, segments=1)
    assert max(level_errors(got, ref, 5, 4)) <= F32_TOL
    one, _ = pair(sk, X[5:6], 4, fold_variant=2, chunks=10, segments=1)
    assert np.array_equal(one[0], got[5])


@pytest.mark.parametrize("G", [2, 3, 4, 8])
def test_cluster_segment_combine(sk, G):
    # opt-in thread-block-cluster (DSMEM) segment combine: same arithmetic and
    # order as the global-scratch combine, hence bitwise the same rows
    X = brownian(10, 1201, 5, seed=300 + G)
    ref = oracle32(X, 4)
    got, st = pair(sk, X, 4, segments=G, cluster=1)
    assert st.segments == G
    assert max(level_errors(got, ref, 5, 4)) <= F32_TOL
    glob, _ = pair(sk, X, 4, segments=G, chunks=st.chunks)
    assert np.array_equal(got, glob)
