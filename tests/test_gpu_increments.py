"""GPU increments / scaled increments (reference kernels.cpp:71-104) against
the compiled reference: fp64 bit-identical (one IEEE subtraction, one
division by the running double factorial); fp32 bit-identical to the same
IEEE operations in numpy."""
import math

import numpy as np
import pytest

from oracle import oracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def need_ref():
    if O.ref() is None:
        pytest.skip("oracle/_ref (the compiled reference) is not built")


@pytest.mark.parametrize("B,L,d", [(1, 2, 1), (3, 7, 2), (5, 100, 5), (2, 1, 3), (65, 33, 10), (7, 50, 4), (3, 9, 8)])
def test_increments_match_reference(sk, B, L, d):
    X = np.random.default_rng(B * L + d).standard_normal((B, L, d))
    got = sk.increments(X)
    ref = O.ref_increments(X)
    assert got.shape == (B, L - 1, d)
    assert np.array_equal(got, ref)
    got32 = sk.increments(X.astype(np.float32))
    X32 = X.astype(np.float32)
    assert np.array_equal(got32, X32[:, 1:] - X32[:, :-1])


@pytest.mark.parametrize("depth", [1, 2, 4, 7])
def test_scaled_increments_match_reference(sk, depth):
    X = np.random.default_rng(depth).standard_normal((4, 50, 3))
    inc = sk.increments(X)
    got = sk.scaled_increments(inc, depth)
    ref = O.ref_scaled_increments(inc, depth)
    assert len(got) == depth - 1 == len(ref)
    for g, r in zip(got, ref):
        assert np.array_equal(g, r)
    if depth > 1:
        assert np.array_equal(got[-1], inc / float(math.factorial(depth)))


def test_increments_device_tensors(sk):
    torch = pytest.importorskip("torch")
    X = torch.randn(8, 300, 5, dtype=torch.float64, device="cuda")
    got = sk.increments(X)
    torch.cuda.synchronize()
    assert torch.equal(got, X[:, 1:] - X[:, :-1])


def test_increments_errors(sk):
    with pytest.raises(sk.DomainError):
        sk.increments(np.zeros((0, 3, 2)))
    with pytest.raises(sk.DomainError):
        sk.scaled_increments(np.zeros((1, 2, 2)), 0)


@pytest.mark.parametrize("L,d,N", [(1, 2, 2), (2, 3, 4), (5, 2, 3), (9, 3, 4), (9, 1, 4), (4, 3, 1)])
def test_bruteforce_matches_reference(sk, L, d, N):
    # reference signature_bruteforce (oracle.cpp:28-96), both tuple classes, fp64 bit-identical
    path = np.random.default_rng(L * 10 + d).standard_normal((L, d))
    assert np.array_equal(sk.signature_bruteforce(path, N), O.ref_bruteforce(path, N))
    assert np.array_equal(sk.signature_bruteforce(path, N, strict=True), O.ref_bruteforce_strict(path, N))


def test_bruteforce_limits(sk):
    with pytest.raises(sk.ResourceError):
        sk.signature_bruteforce(np.zeros((10, 2)), 3)  # 9 segments > 8
    with pytest.raises(sk.ResourceError):
        sk.signature_bruteforce(np.zeros((3, 4)), 2)  # dim 4 > 3
    with pytest.raises(sk.DomainError):
        sk.signature_bruteforce(np.zeros((3, 2)), 0)
    big = sk.signature_bruteforce(np.random.default_rng(0).standard_normal((12, 2)), 5, max_segments=11, max_depth=5)
    assert big.shape == (62,)
