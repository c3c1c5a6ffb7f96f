"""GPU parity of the paper's parallel formulation (KernelKind::Parallel):
sigk_signature_parallel_* runs the per-degree cumulative-sum passes of the
reference's detail::parallel_forward (sig_core.hpp:175-298) as GPU scans.

Checked against the pinned oracle (the sequential fold, the reference's
contract) and against the compiled reference's own
parallel_forward; fp64 <= 1e-12 and fp32 <= 1e-5 per level (north_star).
Also the scratch-lifetime regression of the pair family's segmented plans.
"""
import os

import numpy as np
import pytest

from oracle import oracle as O
from tests.helpers import level_errors

pytestmark = pytest.mark.gpu

THREADS = os.cpu_count() or 1


def brownian(B, L, d, seed=42):
    rng = np.random.default_rng(seed)
    X = np.zeros((B, L, d), np.float64)
    if L > 1:
        X[:, 1:] = np.cumsum(rng.standard_normal((B, L - 1, d)) / np.sqrt(L - 1), axis=1)
    return X


@pytest.mark.parametrize("B,L,d,N", [(3, 2, 3, 4), (5, 17, 1, 5), (4, 64, 2, 6), (3, 130, 5, 4), (2, 33, 10, 3)])
def test_parallel_matches_oracle_and_reference_parallel(sk, B, L, d, N):
    X = brownian(B, L, d, seed=B * L + d)
    st = sk.KernelStats()
    got = sk.signature_parallel(X, N, stats=st)
    assert st.family == sk.FAMILY_SCAN and st.scan_passes == N and st.fold_steps == 0 and st.launches == N
    assert max(level_errors(got, O.signature(X, N), d, N)) <= 1e-12
    if O.ref() is not None:
        assert max(level_errors(got, O.ref_signature(X, N, kernel="parallel"), d, N)) <= 1e-12


def test_parallel_golden_grid(sk, golden):
    # the 800-instance cross-kernel grid's shapes (test_kernels.cpp:128-146)
    for s in golden["grid/seeds"]:
        X, N = golden[f"grid/{s}/X"], int(golden[f"grid/{s}/N"])
        assert max(level_errors(sk.signature_parallel(X, N), golden[f"grid/{s}/seq"], X.shape[2], N)) <= 1e-12, s


def test_parallel_headline_shape_f64_and_f32(sk):
    X = brownian(128, 1000, 5, seed=7)
    ref = O.signature(X, 4, threads=THREADS)
    assert max(level_errors(sk.signature_parallel(X, 4), ref, 5, 4)) <= 1e-12
    X32 = X.astype(np.float32)
    ref32 = O.signature(X32.astype(np.float64), 4, threads=THREADS)
    assert max(level_errors(sk.signature_parallel(X32, 4), ref32, 5, 4)) <= 1e-5


def test_parallel_prefix_rows_match_stream(sk):
    X = brownian(4, 200, 3, seed=11)
    _, ref_rows = O.signature(X, 4, stream=True)
    got = sk.signature_stream(X, 4, kernel=sk.KernelKind.Parallel)
    assert got.shape == ref_rows.shape
    assert np.max(np.abs(got - ref_rows)) <= 1e-12 * np.max(np.abs(ref_rows))
    seq = sk.signature_stream(X, 4, kernel=sk.KernelKind.Sequential)
    assert np.max(np.abs(got - seq)) <= 1e-12 * np.max(np.abs(ref_rows))
    with pytest.raises(sk.DomainError):
        sk.signature_stream(X[:, :1], 4, kernel=sk.KernelKind.Parallel)


def test_parallel_identity_and_memory_cap(sk):
    st = sk.KernelStats()
    out = sk.signature_parallel(np.ones((3, 1, 4)), 3, stats=st)
    assert out.shape == (3, 84) and not out.any() and st.scan_passes == 3
    with pytest.raises(sk.ResourceError, match="parallel kernel: intermediate storage of ~"):
        sk.signature_parallel(brownian(2, 100, 3), 4, memory_cap=1000)
    # the reference's default cap refuses C4 (3.2e9 scalars), like sig_core.hpp:161-173
    with pytest.raises(sk.ResourceError, match="exceeds cap 2147483648"):
        sk.signature_parallel(np.zeros((64, 500, 10), np.float32), 5)


def test_auto_dispatch_follows_caps(sk):
    X = brownian(2, 80, 3, seed=3)
    st = sk.KernelStats()
    sk.signature(X, 3, caps=sk.ExecutionCaps(accelerated=True), stats=st)
    assert st.family == sk.FAMILY_SCAN
    sk.signature(X, 3, caps=sk.ExecutionCaps(accelerated=False), stats=st)
    assert st.family != sk.FAMILY_SCAN and st.path_steps == 79
    sk.signature(X[:, :60], 3, caps=sk.ExecutionCaps(accelerated=True), stats=st)  # 60 < parallel_min_len
    assert st.family != sk.FAMILY_SCAN and st.path_steps == 59


def test_parallel_device_tensors(sk):
    torch = pytest.importorskip("torch")
    X = torch.from_numpy(brownian(16, 300, 4, seed=2)).cuda()
    out = sk.signature_parallel(X, 4)
    ref = O.signature(X.cpu().numpy(), 4)
    assert max(level_errors(out.cpu().numpy(), ref, 4, 4)) <= 1e-12
    rows = sk.signature_stream(X.float(), 3, kernel=sk.KernelKind.Parallel)
    _, ref_rows = O.signature(X.float().cpu().numpy().astype(np.float64), 3, stream=True)
    assert np.max(np.abs(rows.cpu().numpy() - ref_rows)) <= 1e-5 * np.max(np.abs(ref_rows))


def test_segment_scratch_survives_growth_under_graph_replay(sk):
    # A graph captured with a segmented (G > 1) plan keeps the scratch pointer it
    # was captured with; a later, larger call on the same stream grows the scratch.
    # Replaying the graph afterwards must still write into live memory.
    torch = pytest.importorskip("torch")
    s = torch.cuda.Stream()
    X = torch.from_numpy(brownian(8, 2000, 5, seed=31).astype(np.float32)).cuda()
    out = torch.empty((8, 780), device="cuda")
    with torch.cuda.stream(s):
        sk.signature(X, 4, segments=4, out=out)  # allocates the stream's scratch outside the capture
    s.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        sk.signature(X, 4, segments=4, out=out)
    big = torch.from_numpy(brownian(256, 2000, 5, seed=32).astype(np.float32)).cuda()
    with torch.cuda.stream(s):
        big_out = sk.signature(big, 4, segments=4)  # grows the scratch of this stream
        out.zero_()
        for _ in range(3):
            g.replay()
    s.synchronize()
    ref = O.signature(X.cpu().numpy().astype(np.float64), 4)
    assert max(level_errors(out.cpu().numpy(), ref, 5, 4)) <= 1e-5
    ref_big = O.signature(big.cpu().numpy().astype(np.float64)[:16], 4)
    assert max(level_errors(big_out.cpu().numpy()[:16], ref_big, 5, 4)) <= 1e-5


# ---- reverse mode of the parallel formulation (KernelKind::Parallel -> vjp_parallel,
# autodiff.cpp:108-214): GPU suffix scans + per-position contractions (scan_vjp.cuh)

def _rel(a, b):
    return float(np.max(np.abs(a - b)) / max(np.max(np.abs(b)), 1e-300))


@pytest.mark.parametrize("B,L,d,N", [(3, 2, 3, 3), (2, 9, 2, 4), (4, 33, 3, 4), (2, 40, 5, 3), (3, 17, 1, 5), (2, 12, 4, 1)])
def test_parallel_vjp_matches_reference_vjp_parallel(sk, B, L, d, N):
    X = brownian(B, L, d, seed=7 * L + d)
    rng = np.random.default_rng(B + L)
    cot = rng.standard_normal((B, sk.sig_dim(d, N)))
    st = sk.KernelStats()
    g = sk.signature_vjp(X, N, cot, kernel=sk.KernelKind.Parallel, stats=st)
    assert st.family == sk.FAMILY_SCAN and st.scan_passes == 2 * N
    if O.ref() is not None:
        assert _rel(g, O.ref_vjp(X, N, cot, kernel="parallel")) <= 1e-12
    # the two GPU adjoints agree (test_autodiff.cpp:117-130)
    g_seq = sk.signature_vjp(X, N, cot, kernel=sk.KernelKind.Sequential)
    assert _rel(g, g_seq) <= 1e-10


def test_parallel_vjp_headline_shape_f32_and_device(sk):
    torch = pytest.importorskip("torch")
    X = brownian(32, 1000, 5, seed=3)
    cot = np.random.default_rng(3).standard_normal((32, 780))
    g64 = sk.signature_vjp(X, 4, cot, kernel=sk.KernelKind.Parallel)
    g_seq = sk.signature_vjp(X, 4, cot, kernel=sk.KernelKind.Sequential)
    assert _rel(g64, g_seq) <= 1e-10
    Xt = torch.from_numpy(X.astype(np.float32)).cuda()
    ct = torch.from_numpy(cot.astype(np.float32)).cuda()
    g32 = sk.signature_vjp(Xt, 4, ct, kernel=sk.KernelKind.Parallel)
    assert g32.is_cuda and g32.dtype == torch.float32
    assert _rel(g32.cpu().numpy().astype(np.float64), g64) <= 1e-4


def test_parallel_vjp_edges_and_cap(sk):
    cot = np.ones((2, sk.sig_dim(3, 2)))
    g = sk.signature_vjp(np.ones((2, 1, 3)), 2, cot, kernel=sk.KernelKind.Parallel)
    assert g.shape == (2, 1, 3) and not g.any()
    X = brownian(2, 2, 3, seed=5)  # one step: only the diagonal terms
    if O.ref() is not None:
        assert _rel(sk.signature_vjp(X, 2, cot, kernel=sk.KernelKind.Parallel), O.ref_vjp(X, 2, cot, kernel="parallel")) <= 1e-12
    with pytest.raises(sk.ResourceError, match="exceeds cap 2147483648"):
        sk.signature_vjp(np.zeros((64, 500, 10)), 5, np.zeros((64, sk.sig_dim(10, 5))), kernel=sk.KernelKind.Parallel)
    # Auto follows the caps, like the forward
    st = sk.KernelStats()
    sk.signature_vjp(brownian(2, 80, 3), 3, np.ones((2, 39)), caps=sk.ExecutionCaps(accelerated=True), stats=st)
    assert st.family == sk.FAMILY_SCAN
