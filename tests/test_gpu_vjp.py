"""GPU parity of the reverse mode (reference signature_vjp,
/root/reference/proj/src/autodiff.cpp:218-224) against the reference itself
(compiled from its sources into oracle/_ref) and its finite differences
(autodiff.cpp:226-266), mirroring tests/test_autodiff.cpp:73-130 and the
acceptance gate's gradient criterion (acceptance.cpp:211-270).
Bars: fp64 relative 1e-10 against the reference adjoint; fp32 relative 1e-4
(two passes of fp32 accumulation over the path)."""
import numpy as np
import pytest

from oracle import oracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def need_ref():
    if O.ref() is None:
        pytest.skip("oracle/_ref (the compiled reference) is not built")


def walk(B, L, d, seed, scale=None):
    rng = np.random.default_rng(seed)
    X = np.zeros((B, L, d))
    if L > 1:
        X[:, 1:] = np.cumsum(rng.standard_normal((B, L - 1, d)) * (scale or 1 / np.sqrt(L - 1)), axis=1)
    return X


def rel(a, b):
    return float(np.max(np.abs(a - b)) / max(1e-30, np.max(np.abs(b))))


@pytest.mark.parametrize("B,L,d,N", [(2, 2, 3, 3), (3, 7, 2, 4), (2, 33, 3, 3), (2, 50, 5, 4), (1, 20, 1, 5), (2, 40, 10, 3), (5, 70, 4, 4), (3, 64, 6, 3),
                                     (2, 12, 4, 2), (2, 9, 2, 1)])
def test_vjp_f64_matches_reference(sk, B, L, d, N):
    X = walk(B, L, d, seed=B * 100 + L)
    cot = np.random.default_rng(L).standard_normal((B, sk.sig_dim(d, N)))
    got = sk.signature_vjp(X, N, cot)
    ref = O.ref_vjp(X, N, cot)
    assert got.shape == X.shape
    assert rel(got, ref) <= 1e-10, rel(got, ref)


def test_vjp_matches_finite_differences(sk):
    X = walk(2, 6, 3, seed=4)
    cot = np.random.default_rng(5).standard_normal((2, sk.sig_dim(3, 3)))
    got = sk.signature_vjp(X, 3, cot)
    fd = O.ref_finite_diff(X, 3, cot, 1e-5)
    assert np.max(np.abs(got - fd)) <= 1e-6 * (1 + np.max(np.abs(fd)))


def test_vjp_single_point_and_linearity(sk):
    X = walk(2, 1, 3, seed=1)
    assert not sk.signature_vjp(X, 3, np.ones((2, 39))).any()
    X = walk(3, 40, 3, seed=2)
    c1 = np.random.default_rng(3).standard_normal((3, 39))
    c2 = np.random.default_rng(4).standard_normal((3, 39))
    g = sk.signature_vjp(X, 3, 2.0 * c1 - c2)
    assert rel(g, 2.0 * sk.signature_vjp(X, 3, c1) - sk.signature_vjp(X, 3, c2)) <= 1e-11


def test_vjp_f32_headline_shape(sk):
    X = walk(8, 1000, 5, seed=7)
    cot = np.random.default_rng(8).standard_normal((8, 780))
    ref = O.ref_vjp(X.astype(np.float32).astype(np.float64), 4, cot.astype(np.float32).astype(np.float64))
    got = sk.signature_vjp(X.astype(np.float32), 4, cot.astype(np.float32))
    assert rel(got, ref) <= 1e-4, rel(got, ref)


def test_vjp_device_tensors(sk):
    torch = pytest.importorskip("torch")
    X = torch.from_numpy(walk(4, 64, 3, seed=9)).cuda()
    cot = torch.randn(4, 39, dtype=torch.float64, device="cuda")
    g = sk.signature_vjp(X, 3, cot)
    torch.cuda.synchronize()
    ref = O.ref_vjp(X.cpu().numpy(), 3, cot.cpu().numpy())
    assert rel(g.cpu().numpy(), ref) <= 1e-10


def test_vjp_shape_errors(sk):
    with pytest.raises(sk.DomainError):
        sk.signature_vjp(np.zeros((2, 5, 3)), 3, np.zeros((2, 38)))
    with pytest.raises(sk.DomainError):
        sk.signature_vjp(np.zeros((2, 5, 3)), 0, np.zeros((2, 39)))


@pytest.mark.parametrize("chunks", [2, 3, 7])
def test_vjp_chunked_matches_single_walk(sk, chunks):
    # boundary cotangents through chunk signatures == one sequential backward walk
    X = walk(3, 101, 3, seed=21)
    cot = np.random.default_rng(22).standard_normal((3, sk.sig_dim(3, 4)))
    st = sk.KernelStats()
    one = sk.signature_vjp(X, 4, cot, chunks=1, stats=st)
    assert st.chunks == 1
    got = sk.signature_vjp(X, 4, cot, chunks=chunks, stats=st)
    assert st.chunks == chunks
    assert rel(got, one) <= 1e-11
    assert rel(got, O.ref_vjp(X, 4, cot)) <= 1e-10


@pytest.mark.parametrize("chunks", [0, 10, 2])
def test_vjp_f32_long_chunks(sk, chunks):
    # long chunks: the slice adjoint recovers states by inverse steps over up to 5000 steps in fp32
    X = walk(2, 10000, 5, seed=17)
    cot = np.random.default_rng(18).standard_normal((2, 780))
    st = sk.KernelStats()
    got = sk.signature_vjp(X.astype(np.float32), 4, cot.astype(np.float32), stats=st, chunks=chunks)
    ref = O.ref_vjp(X.astype(np.float32).astype(np.float64), 4, cot.astype(np.float32).astype(np.float64))
    print("chunks", st.chunks, "steps per chunk", st.fold_steps, "rel", rel(got, ref))
    assert rel(got, ref) <= 1e-4, rel(got, ref)


def test_vjp_many_chunks_streamed_passes(sk):
    # (U + 4) D fp64 values exceed the chunk pass's shared-memory budget: the
    # chunk signatures are streamed one row per step instead of staged up front
    X = walk(2, 600, 5, seed=23)
    cot = np.random.default_rng(24).standard_normal((2, sk.sig_dim(5, 4)))
    st = sk.KernelStats()
    got = sk.signature_vjp(X, 4, cot, chunks=30, stats=st)
    assert st.chunks == 30
    assert rel(got, O.ref_vjp(X, 4, cot)) <= 1e-10


def test_signature_autograd_gradcheck_and_training_step(sk):
    # torch.autograd over the GPU forward + reverse mode: finite-difference gradcheck
    # (fp64), and the fp32 gradient against the compiled reference's adjoint
    torch = pytest.importorskip("torch")
    g = torch.Generator().manual_seed(5)
    X = torch.randn((2, 9, 3), generator=g, dtype=torch.float64).cumsum(1).mul(0.3).cuda().requires_grad_(True)
    assert torch.autograd.gradcheck(lambda x: sk.signature_autograd(x, 3), (X,), eps=1e-6, atol=1e-7)
    X32 = torch.randn((4, 200, 5), generator=g).cumsum(1).mul(0.05).cuda().requires_grad_(True)
    w = torch.randn(sk.sig_dim(5, 4), generator=g).cuda()
    loss = (sk.signature_autograd(X32, 4) * w).sum()
    loss.backward()
    from oracle import oracle as O

    if O.ref() is not None:
        cot = w.double().cpu().numpy()[None].repeat(4, 0)
        ref = O.ref_vjp(X32.detach().double().cpu().numpy(), 4, cot)
        got = X32.grad.double().cpu().numpy()
        assert np.abs(got - ref).max() <= 1e-4 * np.abs(ref).max()


@pytest.mark.parametrize("B,L,d,N", [(4, 1000, 5, 4), (3, 1200, 3, 4), (2, 800, 2, 5), (5, 900, 4, 3), (4, 1000, 1, 5),
                                     (2, 900, 6, 3), (3, 1500, 8, 2)])
def test_vjp_f32_fold_and_passes_in_one_launch(sk, B, L, d, N):
    # fp32, one wave of paths long enough: one launch folds every path's chunks and runs
    # both chunk passes in shared memory (vjp_prep.cuh), then the walk -- 2 launches
    X = walk(B, L, d, seed=L + d).astype(np.float32)
    cot = np.random.default_rng(d).standard_normal((B, sk.sig_dim(d, N))).astype(np.float32)
    st = sk.KernelStats()
    got = sk.signature_vjp(X, N, cot, stats=st)
    assert st.launches == 2 and st.chunks >= 2, (st.launches, st.chunks)
    ref = O.ref_vjp(X.astype(np.float64), N, cot.astype(np.float64))
    assert rel(got, ref) <= 1e-4, rel(got, ref)
    # the separate chunk-signature and pass launches at the same chunking agree
    sep = sk.signature_vjp(X, N, cot, chunks=st.chunks, stats=st)
    assert st.launches >= 3
    assert rel(got, sep) <= 2e-5, rel(got, sep)


@pytest.mark.parametrize("L", [1000, 300])
def test_vjp_graph_capture_replay(sk, L):
    # reverse mode captured into a CUDA graph (the fold-and-passes launch at L = 1000, the
    # three-launch form at L = 300) replays to the eager result, also after the stream's
    # scratch grew in between
    torch = pytest.importorskip("torch")
    s = torch.cuda.Stream()
    X = torch.from_numpy(walk(8, L, 5, seed=L).astype(np.float32)).cuda()
    cot = torch.from_numpy(np.random.default_rng(L).standard_normal((8, 780)).astype(np.float32)).cuda()
    with torch.cuda.stream(s):
        eager = sk.signature_vjp(X, 4, cot).clone()
    s.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        out = sk.signature_vjp(X, 4, cot)
    big = torch.from_numpy(walk(64, L, 5, seed=L + 1).astype(np.float32)).cuda()
    bcot = torch.randn(64, 780, device="cuda")
    with torch.cuda.stream(s):
        sk.signature_vjp(big, 4, bcot)  # may grow this stream's scratch
        out.zero_()
        g.replay()
    s.synchronize()
    assert torch.equal(out, eager)


def test_vjp_prep_wave_boundary(sk):
    # B = SMs: one fold-and-passes wave; B = SMs + 1: the three-launch form; same gradients
    torch = pytest.importorskip("torch")
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    X = walk(sms + 1, 800, 3, seed=77).astype(np.float32)
    cot = np.random.default_rng(78).standard_normal((sms + 1, sk.sig_dim(3, 4))).astype(np.float32)
    st = sk.KernelStats()
    a = sk.signature_vjp(X[:sms], 4, cot[:sms], stats=st)
    assert st.launches == 2
    b = sk.signature_vjp(X, 4, cot, stats=st)
    assert st.launches >= 3
    assert rel(a, b[:sms]) <= 2e-5


@pytest.mark.parametrize("B,L,d,N", [(16, 1000, 5, 4), (8, 500, 10, 3), (4, 10000, 5, 4)])
def test_vjp_f64_full_length(sk, B, L, d, N):
    # fp64 reverse mode at the BASELINE path lengths (C2 and C3 shapes on a row subset,
    # C4's d = 10 at depth 3: the element-parallel adjoint) against the reference's adjoint
    X = walk(B, L, d, seed=L + d)
    cot = np.random.default_rng(L + 1).standard_normal((B, sk.sig_dim(d, N)))
    got = sk.signature_vjp(X, N, cot)
    assert rel(got, O.ref_vjp(X, N, cot)) <= 1e-10


def test_vjp_very_long_paths(sk):
    # 100K steps per path, two paths: hundreds of chunks per path (the chunk passes
    # stream their rows instead of staging them), fp64 and fp32 against the reference
    X = walk(2, 100001, 3, seed=91)
    cot = np.random.default_rng(92).standard_normal((2, sk.sig_dim(3, 4)))
    st = sk.KernelStats()
    ref = O.ref_vjp(X, 4, cot)
    assert rel(sk.signature_vjp(X, 4, cot, stats=st), ref) <= 1e-10
    assert st.chunks > 100
    g32 = sk.signature_vjp(X.astype(np.float32), 4, cot.astype(np.float32))
    ref32 = O.ref_vjp(X.astype(np.float32).astype(np.float64), 4, cot.astype(np.float32).astype(np.float64))
    assert rel(g32, ref32) <= 1e-4, rel(g32, ref32)


def test_vjp_very_large_batch(sk):
    # 200K short paths in one reverse-mode call, rows sampled against the reference
    X = walk(200000, 12, 3, seed=93)
    cot = np.random.default_rng(94).standard_normal((200000, sk.sig_dim(3, 4)))
    g = sk.signature_vjp(X, 4, cot)
    rows = np.random.default_rng(95).choice(200000, 256, replace=False)
    assert rel(g[rows], O.ref_vjp(X[rows], 4, cot[rows])) <= 1e-10
