"""CPU: the C-ABI library loads, exports every symbol include/sigk.h declares,
and enforces the reference's argument checks without touching a GPU."""
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "sigk.h")).read()
    return sorted(set(re.findall(r"^\s*(?:int|const char\*)\s+(sigk_\w+)\s*\(", src, re.M)))


def test_header_declares_the_boundary():
    syms = declared_symbols()
    for s in ("sigk_sig_dim", "sigk_level_offsets", "sigk_signature_f32", "sigk_signature_f64",
              "sigk_signature_sharded_f32", "sigk_signature_sharded_f64", "sigk_last_error"):
        assert s in syms


def test_library_exports_every_declared_symbol(sk):
    lib = sk.lib()
    for s in declared_symbols():
        assert hasattr(lib, s), s


def test_library_is_built_for_sm100a():
    import subprocess

    so = os.path.join(ROOT, "paper_2501_08455_b200", "libsigk.so")
    r = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", so], capture_output=True, text=True)
    assert "sm_100a" in r.stdout


def test_sig_dim_and_offsets(sk):
    assert sk.sig_dim(10, 4) == 11110 and sk.sig_dim(2, 2) == 6 and sk.sig_dim(6, 3) == 258
    assert sk.level_offsets(5, 4) == [0, 5, 30, 155, 780]
    assert sk.level_sizes(3, 3) == [3, 9, 27]
    with pytest.raises(sk.DomainError):
        sk.sig_dim(0, 2)
    with pytest.raises(sk.DomainError):
        sk.sig_dim(2, 0)


def test_domain_errors_before_any_device_work(sk):
    with pytest.raises(sk.DomainError):
        sk.signature(np.zeros((1, 3, 2)), 0)
    with pytest.raises(sk.DomainError):
        sk.signature(np.zeros((0, 3, 2)), 2)
    with pytest.raises(sk.DomainError):
        sk.signature_parallel(np.zeros((2, 3, 2)), -1)
    with pytest.raises(sk.ResourceError):  # the reference's memory-cap refusal (test_kernels.cpp:265-270)
        sk.signature_parallel(np.zeros((4, 32, 3)), 3, memory_cap=1000)


def test_vjp_refuses_aliased_gradient(sk):
    # grad is written while the paths are still read: overlap is a domain error, raised before device work
    import ctypes as C

    X = np.zeros((2, 5, 3), np.float32)
    cot = np.zeros((2, 39), np.float32)
    lib = sk.lib()
    fp = C.POINTER(C.c_float)
    rc = lib.sigk_signature_vjp_f32(X.ctypes.data_as(fp), C.c_size_t(2), C.c_size_t(5), 3, 3, cot.ctypes.data_as(fp),
                                    X.ctypes.data_as(fp), C.c_uint(0), None, None, None)
    assert rc == 1
    assert b"overlap" in lib.sigk_last_error()


def test_no_silent_cpu_fallback_without_gpu(sk):
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(sk.DeviceError):
        sk.signature(np.zeros((2, 3, 2), np.float32), 2)


def test_fast_variants_cover_the_benchmark_shapes(sk):
    for d, N in ((2, 4), (5, 4), (10, 5), (8, 4)):
        assert sk.has_fast_variant(d, N)[0]
        assert sk.has_fast_variant(d, N, f64=True)[0]
    assert sk.has_fast_variant(5, 4) == (True, 1)
    assert sk.has_fast_variant(10, 5) == (True, 3)


def test_kernel_names_and_dispatch(sk):
    K = sk.KernelKind
    assert sk.kernel_from_name("parallel") is K.Parallel
    with pytest.raises(sk.DomainError):
        sk.kernel_from_name("gpu")
    accel, plain = sk.ExecutionCaps(True), sk.ExecutionCaps(False)
    assert sk.select_kernel(K.Auto, accel, 64) is K.Parallel
    assert sk.select_kernel(K.Auto, accel, 63) is K.Sequential
    assert sk.select_kernel(K.Auto, plain, 1000) is K.Sequential
    assert sk.select_kernel(K.Parallel, plain, 2) is K.Parallel


def test_make_bench_paths_matches_reference(sk):
    # the reference's own generator (bench.cpp:134-161) compiled from its sources
    import ctypes as C

    from oracle import oracle as O

    if O.ref() is None:
        pytest.skip("oracle/_ref (the compiled reference) is not built")
    lib = sk.lib()
    lib.sigk_make_bench_paths.argtypes = [C.c_uint64, C.c_size_t, C.c_size_t, C.c_int, C.c_void_p]
    for seed, B, L, d in ((42, 3, 50, 2), (7, 2, 1, 3), (123456789, 4, 17, 5)):
        got = np.empty((B, L, d))
        assert lib.sigk_make_bench_paths(seed, B, L, d, got.ctypes.data) == 0
        assert np.array_equal(got, O.ref_make_bench_paths(seed, B, L, d))


def test_sigbench_cli_rejects_bad_flags():
    import subprocess

    exe = os.path.join(ROOT, "tools", "sigbench")
    if not os.path.exists(exe):
        pytest.skip("tools/sigbench not built")
    r = subprocess.run([exe, "--dims", "0"], capture_output=True, text=True)
    assert r.returncode == 1 and "--dims entries must be positive" in r.stderr
    r = subprocess.run([exe, "--dtype", "f16"], capture_output=True, text=True)
    assert r.returncode == 1


def test_out_argument_validated_before_any_device_work(sk):
    # a wrong `out` must be refused before its pointer reaches the C ABI
    X = np.zeros((2, 5, 3))
    for bad in (np.empty((2, 38)), np.empty((2, 39), np.float32), np.empty((39, 2)).T):
        with pytest.raises(sk.DomainError):
            sk.signature(X, 3, out=bad)
    with pytest.raises(sk.DomainError):
        sk.signature_stream(X, 3, out=np.empty((2, 5, 39)))
    with pytest.raises(sk.DomainError):
        sk.signature_parallel(X, 3, out=np.empty((2, 4, 39)))


def test_reference_dispatch_defaults(sk, monkeypatch):
    # kernels.hpp:80 (accelerated = false), kernels.cpp:64-69 (detect)
    K = sk.KernelKind
    assert sk.ExecutionCaps().accelerated is False
    monkeypatch.delenv("SIGKIT_ACCELERATED", raising=False)
    assert sk.ExecutionCaps.detect().accelerated is False
    assert sk.select_kernel(K.Auto, sk.ExecutionCaps.detect(), 1000) is K.Sequential
    for v, want in (("1", True), ("yes", True), ("0", False), ("", False)):
        monkeypatch.setenv("SIGKIT_ACCELERATED", v)
        assert sk.ExecutionCaps.detect().accelerated is want, v
