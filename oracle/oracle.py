"""TEST INFRASTRUCTURE ONLY — numpy/ctypes front end of the CPU checkers.

Two checkers live here:

* ``port``: oracle/sig_oracle.c, a plain-C restatement of the reference
  algorithm (``sig_core.hpp:116-147``, ``tensor_algebra.cpp:63-102``,
  ``oracle.cpp:28-96``). Built on demand with gcc (``make -C oracle port``),
  so it exists on the GPU box too.
* ``ref``: the reference itself, compiled from /root/reference/proj/src by
  ``make -C oracle ref`` into oracle/_ref/ (present only where it was built).

Parity is pinned: tests/test_oracle.py requires the port to be bit-identical
to ``ref`` and to the committed golden vectors (tests/golden/).

Only tests/, ``__graft_entry__.smoke()`` and bench.py's CPU-baseline leg may
import this module. The product package never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
import threading

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
PORT_SO = os.path.join(HERE, "_build", "libsig_oracle.so")
REF_SO = os.path.join(HERE, "_ref", "libsigkit_ref.so")

_lock = threading.Lock()
_port = None
_ref = None

_dp = C.POINTER(C.c_double)
_fp = C.POINTER(C.c_float)
_sz = C.c_size_t


def _ptr(a: np.ndarray, t):
    return a.ctypes.data_as(t)


def build_port() -> str:
    src = os.path.join(HERE, "sig_oracle.c")
    if (not os.path.exists(PORT_SO)) or os.path.getmtime(PORT_SO) < os.path.getmtime(src):
        subprocess.run(["make", "-s", "-C", HERE, "port"], check=True)
    return PORT_SO


def build_ref() -> str | None:
    """Compile the reference (only where /root/reference exists), and its acceptance
    gate and doctest unit suites against this repository's drop-in headers and library
    (oracle/_ref/acceptance_dropin, oracle/_ref/unit_tests_dropin)."""
    if os.path.isdir("/root/reference/proj/src"):
        subprocess.run(["make", "-s", "-C", HERE, "ref"], check=True)
        subprocess.run(["make", "-s", "-C", HERE, "acceptance"], check=True)
        subprocess.run(["make", "-s", "-C", HERE, "unittests"], check=True)
    return REF_SO if os.path.exists(REF_SO) else None


def port():
    global _port
    with _lock:
        if _port is None:
            lib = C.CDLL(build_port())
            lib.sigo_sig_dim.restype = _sz
            lib.sigo_sig_dim.argtypes = [C.c_int, C.c_int]
            lib.sigo_sequential_forward_f64.restype = C.c_int64
            lib.sigo_sequential_forward_f64.argtypes = [_dp, _sz, _sz, C.c_int, C.c_int, _dp, _dp, C.c_int]
            lib.sigo_sequential_forward_f32.restype = C.c_int64
            lib.sigo_sequential_forward_f32.argtypes = [_fp, _sz, _sz, C.c_int, C.c_int, _fp, _fp, C.c_int]
            lib.sigo_chen_product_f64.argtypes = [C.c_int, C.c_int, _dp, _dp, _dp]
            lib.sigo_restricted_exp_f64.argtypes = [C.c_int, C.c_int, _dp, _dp]
            lib.sigo_bruteforce_f64.restype = C.c_int
            lib.sigo_bruteforce_f64.argtypes = [_dp, _sz, C.c_int, C.c_int, _dp]
            _port = lib
    return _port


def ref():
    """The compiled reference, or None when oracle/_ref was not built."""
    global _ref
    with _lock:
        if _ref is None and os.path.exists(REF_SO):
            lib = C.CDLL(REF_SO)
            lib.ref_last_error.restype = C.c_char_p
            lib.ref_sig_dim.argtypes = [C.c_int, C.c_int, C.POINTER(_sz)]
            for name in ("ref_signature_sequential", "ref_signature_parallel"):
                getattr(lib, name).argtypes = [_dp, _sz, _sz, C.c_int, C.c_int, _dp, C.POINTER(C.c_int64)]
            lib.ref_signature_stream.argtypes = [_dp, _sz, _sz, C.c_int, C.c_int, _dp]
            lib.ref_sequential_forward_f64.argtypes = [_dp, _sz, _sz, C.c_int, C.c_int, _dp, C.c_int]
            lib.ref_sequential_forward_f32.argtypes = [_fp, _sz, _sz, C.c_int, C.c_int, _fp, C.c_int]
            lib.ref_bruteforce.argtypes = [_dp, _sz, C.c_int, C.c_int, _dp]
            lib.ref_chen_product.argtypes = [C.c_int, C.c_int, _dp, _dp, _dp]
            lib.ref_restricted_exp.argtypes = [C.c_int, C.c_int, _dp, _dp]
            lib.ref_make_bench_paths.argtypes = [C.c_uint64, _sz, _sz, C.c_int, _dp]
            lib.ref_random_paths.argtypes = [C.c_uint64, _sz, _sz, C.c_int, C.c_double, _dp]
            lib.ref_signature_vjp.argtypes = [_dp, _sz, _sz, C.c_int, C.c_int, _dp, C.c_int, _dp]
            lib.ref_finite_diff_grad.argtypes = [_dp, _sz, _sz, C.c_int, C.c_int, _dp, C.c_double, _dp]
            lib.ref_increments.argtypes = [_dp, _sz, _sz, C.c_int, _dp]
            lib.ref_scaled_increments.argtypes = [_dp, _sz, _sz, C.c_int, C.c_int, _dp]
            lib.ref_bruteforce_strict.argtypes = [_dp, _sz, C.c_int, C.c_int, _dp]
            lib.ref_train.argtypes = [_sz, _sz, C.c_int, C.c_int, _sz, C.c_int, C.c_double, C.c_uint64, C.c_int,
                                      C.c_int, _dp]
            _ref = lib
    return _ref


def sig_dim(d: int, N: int) -> int:
    return int(port().sigo_sig_dim(d, N))


def level_offsets(d: int, N: int) -> list[int]:
    off = [0]
    p = 1
    for _ in range(N):
        p *= d
        off.append(off[-1] + p)
    return off


# ---------------------------------------------------------------- the port
def signature(X: np.ndarray, N: int, threads: int = 1, stream: bool = False):
    """detail::sequential_forward on (B,L,d) in X's dtype (f64 or f32)."""
    X = np.ascontiguousarray(X)
    B, L, d = X.shape
    D = sig_dim(d, N)
    lib = port()
    if X.dtype == np.float64:
        out = np.empty((B, D), np.float64)
        so = np.empty((B, L - 1, D), np.float64) if stream else None
        lib.sigo_sequential_forward_f64(_ptr(X, _dp), B, L, d, N, _ptr(out, _dp),
                                        _ptr(so, _dp) if stream else None, threads)
    elif X.dtype == np.float32:
        out = np.empty((B, D), np.float32)
        so = np.empty((B, L - 1, D), np.float32) if stream else None
        lib.sigo_sequential_forward_f32(_ptr(X, _fp), B, L, d, N, _ptr(out, _fp),
                                        _ptr(so, _fp) if stream else None, threads)
    else:
        raise TypeError(X.dtype)
    return (out, so) if stream else out


def chen_product(d: int, N: int, a: np.ndarray, b: np.ndarray) -> np.ndarray:
    a = np.ascontiguousarray(a, np.float64)
    b = np.ascontiguousarray(b, np.float64)
    c = np.empty_like(a)
    port().sigo_chen_product_f64(d, N, _ptr(a, _dp), _ptr(b, _dp), _ptr(c, _dp))
    return c


def restricted_exp(v: np.ndarray, N: int) -> np.ndarray:
    v = np.ascontiguousarray(v, np.float64)
    out = np.empty(sig_dim(len(v), N), np.float64)
    port().sigo_restricted_exp_f64(len(v), N, _ptr(v, _dp), _ptr(out, _dp))
    return out


def bruteforce(path: np.ndarray, N: int) -> np.ndarray:
    path = np.ascontiguousarray(path, np.float64)
    L, d = path.shape
    out = np.empty(sig_dim(d, N), np.float64)
    rc = port().sigo_bruteforce_f64(_ptr(path, _dp), L, d, N, _ptr(out, _dp))
    if rc != 0:
        raise ValueError("bruteforce limits exceeded")
    return out


# ------------------------------------------------------- the reference itself
def _ref_call(rc: int):
    if rc != 0:
        raise RuntimeError(f"reference error {rc}: {ref().ref_last_error().decode()}")


def ref_signature(X: np.ndarray, N: int, kernel: str = "sequential") -> np.ndarray:
    X = np.ascontiguousarray(X, np.float64)
    B, L, d = X.shape
    out = np.empty((B, sig_dim(d, N)), np.float64)
    cnt = C.c_int64(0)
    fn = ref().ref_signature_sequential if kernel == "sequential" else ref().ref_signature_parallel
    _ref_call(fn(_ptr(X, _dp), B, L, d, N, _ptr(out, _dp), C.byref(cnt)))
    return out


def ref_forward(X: np.ndarray, N: int, threads: int = 1) -> np.ndarray:
    """detail::sequential_forward<Real> of the reference on `threads` threads."""
    X = np.ascontiguousarray(X)
    B, L, d = X.shape
    if X.dtype == np.float64:
        out = np.empty((B, sig_dim(d, N)), np.float64)
        _ref_call(ref().ref_sequential_forward_f64(_ptr(X, _dp), B, L, d, N, _ptr(out, _dp), threads))
    else:
        out = np.empty((B, sig_dim(d, N)), np.float32)
        _ref_call(ref().ref_sequential_forward_f32(_ptr(X, _fp), B, L, d, N, _ptr(out, _fp), threads))
    return out


def ref_stream(X: np.ndarray, N: int) -> np.ndarray:
    X = np.ascontiguousarray(X, np.float64)
    B, L, d = X.shape
    out = np.empty((B, L - 1, sig_dim(d, N)), np.float64)
    _ref_call(ref().ref_signature_stream(_ptr(X, _dp), B, L, d, N, _ptr(out, _dp)))
    return out


def ref_bruteforce_strict(path: np.ndarray, N: int) -> np.ndarray:
    """The reference's signature_bruteforce with TupleClass::StrictlyIncreasing."""
    path = np.ascontiguousarray(path, np.float64)
    L, d = path.shape
    out = np.empty(sig_dim(d, N))
    _ref_call(ref().ref_bruteforce_strict(_ptr(path, _dp), L, d, N, _ptr(out, _dp)))
    return out


def ref_bruteforce(path: np.ndarray, N: int) -> np.ndarray:
    path = np.ascontiguousarray(path, np.float64)
    L, d = path.shape
    out = np.empty(sig_dim(d, N), np.float64)
    _ref_call(ref().ref_bruteforce(_ptr(path, _dp), L, d, N, _ptr(out, _dp)))
    return out


def ref_chen_product(d: int, N: int, a: np.ndarray, b: np.ndarray) -> np.ndarray:
    a = np.ascontiguousarray(a, np.float64)
    b = np.ascontiguousarray(b, np.float64)
    c = np.empty_like(a)
    _ref_call(ref().ref_chen_product(d, N, _ptr(a, _dp), _ptr(b, _dp), _ptr(c, _dp)))
    return c


def ref_restricted_exp(v: np.ndarray, N: int) -> np.ndarray:
    v = np.ascontiguousarray(v, np.float64)
    out = np.empty(sig_dim(len(v), N), np.float64)
    _ref_call(ref().ref_restricted_exp(len(v), N, _ptr(v, _dp), _ptr(out, _dp)))
    return out


def ref_random_paths(seed: int, B: int, L: int, d: int, step: float = 1.0) -> np.ndarray:
    out = np.empty((B, L, d), np.float64)
    _ref_call(ref().ref_random_paths(seed, B, L, d, step, _ptr(out, _dp)))
    return out


def ref_make_bench_paths(seed: int, B: int, L: int, d: int) -> np.ndarray:
    out = np.empty((B, L, d), np.float64)
    _ref_call(ref().ref_make_bench_paths(seed, B, L, d, _ptr(out, _dp)))
    return out


def ref_vjp(X: np.ndarray, N: int, cot: np.ndarray, kernel: str = "sequential") -> np.ndarray:
    """The reference's signature_vjp (autodiff.cpp:218-224) on (B, L, d) float64."""
    X = np.ascontiguousarray(X, np.float64)
    cot = np.ascontiguousarray(cot, np.float64)
    B, L, d = X.shape
    g = np.empty_like(X)
    _ref_call(ref().ref_signature_vjp(_ptr(X, _dp), B, L, d, N, _ptr(cot, _dp), 1 if kernel == "parallel" else 0,
                                      _ptr(g, _dp)))
    return g


def ref_increments(X: np.ndarray) -> np.ndarray:
    """The reference's increments (kernels.cpp:71-87)."""
    X = np.ascontiguousarray(X, np.float64)
    B, L, d = X.shape
    out = np.empty((B, L - 1, d))
    _ref_call(ref().ref_increments(_ptr(X, _dp), B, L, d, _ptr(out, _dp)))
    return out


def ref_scaled_increments(inc: np.ndarray, depth: int) -> list:
    """The reference's scaled_increments (kernels.cpp:89-104)."""
    inc = np.ascontiguousarray(inc, np.float64)
    B, S, d = inc.shape
    out = np.empty((max(0, depth - 1), B, S, d))
    _ref_call(ref().ref_scaled_increments(_ptr(inc, _dp), B, S, d, depth, _ptr(out, _dp)))
    return list(out)


def ref_train(n_samples, seq_len, sig_input_size, depth, batch_size, epochs, lr, seed, kernel=0,
              activation=0) -> list[float]:
    """The reference's training loop (model.cpp:222-263); per-epoch mean losses."""
    out = np.empty(max(1, epochs), np.float64)
    _ref_call(ref().ref_train(n_samples, seq_len, sig_input_size, depth, batch_size, epochs, lr, seed, kernel,
                              activation, _ptr(out, _dp)))
    return list(out[:epochs])


def ref_finite_diff(X: np.ndarray, N: int, cot: np.ndarray, h: float = 1e-5) -> np.ndarray:
    X = np.ascontiguousarray(X, np.float64)
    cot = np.ascontiguousarray(cot, np.float64)
    B, L, d = X.shape
    g = np.empty_like(X)
    _ref_call(ref().ref_finite_diff_grad(_ptr(X, _dp), B, L, d, N, _ptr(cot, _dp), h, _ptr(g, _dp)))
    return g
