"""B200-native batched truncated path-signature transform (arXiv 2501.08455).

Python host-side mirror of the reference public API
(/root/reference/proj/include/sigkit/kernels.hpp:12-124,
tensor_algebra.hpp:35-42): ``signature``, ``signature_sequential``,
``signature_parallel``, ``select_kernel``, ``sig_dim``, ``level_offsets``,
``KernelKind``, ``ExecutionCaps``, ``KernelStats`` and the error classes, over
the C ABI of ``libsigk.so`` (include/sigk.h). Every compute call runs the
sm_100a kernels; if the library is missing or no GPU is usable the call
raises — there is no CPU fallback.

Inputs may be numpy arrays (host buffers: the library stages them through
the device and returns numpy) or CUDA torch tensors (device buffers: the call
is asynchronous on the current torch stream and returns a CUDA tensor).
"""
from __future__ import annotations

import ctypes as C
import enum
import os
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# SIGK_LIB_PATH: an alternative build of the same library (tuning experiments)
LIB_PATH = os.environ.get("SIGK_LIB_PATH") or os.path.join(_HERE, "libsigk.so")

SIGK_OK, SIGK_EDOMAIN, SIGK_ERESOURCE, SIGK_EDEVICE, SIGK_ETRAINING = 0, 1, 2, 3, 4
SIGK_X_ON_DEVICE, SIGK_OUT_ON_DEVICE, SIGK_ASYNC_HOST, SIGK_PREFIX_ROWS = 1, 2, 4, 8
DEFAULT_PARALLEL_MEMORY_CAP = 1 << 31  # reference kDefaultParallelMemoryCap (kernels.hpp:93)


class DomainError(ValueError):
    """Bad shapes/arguments (reference errors.hpp:9-12)."""


class ResourceError(RuntimeError):
    """Capacity failure (reference errors.hpp:16-19)."""


class TrainingError(RuntimeError):
    """Reference ``sigkit::TrainingError`` (errors.hpp): non-finite loss; ``epoch`` is 0-based."""

    def __init__(self, msg: str):
        super().__init__(msg)
        tail = msg.rsplit(" ", 1)[-1]
        self.epoch = int(tail) if tail.isdigit() else -1


class DeviceError(RuntimeError):
    """CUDA failure on the device path."""


class _Stats(C.Structure):
    _fields_ = [("fold_steps", C.c_int64), ("scan_passes", C.c_int64), ("chunks", C.c_int32),
                ("prefix_len", C.c_int32), ("threads_per_unit", C.c_int32), ("launches", C.c_int32),
                ("segments", C.c_int32), ("family", C.c_int32), ("path_steps", C.c_int64)]


class _Tuning(C.Structure):
    _fields_ = [("chunks", C.c_int32), ("force_generic", C.c_int32), ("plan_rows", C.c_int64),
                ("fold_event_start", C.c_void_p), ("fold_event_stop", C.c_void_p), ("prefix_len", C.c_int32),
                ("no_overlap", C.c_int32), ("segments", C.c_int32), ("family", C.c_int32),
                ("phase_buf", C.c_void_p), ("mode", C.c_int32), ("fold_variant", C.c_int32),
                ("cluster", C.c_int32)]


MODE_AUTO, MODE_THROUGHPUT, MODE_LATENCY = 0, 1, 2  # sigk_tuning.mode (include/sigk.h SIGK_MODE_*)


@dataclass
class KernelStats:
    """The C ABI's sigk_stats (include/sigk.h), all taken from the launches the
    call made. Reference KernelStats meaning (kernels.hpp:86-91): the chunked
    fold reports ``path_steps`` = fold steps applied per path (= L-1) and
    ``fold_steps`` = steps per chunk unit, ``scan_passes`` = combine rounds; the
    parallel formulation (family FAMILY_SCAN) reports ``scan_passes`` = degree
    passes launched (= depth) and ``fold_steps`` = 0."""
    fold_steps: int = 0
    scan_passes: int = 0
    chunks: int = 0
    prefix_len: int = 0
    threads_per_unit: int = 0
    launches: int = 0
    segments: int = 0
    family: int = 0
    path_steps: int = 0


# fold-kernel families (include/sigk.h SIGK_FAMILY_*)
FAMILY_AUTO, FAMILY_PATH, FAMILY_FLAT, FAMILY_PAIR, FAMILY_GENERIC, FAMILY_PFLAT, FAMILY_SCAN = 0, 1, 2, 3, 4, 5, 6
FAMILY_NAMES = {0: "auto", 1: "path", 2: "flat", 3: "pair", 4: "generic", 5: "pflat", 6: "scan"}


class KernelKind(enum.Enum):
    Sequential = "sequential"
    Parallel = "parallel"
    Auto = "auto"


def kernel_name(kind: KernelKind) -> str:
    return kind.value


def kernel_from_name(name: str) -> KernelKind:
    for k in KernelKind:
        if k.value == name:
            return k
    raise DomainError(f"unknown kernel '{name}', expected sequential, parallel or auto")


@dataclass
class ExecutionCaps:
    """Reference kernels.hpp:76-84 (same defaults): Auto resolves to Parallel
    only when ``accelerated`` and ``seq_len >= parallel_min_len``."""
    accelerated: bool = False
    parallel_min_len: int = 64

    @staticmethod
    def detect() -> "ExecutionCaps":
        """SIGKIT_ACCELERATED set, non-empty and not "0" (kernels.cpp:64-69)."""
        env = os.environ.get("SIGKIT_ACCELERATED")
        return ExecutionCaps(accelerated=env is not None and env not in ("", "0"))


def select_kernel(hint: KernelKind, caps: ExecutionCaps, seq_len: int) -> KernelKind:
    if hint != KernelKind.Auto:
        return hint
    return KernelKind.Parallel if (caps.accelerated and seq_len >= caps.parallel_min_len) else KernelKind.Sequential


_lib = None


def lib():
    """The loaded libsigk.so; raises if it was not built (no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: run `python -c 'import __graft_entry__ as g; g.build()'`")
        L = C.CDLL(LIB_PATH)
        sz, vp = C.c_size_t, C.c_void_p
        L.sigk_sig_dim.argtypes = [C.c_int, C.c_int, C.POINTER(sz)]
        L.sigk_level_offsets.argtypes = [C.c_int, C.c_int, C.POINTER(sz)]
        for n in ("sigk_signature_f32", "sigk_signature_f64"):
            getattr(L, n).argtypes = [vp, sz, sz, C.c_int, C.c_int, vp, C.c_uint, vp, C.POINTER(_Tuning),
                                      C.POINTER(_Stats)]
        for n in ("sigk_signature_stream_f32", "sigk_signature_stream_f64"):
            getattr(L, n).argtypes = [vp, sz, sz, C.c_int, C.c_int, vp, C.c_uint, vp, C.POINTER(_Tuning),
                                      C.POINTER(_Stats)]
        for n in ("sigk_signature_parallel_f32", "sigk_signature_parallel_f64"):
            getattr(L, n).argtypes = [vp, sz, sz, C.c_int, C.c_int, vp, sz, C.c_uint, vp, C.POINTER(_Stats)]
        for n in ("sigk_signature_vjp_parallel_f32", "sigk_signature_vjp_parallel_f64"):
            getattr(L, n).argtypes = [vp, sz, sz, C.c_int, C.c_int, vp, vp, sz, C.c_uint, vp, C.POINTER(_Stats)]
        for n in ("sigk_signature_vjp_f32", "sigk_signature_vjp_f64"):
            getattr(L, n).argtypes = [vp, sz, sz, C.c_int, C.c_int, vp, vp, C.c_uint, vp, C.POINTER(_Tuning),
                                      C.POINTER(_Stats)]
        for n in ("sigk_signature_sharded_f32", "sigk_signature_sharded_f64"):
            getattr(L, n).argtypes = [vp, sz, sz, C.c_int, C.c_int, vp, C.c_int, C.POINTER(_Stats)]
        for n in ("sigk_brownian_f32", "sigk_brownian_f64"):
            getattr(L, n).argtypes = [vp, sz, sz, C.c_int, C.c_uint64, sz, vp]
        L.sigk_has_fast_variant.argtypes = [C.c_int, C.c_int, C.c_int, C.POINTER(C.c_int)]
        L.sigk_plan.argtypes = [sz, sz, C.c_int, C.c_int, C.c_int, C.POINTER(_Tuning), C.POINTER(_Stats)]
        for n in ("sigk_increments_f32", "sigk_increments_f64"):
            getattr(L, n).argtypes = [vp, sz, sz, C.c_int, vp, C.c_uint, vp]
        for n in ("sigk_scaled_increments_f32", "sigk_scaled_increments_f64"):
            getattr(L, n).argtypes = [vp, sz, C.c_int, vp, C.c_uint, vp]
        L.sigk_signature_bruteforce_f64.argtypes = [vp, sz, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, vp]
        L.sigk_train.argtypes = [sz, sz, C.c_int, C.c_int, sz, C.c_int, C.c_double, C.c_uint64, C.c_int, C.c_int,
                                 C.POINTER(C.c_double)]
        L.sigk_last_error.restype = C.c_char_p
        L.sigk_bench_ffma.argtypes = [vp, C.c_int, C.c_int, C.POINTER(C.c_double), vp]
        _lib = L
    return _lib


def _check(rc: int):
    if rc == SIGK_OK:
        return
    msg = lib().sigk_last_error().decode()
    if rc == SIGK_EDOMAIN:
        raise DomainError(msg)
    if rc == SIGK_ERESOURCE:
        raise ResourceError(msg)
    if rc == SIGK_ETRAINING:
        raise TrainingError(msg)
    raise DeviceError(msg)


def sig_dim(dim: int, depth: int) -> int:
    """D = Σ_{n=1..N} d^n (reference tensor_algebra.cpp:10-20)."""
    D = C.c_size_t(0)
    _check(lib().sigk_sig_dim(dim, depth, C.byref(D)))
    return D.value


def level_offsets(dim: int, depth: int) -> list[int]:
    """offsets[n-1] = start of degree n, offsets[N] = D (tensor_algebra.cpp:33-41)."""
    if depth < 1:
        _check(lib().sigk_sig_dim(dim, depth, None))
    off = (C.c_size_t * (depth + 1))()
    _check(lib().sigk_level_offsets(dim, depth, off))
    return list(off)


def level_sizes(dim: int, depth: int) -> list[int]:
    off = level_offsets(dim, depth)
    return [off[i + 1] - off[i] for i in range(depth)]


def has_fast_variant(dim: int, depth: int, f64: bool = False) -> tuple[bool, int]:
    q = C.c_int(0)
    ok = lib().sigk_has_fast_variant(dim, depth, int(f64), C.byref(q))
    return bool(ok), q.value


def _is_torch(x) -> bool:
    return type(x).__module__.startswith("torch")


def _validate_shape(shape, depth):
    if len(shape) != 3:
        raise DomainError(f"paths must have shape (B, L, d), got {tuple(shape)}")
    B, L, d = (int(s) for s in shape)
    if B < 1 or L < 1 or d < 1:
        raise DomainError("paths: batch, len and dim must all be >= 1")
    if depth < 1:
        raise DomainError(f"depth must be >= 1, got {depth}")
    return B, L, d


def plan(B: int, L: int, d: int, depth: int, f64: bool = False, **tuning) -> KernelStats:
    """The launch plan (family, Q, chunks, segments, steps per chunk) a call
    would use on the current device; no kernel runs."""
    st = _Stats()
    tun = _Tuning(**tuning)
    _check(lib().sigk_plan(B, L, d, depth, int(f64), C.byref(tun), C.byref(st)))
    ks = KernelStats()
    for f, _ in _Stats._fields_:
        setattr(ks, f, getattr(st, f))
    return ks


def _copy_stats(st: _Stats, stats: KernelStats | None):
    if stats is not None:
        for f, _ in _Stats._fields_:
            setattr(stats, f, getattr(st, f))


def _torch_dtype_ok(X):
    import torch

    if X.dtype not in (torch.float32, torch.float64):
        raise DomainError(f"unsupported dtype {X.dtype} (float32 or float64)")


def _host_array(paths, depth: int):
    X = np.asarray(paths)
    B, L, d = _validate_shape(X.shape, depth)
    if X.dtype not in (np.float32, np.float64):
        X = X.astype(np.float64)
    return np.ascontiguousarray(X), B, L, d


def _check_out(out, shape, like, *, pinned: bool = False):
    """Validate a caller-provided ``out`` before its pointer reaches the C ABI:
    exact shape, the input's dtype, same device (pinned host memory for the
    asynchronous host mode), contiguous."""
    if tuple(out.shape) != tuple(shape):
        raise DomainError(f"out has shape {tuple(out.shape)}, expected {tuple(shape)}")
    if out.dtype != like.dtype:
        raise DomainError(f"out has dtype {out.dtype}, expected {like.dtype}")
    if _is_torch(out) != _is_torch(like):
        raise DomainError("out must be the same kind of array as the paths (numpy or torch)")
    if _is_torch(out):
        if out.device != like.device:
            raise DomainError(f"out is on {out.device}, paths on {like.device}")
        if not out.is_contiguous():
            raise DomainError("out must be contiguous")
        if pinned and not out.is_pinned():
            raise DomainError("async host mode needs a pinned CPU `out`")
    elif not (out.flags["C_CONTIGUOUS"] and out.flags["WRITEABLE"]):
        raise DomainError("out must be a writeable C-contiguous array")
    return out


def _run(paths, depth: int, stats: KernelStats | None, chunks: int = 0, force_generic: bool = False,
         out=None, plan_rows: int = 0, prefix_len: int = 0, segments: int = 0, family: int = 0, mode: int = 0,
         fold_variant: int = 0, cluster: int = 0):
    st = _Stats()
    tun = _Tuning(chunks=chunks, force_generic=int(force_generic), plan_rows=plan_rows, prefix_len=prefix_len,
                  segments=segments, family=family, mode=mode, fold_variant=fold_variant, cluster=cluster)
    if _is_torch(paths):
        import torch

        B, L, d = _validate_shape(paths.shape, depth)
        _torch_dtype_ok(paths)
        fn = lib().sigk_signature_f32 if paths.dtype == torch.float32 else lib().sigk_signature_f64
        D = sig_dim(d, depth)
        if not paths.is_cuda:
            # page-locked host tensors: asynchronous host mode on the current CUDA
            # stream (SIGK_ASYNC_HOST); `out` is valid once that stream is synchronised.
            # The input must be the caller's own contiguous pinned buffer: a temporary
            # copy could be recycled by the pinned-memory cache while the H2D is queued.
            if not paths.is_pinned():
                raise DomainError("torch CPU input must be pinned (async host mode); use numpy for plain host buffers")
            if not paths.is_contiguous():
                raise DomainError("async host mode needs a contiguous pinned input (copies could be freed "
                                  "before the queued host-to-device copy runs)")
            X = paths
            if out is None:
                out = torch.empty((B, D), dtype=X.dtype, pin_memory=True)
            if out.is_cuda:
                raise DomainError("async host mode needs a pinned CPU `out`")
            _check_out(out, (B, D), X, pinned=True)
            s = torch.cuda.current_stream().cuda_stream
            _check(fn(X.data_ptr(), B, L, d, depth, out.data_ptr(), SIGK_ASYNC_HOST, s, C.byref(tun), C.byref(st)))
            _copy_stats(st, stats)
            return out
        X = paths.contiguous()
        out = torch.empty((B, D), dtype=X.dtype, device=X.device) if out is None else _check_out(out, (B, D), X)
        with torch.cuda.device(X.device):
            s = torch.cuda.current_stream(X.device).cuda_stream
            _check(fn(X.data_ptr(), B, L, d, depth, out.data_ptr(), SIGK_X_ON_DEVICE | SIGK_OUT_ON_DEVICE,
                      s, C.byref(tun), C.byref(st)))
    else:
        X, B, L, d = _host_array(paths, depth)
        D = sig_dim(d, depth)
        out = np.empty((B, D), dtype=X.dtype) if out is None else _check_out(out, (B, D), X)
        fn = lib().sigk_signature_f32 if X.dtype == np.float32 else lib().sigk_signature_f64
        _check(fn(X.ctypes.data, B, L, d, depth, out.ctypes.data, 0, None, C.byref(tun), C.byref(st)))
    _copy_stats(st, stats)
    return out


def _run_parallel(paths, depth: int, stats: KernelStats | None, memory_cap: int, prefix_rows: bool, out=None):
    """The paper's per-degree scan formulation on the GPU (sigk_signature_parallel_*)."""
    st = _Stats()
    flags = SIGK_PREFIX_ROWS if prefix_rows else 0
    if _is_torch(paths):
        import torch

        if not paths.is_cuda:
            raise DomainError("torch input must be a CUDA tensor (use numpy for host buffers)")
        B, L, d = _validate_shape(paths.shape, depth)
        _torch_dtype_ok(paths)
        X = paths.contiguous()
        shape = (B, max(L - 1, 0), sig_dim(d, depth)) if prefix_rows else (B, sig_dim(d, depth))
        out = torch.empty(shape, dtype=X.dtype, device=X.device) if out is None else _check_out(out, shape, X)
        fn = lib().sigk_signature_parallel_f32 if X.dtype == torch.float32 else lib().sigk_signature_parallel_f64
        with torch.cuda.device(X.device):
            s = torch.cuda.current_stream(X.device).cuda_stream
            _check(fn(X.data_ptr(), B, L, d, depth, out.data_ptr(), memory_cap,
                      flags | SIGK_X_ON_DEVICE | SIGK_OUT_ON_DEVICE, s, C.byref(st)))
    else:
        X, B, L, d = _host_array(paths, depth)
        shape = (B, max(L - 1, 0), sig_dim(d, depth)) if prefix_rows else (B, sig_dim(d, depth))
        out = np.empty(shape, dtype=X.dtype) if out is None else _check_out(out, shape, X)
        fn = lib().sigk_signature_parallel_f32 if X.dtype == np.float32 else lib().sigk_signature_parallel_f64
        _check(fn(X.ctypes.data, B, L, d, depth, out.ctypes.data if out.size else None, memory_cap, flags, None,
                  C.byref(st)))
    _copy_stats(st, stats)
    return out


def _seq_len(paths) -> int:
    return int(np.shape(paths)[1]) if len(np.shape(paths)) == 3 else 0


def signature(paths, depth: int, kernel: KernelKind = KernelKind.Auto, caps: ExecutionCaps | None = None,
              stats: KernelStats | None = None, *, chunks: int = 0, out=None, plan_rows: int = 0,
              prefix_len: int = 0, segments: int = 0, family: int = 0, mode: int = MODE_AUTO,
              fold_variant: int = 0, cluster: int = 0):
    """Reference ``sigkit::signature`` (kernels.cpp:200-206): (B, L, d) -> (B, D).

    ``kernel``/``caps`` dispatch like the reference (select_kernel,
    kernels.cpp:150-154): Parallel runs the paper's per-degree scan
    formulation on the GPU (``signature_parallel``), Sequential the chunked
    Chen fold. ``chunks`` forces the sequence split of the fold (0 = planned);
    ``plan_rows`` plans the split as if the batch had that many rows (results
    are bitwise independent of batch composition at equal chunking);
    ``segments``/``family``/``prefix_len`` pin the rest of the plan (tests, tuning);
    ``mode`` picks what the plan optimises (MODE_THROUGHPUT: back-to-back calls,
    MODE_LATENCY: a call that runs alone; MODE_AUTO: latency for numpy inputs,
    throughput for device tensors); ``fold_variant`` pins the pair family's fold
    (1 register table, 2 position table with a producer warp; 0 planned); ``cluster=1``
    combines 2..8 segments of a path inside a thread-block cluster (opt-in).
    """
    if select_kernel(kernel, caps or ExecutionCaps.detect(), _seq_len(paths)) == KernelKind.Parallel:
        return signature_parallel(paths, depth, stats, out=out)
    return _run(paths, depth, stats, chunks=chunks, out=out, plan_rows=plan_rows, prefix_len=prefix_len,
                segments=segments, family=family, mode=mode, fold_variant=fold_variant, cluster=cluster)


def signature_stream(paths, depth: int, kernel: KernelKind = KernelKind.Auto, caps: ExecutionCaps | None = None,
                     stats: KernelStats | None = None, *, out=None, family: int = 0, chunks: int = 0,
                     segments: int = 0):
    """Reference ``sigkit::signature_stream`` (kernels.cpp:156-198): (B, L, d) -> (B, L-1, D),
    row (b, t) = signature of X[b, 0..t+1]. L < 2 raises DomainError. The Parallel kind reads
    every position of the per-degree scan formulation (kernels.cpp:183-197)."""
    if select_kernel(kernel, caps or ExecutionCaps.detect(), _seq_len(paths)) == KernelKind.Parallel:
        return _run_parallel(paths, depth, stats, DEFAULT_PARALLEL_MEMORY_CAP, True, out=out)
    st = _Stats()
    tun = _Tuning(family=family, chunks=chunks, segments=segments)
    if _is_torch(paths):
        import torch

        if not paths.is_cuda:
            raise DomainError("torch input must be a CUDA tensor (use numpy for host buffers)")
        B, L, d = _validate_shape(paths.shape, depth)
        _torch_dtype_ok(paths)
        X = paths.contiguous()
        shape = (B, max(L - 1, 0), sig_dim(d, depth))
        out = torch.empty(shape, dtype=X.dtype, device=X.device) if out is None else _check_out(out, shape, X)
        fn = lib().sigk_signature_stream_f32 if X.dtype == torch.float32 else lib().sigk_signature_stream_f64
        with torch.cuda.device(X.device):
            s = torch.cuda.current_stream(X.device).cuda_stream
            _check(fn(X.data_ptr(), B, L, d, depth, out.data_ptr(), SIGK_X_ON_DEVICE | SIGK_OUT_ON_DEVICE,
                      s, C.byref(tun), C.byref(st)))
    else:
        X, B, L, d = _host_array(paths, depth)
        shape = (B, max(L - 1, 0), sig_dim(d, depth))
        out = np.empty(shape, dtype=X.dtype) if out is None else _check_out(out, shape, X)
        fn = lib().sigk_signature_stream_f32 if X.dtype == np.float32 else lib().sigk_signature_stream_f64
        _check(fn(X.ctypes.data, B, L, d, depth, out.ctypes.data, 0, None, C.byref(tun), C.byref(st)))
    _copy_stats(st, stats)
    return out


def signature_vjp(paths, depth: int, cotangent, kernel: KernelKind = KernelKind.Auto,
                  caps: ExecutionCaps | None = None, stats: KernelStats | None = None, *, chunks: int = 0):
    """Reference ``sigkit::signature_vjp`` (autodiff.cpp:218-224): d<cotangent, Sig(X)>/dX,
    (B, L, d), for a (B, D) cotangent. numpy in -> numpy out; CUDA tensors in -> CUDA tensor out.
    ``chunks`` pins the number of backward chunks per path (0: planned; 1: one sequential walk).
    As the reference, the selected kind picks the adjoint: Parallel runs the adjoint of the
    per-degree scan passes (vjp_parallel, autodiff.cpp:108-214; sigk_signature_vjp_parallel_*,
    with the forward formulation's storage cap), otherwise the fold adjoint (vjp_sequential,
    :31-107). The two are independent GPU routes to the same gradient (test_autodiff.cpp:117-130)."""
    kind = select_kernel(kernel, caps or ExecutionCaps.detect(), _seq_len(paths))
    st = _Stats()
    tun = C.byref(_Tuning(chunks=chunks)) if chunks else None
    par = kind == KernelKind.Parallel

    def call(fn32, fn64, is32, *a):
        if par:
            fn = lib().sigk_signature_vjp_parallel_f32 if is32 else lib().sigk_signature_vjp_parallel_f64
            xp, B_, L_, d_, n_, cp, gp, flags, s = a
            return fn(xp, B_, L_, d_, n_, cp, gp, DEFAULT_PARALLEL_MEMORY_CAP, flags, s, C.byref(st))
        return (fn32 if is32 else fn64)(*a, tun, C.byref(st))
    if _is_torch(paths):
        import torch

        if not paths.is_cuda:
            raise DomainError("torch input must be a CUDA tensor (use numpy for host buffers)")
        B, L, d = _validate_shape(paths.shape, depth)
        _torch_dtype_ok(paths)
        X = paths.contiguous()
        cot = cotangent.to(device=X.device, dtype=X.dtype).contiguous()
        if tuple(cot.shape) != (B, sig_dim(d, depth)):
            raise DomainError("signature_vjp: cotangent shape does not match paths/depth")
        grad = torch.empty_like(X)
        with torch.cuda.device(X.device):
            s = torch.cuda.current_stream(X.device).cuda_stream
            _check(call(lib().sigk_signature_vjp_f32, lib().sigk_signature_vjp_f64, X.dtype == torch.float32,
                        X.data_ptr(), B, L, d, depth, cot.data_ptr(), grad.data_ptr(), SIGK_X_ON_DEVICE, s))
    else:
        X, B, L, d = _host_array(paths, depth)
        cot = np.ascontiguousarray(cotangent, dtype=X.dtype)
        if cot.shape != (B, sig_dim(d, depth)):
            raise DomainError("signature_vjp: cotangent shape does not match paths/depth")
        grad = np.empty_like(X)
        _check(call(lib().sigk_signature_vjp_f32, lib().sigk_signature_vjp_f64, X.dtype == np.float32,
                    X.ctypes.data, B, L, d, depth, cot.ctypes.data, grad.ctypes.data, 0, None))
    _copy_stats(st, stats)
    return grad


class _SignatureFn:
    """torch.autograd.Function over the GPU forward and reverse mode (built lazily so
    importing the package does not import torch)."""
    _cls = None

    @classmethod
    def get(cls):
        if cls._cls is None:
            import torch

            class SignatureFunction(torch.autograd.Function):
                @staticmethod
                def forward(ctx, X, depth):
                    ctx.depth = depth
                    ctx.save_for_backward(X)
                    return _run(X, depth, None)

                @staticmethod
                def backward(ctx, grad_out):
                    (X,) = ctx.saved_tensors
                    return signature_vjp(X, ctx.depth, grad_out.contiguous()), None

            cls._cls = SignatureFunction
        return cls._cls


def signature_autograd(paths, depth: int):
    """Differentiable signature for CUDA torch tensors (B, L, d) -> (B, D): the forward
    is ``signature`` (chunked GPU fold), the backward ``signature_vjp`` (GPU reverse
    mode) — the signature layer of the paper's training setup (§3.2) as a
    ``torch.autograd.Function``; float32 or float64."""
    if not _is_torch(paths) or not paths.is_cuda:
        raise DomainError("signature_autograd needs a CUDA torch tensor")
    _validate_shape(paths.shape, depth)
    _torch_dtype_ok(paths)
    return _SignatureFn.get().apply(paths.contiguous(), depth)


def signature_sequential(paths, depth: int, stats: KernelStats | None = None, **kw):
    """Reference ``signature_sequential`` (kernels.cpp:106-122): the chunked Chen fold."""
    return _run(paths, depth, stats, **kw)


def signature_parallel(paths, depth: int, stats: KernelStats | None = None,
                       memory_cap: int = DEFAULT_PARALLEL_MEMORY_CAP, *, out=None):
    """Reference ``signature_parallel`` (kernels.cpp:124-148): the paper's per-degree
    cumulative-sum formulation (sig_core.hpp:175-298) as N GPU scan passes, including
    its ResourceError refusal above ``memory_cap`` scalars (sig_core.hpp:161-173)."""
    return _run_parallel(paths, depth, stats, memory_cap, False, out=out)


def signature_generic(paths, depth: int, stats: KernelStats | None = None):
    """Force the shape-generic GPU kernel (cross-check of the sliced variants)."""
    return _run(paths, depth, stats, force_generic=True)


def signature_sharded(paths: np.ndarray, depth: int, num_gpus: int = 0, stats: KernelStats | None = None):
    """Host buffers in/out, batch rows sharded across ``num_gpus`` devices."""
    X = np.ascontiguousarray(paths)
    B, L, d = _validate_shape(X.shape, depth)
    if X.dtype not in (np.float32, np.float64):
        X = X.astype(np.float64)
    out = np.empty((B, sig_dim(d, depth)), dtype=X.dtype)
    st = _Stats()
    fn = lib().sigk_signature_sharded_f32 if X.dtype == np.float32 else lib().sigk_signature_sharded_f64
    _check(fn(X.ctypes.data, B, L, d, depth, out.ctypes.data, num_gpus, C.byref(st)))
    if stats is not None:
        for f, _ in _Stats._fields_:
            setattr(stats, f, getattr(st, f))
    return out


def brownian(out, seed: int = 42, row0: int = 0):
    """Fill a CUDA tensor (B, L, d) with synthetic Brownian paths (sigk_brownian_*)."""
    import torch

    B, L, d = out.shape
    fn = lib().sigk_brownian_f32 if out.dtype == torch.float32 else lib().sigk_brownian_f64
    with torch.cuda.device(out.device):
        _check(fn(out.data_ptr(), B, L, d, seed, row0, torch.cuda.current_stream(out.device).cuda_stream))
    return out


def increments(paths):
    """Reference ``increments`` (kernels.cpp:71-87): X[:, k+1] - X[:, k], (B, L-1, d), on the GPU.
    numpy in -> numpy out; CUDA tensors in -> CUDA tensor out."""
    if _is_torch(paths):
        import torch

        B, L, d = _validate_shape(paths.shape, 1)
        X = paths.contiguous()
        out = torch.empty((B, L - 1, d), dtype=X.dtype, device=X.device)
        fn = lib().sigk_increments_f32 if X.dtype == torch.float32 else lib().sigk_increments_f64
        with torch.cuda.device(X.device):
            _check(fn(X.data_ptr(), B, L, d, out.data_ptr(), SIGK_X_ON_DEVICE | SIGK_OUT_ON_DEVICE,
                      torch.cuda.current_stream(X.device).cuda_stream))
        return out
    X = np.asarray(paths)
    B, L, d = _validate_shape(X.shape, 1)
    X = np.ascontiguousarray(X if X.dtype in (np.float32, np.float64) else X.astype(np.float64))
    out = np.empty((B, L - 1, d), X.dtype)
    fn = lib().sigk_increments_f32 if X.dtype == np.float32 else lib().sigk_increments_f64
    _check(fn(X.ctypes.data, B, L, d, out.ctypes.data if out.size else None, 0, None))
    return out


def signature_bruteforce(path, depth: int, max_segments: int = 8, max_depth: int = 4, max_dim: int = 3,
                         strict: bool = False) -> np.ndarray:
    """Reference ``signature_bruteforce`` (oracle.cpp:28-96): one (L, d) path by tuple enumeration, on the GPU
    (fp64, bit-identical). Limits as the reference's OracleLimits (ResourceError beyond them)."""
    p = np.ascontiguousarray(path, np.float64)
    if p.ndim != 2:
        raise DomainError("signature_bruteforce: path must have shape (L, d)")
    L, d = p.shape
    out = np.empty(sig_dim(d, depth) if d >= 1 and depth >= 1 else 0)
    _check(lib().sigk_signature_bruteforce_f64(p.ctypes.data if p.size else None, L, d, depth, max_segments,
                                               max_depth, max_dim, int(strict), out.ctypes.data if out.size else None))
    return out


def scaled_increments(inc, depth: int) -> list:
    """Reference ``scaled_increments`` (kernels.cpp:89-104): [inc / m! for m = 2..depth] on the GPU."""
    a = np.ascontiguousarray(inc if np.asarray(inc).dtype in (np.float32, np.float64) else np.asarray(inc, np.float64))
    out = np.empty((max(0, depth - 1),) + a.shape, a.dtype)
    fn = lib().sigk_scaled_increments_f32 if a.dtype == np.float32 else lib().sigk_scaled_increments_f64
    _check(fn(a.ctypes.data if a.size else None, a.size, depth, out.ctypes.data if out.size else None, 0, None))
    return list(out)


@dataclass
class TrainConfig:
    """Reference ``sigkit::TrainConfig`` (include/sigkit/model.hpp:39-50)."""
    n_samples: int = 1024
    seq_len: int = 100
    sig_input_size: int = 4
    depth: int = 3
    batch_size: int = 128
    epochs: int = 10
    learning_rate: float = 0.05
    seed: int = 42
    kernel: KernelKind = KernelKind.Auto
    activation: str = "tanh"


def train(config: TrainConfig) -> list[float]:
    """Reference ``sigkit::train`` (model.cpp:222-263; paper §3.2): Dense(20->d) -> act -> signature ->
    Dense(D->10) trained by SGD on MSE against a frozen teacher; signature forward and VJP run on the GPU.
    Returns the per-epoch mean losses."""
    if config.activation not in ("tanh", "identity"):
        raise DomainError(f"unknown activation '{config.activation}', expected tanh or identity")
    kern = {KernelKind.Sequential: 0, KernelKind.Parallel: 1}.get(config.kernel, 2)
    losses = (C.c_double * max(1, config.epochs))()
    _check(lib().sigk_train(config.n_samples, config.seq_len, config.sig_input_size, config.depth,
                            config.batch_size, config.epochs, config.learning_rate, config.seed, kern,
                            0 if config.activation == "tanh" else 1, losses))
    return list(losses[:config.epochs])


__all__ = [
    "DomainError", "ResourceError", "TrainingError", "DeviceError", "KernelKind", "KernelStats", "ExecutionCaps", "kernel_name",
    "kernel_from_name", "select_kernel", "sig_dim", "level_offsets", "level_sizes", "signature",
    "signature_sequential", "signature_parallel", "signature_generic", "signature_sharded", "brownian",
    "signature_stream", "signature_vjp", "signature_autograd", "TrainConfig", "train", "increments", "scaled_increments", "signature_bruteforce",
    "has_fast_variant", "lib", "plan", "FAMILY_AUTO", "FAMILY_PATH", "FAMILY_FLAT", "FAMILY_PAIR",
    "FAMILY_GENERIC", "FAMILY_PFLAT", "FAMILY_SCAN", "FAMILY_NAMES", "MODE_AUTO", "MODE_THROUGHPUT", "MODE_LATENCY", "SIGK_X_ON_DEVICE", "SIGK_OUT_ON_DEVICE",
    "SIGK_ASYNC_HOST", "SIGK_PREFIX_ROWS", "DEFAULT_PARALLEL_MEMORY_CAP",
]
