"""Build recipe for libsigk.so (sm_100a kernels + C ABI + C++ drop-in API).

Every translation unit is compiled in-tree with
``nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo`` in parallel;
the fold variants are split one TU per (precision, d) so the build scales
with cores. Objects go to paper_2501_08455_b200/_build/, the shared library
to paper_2501_08455_b200/libsigk.so (git-ignored; travels with gpurun).
"""
from __future__ import annotations

import concurrent.futures as cf
import hashlib
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
# experiment builds: SIGK_DEFS="-DX=1 ..." and SIGK_LIB_OUT=path build a separate library
DEFS = os.environ.get("SIGK_DEFS", "").split()
OBJ = os.path.join(PKG, "_build" + ("_" + hashlib.sha1(" ".join(DEFS).encode()).hexdigest()[:8] if DEFS else ""))
LIB = os.environ.get("SIGK_LIB_OUT") or os.path.join(PKG, "libsigk.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVFLAGS = ["-std=c++17", "-O3", "-lineinfo", "-Xcompiler", "-fPIC,-O3", "-Xptxas", "-v",
           "-I" + os.path.join(ROOT, "include"), "-I" + CSRC] + DEFS
DIMS = [1, 2, 3, 4, 5, 6, 7, 8, 10]
HEADERS = ["sigk_common.cuh", "fold.cuh", "merge.cuh", "pair_kernel.cuh", "ipair_kernel.cuh", "stream_kernel.cuh", "vjp_kernel.cuh", "vjp_slice.cuh", "increments.cuh", "scan_kernel.cuh", "scan_vjp.cuh", "vjp_prep.cuh", "pos_fold.cuh", "ppair_kernel.cuh", "generic.cuh", "variants.cuh", "variants.h"]


def _units():
    units = [("sigk_abi", os.path.join(CSRC, "sigk_abi.cu"), []),
             ("microbench", os.path.join(CSRC, "microbench.cu"), [])]
    for real in ("float", "double"):
        for d in DIMS:
            units.append((f"variants_{real}_d{d}", os.path.join(CSRC, "variants_inst.cu"),
                          [f"-DSIGK_REAL={real}", f"-DSIGK_DIM={d}"]))
    units.append(("vjp_f32", os.path.join(CSRC, "vjp_inst.cu"), ["-DSIGK_VJP_REAL_F32=1"]))
    units.append(("vjp_f64", os.path.join(CSRC, "vjp_inst.cu"), ["-DSIGK_VJP_REAL_F32=0"]))
    units.append(("sigkit_api", os.path.join(CSRC, "sigkit_api.cpp"), []))
    units.append(("bench_api", os.path.join(CSRC, "bench_api.cpp"), []))
    units.append(("model_api", os.path.join(CSRC, "model_api.cpp"), []))
    units.append(("model_gpu", os.path.join(CSRC, "model_gpu.cu"), []))
    return units


def _stamp(src: str, extra: list[str]) -> str:
    h = hashlib.sha1()
    incs = [os.path.join(ROOT, "include", "sigk.h")] + [os.path.join(ROOT, "include", "sigkit", x)
                                                         for x in sorted(os.listdir(os.path.join(ROOT, "include", "sigkit")))]
    for p in [src] + [os.path.join(CSRC, x) for x in HEADERS] + incs:
        with open(p, "rb") as f:
            h.update(f.read())
    h.update(" ".join(NVFLAGS + ARCH + extra).encode())
    return h.hexdigest()


def _compile(unit):
    name, src, extra = unit
    obj = os.path.join(OBJ, name + ".o")
    stamp = obj + ".sha"
    key = _stamp(src, extra)
    if os.path.exists(obj) and os.path.exists(stamp) and open(stamp).read() == key:
        return name, "cached", ""
    if src.endswith(".cpp"):
        cmd = ["g++", "-std=c++17", "-O3", "-fPIC", "-I" + os.path.join(ROOT, "include"),
               "-I/usr/local/cuda/include", "-c", src, "-o", obj]
    else:
        cmd = [NVCC] + ARCH + NVFLAGS + extra + ["-c", src, "-o", obj]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"compile failed: {' '.join(cmd)}\n{r.stdout}\n{r.stderr}")
    with open(stamp, "w") as f:
        f.write(key)
    with open(obj + ".log", "w") as f:
        f.write(r.stderr)
    return name, "built", r.stderr


def build(verbose: bool = False, jobs: int | None = None) -> str:
    os.makedirs(OBJ, exist_ok=True)
    units = _units()
    jobs = jobs or max(1, os.cpu_count() or 1)
    with cf.ThreadPoolExecutor(jobs) as ex:
        results = list(ex.map(_compile, units))
    if verbose:
        for name, status, _ in results:
            print(f"  {status:6s} {name}")
    objs = [os.path.join(OBJ, u[0] + ".o") for u in units]
    newest = max(os.path.getmtime(o) for o in objs)
    if not os.path.exists(LIB) or os.path.getmtime(LIB) < newest:
        cmd = [NVCC] + ARCH + ["-shared", "-o", LIB] + objs + ["-lcudart_static", "-lpthread", "-ldl", "-lrt"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed: {' '.join(cmd)}\n{r.stdout}\n{r.stderr}")
    if not DEFS:
        _build_cli(verbose)
    return LIB


def _build_cli(verbose: bool = False) -> None:
    """tools/sigbench: the reference sigbench CLI over the B200 library."""
    src = os.path.join(ROOT, "tools", "sigbench.cpp")
    exe = os.path.join(ROOT, "tools", "sigbench")
    if not os.path.exists(src):
        return
    if os.path.exists(exe) and os.path.getmtime(exe) >= max(os.path.getmtime(src), os.path.getmtime(LIB)):
        return
    cmd = ["g++", "-std=c++17", "-O2", "-I" + os.path.join(ROOT, "include"), src, "-o", exe, LIB,
           "-Wl,-rpath,$ORIGIN/../paper_2501_08455_b200"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"sigbench build failed: {' '.join(cmd)}\n{r.stderr}")
    if verbose:
        print("  built  tools/sigbench")


if __name__ == "__main__":
    print(build(verbose=True, jobs=int(sys.argv[1]) if len(sys.argv) > 1 else None))
