"""Generate tests/golden/golden.npz from the REFERENCE ITSELF.

Run here (where /root/reference exists): ``python tests/golden/make_golden.py``.
Every output below comes from the reference compiled from its own sources
(oracle/_ref, built by ``make -C oracle ref``): inputs from the reference
test/bench generators (tests/helpers.hpp:16-36 random_paths,
src/bench.cpp:134-161 make_bench_paths — libstdc++'s normal_distribution is
implementation-defined, so the inputs are stored, not re-derived), outputs
from signature_sequential (kernels.cpp:106-122), signature_bruteforce
(oracle.cpp:28-96), chen_product (tensor_algebra.cpp:80-102),
restricted_exp (:63-78), signature_stream (kernels.cpp:156-198) and the
float instantiation of sequential_forward (sig_core.hpp:120-147).
"""
from __future__ import annotations

import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from oracle import oracle as O  # noqa: E402


def main():
    O.build_ref()
    assert O.ref() is not None, "oracle/_ref not built"
    g: dict[str, np.ndarray] = {}

    # 1. the worked example (acceptance.cpp:195-209, test_oracle.cpp:27-33)
    corner = np.array([[[0.0, 0.0], [1.0, 0.0], [1.0, 1.0]]])
    g["corner/X"] = corner
    g["corner/sig2"] = O.ref_signature(corner, 2)

    # 2. oracle-equivalence grid (acceptance.cpp:60-85): L 2..7, d 1..3, N 1..4
    seed = 1
    cases = []
    for L in range(2, 8):
        for d in range(1, 4):
            for N in range(1, 5):
                X = O.ref_random_paths(seed, 1, L, d, 0.7)
                key = f"brute/{seed}"
                g[key + "/X"] = X
                g[key + "/N"] = np.array(N)
                g[key + "/brute"] = O.ref_bruteforce(X[0], N)
                g[key + "/seq"] = O.ref_signature(X, N)
                cases.append(seed)
                seed += 1
    g["brute/seeds"] = np.array(cases)

    # 3. cross-kernel shape grid (test_kernels.cpp:128-146): B {1,3}, L {2,5,17,64}, d {1,2,3,5}, N 1..5
    seed = 1000
    cases = []
    for B in (1, 3):
        for L in (2, 5, 17, 64):
            for d in (1, 2, 3, 5):
                for N in range(1, 6):
                    X = O.ref_random_paths(seed, B, L, d, 0.5)
                    key = f"grid/{seed}"
                    g[key + "/X"] = X
                    g[key + "/N"] = np.array(N)
                    g[key + "/seq"] = O.ref_signature(X, N)
                    cases.append(seed)
                    seed += 1
    g["grid/seeds"] = np.array(cases)

    # 4. wide rows (test_kernels.cpp:119-126): d=10, N=4 -> 11110 per row
    X = O.ref_random_paths(26, 1, 3, 10)
    g["wide/X"] = X
    g["wide/seq"] = O.ref_signature(X, 4)

    # 5. batch-composition invariance (test_kernels.cpp:252-263): B=65
    X = O.ref_random_paths(130, 65, 9, 2)
    g["b65/X"] = X
    g["b65/seq"] = O.ref_signature(X, 3)

    # 6. Chen product and restricted exponential
    rng = np.random.default_rng(7)
    for d, N in ((2, 4), (3, 3), (5, 4)):
        D = O.sig_dim(d, N)
        a, b = rng.standard_normal(D), rng.standard_normal(D)
        v = rng.standard_normal(d)
        g[f"chen/{d}_{N}/a"], g[f"chen/{d}_{N}/b"] = a, b
        g[f"chen/{d}_{N}/c"] = O.ref_chen_product(d, N, a, b)
        g[f"chen/{d}_{N}/v"] = v
        g[f"chen/{d}_{N}/exp"] = O.ref_restricted_exp(v, N)

    # 7. the C1 headline-plumbing case on the reference bench input (seed 42)
    X = O.ref_make_bench_paths(42, 32, 100, 2)
    g["c1/X"] = X
    g["c1/seq"] = O.ref_signature(X, 4)
    X32 = X.astype(np.float32)
    g["c1/X32"] = X32
    g["c1/f32"] = O.ref_forward(X32, 4)  # sequential_forward<float>

    # 8. prefix stream (test_kernels.cpp:272-292)
    X = O.ref_random_paths(150, 2, 9, 2)
    g["stream/X"] = X
    g["stream/N3"] = O.ref_stream(X, 3)

    out = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden.npz")
    np.savez_compressed(out, **g)
    print(out, os.path.getsize(out), "bytes,", len(g), "arrays")


if __name__ == "__main__":
    main()
