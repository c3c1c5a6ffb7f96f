"""Determinism / agreement check of the reverse-mode kernels (debug tool):
repeated calls with pinned chunk counts, slice vs element-parallel kernel."""
import os, sys, numpy as np
sys.path.insert(0, ".")
import paper_2501_08455_b200 as sk
from oracle import oracle as O

def walk(B, L, d, seed):
    rng = np.random.default_rng(seed); X = np.zeros((B, L, d))
    X[:, 1:] = np.cumsum(rng.standard_normal((B, L - 1, d)) / np.sqrt(L - 1), axis=1); return X

X = walk(3, 101, 3, 21)
cot = np.random.default_rng(22).standard_normal((3, sk.sig_dim(3, 4)))
ref = O.ref_vjp(X, 4, cot) if O.ref() is not None else None
for mode in ("slice", "element"):
    if mode == "element": os.environ["SIGK_VJP_ELEMENT"] = "1"
    for U in (1, 2, 3, 7):
        outs = [sk.signature_vjp(X, 4, cot, chunks=U) for _ in range(4)]
        same = all(np.array_equal(outs[0], o) for o in outs[1:])
        r = np.abs(outs[0] - ref).max() / np.abs(ref).max() if ref is not None else None
        print(mode, "U", U, "deterministic", same, "rel vs reference", r, [np.abs(o - ref).max() / np.abs(ref).max() for o in outs[1:]])
