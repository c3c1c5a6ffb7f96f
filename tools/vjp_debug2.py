import os, sys, numpy as np
sys.path.insert(0, ".")
import paper_2501_08455_b200 as sk
from oracle import oracle as O
def walk(B, L, d, seed):
    rng = np.random.default_rng(seed); X = np.zeros((B, L, d))
    X[:, 1:] = np.cumsum(rng.standard_normal((B, L - 1, d)) / np.sqrt(L - 1), axis=1); return X
X = walk(3, 101, 3, 21)
cot = np.random.default_rng(22).standard_normal((3, sk.sig_dim(3, 4)))
ref = O.ref_vjp(X, 4, cot)
for U in (3, 7, 5):
    g = sk.signature_vjp(X, 4, cot, chunks=U)
    err = np.abs(g - ref).max(axis=2) / np.abs(ref).max()
    bad = np.argwhere(err > 1e-12)
    print("U", U, "bad count", len(bad), "rows", sorted(set(bad[:, 0].tolist())), "t range", bad[:, 1].min() if len(bad) else None, bad[:, 1].max() if len(bad) else None)
    g2 = sk.signature_vjp(X, 4, cot, chunks=U)
    print("   second call bad", int((np.abs(g2 - ref).max(axis=2) / np.abs(ref).max() > 1e-12).sum()))
