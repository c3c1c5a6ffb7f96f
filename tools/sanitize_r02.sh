#!/bin/bash
# compute-sanitizer over the round-2 device paths: the parallel (per-degree scan)
# formulation and its reverse mode, the chunked reverse mode (in-place chunk
# signatures, by-degree chunk passes, the one-launch fold-and-passes), the cluster (DSMEM) segment combine, the position-table fold with its
# producer warp (mbarrier pipeline), and the scratch-lifetime graph test.
S=/usr/local/cuda/bin/compute-sanitizer
cat > /tmp/san_r02.py <<'PY'
import numpy as np, torch, sys
sys.path.insert(0, ".")
import paper_2501_08455_b200 as sk
from oracle import oracle as O
rng = np.random.default_rng(3)
X = np.cumsum(rng.standard_normal((6, 301, 5)) * 0.05, axis=1).astype(np.float32)
ref = O.signature(X.astype(np.float64), 4)
for kw in ({"segments": 2}, {"segments": 4, "chunks": 6}, {"segments": 8}, {"fold_variant": 2, "chunks": 10},
           {"fold_variant": 2, "segments": 3, "chunks": 4}, {"fold_variant": 2, "segments": 12, "chunks": 2}):
    got = sk.signature(X, 4, family=sk.FAMILY_PAIR, **kw)
    err = np.abs(got - ref).max() / np.abs(ref).max()
    assert err < 1e-5, (kw, err)
p = sk.signature_parallel(X.astype(np.float64), 4)
assert np.abs(p - ref).max() < 1e-10
rows = sk.signature_stream(X[:2].astype(np.float64), 3, kernel=sk.KernelKind.Parallel)
# reverse modes: the parallel formulation's adjoint (scan_vjp.cuh) and the chunked fold adjoint
# with in-place chunk signatures and the by-degree chunk passes
cot = rng.standard_normal((3, 155))
gp = sk.signature_vjp(X[:3].astype(np.float64), 3, cot, kernel=sk.KernelKind.Parallel)
gs = sk.signature_vjp(X[:3].astype(np.float64), 3, cot, kernel=sk.KernelKind.Sequential)
assert np.abs(gp - gs).max() <= 1e-10 * np.abs(gs).max()
g32 = sk.signature_vjp(X[:3], 3, cot.astype(np.float32), chunks=6)
assert np.abs(g32 - gs).max() <= 1e-4 * np.abs(gs).max()
# fp32 fold-and-passes in one launch (vjp_prep.cuh): one wave of paths of >= 750 steps
X2 = np.cumsum(rng.standard_normal((3, 801, 5)) * 0.03, axis=1).astype(np.float32)
c2 = rng.standard_normal((3, 780)).astype(np.float32)
st = sk.KernelStats()
gp2 = sk.signature_vjp(X2, 4, c2, stats=st)
assert st.launches == 2
gs2 = sk.signature_vjp(X2.astype(np.float64), 4, c2.astype(np.float64))
assert np.abs(gp2 - gs2).max() <= 1e-4 * np.abs(gs2).max()
print("sanitized paths ok")
PY
for tool in memcheck racecheck synccheck; do
  echo "== $tool round-2 paths"; timeout 900 $S --tool $tool python /tmp/san_r02.py 2>&1 | tail -2
done
echo "== memcheck graph-replay scratch test"
timeout 900 $S --tool memcheck python -m pytest tests/test_gpu_parallel.py -q -k "scratch" 2>&1 | tail -2
