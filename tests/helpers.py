"""Shared test metrics (the reference's testutil helpers, tests/helpers.hpp:38-55,
plus the per-level relative error of SURVEY.md §8c)."""
from __future__ import annotations

import numpy as np


def level_offsets(d: int, N: int) -> list[int]:
    off, p = [0], 1
    for _ in range(N):
        p *= d
        off.append(off[-1] + p)
    return off


def max_abs_diff(a, b) -> float:
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    return float(np.max(np.abs(a - b))) if a.size else 0.0


def rel_diff(a, b) -> float:
    """max|a-b| / (1 + max|a|)  (reference helpers.hpp:51-55)."""
    a = np.asarray(a, np.float64)
    return max_abs_diff(a, b) / (1.0 + (float(np.max(np.abs(a))) if a.size else 0.0))


def level_errors(got, ref, d: int, N: int) -> list[float]:
    """err_n = max_{b, i in level n} |g - r| / max |r|."""
    g = np.asarray(got, np.float64).reshape(-1, level_offsets(d, N)[-1])
    r = np.asarray(ref, np.float64).reshape(g.shape)
    off = level_offsets(d, N)
    errs = []
    for n in range(N):
        gs, rs = g[:, off[n]:off[n + 1]], r[:, off[n]:off[n + 1]]
        scale = float(np.max(np.abs(rs)))
        diff = float(np.max(np.abs(gs - rs)))
        errs.append(diff / scale if scale > 0 else diff)
    return errs
