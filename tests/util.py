"""Comparison helpers for tests (test infrastructure; no method arithmetic).

Error metric (reading R10): per-channel normwise relative error
  e = max_c max_{i in c} |g_i - r_i| / max(max_{i in c} |r_i|, tiny)
for activations/gradients, and max_c |g_c - r_c| / max_c |r_c| for [C] vectors.
"""
from __future__ import annotations

import numpy as np


def chan_err(got, ref, channel_axis: int, mask=None) -> float:
    """Per-channel normwise relative error; ``mask`` (same shape, bool) marks
    elements to exclude (ambiguous activation branch, R16)."""
    g = np.asarray(got, dtype=np.float64)
    r = np.asarray(ref, dtype=np.float64)
    assert g.shape == r.shape, (g.shape, r.shape)
    d = np.abs(g - r)
    a = np.abs(r)
    if mask is not None:
        d = np.where(mask, 0.0, d)
    axes = tuple(i for i in range(g.ndim) if i != channel_axis % g.ndim)
    dmax = d.max(axis=axes) if axes else d
    amax = a.max(axis=axes) if axes else a
    return float(np.max(dmax / np.maximum(amax, 1e-30)))


def vec_err(got, ref) -> float:
    g = np.asarray(got, dtype=np.float64).ravel()
    r = np.asarray(ref, dtype=np.float64).ravel()
    return float(np.max(np.abs(g - r)) / max(float(np.max(np.abs(r))), 1e-30))


def rel_err(got, ref) -> float:
    """Global normwise relative error."""
    g = np.asarray(got, dtype=np.float64)
    r = np.asarray(ref, dtype=np.float64)
    return float(np.max(np.abs(g - r)) / max(float(np.max(np.abs(r))), 1e-30))
