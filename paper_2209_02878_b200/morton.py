"""Host-side Morton helpers for the optional `sort_rays` reordering
(reference: morton.py:34-146, engine.py:125-147).  The BVH's own keys are
computed on device (csrc/rs_build.cu); this module only orders segment
midpoints on the host when a caller asks for sort_rays on numpy input."""

from __future__ import annotations

import numpy as np

GRID_BITS = 21
GRID_MAX = (1 << GRID_BITS) - 1
_MASKS = (0x1F00000000FFFF, 0x1F0000FF0000FF, 0x100F00F00F00F00F, 0x10C30C30C30C30C3,
          0x1249249249249249)
_SHIFTS = (32, 16, 8, 4, 2)


def quantize(points: np.ndarray) -> np.ndarray:
    """Per-axis floor((p - min) / extent * (2^21 - 1)), clipped; flat axis -> 0
    (morton.py:48-63) on the points' own support (morton.py:40-45)."""
    p = np.asarray(points, dtype=np.float64)
    lo, hi = p.min(axis=0), p.max(axis=0)
    q = np.zeros(p.shape, dtype=np.uint32)
    for k in range(3):
        ext = hi[k] - lo[k]
        if ext > 0.0:
            s = np.floor((p[:, k] - lo[k]) / ext * float(GRID_MAX))
            q[:, k] = np.clip(s, 0.0, float(GRID_MAX)).astype(np.uint32)
    return q


def encode(q: np.ndarray) -> np.ndarray:
    """63-bit interleave, x -> bit 0, y -> bit 1, z -> bit 2 (morton.py:117-128)."""
    codes = np.zeros(q.shape[0], dtype=np.uint64)
    for k in range(3):
        v = q[:, k].astype(np.uint64)
        for sh, m in zip(_SHIFTS, _MASKS):
            v = (v | v << np.uint64(sh)) & np.uint64(m)
        codes |= v << np.uint64(k)
    return codes


def order_points(points: np.ndarray) -> np.ndarray:
    """Stable Z-order permutation: ascending (code, index) (morton.py:131-146)."""
    codes = encode(quantize(points))
    return np.lexsort((np.arange(codes.shape[0]), codes))
