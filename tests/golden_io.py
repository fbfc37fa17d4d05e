"""Loader for the committed golden fixtures (tests/golden/*.npz)."""

from __future__ import annotations

from pathlib import Path

import numpy as np

GOLDEN = Path(__file__).resolve().parent / "golden"
MODES = ("boolean", "barycentric", "count")
RESULT_FIELDS = ("crossing", "counts", "ray_index", "distance", "triangle_id", "point")
TREE_FIELDS = (
    "internal_bounds", "internal_child_left", "internal_child_right",
    "internal_range_left", "internal_range_right", "internal_triangle_id",
    "internal_visit", "leaf_bounds", "leaf_triangle_id", "leaf_range_left",
    "leaf_range_right", "sorted_triangle_ids",
)
SCENES = ("c1", "s19", "s77", "full", "none", "dup")  # dup: every triangle repeated (equal Morton codes)
SOUPS = ("17", "20")
OVERFLOWS = ("ovf21", "ovf31", "ovfshort")
TREE_SIZES = (1, 2, 3, 7, 8, 100, 5000, "dup5")  # dup5: all codes equal (test_backends.py:70-84)


def load(name: str) -> dict:
    with np.load(GOLDEN / f"{name}.npz") as z:
        return {k: z[k] for k in z.files}


def expected(fx: dict, prefix: str, mode: str) -> dict:
    """The reference ResultSet fields stored under `prefix_mode_*`."""
    out = {}
    for f in RESULT_FIELDS:
        key = f"{prefix}_{mode}_{f}"
        if key in fx:
            out[f] = fx[key]
    return out


def assert_result_fields(got: dict, want: dict, context: str = "", float_tol: float = 0.0):
    """tests/helpers.py:65-82 semantics: exact, floats optionally to float_tol."""
    for f, w in want.items():
        if f == "mode":
            continue
        g = got.get(f)
        assert g is not None, f"{context}: missing {f}"
        g = np.asarray(g)
        assert g.shape == w.shape, f"{context}: {f} shape {g.shape} vs {w.shape}"
        if float_tol > 0 and f in ("distance", "point"):
            assert np.allclose(g, w, atol=float_tol, rtol=0), f"{context}: {f} beyond {float_tol}"
        else:
            assert np.array_equal(g, w), f"{context}: {f} differs"
