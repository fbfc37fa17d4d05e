"""Host view of a device-built BVH, field-compatible with the reference's
BvhTree (raysurf/lbvh.py:39-83).  Produced by the plugin's build_tree via
rs_tree_download; the traversal itself never reads these host arrays."""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

TREE_FIELDS = (
    "internal_bounds", "internal_child_left", "internal_child_right",
    "internal_range_left", "internal_range_right", "internal_triangle_id",
    "internal_visit", "leaf_bounds", "leaf_triangle_id", "leaf_range_left",
    "leaf_range_right", "sorted_triangle_ids",
)


@dataclass
class BvhTree:
    num_triangles: int
    internal_bounds: np.ndarray
    internal_child_left: np.ndarray
    internal_child_right: np.ndarray
    internal_range_left: np.ndarray
    internal_range_right: np.ndarray
    internal_triangle_id: np.ndarray
    internal_visit: np.ndarray
    leaf_bounds: np.ndarray
    leaf_triangle_id: np.ndarray
    leaf_range_left: np.ndarray
    leaf_range_right: np.ndarray
    sorted_triangle_ids: np.ndarray
    device: object = field(default=None, repr=False, compare=False)  # DeviceTree handle

    @property
    def num_internal(self) -> int:
        return self.num_triangles - 1

    @property
    def root(self) -> int:
        return int(self.internal_child_left[self.num_triangles - 1])

    def is_leaf_ref(self, ref: int) -> bool:
        return ref >= self.num_internal

    def leaf_index(self, ref: int) -> int:
        return ref - self.num_internal

    def node_bounds(self, ref: int) -> np.ndarray:
        if ref < self.num_internal:
            return self.internal_bounds[ref]
        return self.leaf_bounds[ref - self.num_internal]

    def node_range(self, ref: int) -> tuple[int, int]:
        if ref < self.num_internal:
            return int(self.internal_range_left[ref]), int(self.internal_range_right[ref])
        i = ref - self.num_internal
        return int(self.leaf_range_left[i]), int(self.leaf_range_right[i])

    @classmethod
    def empty(cls, n: int) -> "BvhTree":
        f = {k: np.empty((n, 6) if k.endswith("bounds") else n,
                         np.float32 if k.endswith("bounds") else np.int32) for k in TREE_FIELDS}
        return cls(num_triangles=n, **f)
