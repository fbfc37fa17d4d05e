"""The B200 kernel backend behind the reference's plugin protocol.

Module protocol (raysurf/_backend/__init__.py:15-51, _compiled.py:27-140):
    NAME
    build_tree(mesh, sorted_codes, sorted_ids, workers=1) -> (BvhTree, reset_s, construct_s)
    batch_query(mesh, tree, segments, seg_boxes, mode, max_collisions,
                max_stack, lo, hi, out) -> None
    batch_baseline(mesh, tri_boxes, segments, seg_boxes, mode, lo, hi, out) -> None

A maintainer registers it with `_BACKENDS["b200"] = b200`.
The trees it returns are built on the GPU from the caller's sorted keys and
are bit-identical to the reference's; batch_query runs with the reference's
exact flush/overflow semantics on that tree.  Every call goes through the C
ABI; there is no CPU path.
"""

from __future__ import annotations

import ctypes as C

import numpy as np

from .. import _lib
from ..mesh import is_device_array
from ..tree import BvhTree

NAME = "b200"


def _torch():
    import torch

    if not torch.cuda.is_available():
        raise RuntimeError("the b200 backend needs a CUDA device (no CPU fallback)")
    return torch


def _dev(a, dtype):
    """Device tensor view/copy of a numpy array or CUDA tensor."""
    torch = _torch()
    if is_device_array(a):
        return a.to(dtype).contiguous()
    return torch.from_numpy(np.ascontiguousarray(a)).to(device="cuda", dtype=dtype, non_blocking=False)


def _p(t):
    return C.c_void_p(0 if t is None else t.data_ptr())


def _stream():
    return C.c_void_p(_torch().cuda.current_stream().cuda_stream)


class DeviceTree:
    """Owns an `rs_tree*` and the device mesh it was built over."""

    def __init__(self, mesh, kind: str = "reference", sorted_codes=None, sorted_ids=None):
        torch = _torch()
        self.V = _dev(mesh.vertices, torch.float32)
        self.T = _dev(mesh.triangles, torch.int32)
        self.n = int(mesh.num_triangles)
        self.kind = kind
        self._h = C.c_void_p()
        lib = _lib.lib()
        if sorted_codes is not None:
            codes = _dev(np.asarray(sorted_codes, np.uint64).view(np.int64), torch.int64)
            ids = _dev(np.asarray(sorted_ids, np.int32), torch.int32)
            st = lib.rs_build_from_sorted(_p(self.V), self.V.shape[0], _p(self.T), self.n,
                                          _p(codes), _p(ids), _stream(), C.byref(self._h))
            self._keep = (codes, ids)
            self.kind = "reference"
        else:
            st = lib.rs_build(_p(self.V), self.V.shape[0], _p(self.T), self.n,
                              _lib.TREE_KINDS[kind], _stream(), C.byref(self._h))
        _lib.check(st)

    def info(self) -> dict:
        n, root, height, kind = C.c_int64(), C.c_int32(), C.c_int32(), C.c_int32()
        _lib.check(_lib.lib().rs_tree_info(self._h, C.byref(n), C.byref(root), C.byref(height),
                                           C.byref(kind), _stream()))
        return {"num_triangles": n.value, "root": root.value, "height": height.value,
                "kind": ("reference", "fast")[kind.value]}

    def download(self) -> BvhTree:
        t = BvhTree.empty(self.n)
        arrs = [t.internal_bounds, t.internal_child_left, t.internal_child_right,
                t.internal_range_left, t.internal_range_right, t.internal_triangle_id,
                t.internal_visit, t.leaf_bounds, t.leaf_triangle_id, t.leaf_range_left,
                t.leaf_range_right, t.sorted_triangle_ids]
        _lib.check(_lib.lib().rs_tree_download(
            self._h, *[C.c_void_p(a.ctypes.data) for a in arrs], _stream()))
        t.device = self
        return t

    def query_dense(self, starts, ends, mode: str, max_collisions: int, max_stack: int,
                    ref_semantics: bool = True) -> dict:
        """Dense rows for every segment (device tensors)."""
        torch = _torch()
        s = _dev(starts, torch.float32)
        e = _dev(ends, torch.float32)
        n = int(s.shape[0])
        out = {"detected": torch.zeros(n, dtype=torch.int32, device="cuda"),
               "counts": torch.zeros(n, dtype=torch.int32, device="cuda"),
               "tri": torch.full((n,), -1, dtype=torch.int32, device="cuda"),
               "dist": torch.zeros(n, dtype=torch.float32, device="cuda"),
               "points": torch.zeros((n, 3), dtype=torch.float32, device="cuda")}
        bad = C.c_int64(-1)
        st = _lib.lib().rs_query(self._h, _p(s), _p(e), n, _lib.MODE_TAGS[mode], max_collisions,
                                 max_stack, int(ref_semantics), _p(out["detected"]),
                                 _p(out["counts"]), _p(out["tri"]), _p(out["dist"]),
                                 _p(out["points"]), C.byref(bad), _stream())
        _lib.check(st, bad.value, max_stack)
        return out

    def query_compact(self, starts, ends, max_collisions: int = 32, max_stack: int = 64,
                      ref_semantics: bool = False) -> dict:
        torch = _torch()
        s = _dev(starts, torch.float32)
        e = _dev(ends, torch.float32)
        n = int(s.shape[0])
        ray = torch.empty(n, dtype=torch.int32, device="cuda")
        dist = torch.empty(n, dtype=torch.float32, device="cuda")
        tri = torch.empty(n, dtype=torch.int32, device="cuda")
        pt = torch.empty((n, 3), dtype=torch.float32, device="cuda")
        k, bad = C.c_int64(0), C.c_int64(-1)
        st = _lib.lib().rs_query_compact(self._h, _p(s), _p(e), n, max_collisions, max_stack,
                                         int(ref_semantics), _p(ray), _p(dist), _p(tri), _p(pt),
                                         C.byref(k), C.byref(bad), _stream())
        _lib.check(st, bad.value, max_stack)
        m = k.value
        return {"ray_index": ray[:m], "distance": dist[:m], "triangle_id": tri[:m], "point": pt[:m]}

    def stats(self, starts, ends, mode: str = "boolean", max_collisions: int = 32,
              max_stack: int = 64, ref_semantics: bool = False) -> dict:
        torch = _torch()
        s = _dev(starts, torch.float32)
        e = _dev(ends, torch.float32)
        v, m = C.c_int64(0), C.c_int64(0)
        _lib.check(_lib.lib().rs_query_stats(self._h, _p(s), _p(e), int(s.shape[0]),
                                             _lib.MODE_TAGS[mode], max_collisions, max_stack,
                                             int(ref_semantics), C.byref(v), C.byref(m), _stream()))
        return {"internal_visits": v.value, "exact_tests": m.value}

    def close(self):
        if self._h:
            _lib.lib().rs_free(self._h, _stream())
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


# ---------------------------------------------------------------- protocol --

def build_tree(mesh, sorted_codes, sorted_ids, workers: int = 1):
    """_compiled.py:27-69: returns (tree, reset_s, construct_s), the device
    times of the reset (k_prep: tree reset fused with the triangle boxes) and
    of the climb, from CUDA events (rs_last_phases)."""
    dt = DeviceTree(mesh, sorted_codes=sorted_codes, sorted_ids=sorted_ids)
    ph = _lib.last_phases()  # before download: the build's marks
    tree = dt.download()
    return tree, ph.get("reset", 0.0), ph.get("construct", 0.0)


def _device_tree_for(mesh, tree: BvhTree) -> DeviceTree:
    dt = getattr(tree, "device", None)
    if isinstance(dt, DeviceTree):
        return dt
    # a tree built elsewhere (e.g. by the reference's own backend): rebuild it
    # on device from the mesh (device keys + sort, reference kind); the climb
    # reproduces it exactly when it came from this mesh's Morton order.
    dt = DeviceTree(mesh, kind="reference")
    if not np.array_equal(np.asarray(dt.download().sorted_triangle_ids),
                          np.asarray(tree.sorted_triangle_ids)):
        raise ValueError("tree was not built from this mesh's Morton order")
    tree.device = dt
    return dt


def _as_host_error(exc: Exception) -> Exception:
    """The error in the calling package's own classes: registered inside the
    reference (`raysurf._backend`), its engine and tests catch
    raysurf.exceptions.TraversalStackOverflow / ValidationError
    (_compiled.py:108-112 raises those), not this package's."""
    import sys

    from .. import exceptions as ours

    host = sys.modules.get("raysurf.exceptions")
    if host is None or host is ours:
        return exc
    if isinstance(exc, ours.TraversalStackOverflow):
        return host.TraversalStackOverflow(str(exc), segment_index=exc.segment_index)
    if isinstance(exc, ours.ValidationError):
        return host.ValidationError(str(exc))
    return exc


def batch_query(mesh, tree, segments, seg_boxes, mode, max_collisions, max_stack, lo, hi, out):
    """_compiled.py:72-112: rows [lo, hi) of `out`; seg_boxes are recomputed
    on device from the endpoints (engine.py:115-122 gives the same boxes)."""
    if hi <= lo:
        return
    dt = _device_tree_for(mesh, tree)
    try:
        res = dt.query_dense(segments.starts[lo:hi], segments.ends[lo:hi], mode, max_collisions,
                             max_stack, ref_semantics=True)
    except Exception as exc:
        from ..exceptions import TraversalStackOverflow

        if isinstance(exc, TraversalStackOverflow) and exc.segment_index is not None:
            exc.segment_index += lo
        host = _as_host_error(exc)
        if host is exc:
            raise
        raise host from exc
    _store(out, lo, hi, mode, res)


def batch_baseline(mesh, tri_boxes, segments, seg_boxes, mode, lo, hi, out):
    """_compiled.py:115-140: rows [lo, hi) of `out`."""
    if hi <= lo:
        return
    res = baseline_dense(mesh, type(segments)(segments.starts[lo:hi], segments.ends[lo:hi]), mode)
    _store(out, lo, hi, mode, res)


def _store(out, lo, hi, mode, res):
    keys = {"boolean": ("detected",), "count": ("counts",),
            "barycentric": ("detected", "tri", "dist", "points")}[mode]
    for k in keys:
        v = res[k]
        out[k][lo:hi] = v.cpu().numpy() if is_device_array(v) else v


def baseline_compact(mesh, segments):
    """All-pairs barycentric on device tensors with the ordered compaction
    (rs_baseline_compact); returns a ResultSet of CUDA tensors."""
    from ..engine import MODE_BARYCENTRIC, ResultSet

    torch = _torch()
    V = _dev(mesh.vertices, torch.float32)
    T = _dev(mesh.triangles, torch.int32)
    s = _dev(segments.starts, torch.float32)
    e = _dev(segments.ends, torch.float32)
    n = int(s.shape[0])
    ray = torch.empty(n, dtype=torch.int32, device=s.device)
    dist = torch.empty(n, dtype=torch.float32, device=s.device)
    tri = torch.empty(n, dtype=torch.int32, device=s.device)
    pt = torch.empty((n, 3), dtype=torch.float32, device=s.device)
    k = C.c_int64(0)
    _lib.check(_lib.lib().rs_baseline_compact(
        _p(V), int(V.shape[0]), _p(T), int(T.shape[0]), _p(s), _p(e), n, _p(ray), _p(dist), _p(tri),
        _p(pt), C.byref(k), _stream()))
    m = k.value
    return ResultSet(MODE_BARYCENTRIC, n, ray_index=ray[:m], distance=dist[:m], triangle_id=tri[:m],
                     point=pt[:m])


def baseline_dense(mesh, segments, mode: str) -> dict:
    """All-pairs on device; returns numpy rows for host inputs, tensors for
    device inputs."""
    torch = _torch()
    host = not is_device_array(segments.starts)
    V = _dev(mesh.vertices, torch.float32)
    T = _dev(mesh.triangles, torch.int32)
    s = _dev(segments.starts, torch.float32)
    e = _dev(segments.ends, torch.float32)
    n = int(s.shape[0])
    out = {"detected": torch.zeros(n, dtype=torch.int32, device="cuda"),
           "counts": torch.zeros(n, dtype=torch.int32, device="cuda"),
           "tri": torch.full((n,), -1, dtype=torch.int32, device="cuda"),
           "dist": torch.zeros(n, dtype=torch.float32, device="cuda"),
           "points": torch.zeros((n, 3), dtype=torch.float32, device="cuda")}
    st = _lib.lib().rs_baseline(_p(V), int(V.shape[0]), _p(T), int(T.shape[0]), _p(s), _p(e), n,
                                _lib.MODE_TAGS[mode], _p(out["detected"]), _p(out["counts"]),
                                _p(out["tri"]), _p(out["dist"]), _p(out["points"]), _stream())
    _lib.check(st)
    if host:
        return {k: v.cpu().numpy() for k, v in out.items()}
    return out
