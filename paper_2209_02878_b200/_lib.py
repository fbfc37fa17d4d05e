"""ctypes binding of the engine's C ABI (include/raysurf_b200.h).

The shared library is built in-tree by `make -C paper_2209_02878_b200/csrc`
(or `__graft_entry__.build()`).  There is no fallback: if the library is
missing or no CUDA device is present, every compute call raises.
"""

from __future__ import annotations

import contextlib
import ctypes as C
import re
from pathlib import Path

from .exceptions import TraversalStackOverflow, ValidationError

PKG = Path(__file__).resolve().parent
import os as _os

LIB_PATH = Path(_os.environ.get("RS_LIB", PKG / "lib" / "libraysurf_b200.so"))  # RS_LIB: A/B builds
HEADER = PKG.parent / "include" / "raysurf_b200.h"

RS_OK, RS_STACK_OVERFLOW, RS_CUDA_ERROR, RS_INVALID_ARG, RS_INTERNAL = range(5)
MODE_TAGS = {"boolean": 0, "barycentric": 1, "count": 2}
TREE_KINDS = {"reference": 0, "fast": 1}

p, i32, i64 = C.c_void_p, C.c_int, C.c_int64
_SIGS = {
    "rs_abi_version": (i32, []),
    "rs_last_error": (C.c_char_p, []),
    "rs_build": (i32, [p, i64, p, i64, i32, p, p]),
    "rs_build_from_sorted": (i32, [p, i64, p, i64, p, p, p, p]),
    "rs_tree_info": (i32, [p, p, p, p, p, p]),
    "rs_tree_download": (i32, [p] + [p] * 12 + [p]),
    "rs_free": (i32, [p, p]),
    "rs_query": (i32, [p, p, p, i64, i32, i32, i32, i32, p, p, p, p, p, p, p]),
    "rs_query_compact": (i32, [p, p, p, i64, i32, i32, i32, p, p, p, p, p, p, p]),
    "rs_query_stats": (i32, [p, p, p, i64, i32, i32, i32, i32, p, p, p]),
    "rs_baseline": (i32, [p, i64, p, i64, p, p, i64, i32, p, p, p, p, p, p]),
    "rs_run_batch_device": (i32, [p, i64, p, i64, p, p, i64, i32, i32, i32, i32,
                                  p, p, p, p, p, p, p, p]),
    "rs_run_batch_host": (i32, [p, i64, p, i64, p, p, i64, i32, i32, i32, i32, i64,
                                p, p, p, p, p, p, p, p]),
    "rs_set_timing": (i32, [i32]),
    "rs_last_timings": (i32, [p, p, p]),
    "rs_last_phases": (i32, [p, i32]),
    "rs_stage_times": (i32, [p, i32]),
    "rs_kernel_launches": (C.c_longlong, []),
    "rs_last_status": (i32, [p]),
    "rs_set_option": (i32, [C.c_char_p, C.c_longlong, p]),
    "rs_hot_kernel": (C.c_char_p, []),
    "rs_sort_segments": (i32, [p, p, i64, p, p, p, p]),
    "rs_baseline_compact": (i32, [p, i64, p, i64, p, p, i64, p, p, p, p, p, p]),
    "rs_unpermute_dense": (i32, [p, i64, p, p, p]),
    "rs_segment_boxes": (i32, [p, p, i64, p, p]),
    "rs_oracle_intersect": (i32, [p, i64, p, i64, p, p, i64, i32, p, p, p, p, p, p, p]),
    "rs_unpermute_rows": (i32, [p, i64, p, p, p, p, i64, p, p, p, p, p]),
    "rs_generate_segments": (i32, [p, p, i64, C.c_double, C.c_double, C.c_double, C.c_double,
                                   C.c_double, C.c_uint64, i64, i64, p, p, p, p]),
}

_lib = None


def header_symbols() -> list[str]:
    """Every entry point include/raysurf_b200.h declares."""
    return re.findall(r"RS_API\s+[^()]*?\b(rs_\w+)\s*\(", HEADER.read_text())


def lib() -> C.CDLL:
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise ImportError(
                f"{LIB_PATH} is missing: build it with `make -C {PKG / 'csrc'}` "
                "(the engine has no CPU fallback)")
        dll = C.CDLL(str(LIB_PATH))
        for name, (res, args) in _SIGS.items():
            if "RS_LIB" in _os.environ and not hasattr(dll, name):
                continue  # an older A/B build without a newer diagnostic entry point
            fn = getattr(dll, name)
            fn.restype = res
            fn.argtypes = args
        _lib = dll
    return _lib


@contextlib.contextmanager
def option(name: str, value: int):
    """Temporarily set a fast-path tuning knob (rs_set_option)."""
    old = C.c_longlong()
    check(lib().rs_set_option(name.encode(), int(value), C.byref(old)))
    try:
        yield
    finally:
        lib().rs_set_option(name.encode(), old.value, None)


# ResultSet.timings keys filled from device events (engine.py:238-288), in
# rs_last_phases order; "ray sort" is timed by the engine around its sort.
PHASES = ("ray boxes", "quantization", "encoding", "sorting", "reset", "construct", "query")


def last_phases() -> dict:
    """Seconds per reference phase of the calling thread's last native call
    (phases that did not run are absent)."""
    arr = (C.c_float * len(PHASES))()
    if lib().rs_last_phases(arr, len(PHASES)) != RS_OK:
        return {}
    return {k: arr[i] / 1e3 for i, k in enumerate(PHASES) if arr[i] >= 0}


def last_error() -> str:
    msg = lib().rs_last_error()
    return msg.decode() if msg else ""


def check(status: int, bad_segment: int | None = None, max_stack: int | None = None) -> None:
    """Map an RS_* status onto the reference's exception contract
    (exceptions.py:4-26, _compiled.py:108-112)."""
    if status == RS_OK:
        return
    if status == RS_STACK_OVERFLOW:
        raise TraversalStackOverflow(
            f"traversal stack overflow (capacity {max_stack})", segment_index=bad_segment)
    if status == RS_INVALID_ARG:
        raise ValidationError(last_error())
    if status == RS_CUDA_ERROR and "memory" in last_error():
        raise MemoryError(last_error())
    raise RuntimeError(f"raysurf_b200 status {status}: {last_error()}")
