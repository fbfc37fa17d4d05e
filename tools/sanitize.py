"""Small workloads for compute-sanitizer (memcheck / racecheck / synccheck).

Every default kernel of the product path runs at least once, on device and
host inputs, and through a captured graph:
  build:      k_prep, k_keys, k_sort_hist, k_onesweep, k_climb_lean (fast
              query-only trees), k_climb (reference / downloadable trees)
  binning:    k_seg_sample, k_bin_count_tma, k_bin_scan1, k_bin_scatter
  traversal:  k_trav_tile (dense batch), k_trav_sorted_bin (sparse batch),
              k_query_dense (reference semantics)
  output:     k_bary_compact, k_status_out, k_baseline (dense and compacted)
  round 2:    k_generate (device segments), k_expand_bits (hit bitmap of
              large boolean batches, forced on small ones via hitbits_min),
              the device-chunked loop (device_chunk), k_unpermute_dense /
              k_rows_inverse / k_gather_compact (sort_rays on device),
              k_segment_boxes, inside_closed_surface (count mode)
Exits non-zero if any result differs from the generator's ground truth.

usage: compute-sanitizer --tool memcheck python tools/sanitize.py [small]
"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch

import paper_2209_02878_b200 as rs

small = len(sys.argv) > 1 and sys.argv[1] == "small"


def dev(sc):
    t = lambda a: torch.from_numpy(a).cuda()  # noqa: E731
    return (rs.Mesh.from_arrays(t(sc.mesh.vertices), t(sc.mesh.triangles)),
            rs.SegmentBatch.from_arrays(t(sc.segments.starts), t(sc.segments.ends)))


def check(r, truth, mode, what):
    if mode == "boolean":
        got = r.crossing
    elif mode == "count":
        got = r.counts
    else:
        got = r.ray_index
        truth = np.nonzero(truth)[0]
    got = got.cpu().numpy() if hasattr(got, "cpu") else np.asarray(got)
    assert np.array_equal(got, truth.astype(got.dtype)), what


# dense: >= 16 segments per triangle -> k_trav_tile; sparse -> k_trav_sorted_bin
cases = [(500, 20_000 if small else 60_000, "dense"), (4000, 5000, "sparse")]
for n_tri, n_seg, tag in cases:
    sc = rs.generate_scene(n_tri, n_seg, 0.5, seed=3)
    truth = sc.expected_crossings.astype(np.int32)
    dm, db = dev(sc)
    for mode in rs.MODES:
        for rep in range(3):  # call 2 captures the graph, call 3 replays it
            check(rs.run_batch(dm, db, rs.EngineConfig(mode=mode)), truth, mode, f"{tag} dev {mode}")
        check(rs.run_batch(sc.mesh, sc.segments, rs.EngineConfig(mode=mode)), truth, mode, f"{tag} host {mode}")
        check(rs.run_batch(sc.mesh, sc.segments, rs.EngineConfig(mode=mode, tree="reference")), truth, mode,
              f"{tag} reference {mode}")
    from paper_2209_02878_b200._backend import b200
    b200.DeviceTree(sc.mesh, kind="fast").download()
    b200.DeviceTree(sc.mesh, kind="reference").download()

sc = rs.generate_scene(300, 3000, 0.5, seed=4)
truth = sc.expected_crossings.astype(np.int32)
for mode in rs.MODES:
    check(rs.run_baseline_allpairs(sc.mesh, sc.segments, rs.EngineConfig(mode=mode)), truth, mode, f"baseline {mode}")
    check(rs.run_batch(sc.mesh, sc.segments, rs.EngineConfig(mode=mode, sort_rays=True)), truth, mode, f"sort_rays {mode}")
from paper_2209_02878_b200 import _lib

# device generator + hit bitmap + device-chunked loop
mesh = rs.generate_scene(2000, 0, 0.5, seed=2022).mesh
dmesh = rs.Mesh.from_arrays(torch.from_numpy(mesh.vertices).cuda(), torch.from_numpy(mesh.triangles).cuda())
segs, flags = rs.generate_segments_device(dmesh, 40_000 if small else 200_000, 0.5, seed=9, first=123)
truth = flags.cpu().numpy().astype(np.int32)
with _lib.option("hitbits_min", 1):
    check(rs.run_batch(dmesh, segs, rs.EngineConfig(mode="boolean")), truth, "boolean", "bitmap")
    with _lib.option("device_chunk", 8192):
        check(rs.run_batch(dmesh, segs, rs.EngineConfig(mode="boolean")), truth, "boolean", "chunked bitmap")
with _lib.option("device_chunk", 8192):
    for mode in ("count", "barycentric"):
        check(rs.run_batch(dmesh, segs, rs.EngineConfig(mode=mode)), truth, mode, f"chunked {mode}")
# sort_rays on device tensors (un-permutation kernels), segment boxes
for mode in rs.MODES:
    check(rs.run_batch(dmesh, segs, rs.EngineConfig(mode=mode, sort_rays=True)), truth, mode, f"dev sort_rays {mode}")
    check(rs.run_baseline_allpairs(dmesh, rs.SegmentBatch(segs.starts[:3000], segs.ends[:3000]),
                                   rs.EngineConfig(mode=mode, sort_rays=True)), truth[:3000], mode,
          f"dev baseline sort_rays {mode}")
rs.compute_segment_boxes(segs)
# odd parity on a closed cube
v = np.array([[x, y, z] for x in (-0.5, 0.5) for y in (-0.5, 0.5) for z in (-0.5, 0.5)], np.float32)
quads = [(0, 1, 3, 2), (4, 6, 7, 5), (0, 4, 5, 1), (2, 3, 7, 6), (0, 2, 6, 4), (1, 5, 7, 3)]
t = np.array([tri for a, b, c, d in quads for tri in ((a, b, c), (a, c, d))], np.int32)
pts = np.array([[0, 0, 0], [2, 0, 0]], np.float32)
assert rs.inside_closed_surface(pts, rs.Mesh.from_arrays(v, t)).tolist() == [True, False]
torch.cuda.synchronize()
print("sanitize workload ok")
