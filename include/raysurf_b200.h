/*
 * raysurf_b200.h -- C ABI of the B200 segment/triangle intersection engine.
 *
 * This is the drop-in boundary for the reference's kernel-backend plugin
 * (raysurf/_backend/__init__.py:15-51, module protocol build_tree /
 * batch_query / batch_baseline, and the native _core it wraps).  Plain
 * pointers and sizes only; no torch types.  Every entry point returns an
 * RS_* status; rs_last_error() gives the message for the calling thread.
 *
 * Pointer conventions: `d_` = device (CUDA global memory), `h_` = host
 * (pinned or pageable).  Arrays are C-contiguous little-endian:
 *   vertices (n_v,3) f32, triangles (n_t,3) i32, segment starts/ends
 *   (n_r,3) f32 -- the reference's Mesh / SegmentBatch layouts
 *   (mesh.py:20-32, engine.py:35-48).
 * `stream` is a cudaStream_t (NULL = legacy default stream).
 *
 * Mapping to the reference (paths under raysurf/):
 *   rs_build_from_sorted  <- _backend/_compiled.py:27-69 build_tree(mesh, sorted_codes, sorted_ids)
 *                            and _core.pyx:117-184 construct_range/_climb
 *   rs_build              <- engine.py:250-268 (centroids, support, quantise,
 *                            encode, sort) + build_tree, all on device
 *   rs_query              <- _backend/_compiled.py:72-112 batch_query /
 *                            _core.pyx:195-352 (dense per-segment rows)
 *   rs_query_compact      <- batch_query + engine.py:206-215 _assemble
 *                            (barycentric rows, ascending ray index)
 *   rs_baseline           <- _backend/_compiled.py:115-140 batch_baseline /
 *                            _core.pyx:355-433
 *   rs_tree_download      <- the 12 BvhTree fields (lbvh.py:39-55)
 *   rs_run_batch_host     <- engine.py:222-290 run_batch on host arrays
 *                            (copies, build, query, compaction, copies back)
 */
#ifndef RAYSURF_B200_H
#define RAYSURF_B200_H

#include <stdint.h>

#if defined(__GNUC__)
#define RS_API __attribute__((visibility("default")))
#else
#define RS_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

/* status codes */
#define RS_OK 0
#define RS_STACK_OVERFLOW 1 /* -> TraversalStackOverflow(segment_index) (exceptions.py:21-26) */
#define RS_CUDA_ERROR 2     /* CUDA error or out of device memory (-> MemoryError / RuntimeError) */
#define RS_INVALID_ARG 3    /* -> ValidationError (exceptions.py:15-18) */
#define RS_INTERNAL 4       /* internal capacity exceeded (never expected) */

/* modes (_backend/_compiled.py:17-21) */
#define RS_MODE_BOOLEAN 0
#define RS_MODE_BARYCENTRIC 1
#define RS_MODE_COUNT 2

/* tree kinds */
#define RS_TREE_REFERENCE 0 /* per-axis 63-bit Morton: bit-identical to the reference tree */
#define RS_TREE_FAST 1      /* isotropic 30-bit Morton: same results, fewer node visits */

typedef struct rs_tree rs_tree;

RS_API int rs_abi_version(void);
RS_API const char *rs_last_error(void);

/* Build a BVH over a device-resident mesh (all keys computed on device). */
RS_API int rs_build(const float *d_verts, int64_t n_v, const int32_t *d_tris, int64_t n_t,
             int tree_kind, void *stream, rs_tree **out);

/* Build from caller-sorted Morton keys (device arrays of length n_t):
 * reproduces _compiled.build_tree field for field. */
RS_API int rs_build_from_sorted(const float *d_verts, int64_t n_v, const int32_t *d_tris, int64_t n_t,
                         const uint64_t *d_sorted_codes, const int32_t *d_sorted_ids,
                         void *stream, rs_tree **out);

/* Synchronises `stream`; returns triangle count, root ref, height, kind. */
RS_API int rs_tree_info(const rs_tree *tree, int64_t *n_tri, int32_t *root, int32_t *height,
                 int32_t *kind, void *stream);

/* Copy the 12 BvhTree fields into host arrays (sizes per lbvh.py:39-55:
 * bounds (n,6) f32, the rest (n,) i32).  Any pointer may be NULL. */
RS_API int rs_tree_download(const rs_tree *tree, float *h_internal_bounds, int32_t *h_child_left,
                     int32_t *h_child_right, int32_t *h_range_left, int32_t *h_range_right,
                     int32_t *h_internal_triangle_id, int32_t *h_internal_visit,
                     float *h_leaf_bounds, int32_t *h_leaf_triangle_id,
                     int32_t *h_leaf_range_left, int32_t *h_leaf_range_right,
                     int32_t *h_sorted_triangle_ids, void *stream);

/* Release a tree (stream-ordered). */
RS_API int rs_free(rs_tree *tree, void *stream);

/* Dense per-segment query, device arrays of n_r rows (row i of each output
 * is written; unused outputs may be NULL: boolean writes d_detected, count
 * writes d_counts, barycentric writes d_detected/d_tri/d_dist/d_points).
 * ref_semantics=1 reproduces the reference's max_collisions flush points
 * and max_stack overflow exactly (use with a RS_TREE_REFERENCE tree).
 * Synchronises `stream`.  On RS_STACK_OVERFLOW *bad_segment is the lowest
 * overflowing row. */
RS_API int rs_query(const rs_tree *tree, const float *d_starts, const float *d_ends, int64_t n_r,
             int mode, int max_collisions, int max_stack, int ref_semantics,
             int32_t *d_detected, int32_t *d_counts, int32_t *d_tri, float *d_dist,
             float *d_points, int64_t *bad_segment, void *stream);

/* Barycentric query with fused ordered compaction: rows for intersecting
 * segments only, ray indices ascending (engine.py:206-215).  Output arrays
 * must hold n_r rows; *n_hits receives the row count.  Synchronises. */
RS_API int rs_query_compact(const rs_tree *tree, const float *d_starts, const float *d_ends,
                     int64_t n_r, int max_collisions, int max_stack, int ref_semantics,
                     int32_t *d_ray_index, float *d_distance, int32_t *d_triangle_id,
                     float *d_point, int64_t *n_hits, int64_t *bad_segment, void *stream);

/* Traversal statistics (internal-node visits and exact tests, summed over
 * segments) for the roofline's W32/W64 units.  Synchronises. */
RS_API int rs_query_stats(const rs_tree *tree, const float *d_starts, const float *d_ends, int64_t n_r,
                   int mode, int max_collisions, int max_stack, int ref_semantics,
                   int64_t *internal_visits, int64_t *exact_tests, void *stream);

/* sort_segments_by_morton (reference engine.py:125-147) on device: writes
 * the segments in Z-order of their f64 midpoints (per-axis 21-bit
 * quantisation over the midpoints' support, 63-bit interleave, stable by
 * (code, index)) and perm[k] = original index of sorted slot k (int64, as
 * the reference's np.lexsort result).  Stream-ordered; does not synchronise. */
RS_API int rs_sort_segments(const float *d_starts, const float *d_ends, int64_t n,
                            float *d_out_starts, float *d_out_ends, int64_t *d_perm, void *stream);

/* Synthetic terrain segments generated on device (BASELINE configs[4]: 1B
 * segments cannot come through PCIe from the reference's numpy generator,
 * raysurf/oracle.py:167-274).  Restates that generator's distribution
 * (oracle.py:228-271) with a Philox-4x32-10 stream keyed by (seed, global
 * segment index): rows [first, first + n) of the batch are written to
 * d_starts/d_ends (n,3) f32, and d_flags (n,) u8 (may be NULL) receives the
 * ground truth (1 = crosses the terrain exactly once, 0 = misses).  Any
 * sharding of a batch yields the same rows.  The mesh is a generate_scene
 * height field: z_lo/z_hi its vertex z range, x_hi/y_hi = grid extent + 1.
 * Stream-ordered; does not synchronise. */
RS_API int rs_generate_segments(const float *d_verts, const int32_t *d_tris, int64_t n_t,
                                double z_lo, double z_hi, double x_hi, double y_hi,
                                double crossing_fraction, uint64_t seed, int64_t first, int64_t n,
                                float *d_starts, float *d_ends, uint8_t *d_flags, void *stream);

/* All-pairs baseline (no BVH), device arrays, dense outputs as rs_query. */
RS_API int rs_baseline(const float *d_verts, int64_t n_v, const int32_t *d_tris, int64_t n_t,
                const float *d_starts, const float *d_ends, int64_t n_r, int mode,
                int32_t *d_detected, int32_t *d_counts, int32_t *d_tri, float *d_dist,
                float *d_points, void *stream);

/* All-pairs barycentric with ordered compaction (engine.py:320-335 +
 * _assemble): rows for intersecting segments only, ray index ascending;
 * output arrays hold n_r rows, *n_hits receives the count.  Synchronises. */
RS_API int rs_baseline_compact(const float *d_verts, int64_t n_v, const int32_t *d_tris, int64_t n_t,
                               const float *d_starts, const float *d_ends, int64_t n_r,
                               int32_t *d_ray_index, float *d_distance, int32_t *d_triangle_id,
                               float *d_point, int64_t *n_hits, void *stream);

/* oracle_intersect (oracle.py:30-158): the reference's independent
 * verification oracle on device -- all pairs, plane intersection + three
 * edge sign tests in f64 (no Moller-Trumbore, no box prescreen).  boolean /
 * count -> d_flags (n_r rows); barycentric -> compacted rows, *n_hits.
 * Synchronises. */
RS_API int rs_oracle_intersect(const float *d_verts, int64_t n_v, const int32_t *d_tris, int64_t n_t,
                               const float *d_starts, const float *d_ends, int64_t n_r, int mode,
                               int32_t *d_flags, int32_t *d_ray_index, float *d_distance,
                               int32_t *d_triangle_id, float *d_point, int64_t *n_hits, void *stream);

/* compute_segment_boxes (engine.py:115-122): d_boxes (n,6) f32
 * [xmin,xmax,ymin,ymax,zmin,zmax] per segment.  Stream-ordered. */
RS_API int rs_segment_boxes(const float *d_starts, const float *d_ends, int64_t n, float *d_boxes,
                            void *stream);

/* sort_rays un-permutation (engine.py:191-198) on device, perm[k] = original
 * index of sorted slot k (rs_sort_segments).  Dense rows: d_out[perm[k]] =
 * d_in[k].  Barycentric rows (k of them, ray index = sorted slot): written
 * to o_* ascending by original index perm[ray].  Stream-ordered. */
RS_API int rs_unpermute_dense(const int64_t *d_perm, int64_t n, const int32_t *d_in, int32_t *d_out,
                              void *stream);
RS_API int rs_unpermute_rows(const int64_t *d_perm, int64_t n, const int32_t *d_ray_index,
                             const float *d_distance, const int32_t *d_triangle_id,
                             const float *d_point, int64_t k, int32_t *o_ray_index,
                             float *o_distance, int32_t *o_triangle_id, float *o_point, void *stream);

/* Whole run_batch on device arrays: build (tree_kind) + query (+ compaction
 * for barycentric).  boolean -> d_flags = crossing, count -> d_flags = counts;
 * barycentric -> d_ray_index/d_distance/d_triangle_id/d_point (n_r rows
 * capacity), *n_hits.  Synchronises. */
RS_API int rs_run_batch_device(const float *d_verts, int64_t n_v, const int32_t *d_tris, int64_t n_t,
                        const float *d_starts, const float *d_ends, int64_t n_r, int mode,
                        int tree_kind, int max_collisions, int max_stack, int32_t *d_flags,
                        int32_t *d_ray_index, float *d_distance, int32_t *d_triangle_id,
                        float *d_point, int64_t *n_hits, int64_t *bad_segment, void *stream);

/* Whole run_batch on HOST arrays: mesh H2D, device build, rays streamed in
 * chunks (H2D / query / D2H overlapped on two streams), results D2H.
 * Outputs as rs_run_batch_device but host arrays (barycentric rows capacity
 * n_r).  chunk_rays <= 0 picks the default. */
RS_API int rs_run_batch_host(const float *h_verts, int64_t n_v, const int32_t *h_tris, int64_t n_t,
                      const float *h_starts, const float *h_ends, int64_t n_r, int mode,
                      int tree_kind, int max_collisions, int max_stack, int64_t chunk_rays,
                      int32_t *h_flags, int32_t *h_ray_index, float *h_distance,
                      int32_t *h_triangle_id, float *h_point, int64_t *n_hits,
                      int64_t *bad_segment, void *stream);

/* Device phase timing (the reference's ResultSet.timings, engine.py:238-288,
 * measured with CUDA events on the device).  Thread-local level, default 1
 * (env RS_TIMING overrides): 0 off; 1 the reference's phases plus the
 * traversal kernel; 2 the traversal kernel only (the lightest: bench.py's
 * timed region); 3 every stage (diagnostics).  Inside a captured graph the
 * marks are side-branch nodes, off the kernel chain.
 *
 * rs_last_phases fills up to n of, in this order (ms; -1 = phase not run):
 *   0 "ray boxes"    segment boxes + spatial binning (k_seg_sample ..
 *                    scatter; runs beside the build on a second stream)
 *   1 "quantization" centroid quantisation and Morton encoding (k_keys:
 *   2 "encoding"     one fused kernel, so "encoding" reads 0)
 *   3 "sorting"      the device radix sort of the keys
 *   4 "reset"        tree reset fused with triangle boxes, centroids, support (k_prep)
 *   5 "construct"    the Apetrei climb
 *   6 "query"        traversal + exact tests + compaction (summed over chunks
 *                    on the host path)
 * for the calling thread's last call of rs_build, rs_build_from_sorted,
 * rs_query*, rs_run_batch_device or rs_run_batch_host.
 * rs_last_timings gives build (start .. climb done), query and the traversal
 * kernel alone.  rs_stage_times (level 3) fills ms[k] = time from the call's
 * start to stage mark k (-1 when not reached): 0 prep done, 1 keys+sort done,
 * 2 climb done, 4 binning start, 5 sample done, 6 histogram done, 7 scan
 * done, 8 binning done, 9 status copied, 10 frees done, 13 keys done, 14
 * traversal start, 15 traversal end; 11 and 12 are the host milliseconds
 * spent in the graph launch and in the wait. */
RS_API int rs_set_timing(int enable);
RS_API int rs_last_phases(float *ms, int n);
RS_API int rs_last_timings(float *build_ms, float *query_ms, float *hot_kernel_ms);
RS_API int rs_stage_times(float *ms, int n);

/* Cumulative number of kernels this library has launched. */
RS_API long long rs_kernel_launches(void);

/* Tuning knobs of the fast-tree query (A/B experiments and tests that pin a
 * traversal variant): "trav" (0 auto, 1 per-thread binary, 2 per-thread
 * 4-wide, 3 tile), "tile_density", "tile_balance", "tile_area",
 * "bin_occupancy".  A negative value only reads; the previous value is
 * returned in *old_value.  Results never depend on these. */
RS_API int rs_set_option(const char *name, long long value, long long *old_value);

/* Name of the traversal kernel the fast path chose on its last launch (the
 * dominant kernel bench.py's roofline is quoted on). */
RS_API const char *rs_hot_kernel(void);

/* Diagnostics: the 8 device status words (bad, internal, hits, tile_counter,
 * visits, mts, cand_count, pad) of the calling thread's last
 * rs_run_batch_device call when that call ran a captured graph; all zeros
 * when it ran the direct launches (a graph is captured on an argument set's
 * second call). */
RS_API int rs_last_status(unsigned long long *out8);

#ifdef __cplusplus
}
#endif
#endif /* RAYSURF_B200_H */
