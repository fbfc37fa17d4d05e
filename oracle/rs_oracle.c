/*
 * rs_oracle.c -- CPU restatement of the reference `raysurf` run_batch path.
 *
 * TEST INFRASTRUCTURE ONLY.  Nothing in the product (paper_2209_02878_b200)
 * links, loads or calls this file.  It is the parity checker used by tests/,
 * __graft_entry__.smoke() and the cpu_baseline leg of bench.py.
 *
 * Every function cites the reference file:line it restates (paths relative to
 * the reference package root, /root/reference/pkg/src/raysurf/).  The
 * arithmetic is kept in the reference's operation order and this file must be
 * compiled with -ffp-contract=off (mirrors setup.py:24-26) so the f64
 * Moller-Trumbore and the f64 Morton quantisation round identically.
 *
 * Parity pinning: tests/test_oracle_golden.py checks these functions against
 * fixtures produced by running the reference itself (tests/golden/make_golden.py).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define RO_EMPTY (-1)
#define RO_DET_EPS 1e-9  /* geometry.py:14-15 */
#define RO_BARY_EPS 1e-7 /* geometry.py:16-17 */
#define RO_GRID_MAX 2097151.0 /* morton.py:15-16 (2^21 - 1) */

enum { RO_BOOLEAN = 0, RO_BARYCENTRIC = 1, RO_COUNT = 2 }; /* _compiled.py:17-21 */

/* ---------------------------------------------------------------- mesh ---- */

/* mesh.py:69-79: per-triangle AABB [xmin,xmax,ymin,ymax,zmin,zmax], f32. */
void ro_tri_boxes(const float *V, const int32_t *T, int64_t nt, float *boxes) {
    for (int64_t j = 0; j < nt; ++j) {
        const float *a = V + 3 * (int64_t)T[3 * j];
        const float *b = V + 3 * (int64_t)T[3 * j + 1];
        const float *c = V + 3 * (int64_t)T[3 * j + 2];
        for (int k = 0; k < 3; ++k) {
            float lo = fminf(a[k], b[k]), hi = fmaxf(a[k], b[k]);
            lo = fminf(lo, c[k]);
            hi = fmaxf(hi, c[k]);
            boxes[6 * j + 2 * k] = lo;
            boxes[6 * j + 2 * k + 1] = hi;
        }
    }
}

/* engine.py:115-122: per-segment AABB, same layout. */
static inline void seg_box(const float *s, const float *e, float *box) {
    for (int k = 0; k < 3; ++k) {
        box[2 * k] = s[k] < e[k] ? s[k] : e[k];
        box[2 * k + 1] = s[k] > e[k] ? s[k] : e[k];
    }
}

/* ---------------------------------------------------------------- morton -- */

/* morton.py:34-37: ((va + vb) + vc) / 3.0 in f64. */
void ro_centroids(const float *V, const int32_t *T, int64_t nt, double *c) {
    for (int64_t j = 0; j < nt; ++j)
        for (int k = 0; k < 3; ++k) {
            double a = V[3 * (int64_t)T[3 * j] + k];
            double b = V[3 * (int64_t)T[3 * j + 1] + k];
            double d = V[3 * (int64_t)T[3 * j + 2] + k];
            c[3 * j + k] = ((a + b) + d) / 3.0;
        }
}

/* morton.py:40-45: componentwise min / max. */
void ro_support(const double *p, int64_t n, double *lo, double *hi) {
    for (int k = 0; k < 3; ++k) { lo[k] = p[k]; hi[k] = p[k]; }
    for (int64_t i = 1; i < n; ++i)
        for (int k = 0; k < 3; ++k) {
            if (p[3 * i + k] < lo[k]) lo[k] = p[3 * i + k];
            if (p[3 * i + k] > hi[k]) hi[k] = p[3 * i + k];
        }
}

static inline uint32_t quant1(double p, double lo, double ext, double gmax) {
    double s = floor((p - lo) / ext * gmax);
    if (s < 0.0) s = 0.0;
    if (s > gmax) s = gmax;
    return (uint32_t)s;
}

/* morton.py:48-63: per-axis floor((p - lo) / ext * (2^21-1)), clipped; ext == 0 -> 0. */
void ro_quantize(const double *p, int64_t n, const double *lo, const double *hi, uint32_t *q) {
    for (int k = 0; k < 3; ++k) {
        double ext = hi[k] - lo[k];
        for (int64_t i = 0; i < n; ++i)
            q[3 * i + k] = ext > 0.0 ? quant1(p[3 * i + k], lo[k], ext, RO_GRID_MAX) : 0u;
    }
}

/* NOT a reference function: the "fast" tree's isotropic quantiser (DESIGN.md
 * section 3).  One extent (the largest axis) for all three axes, grid of
 * 2^bits - 1 cells.  Kept here so GPU fast trees can be compared bitwise. */
void ro_quantize_iso(const double *p, int64_t n, const double *lo, const double *hi, int bits,
                     uint32_t *q) {
    double ext = 0.0;
    for (int k = 0; k < 3; ++k)
        if (hi[k] - lo[k] > ext) ext = hi[k] - lo[k];
    double gmax = (double)((1u << bits) - 1u);
    for (int64_t i = 0; i < n; ++i)
        for (int k = 0; k < 3; ++k)
            q[3 * i + k] = ext > 0.0 ? quant1(p[3 * i + k], lo[k], ext, gmax) : 0u;
}

/* morton.py:72-80 (magic masks), x -> bit 0, y -> bit 1, z -> bit 2. */
static inline uint64_t split21(uint64_t v) {
    v &= 0x1FFFFFull;
    v = (v | v << 32) & 0x1F00000000FFFFull;
    v = (v | v << 16) & 0x1F0000FF0000FFull;
    v = (v | v << 8) & 0x100F00F00F00F00Full;
    v = (v | v << 4) & 0x10C30C30C30C30C3ull;
    v = (v | v << 2) & 0x1249249249249249ull;
    return v;
}

/* morton.py:117-128. */
void ro_morton_codes(const uint32_t *q, int64_t n, uint64_t *codes) {
    for (int64_t i = 0; i < n; ++i)
        codes[i] = split21(q[3 * i]) | split21(q[3 * i + 1]) << 1 | split21(q[3 * i + 2]) << 2;
}

typedef struct { uint64_t code; int32_t id; } key_t_;

static int key_cmp(const void *pa, const void *pb) {
    const key_t_ *a = (const key_t_ *)pa, *b = (const key_t_ *)pb;
    if (a->code != b->code) return a->code < b->code ? -1 : 1;
    return (a->id > b->id) - (a->id < b->id);
}

/* morton.py:131-146: np.lexsort((ids, codes)) == ascending by (code, id).
 * Sorts in place. */
void ro_sort(uint64_t *codes, int32_t *ids, int64_t n) {
    key_t_ *k = (key_t_ *)malloc(sizeof(key_t_) * (size_t)(n ? n : 1));
    for (int64_t i = 0; i < n; ++i) { k[i].code = codes[i]; k[i].id = ids[i]; }
    qsort(k, (size_t)n, sizeof(key_t_), key_cmp);
    for (int64_t i = 0; i < n; ++i) { codes[i] = k[i].code; ids[i] = k[i].id; }
    free(k);
}

/* ------------------------------------------------------------------ tree -- */

/* lbvh.py:39-55 BvhTree field set, all C-contiguous, caller-owned. */
typedef struct {
    float *int_bounds;   /* (n,6) */
    int32_t *child_l, *child_r, *range_l, *range_r, *int_tri, *visit; /* (n,) */
    float *leaf_bounds;  /* (n,6) */
    int32_t *leaf_tri, *leaf_range_l, *leaf_range_r, *sorted_ids;     /* (n,) */
} ro_tree;

/* lbvh.py:130-145 / _core.pyx:52-64. */
static inline int delta_less(const uint64_t *codes, const int32_t *ids, int64_t a, int64_t b) {
    uint64_t xa = codes[a] ^ codes[a + 1], xb = codes[b] ^ codes[b + 1];
    if (xa != xb) return xa < xb;
    int32_t ia = ids[a] ^ ids[a + 1], ib = ids[b] ^ ids[b + 1];
    if (ia != ib) return ia < ib;
    return a < b;
}

static inline const float *bounds_of(const ro_tree *t, int32_t ref, int32_t n_int) {
    return ref < n_int ? t->int_bounds + 6 * (int64_t)ref : t->leaf_bounds + 6 * (int64_t)(ref - n_int);
}

/* lbvh.py:175-195 (_reset_tree) + lbvh.py:148-172 / _core.pyx:117-184 (climb).
 * tri_boxes are the unsorted per-triangle boxes (mesh.py:69-79).
 * Sequential climb in leaf order: the tree is schedule independent
 * (test_backends.py:58-68), so the order does not matter. */
void ro_build(int64_t n, const uint64_t *codes, const int32_t *ids, const float *tri_boxes,
              ro_tree *t) {
    int32_t n_int = (int32_t)(n - 1);
    memset(t->int_bounds, 0, sizeof(float) * 6 * (size_t)n);
    for (int64_t i = 0; i < n; ++i) {
        t->child_l[i] = RO_EMPTY; t->child_r[i] = RO_EMPTY;
        t->range_l[i] = -1; t->range_r[i] = -1;
        t->int_tri[i] = -1; t->visit[i] = 0;
        memcpy(t->leaf_bounds + 6 * i, tri_boxes + 6 * (int64_t)ids[i], 6 * sizeof(float));
        t->leaf_tri[i] = ids[i];
        t->leaf_range_l[i] = (int32_t)i; t->leaf_range_r[i] = (int32_t)i;
        t->sorted_ids[i] = ids[i];
    }
    if (n == 1) { t->child_l[0] = n_int; return; } /* lbvh.py:163-166 */
    for (int64_t i = 0; i < n; ++i) {
        int64_t left = i, right = i;
        int32_t node = n_int + (int32_t)i;
        for (;;) {
            if (left == 0 && right == n - 1) {
                t->child_l[n - 1] = node;
                if (node < n_int) t->int_tri[node] = -2;
                break;
            }
            int64_t parent;
            if (left == 0 || (right != n - 1 && delta_less(codes, ids, right, left - 1))) {
                parent = right;
                t->child_l[parent] = node;
                t->range_l[parent] = (int32_t)left;
            } else {
                parent = left - 1;
                t->child_r[parent] = node;
                t->range_r[parent] = (int32_t)right;
            }
            if (t->visit[parent]++ == 0) break;
            left = t->range_l[parent];
            right = t->range_r[parent];
            const float *lb = bounds_of(t, t->child_l[parent], n_int);
            const float *rb = bounds_of(t, t->child_r[parent], n_int);
            float *pb = t->int_bounds + 6 * parent;
            for (int k = 0; k < 3; ++k) {
                pb[2 * k] = lb[2 * k] < rb[2 * k] ? lb[2 * k] : rb[2 * k];
                pb[2 * k + 1] = lb[2 * k + 1] > rb[2 * k + 1] ? lb[2 * k + 1] : rb[2 * k + 1];
            }
            node = (int32_t)parent;
        }
    }
}

/* ------------------------------------------------------------- geometry -- */

/* _core.pyx:44-49 / geometry.py:69-79: touching counts as overlap. */
static inline int overlap(const float *a, const float *b) {
    return a[0] <= b[1] && a[1] >= b[0] && a[2] <= b[3] && a[3] >= b[2] && a[4] <= b[5] &&
           a[5] >= b[4];
}

/* geometry.py:82-137 / _core.pyx:67-114: f64 Moller-Trumbore, reference op order. */
int ro_mt_hit(const float *va, const float *vb, const float *vc, const float *s, const float *e,
              double *t_out, double *u_out, double *v_out) {
    double ax = va[0], ay = va[1], az = va[2];
    double sx = s[0], sy = s[1], sz = s[2];
    double e1x = (double)vb[0] - ax, e1y = (double)vb[1] - ay, e1z = (double)vb[2] - az;
    double e2x = (double)vc[0] - ax, e2y = (double)vc[1] - ay, e2z = (double)vc[2] - az;
    double dx = (double)e[0] - sx, dy = (double)e[1] - sy, dz = (double)e[2] - sz;
    double px = dy * e2z - dz * e2y;
    double py = dz * e2x - dx * e2z;
    double pz = dx * e2y - dy * e2x;
    double det = e1x * px + e1y * py + e1z * pz;
    if (fabs(det) < RO_DET_EPS) return 0;
    double inv_det = 1.0 / det;
    double tx = sx - ax, ty = sy - ay, tz = sz - az;
    double u = (tx * px + ty * py + tz * pz) * inv_det;
    if (u < -RO_BARY_EPS || u > 1.0 + RO_BARY_EPS) return 0;
    double qx = ty * e1z - tz * e1y;
    double qy = tz * e1x - tx * e1z;
    double qz = tx * e1y - ty * e1x;
    double v = (dx * qx + dy * qy + dz * qz) * inv_det;
    if (v < -RO_BARY_EPS || u + v > 1.0 + RO_BARY_EPS) return 0;
    double t = (e2x * qx + e2y * qy + e2z * qz) * inv_det;
    if (t < 0.0 || t > 1.0) return 0;
    *t_out = t; *u_out = u; *v_out = v;
    return 1;
}

/* _core.pyx:330-348: point = s + t*d in f64, distance = f32(sqrt(|p - s|^2)). */
static inline void write_bary(const float *sp, const float *ep, double best_t, int32_t best_tri,
                              int64_t i, int32_t *detected, int32_t *tri_out, float *dist_out,
                              float *points_out) {
    double sx = sp[0], sy = sp[1], sz = sp[2];
    double dx = (double)ep[0] - sx, dy = (double)ep[1] - sy, dz = (double)ep[2] - sz;
    double px = sx + best_t * dx, py = sy + best_t * dy, pz = sz + best_t * dz;
    double ddx = px - sx, ddy = py - sy, ddz = pz - sz;
    detected[i] = 1;
    tri_out[i] = best_tri;
    dist_out[i] = (float)sqrt(ddx * ddx + ddy * ddy + ddz * ddz);
    points_out[3 * i] = (float)px;
    points_out[3 * i + 1] = (float)py;
    points_out[3 * i + 2] = (float)pz;
}

/* --------------------------------------------------------------- queries -- */

/* _core.pyx:195-352 (batch_query): coarse traversal into a max_coll buffer
 * with suspend/resume, then exact tests; boolean early exit; min-(t, tid)
 * tie-break.  Returns 0 or 1 (stack overflow); *bad_segment is the lowest
 * overflowing segment in [lo, hi) (engine.py:179-180 chunk-order semantics).
 * stats (optional, length 2): summed internal-node visits and MT calls. */
int ro_query(const float *V, const int32_t *T, const float *starts, const float *ends,
             const ro_tree *t, int32_t root, int64_t n_tri, int mode, int max_coll, int max_stack,
             int64_t lo, int64_t hi, int32_t *detected, int32_t *counts, int32_t *tri_out,
             float *dist_out, float *points_out, int64_t *bad_segment, int nthreads,
             int64_t *stats) {
    const int32_t n_int = (int32_t)(n_tri - 1);
    int64_t bad = INT64_MAX;
    int64_t tot_visit = 0, tot_mt = 0;
#ifdef _OPENMP
    if (nthreads <= 0) nthreads = omp_get_max_threads();
#pragma omp parallel num_threads(nthreads) reduction(+ : tot_visit, tot_mt)
#endif
    {
        int32_t *stack = (int32_t *)malloc(sizeof(int32_t) * (size_t)(max_stack > 0 ? max_stack : 1));
        int32_t *buf = (int32_t *)malloc(sizeof(int32_t) * (size_t)max_coll);
#ifdef _OPENMP
#pragma omp for schedule(dynamic, 1024)
#endif
        for (int64_t i = lo; i < hi; ++i) {
            int64_t cur_bad;
#ifdef _OPENMP
#pragma omp atomic read
#endif
            cur_bad = bad;
            if (i > cur_bad) continue;
            const float *sp = starts + 3 * i, *ep = ends + 3 * i;
            float qbox[6];
            seg_box(sp, ep, qbox);
            stack[0] = RO_EMPTY;
            int top = 1;
            int32_t node = root;
            int det_flag = 0, has_best = 0, n_hits = 0, overflow = 0;
            double best_t = 0.0;
            int32_t best_tri = -1;
            for (;;) {
                int count = 0, full = 0;
                while (node != RO_EMPTY && !full) {
                    if (node >= n_int) { /* _core.pyx:260-267 leaf root */
                        if (overlap(qbox, t->leaf_bounds + 6 * (int64_t)(node - n_int))) {
                            buf[count++] = t->leaf_tri[node - n_int];
                            full = count >= max_coll - 1;
                        }
                        node = stack[--top];
                        continue;
                    }
                    ++tot_visit;
                    int32_t ca = t->child_l[node], cb = t->child_r[node];
                    int la = ca >= n_int, lb = cb >= n_int;
                    int oa = overlap(qbox, bounds_of(t, ca, n_int));
                    int ob = overlap(qbox, bounds_of(t, cb, n_int));
                    if (oa && la) { buf[count++] = t->leaf_tri[ca - n_int]; full = count >= max_coll - 1; }
                    if (ob && lb) { buf[count++] = t->leaf_tri[cb - n_int]; full = full || count >= max_coll - 1; }
                    int ta = oa && !la, tb = ob && !lb;
                    if (!ta && !tb) {
                        node = stack[--top];
                    } else {
                        node = ta ? ca : cb;
                        if (ta && tb) {
                            if (top >= max_stack) { overflow = 1; break; }
                            stack[top++] = cb;
                        }
                    }
                }
                if (overflow) break;
                for (int k = 0; k < count; ++k) {
                    if (mode == RO_BOOLEAN && det_flag) break;
                    int32_t tid = buf[k];
                    double tt, uu, vv;
                    ++tot_mt;
                    if (ro_mt_hit(V + 3 * (int64_t)T[3 * tid], V + 3 * (int64_t)T[3 * tid + 1],
                                  V + 3 * (int64_t)T[3 * tid + 2], sp, ep, &tt, &uu, &vv)) {
                        det_flag = 1;
                        ++n_hits;
                        if (!has_best || tt < best_t || (tt == best_t && tid < best_tri)) {
                            has_best = 1; best_t = tt; best_tri = tid;
                        }
                    }
                }
                if (node == RO_EMPTY || (mode == RO_BOOLEAN && det_flag)) break;
            }
            if (overflow) {
#ifdef _OPENMP
#pragma omp critical
#endif
                { if (i < bad) bad = i; }
                continue;
            }
            if (mode == RO_BOOLEAN) detected[i] = det_flag;
            else if (mode == RO_COUNT) counts[i] = n_hits;
            else if (has_best) write_bary(sp, ep, best_t, best_tri, i, detected, tri_out, dist_out, points_out);
        }
        free(stack);
        free(buf);
    }
    if (stats) { stats[0] = tot_visit; stats[1] = tot_mt; }
    if (bad != INT64_MAX) { *bad_segment = bad; return 1; }
    *bad_segment = -1;
    return 0;
}

/* _core.pyx:355-433 (batch_baseline): every (segment, triangle) pair with
 * the AABB prescreen; boolean breaks at the first hit; tie-break j < best. */
void ro_baseline(const float *V, const int32_t *T, int64_t n_tri, const float *tri_boxes,
                 const float *starts, const float *ends, int mode, int64_t lo, int64_t hi,
                 int32_t *detected, int32_t *counts, int32_t *tri_out, float *dist_out,
                 float *points_out, int nthreads) {
#ifdef _OPENMP
    if (nthreads <= 0) nthreads = omp_get_max_threads();
#pragma omp parallel for num_threads(nthreads) schedule(dynamic, 64)
#endif
    for (int64_t i = lo; i < hi; ++i) {
        const float *sp = starts + 3 * i, *ep = ends + 3 * i;
        float qbox[6];
        seg_box(sp, ep, qbox);
        int det_flag = 0, has_best = 0, n_hits = 0;
        double best_t = 0.0;
        int32_t best_tri = -1;
        for (int64_t j = 0; j < n_tri; ++j) {
            if (!overlap(qbox, tri_boxes + 6 * j)) continue;
            double tt, uu, vv;
            if (!ro_mt_hit(V + 3 * (int64_t)T[3 * j], V + 3 * (int64_t)T[3 * j + 1],
                           V + 3 * (int64_t)T[3 * j + 2], sp, ep, &tt, &uu, &vv))
                continue;
            det_flag = 1;
            ++n_hits;
            if (mode == RO_BOOLEAN) break;
            if (!has_best || tt < best_t || (tt == best_t && j < best_tri)) {
                has_best = 1; best_t = tt; best_tri = (int32_t)j;
            }
        }
        if (mode == RO_BOOLEAN) detected[i] = det_flag;
        else if (mode == RO_COUNT) counts[i] = n_hits;
        else if (has_best) write_bary(sp, ep, best_t, best_tri, i, detected, tri_out, dist_out, points_out);
    }
}
