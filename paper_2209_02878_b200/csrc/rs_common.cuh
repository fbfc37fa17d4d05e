// rs_common.cuh -- shared device types and helpers for the raysurf B200 engine.
//
// HBM layout (one BVH per device):
//   RsNode  nodes[N_t - 1]  64 B  internal node = both children's f32 AABBs
//                                  + both child refs; one 64-B line per visit
//   RsLeaf  leaves[N_t]     48 B  Morton-ordered triangle: 9 vertex floats +
//                                  original triangle id (for the exact test)
//   the reference's SoA BvhTree fields (lbvh.py:39-55) are kept beside them
//   so a built tree can be downloaded field-for-field (rs_tree_download).
//
// Node references use the reference's tagging (lbvh.py:1-17): ref < N_t - 1
// is an internal node, otherwise leaf ref - (N_t - 1); -1 is empty.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace rs {

constexpr int kEmpty = -1;
constexpr double kDetEps = 1e-9;   // geometry.py:14-15
constexpr double kBaryEps = 1e-7;  // geometry.py:16-17
constexpr double kGridMax21 = 2097151.0;  // morton.py:15-16
constexpr int kIsoBits = 10;       // fast tree: 30-bit isotropic Morton

enum Mode { kBoolean = 0, kBarycentric = 1, kCount = 2 };  // _compiled.py:17-21
enum TreeKind { kTreeReference = 0, kTreeFast = 1 };

struct __align__(16) RsNode {
    float4 a;  // l.xmin l.xmax l.ymin l.ymax
    float4 b;  // l.zmin l.zmax r.xmin r.xmax
    float4 c;  // r.ymin r.ymax r.zmin r.zmax
    int4 d;    // lref rref - -
};

// 4-wide node: one 32-B slot per child, read by the 4 lanes of a segment's
// lane group with one 256-bit load each (one 128-B line per node visit).
struct __align__(32) RsSlot {
    float lo_x, hi_x, lo_y, hi_y, lo_z, hi_z;  // exact f32 child AABB
    int ref;                                   // child ref (-1 = empty slot)
    int pad;
};
struct __align__(128) RsNode4 {
    RsSlot s[4];
};

struct __align__(16) RsLeaf {
    float4 p0;  // a.x a.y a.z b.x
    float4 p1;  // b.y b.z c.x c.y
    float4 p2;  // c.z tid(bits) - -
};

// Per-tree device header (zeroed with one memset before a build).
struct RsHeader {
    unsigned long long smin[3];  // ~ordered(min centroid)  (atomicMax of complement)
    unsigned long long smax[3];  //  ordered(max centroid)
    int root;
    int height;
    unsigned bmin[3];            // ~ordered32(min triangle-box coordinate) = root box
    unsigned bmax[3];            //  ordered32(max triangle-box coordinate)
    unsigned tsize[3];           // largest triangle-box side per axis (f32 bits, >= 0)
    float parea;                 // sum over triangles of the box's three projected face areas
};

// Per-query device status (zeroed before a query).
struct RsStatus {
    unsigned long long bad;       // ~lowest overflowing segment (0 = none)
    unsigned long long internal;  // internal-capacity overflow (should stay 0)
    unsigned long long hits;      // barycentric: number of compacted rows
    unsigned long long tile_counter;
    unsigned long long visits;    // optional stats
    unsigned long long mts;
    unsigned long long cand_count;  // collision-buffer entries claimed (may exceed capacity)
    unsigned long long dropped;     // collision buffer overflowed: candidates dropped, re-launch
};

constexpr int kCandChunk = 128;  // collision-buffer entries claimed per warp atomic

// ---- ordered encodings so atomics on u64 give min/max of doubles ----------
__device__ __forceinline__ unsigned long long ord_of(double d) {
    unsigned long long u = __double_as_longlong(d);
    return (u & 0x8000000000000000ull) ? ~u : (u | 0x8000000000000000ull);
}
__host__ __device__ __forceinline__ double from_ord(unsigned long long o) {
    unsigned long long u = (o & 0x8000000000000000ull) ? (o & ~0x8000000000000000ull) : ~o;
#ifdef __CUDA_ARCH__
    return __longlong_as_double(u);
#else
    double d;
    __builtin_memcpy(&d, &u, 8);
    return d;
#endif
}

__device__ __forceinline__ unsigned ord32(float f) {
    const unsigned u = __float_as_uint(f);
    return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
__device__ __forceinline__ float from_ord32(unsigned o) {
    return __uint_as_float((o & 0x80000000u) ? (o & 0x7fffffffu) : ~o);
}

// ---- Morton keys (morton.py:48-63,117-128) -------------------------------
__device__ __forceinline__ unsigned long long split21(unsigned long long v) {
    v &= 0x1FFFFFull;
    v = (v | v << 32) & 0x1F00000000FFFFull;
    v = (v | v << 16) & 0x1F0000FF0000FFull;
    v = (v | v << 8) & 0x100F00F00F00F00Full;
    v = (v | v << 4) & 0x10C30C30C30C30C3ull;
    v = (v | v << 2) & 0x1249249249249249ull;
    return v;
}

__device__ __forceinline__ unsigned quant1(double p, double lo, double ext, double gmax) {
    double s = floor(__dmul_rn(__ddiv_rn(__dsub_rn(p, lo), ext), gmax));
    s = s < 0.0 ? 0.0 : (s > gmax ? gmax : s);  // np.clip (morton.py:62)
    return (unsigned)s;
}

// ---- f32 box test: touching counts (geometry.py:69-79, _core.pyx:44-49) ---
__device__ __forceinline__ bool overlap6(const float q[6], float x0, float x1, float y0, float y1,
                                         float z0, float z1) {
    return q[0] <= x1 && q[1] >= x0 && q[2] <= y1 && q[3] >= y0 && q[4] <= z1 && q[5] >= z0;
}

// ---- f64 Moller-Trumbore in the reference op order (geometry.py:82-137,
// _core.pyx:67-114).  Explicit _rn intrinsics: no FMA contraction, so the
// result is bit-identical to the -ffp-contract=off CPU reference. ----------
// mt_hit_pre takes the triangle's first vertex and both edges already in f64
// (e1 = b - a, e2 = c - a, each one rounded f64 subtraction of f32 inputs,
// exactly as the reference forms them), so a caller testing one triangle
// against many segments forms them once.
__device__ __forceinline__ bool mt_hit_pre(double ax, double ay, double az, double e1x,
                                           double e1y, double e1z, double e2x, double e2y,
                                           double e2z, double sx, double sy, double sz, double dx,
                                           double dy, double dz, double* t_out) {
    const double px = __dsub_rn(__dmul_rn(dy, e2z), __dmul_rn(dz, e2y));
    const double py = __dsub_rn(__dmul_rn(dz, e2x), __dmul_rn(dx, e2z));
    const double pz = __dsub_rn(__dmul_rn(dx, e2y), __dmul_rn(dy, e2x));
    const double det =
        __dadd_rn(__dadd_rn(__dmul_rn(e1x, px), __dmul_rn(e1y, py)), __dmul_rn(e1z, pz));
    if (fabs(det) < kDetEps) return false;
    const double tx = __dsub_rn(sx, ax), ty = __dsub_rn(sy, ay), tz = __dsub_rn(sz, az);
    const double un = __dadd_rn(__dadd_rn(__dmul_rn(tx, px), __dmul_rn(ty, py)), __dmul_rn(tz, pz));
    const double qx = __dsub_rn(__dmul_rn(ty, e1z), __dmul_rn(tz, e1y));
    const double qy = __dsub_rn(__dmul_rn(tz, e1x), __dmul_rn(tx, e1z));
    const double qz = __dsub_rn(__dmul_rn(tx, e1y), __dmul_rn(ty, e1x));
    const double vn = __dadd_rn(__dadd_rn(__dmul_rn(dx, qx), __dmul_rn(dy, qy)), __dmul_rn(dz, qz));
    const double tn = __dadd_rn(__dadd_rn(__dmul_rn(e2x, qx), __dmul_rn(e2y, qy)), __dmul_rn(e2z, qz));
    // Division-free rejection of clear misses.  u = fl(un * fl(1/det)) is
    // un/det to within 2.3e-16 relative, so comparing un*sign(det) against
    // the bounds scaled by |det| with a 1e-9 relative margin only rejects
    // segments the exact tests below reject too.  (t < 0 needs |t/det| >
    // 1e-300 so that t cannot round to -0.0, which the reference accepts.)
    {
        const double ad = fabs(det);
        const double su = det < 0.0 ? -un : un, sv = det < 0.0 ? -vn : vn, st = det < 0.0 ? -tn : tn;
        const double m = ad * (1.0 + 1e-9);
        if (su < -kBaryEps * m || su > (1.0 + kBaryEps) * m || sv < -kBaryEps * m ||
            st < -1e-300 * ad || st > m)
            return false;
    }
    const double inv_det = __ddiv_rn(1.0, det);
    const double u = __dmul_rn(un, inv_det);
    if (u < -kBaryEps || u > 1.0 + kBaryEps) return false;
    const double v = __dmul_rn(vn, inv_det);
    if (v < -kBaryEps || __dadd_rn(u, v) > 1.0 + kBaryEps) return false;
    const double t = __dmul_rn(tn, inv_det);
    if (t < 0.0 || t > 1.0) return false;
    *t_out = t;
    return true;
}

__device__ __forceinline__ bool mt_hit(float ax_, float ay_, float az_, float bx, float by,
                                       float bz, float cx, float cy, float cz, double sx,
                                       double sy, double sz, double dx, double dy, double dz,
                                       double* t_out) {
    const double ax = ax_, ay = ay_, az = az_;
    const double e1x = __dsub_rn((double)bx, ax), e1y = __dsub_rn((double)by, ay),
                 e1z = __dsub_rn((double)bz, az);
    const double e2x = __dsub_rn((double)cx, ax), e2y = __dsub_rn((double)cy, ay),
                 e2z = __dsub_rn((double)cz, az);
    return mt_hit_pre(ax, ay, az, e1x, e1y, e1z, e2x, e2y, e2z, sx, sy, sz, dx, dy, dz, t_out);
}

// _core.pyx:330-348: point = s + t*d (f64), distance = f32(sqrt(|p - s|^2)).
__device__ __forceinline__ void hit_point(double sx, double sy, double sz, double dx, double dy,
                                          double dz, double t, float* px_, float* py_,
                                          float* pz_, float* dist) {
    const double px = __dadd_rn(sx, __dmul_rn(t, dx));
    const double py = __dadd_rn(sy, __dmul_rn(t, dy));
    const double pz = __dadd_rn(sz, __dmul_rn(t, dz));
    const double ddx = __dsub_rn(px, sx), ddy = __dsub_rn(py, sy), ddz = __dsub_rn(pz, sz);
    const double s2 =
        __dadd_rn(__dadd_rn(__dmul_rn(ddx, ddx), __dmul_rn(ddy, ddy)), __dmul_rn(ddz, ddz));
    *dist = __double2float_rn(__dsqrt_rn(s2));
    *px_ = __double2float_rn(px);
    *py_ = __double2float_rn(py);
    *pz_ = __double2float_rn(pz);
}

// ---- warp-parallel decoupled look-back --------------------------------------
// status[t] = flag << 62 | value; flag 1 = tile aggregate, 2 = inclusive
// prefix.  Called by all 32 lanes of one warp for tile `tile` with its
// aggregate; returns the exclusive prefix (same value in every lane).  Each
// round reads the 32 preceding tiles at once, so a walk over k still-running
// predecessors costs k/32 L2 round trips instead of k.
__device__ __forceinline__ unsigned long long lookback_warp(unsigned long long* status, long long tile,
                                                            unsigned long long agg) {
    const unsigned kAll = 0xffffffffu;
    const int lane = threadIdx.x & 31;
    const unsigned long long kMask = (1ull << 62) - 1;
    volatile unsigned long long* st = status;
    if (tile == 0) {
        if (lane == 0) {
            __threadfence();
            st[0] = (2ull << 62) | agg;
        }
        return 0;
    }
    if (lane == 0) {
        __threadfence();
        st[tile] = (1ull << 62) | agg;
    }
    unsigned long long excl = 0;
    long long j = tile - 1;
    for (;;) {
        const long long k = j - lane;
        const unsigned long long v = k >= 0 ? st[k] : (2ull << 62);
        const unsigned flag = (unsigned)(v >> 62);
        const unsigned incl = __ballot_sync(kAll, flag == 2);
        const int first = incl ? __ffs(incl) - 1 : 32;
        const unsigned upto = first >= 31 ? kAll : ((2u << first) - 1u);
        if (__ballot_sync(kAll, flag == 0) & upto) continue;  // a predecessor is not ready: re-read
        unsigned long long c = (lane <= first && k >= 0) ? (v & kMask) : 0ull;
        for (int o = 16; o; o >>= 1) c += __shfl_xor_sync(kAll, c, o);
        excl += c;
        if (first < 32) break;
        j -= 32;
    }
    __threadfence();
    if (lane == 0) st[tile] = (2ull << 62) | (excl + agg);
    return excl;
}

}  // namespace rs
