// rs_trav.cu -- the fast-tree hot path: 4-lane group traversal of the 4-wide
// BVH that emits (segment, leaf) candidates into a collision buffer, then a
// SIMD-dense exact-test pass over the buffer.
//
//   k_trav_quad   one segment per 4-lane group, one child slot per lane: a
//                 node visit is one 256-bit load per lane (the group reads one
//                 128-B line).  Leaf children whose exact f32 AABB overlaps the
//                 segment AABB are appended to the collision buffer (staged
//                 per warp in shared memory, flushed 32 per atomic);
//                 internal hits are pushed in parallel onto the group's
//                 shared-memory stack.  Segments are fed through a per-warp
//                 queue of 32 prefetched ids/boxes (one atomic per 32).
//   k_exact       one candidate per thread: f64 Moller-Trumbore in reference
//                 op order, then boolean store / count atomicAdd /
//                 barycentric atomicMin on the t key.
//   k_tiebreak    barycentric: among hits with t == min t, atomicMin of the
//                 triangle id (_core.pyx:317-320 (t, tid) order).
//   k_bary_compact ordered compaction of barycentric rows (decoupled
//                 look-back), point/distance computed from the winning t.
//
// Candidates are staged per warp in shared memory and written 32 at a time
// behind one atomicAdd, so the buffer is dense (no gaps).  Capacity: the
// buffer is pre-sized (2 x segments by default); the append counter keeps
// counting past the end, so the host sees the true size and re-launches with
// a buffer that fits (rs_capi.cu).
#include <cuda/atomic>

#include "rs_common.cuh"
#include "rs_internal.h"

namespace rs {

constexpr int kTravThreads = 128;
constexpr int kTravGroups = kTravThreads / 4;
constexpr int kTravStack = 96;  // 4-wide depth <= 31 x 3 pending pushes
constexpr unsigned kFull = 0xffffffffu;

__device__ __forceinline__ void ld_slot8(const RsSlot* p, float f[8]) {
    asm("ld.global.nc.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=f"(f[0]), "=f"(f[1]), "=f"(f[2]), "=f"(f[3]), "=f"(f[4]), "=f"(f[5]),
                   "=f"(f[6]), "=f"(f[7])
                 : "l"(p));
}

template <bool STATS>
__global__ void __launch_bounds__(kTravThreads) k_trav_quad(TravArgs a) {
    __shared__ int stk[kTravStack + 4][kTravGroups];
    __shared__ float4 qs[kTravThreads / 32][32][2];  // per-warp queue: box + segment id
    __shared__ int2 cs[kTravThreads / 32][64];       // per-warp candidate staging
    const int lane = threadIdx.x & 31;
    const int warp = threadIdx.x >> 5;
    const int q = lane & 3;
    const int gshift = lane & ~3;
    const unsigned lt = (1u << lane) - 1u;
    const unsigned lt_in_group = (1u << q) - 1u;
    const unsigned kGroupBits = 0x11111111u;
    const int n_int = a.n_int;
    const int root = n_int > 0 ? __ldg(&a.hdr->root) : 0;
    int* const my_stk = &stk[0][threadIdx.x >> 2];  // this group's column, stride kTravGroups
    int2* const my_cs = cs[warp];
    const RsSlot* const slots = &a.nodes4[0].s[q];  // + 4 * node

    int qhead = 0, qcount = 0;  // live segments queued in qs[warp][qhead, qcount)
    bool exhausted = false;
    int cn = 0;                 // staged candidates (warp-uniform)
    // per-group traversal state (replicated in the group's 4 lanes)
    int ray = -1, node = root, top = 0;
    float b0 = INFINITY, b1 = -INFINITY, b2 = INFINITY, b3 = -INFINITY, b4 = INFINITY,
          b5 = -INFINITY;  // empty box: overlaps nothing
    unsigned long long visits = 0;

    for (;;) {
        const unsigned idle = __ballot_sync(kFull, ray < 0) & kGroupBits;
        if (idle) {
            // refill: claim 32 segments, cull those that miss every child of
            // the root (their result is the pre-zeroed default), queue the rest
            while (qhead == qcount && !exhausted) {
                unsigned long long base = 0;
                if (lane == 0) base = atomicAdd(&a.status->tile_counter, 32ull);
                base = __shfl_sync(kFull, base, 0);
                exhausted = (long long)base + 32 >= a.n_r;
                const long long rid = (long long)base + lane;
                bool live = false;
                float bx[6];
                if (rid < a.n_r) {
                    const float* sp = a.starts + 3 * rid;
                    const float* ep = a.ends + 3 * rid;
                    const float s0 = __ldg(sp), s1 = __ldg(sp + 1), s2 = __ldg(sp + 2);
                    const float e0 = __ldg(ep), e1 = __ldg(ep + 1), e2 = __ldg(ep + 2);
                    bx[0] = fminf(s0, e0); bx[1] = fmaxf(s0, e0);  // engine.py:115-122
                    bx[2] = fminf(s1, e1); bx[3] = fmaxf(s1, e1);
                    bx[4] = fminf(s2, e2); bx[5] = fmaxf(s2, e2);
#pragma unroll
                    for (int j = 0; j < 4; ++j) {
                        float f[8];
                        ld_slot8(&a.nodes4[root].s[j], f);
                        live |= __float_as_int(f[6]) >= 0 && bx[0] <= f[1] && bx[1] >= f[0] &&
                                bx[2] <= f[3] && bx[3] >= f[2] && bx[4] <= f[5] && bx[5] >= f[4];
                    }
                }
                const unsigned lm = __ballot_sync(kFull, live);
                if (live) {
                    const int at = __popc(lm & lt);
                    qs[warp][at][0] = make_float4(bx[0], bx[1], bx[2], bx[3]);
                    qs[warp][at][1] = make_float4(bx[4], bx[5], __int_as_float((int)rid), 0.f);
                }
                qhead = 0;
                qcount = __popc(lm);
                __syncwarp();
            }
            const int avail = qcount - qhead;
            if (avail <= 0 && exhausted && idle == kGroupBits) break;
            const int nidle = __popc(idle);
            const int take = nidle < avail ? nidle : avail;
            const int rank = __popc(idle & ((1u << gshift) - 1u));
            if (ray < 0 && rank < take) {
                const float4 u = qs[warp][qhead + rank][0];
                const float4 v = qs[warp][qhead + rank][1];
                b0 = u.x; b1 = u.y; b2 = u.z; b3 = u.w; b4 = v.x; b5 = v.y;
                ray = __float_as_int(v.z);
                node = root;
                top = 0;
            }
            qhead += take > 0 ? take : 0;
            __syncwarp();
        }
        // ---- one node visit per group: one 256-bit slot load per lane ----
        // (idle groups keep an empty box and re-read the root slot: no branch)
        float f[8];
        ld_slot8(slots + 4 * node, f);
        const int ref = __float_as_int(f[6]);
        const bool hit = ref >= 0 && b0 <= f[1] && b1 >= f[0] && b2 <= f[3] && b3 >= f[2] &&
                         b4 <= f[5] && b5 >= f[4];
        if (STATS && q == 0 && ray >= 0) ++visits;
        const bool leafhit = hit && ref >= n_int;
        const bool ihit = hit && ref < n_int;
        // ---- stage leaf candidates; flush 32 at a time (one atomic each) ----
        const unsigned lb = __ballot_sync(kFull, leafhit);
        if (leafhit) my_cs[cn + __popc(lb & lt)] = make_int2(ray, ref - n_int);
        cn += __popc(lb);
        if (cn >= 32) {
            __syncwarp();
            unsigned long long base = 0;
            if (lane == 0) base = atomicAdd(&a.status->cand_count, 32ull);
            base = __shfl_sync(kFull, base, 0);
            const int2 c = my_cs[lane];
            const int2 rest = my_cs[32 + lane];
            if (base + lane < (unsigned long long)a.cand_cap) a.cand[base + lane] = c;
            __syncwarp();
            cn -= 32;
            if (lane < cn) my_cs[lane] = rest;
        }
        // ---- push internal hits in parallel, pop the next node ----
        const unsigned gm = (__ballot_sync(kFull, ihit) >> gshift) & 0xFu;
        if (ihit) my_stk[(top + __popc(gm & lt_in_group)) * kTravGroups] = ref;
        top += __popc(gm);
        __syncwarp();
        if (ray >= 0) {
            if (top == 0) {
                ray = -1;
                b0 = b2 = b4 = INFINITY; b1 = b3 = b5 = -INFINITY;
                node = root;
            } else if (top > kTravStack) {  // cannot happen for fast trees (height <= 61)
                if (q == 0) atomicAdd(&a.status->internal, 1ull);
                ray = -1;
                top = 0;
                b0 = b2 = b4 = INFINITY; b1 = b3 = b5 = -INFINITY;
                node = root;
            } else {
                node = my_stk[--top * kTravGroups];
            }
        } else {
            top = 0;
        }
    }
    // flush the staged tail
    __syncwarp();
    if (cn > 0) {
        unsigned long long base = 0;
        if (lane == 0) base = atomicAdd(&a.status->cand_count, (unsigned long long)cn);
        base = __shfl_sync(kFull, base, 0);
        if (lane < cn && base + lane < (unsigned long long)a.cand_cap) a.cand[base + lane] = my_cs[lane];
    }
    if (STATS) {
        for (int o = 16; o; o >>= 1) visits += __shfl_xor_sync(kFull, visits, o);
        if (lane == 0) atomicAdd(&a.status->visits, visits);
    }
}

// t >= 0 for every hit, so the IEEE bits order like the values; -0.0 is
// folded onto +0.0 (they compare equal in the reference's `t < best_t`).
__device__ __forceinline__ unsigned long long t_key(double t) {
    return t == 0.0 ? 0ull : (unsigned long long)__double_as_longlong(t);
}

template <int MODE, bool STATS>
__global__ void __launch_bounds__(256) k_exact(ExactArgs a) {
    const unsigned long long n = *a.cand_count < (unsigned long long)a.cand_cap
                                     ? *a.cand_count : (unsigned long long)a.cand_cap;
    unsigned long long mts = 0;
    for (unsigned long long i = blockIdx.x * 256ull + threadIdx.x; i < n; i += gridDim.x * 256ull) {
        const int2 c = a.cand[i];
        const float* s = a.starts + 3ll * c.x;
        const float* e = a.ends + 3ll * c.x;
        const double sx = __ldg(s), sy = __ldg(s + 1), sz = __ldg(s + 2);
        const double dx = __dsub_rn((double)__ldg(e), sx), dy = __dsub_rn((double)__ldg(e + 1), sy),
                     dz = __dsub_rn((double)__ldg(e + 2), sz);
        const float4 p0 = __ldg(&a.leaves[c.y].p0), p1 = __ldg(&a.leaves[c.y].p1),
                     p2 = __ldg(&a.leaves[c.y].p2);
        double t;
        ++mts;
        const bool hit = mt_hit(p0.x, p0.y, p0.z, p0.w, p1.x, p1.y, p1.z, p1.w, p2.x, sx, sy, sz,
                                dx, dy, dz, &t);
        if (MODE == kBoolean) {
            if (hit) a.flags[c.x] = 1;
        } else if (MODE == kCount) {
            if (hit) atomicAdd(a.flags + c.x, 1);
        } else {
            const unsigned long long k = hit ? t_key(t) : ~0ull;
            a.cand_t[i] = k;
            if (hit) atomicMin(a.best_t + c.x, k);
        }
    }
    if (STATS) {
        for (int o = 16; o; o >>= 1) mts += __shfl_xor_sync(kFull, mts, o);
        if ((threadIdx.x & 31) == 0) atomicAdd(a.mts, mts);
    }
}

__global__ void __launch_bounds__(256) k_tiebreak(ExactArgs a) {
    const unsigned long long n = *a.cand_count < (unsigned long long)a.cand_cap
                                     ? *a.cand_count : (unsigned long long)a.cand_cap;
    for (unsigned long long i = blockIdx.x * 256ull + threadIdx.x; i < n; i += gridDim.x * 256ull) {
        const unsigned long long k = a.cand_t[i];
        if (k == ~0ull) continue;
        const int2 c = a.cand[i];
        if (k == a.best_t[c.x])  // unsigned min: the 0xFFFFFFFF (-1) preset is the largest key
            atomicMin(reinterpret_cast<unsigned*>(a.best_tri) + c.x,
                      (unsigned)__float_as_int(__ldg(&a.leaves[c.y].p2.y)));
    }
}

// Ordered barycentric compaction over segments (engine.py:206-215): block scan
// of hit flags + decoupled look-back across tiles; point/distance from the
// winning t in reference op order (_core.pyx:330-348).
constexpr int kCompactThreads = 256;

__global__ void __launch_bounds__(kCompactThreads) k_bary_compact(CompactArgs a) {
    __shared__ unsigned s_warp[kCompactThreads / 32];
    __shared__ unsigned long long s_prefix;
    __shared__ int s_tile;
    if (threadIdx.x == 0) s_tile = (int)atomicAdd(a.tile_counter, 1ull);
    __syncthreads();
    const int tile = s_tile;
    const long long i = (long long)tile * kCompactThreads + threadIdx.x;
    int tri = -1;
    if (i < a.n_r) tri = a.best_tri[i];
    const bool hit = tri >= 0;
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    const unsigned ball = __ballot_sync(kFull, hit);
    if (l == 0) s_warp[w] = __popc(ball);
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned agg = 0;
        for (int k = 0; k < kCompactThreads / 32; ++k) {
            const unsigned c = s_warp[k];
            s_warp[k] = agg;
            agg += c;
        }
        cuda::atomic_ref<unsigned long long, cuda::thread_scope_device> me(a.tile_status[tile]);
        unsigned long long excl = 0;
        if (tile == 0) {
            me.store((2ull << 62) | agg, cuda::memory_order_release);
        } else {
            me.store((1ull << 62) | agg, cuda::memory_order_release);
            for (int j = tile - 1; j >= 0;) {
                cuda::atomic_ref<unsigned long long, cuda::thread_scope_device> prev(a.tile_status[j]);
                const unsigned long long v = prev.load(cuda::memory_order_acquire);
                const unsigned flag = (unsigned)(v >> 62);
                if (flag == 0) continue;
                excl += v & ((1ull << 62) - 1);
                if (flag == 2) break;
                --j;
            }
            me.store((2ull << 62) | (excl + agg), cuda::memory_order_release);
        }
        s_prefix = excl;
        if ((long long)(tile + 1) * kCompactThreads >= a.n_r) *a.n_hits = excl + agg;
    }
    __syncthreads();
    if (hit) {
        const unsigned long long pos = s_prefix + s_warp[w] + __popc(ball & ((1u << l) - 1u));
        const unsigned long long k = a.best_t[i];
        const double t = k == 0ull ? 0.0 : __longlong_as_double((long long)k);
        const float* s = a.starts + 3 * i;
        const float* e = a.ends + 3 * i;
        const double sx = s[0], sy = s[1], sz = s[2];
        float px, py, pz, d;
        hit_point(sx, sy, sz, __dsub_rn((double)e[0], sx), __dsub_rn((double)e[1], sy),
                  __dsub_rn((double)e[2], sz), t, &px, &py, &pz, &d);
        a.ray[pos] = (int)(i + a.ray_offset);
        a.dist[pos] = d;
        a.tri[pos] = tri;
        a.point[3 * pos] = px;
        a.point[3 * pos + 1] = py;
        a.point[3 * pos + 2] = pz;
    }
}

// Dense barycentric rows from (best_t, best_tri) (plugin protocol path).
__global__ void __launch_bounds__(256) k_bary_dense(CompactArgs a, int* detected, int* tri_out,
                                                    float* dist, float* points) {
    const long long i = blockIdx.x * 256ll + threadIdx.x;
    if (i >= a.n_r) return;
    const int tri = a.best_tri[i];
    float px = 0.f, py = 0.f, pz = 0.f, d = 0.f;
    if (tri >= 0) {
        const unsigned long long k = a.best_t[i];
        const double t = k == 0ull ? 0.0 : __longlong_as_double((long long)k);
        const float* s = a.starts + 3 * i;
        const float* e = a.ends + 3 * i;
        const double sx = s[0], sy = s[1], sz = s[2];
        hit_point(sx, sy, sz, __dsub_rn((double)e[0], sx), __dsub_rn((double)e[1], sy),
                  __dsub_rn((double)e[2], sz), t, &px, &py, &pz, &d);
    }
    detected[i] = tri >= 0;
    tri_out[i] = tri;
    dist[i] = d;
    points[3 * i] = px;
    points[3 * i + 1] = py;
    points[3 * i + 2] = pz;
}

// ------------------------------------------------------------ host glue ---

static int sm_count() {
    static int sms = 0;
    if (!sms) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    }
    return sms;
}

void launch_trav(const TravArgs& a, bool stats, cudaStream_t s) {
    if (a.n_r <= 0) return;
    count_launches(1);
    auto k = stats ? k_trav_quad<true> : k_trav_quad<false>;
    static int occ[2] = {0, 0};
    int& o = occ[stats ? 1 : 0];
    if (!o) cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, k, kTravThreads, 0);
    const long long want = (a.n_r + kTravGroups - 1) / kTravGroups;
    const long long pg = (long long)sm_count() * (o > 0 ? o : 1);
    k<<<(unsigned)(want < pg ? want : pg), kTravThreads, 0, s>>>(a);
}

void launch_exact(const ExactArgs& a, int mode, bool stats, cudaStream_t s) {
    count_launches(mode == kBarycentric ? 2 : 1);
    const unsigned grid = (unsigned)sm_count() * 8;
    if (mode == kBoolean) {
        if (stats) k_exact<kBoolean, true><<<grid, 256, 0, s>>>(a);
        else k_exact<kBoolean, false><<<grid, 256, 0, s>>>(a);
    } else if (mode == kCount) {
        if (stats) k_exact<kCount, true><<<grid, 256, 0, s>>>(a);
        else k_exact<kCount, false><<<grid, 256, 0, s>>>(a);
    } else {
        if (stats) k_exact<kBarycentric, true><<<grid, 256, 0, s>>>(a);
        else k_exact<kBarycentric, false><<<grid, 256, 0, s>>>(a);
        k_tiebreak<<<grid, 256, 0, s>>>(a);
    }
}

size_t bary_compact_scratch(long long n_r) {
    return (size_t)((n_r + kCompactThreads - 1) / kCompactThreads) * 8 + 8;
}

void launch_bary_compact(const CompactArgs& a, cudaStream_t s) {
    if (a.n_r <= 0) return;
    count_launches(1);
    k_bary_compact<<<(unsigned)((a.n_r + kCompactThreads - 1) / kCompactThreads), kCompactThreads,
                     0, s>>>(a);
}

void launch_bary_dense(const CompactArgs& a, int* detected, int* tri, float* dist, float* points,
                       cudaStream_t s) {
    if (a.n_r <= 0) return;
    count_launches(1);
    k_bary_dense<<<(unsigned)((a.n_r + 255) / 256), 256, 0, s>>>(a, detected, tri, dist, points);
}

}  // namespace rs
