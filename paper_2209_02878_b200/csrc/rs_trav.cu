// rs_trav.cu -- the collision-buffer path (option fast_path=1, north_star's
// buffer manager; the default hot path is the tile traversal in
// rs_sorted.cu): 4-lane group traversal of the 4-wide BVH that emits
// (segment, leaf) candidates into a collision buffer, then a SIMD-dense
// exact-test pass over the buffer.  Also the barycentric compaction and the
// sort_rays un-permutation that every path uses.
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
//   k_bary_compact ordered compaction of barycentric rows (per-tile counts,
//                 one-CTA scan, placement), point/distance from the winning t.
//
// Candidates are staged per warp in shared memory and written 32 at a time
// behind one atomicAdd, so the buffer is dense (no gaps).  Capacity: the
// buffer is pre-sized (2 x segments by default); the append counter keeps
// counting past the end, so the host sees the true size and re-launches with
// a buffer that fits (rs_capi.cu).
#include <cuda/atomic>

#include "rs_common.cuh"
#include "rs_internal.h"

#include <cstdlib>

namespace rs {

constexpr int kTravThreads = 128;
constexpr int kTravStack = 96;  // 4-wide depth <= 31 x 3 pending pushes
constexpr int kSmemStack = 12;  // entries kept in shared memory; deeper ones in global
constexpr int kPairStack = 32;  // pair kernel: shared-memory stack entries per segment
constexpr unsigned kFull = 0xffffffffu;

__device__ __forceinline__ void ld_slot8(const RsSlot* p, float f[8]) {
    asm("ld.global.nc.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=f"(f[0]), "=f"(f[1]), "=f"(f[2]), "=f"(f[3]), "=f"(f[4]), "=f"(f[5]),
                   "=f"(f[6]), "=f"(f[7])
                 : "l"(p));
}

// G lanes per segment (G = 2: "pairs", each lane tests 2 of the 4 slots;
// G = 4: "quads", one slot per lane).  A visit is G x (4/G) 256-bit loads
// within one 128-B node line.
template <int G, bool STATS>
__global__ void __launch_bounds__(kTravThreads) k_trav_group(TravArgs a) {
    constexpr int SL = 4 / G;                 // slots per lane
    constexpr int GPW = 32 / G;               // groups per warp
    constexpr int GPC = kTravThreads / G;     // groups per CTA
    constexpr unsigned kGroupBits = G == 2 ? 0x55555555u : 0x11111111u;
    __shared__ int stk[kSmemStack][GPC];
    __shared__ float4 qs[kTravThreads / 32][32][2];  // per-warp queue: box + segment id
    __shared__ int2 cs[kTravThreads / 32][64 + 32 * SL];  // per-warp candidate staging
    const int lane = threadIdx.x & 31;
    const int warp = threadIdx.x >> 5;
    const int h = lane & (G - 1);             // lane within the group
    const int gshift = lane & ~(G - 1);
    const unsigned lt = (1u << lane) - 1u;
    const int n_int = a.n_int;
    const int root = n_int > 0 ? __ldg(&a.hdr->root) : 0;
    int* const my_stk = &stk[0][threadIdx.x / G];
    int* const my_gstk = a.gstack + ((long long)blockIdx.x * GPC + threadIdx.x / G) * kTravStack;
    int2* const my_cs = cs[warp];
    const RsSlot* const slots = &a.nodes4[0].s[h * SL];

    int qhead = 0, qcount = 0;
    bool exhausted = false;
    int cn = 0;
    int ray = -1, node = root, top = 0;
    float b0 = 0.f, b1 = 0.f, b2 = 0.f, b3 = 0.f, b4 = 0.f, b5 = 0.f;
    unsigned long long visits = 0;
    (void)GPW;

    for (;;) {
        const unsigned idle = __ballot_sync(kFull, ray < 0) & kGroupBits;
        if (idle) {
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
            const int take = nidle < avail ? nidle : (avail > 0 ? avail : 0);
            const int rank = __popc(idle & ((1u << gshift) - 1u));
            if (ray < 0 && rank < take) {
                const float4 u = qs[warp][qhead + rank][0];
                const float4 v = qs[warp][qhead + rank][1];
                b0 = u.x; b1 = u.y; b2 = u.z; b3 = u.w; b4 = v.x; b5 = v.y;
                ray = __float_as_int(v.z);
                node = root;
                top = 0;
            }
            qhead += take;
            __syncwarp();
        }
        const bool live = ray >= 0;
        // ---- one node visit: SL 256-bit slot loads per lane ----
        unsigned lbits = 0, ibits = 0;
        int refs[SL];
#pragma unroll
        for (int j = 0; j < SL; ++j) {
            float f[8];
            ld_slot8(slots + 4 * node + j, f);
            refs[j] = __float_as_int(f[6]);
            const bool hit = live && refs[j] >= 0 && b0 <= f[1] && b1 >= f[0] && b2 <= f[3] &&
                             b3 >= f[2] && b4 <= f[5] && b5 >= f[4];
            lbits |= (hit && refs[j] >= n_int) ? (1u << j) : 0u;
            ibits |= (hit && refs[j] < n_int) ? (1u << j) : 0u;
        }
        if (STATS && h == 0 && live) ++visits;
        // ---- stage leaf candidates (warp prefix over per-lane counts) ----
        {
            const int c = __popc(lbits);
            unsigned pre = 0, tot = 0;
#pragma unroll
            for (int bit = 0; bit < (SL == 2 ? 2 : 1); ++bit) {
                const unsigned bm = __ballot_sync(kFull, (c >> bit) & 1);
                pre += __popc(bm & lt) << bit;
                tot += __popc(bm) << bit;
            }
            if (c) {
                int at = cn + pre;
#pragma unroll
                for (int j = 0; j < SL; ++j)
                    if (lbits & (1u << j)) my_cs[at++] = make_int2(ray, refs[j] - n_int);
            }
            cn += tot;
        }
        if (cn >= 32) {
            __syncwarp();
            unsigned long long base = 0;
            if (lane == 0) base = atomicAdd(&a.status->cand_count, 32ull);
            base = __shfl_sync(kFull, base, 0);
            const int2 c0 = my_cs[lane];
            const int2 c1 = my_cs[32 + lane];
            const int2 c2 = SL == 2 ? my_cs[64 + lane] : make_int2(0, 0);
            if (base + lane < (unsigned long long)a.cand_cap) a.cand[base + lane] = c0;
            __syncwarp();
            cn -= 32;
            if (lane < cn) my_cs[lane] = c1;
            if (SL == 2 && lane + 32 < cn) my_cs[32 + lane] = c2;
        }
        // ---- next node: the first internal hit (in registers); the other
        //      internal hits are pushed; pop only when nothing was hit ----
        unsigned gm;
        if (G == 2) {
            const unsigned o = __shfl_xor_sync(kFull, ibits, 1);
            gm = h ? (o | (ibits << 2)) : (ibits | (o << 2));
        } else {
            gm = (__ballot_sync(kFull, ibits != 0) >> gshift) & 0xFu;
        }
        const int first = gm ? __ffs(gm) - 1 : 0;
        const int nxt = __shfl_sync(kFull, SL == 2 ? ((first & 1) ? refs[SL - 1] : refs[0]) : refs[0],
                                    gshift + first / SL);
        const unsigned rest = gm & (gm - 1u);
        if (rest) {
#pragma unroll
            for (int j = 0; j < SL; ++j) {
                const int bit = h * SL + j;
                if (rest & (1u << bit)) {
                    const int pos = top + __popc(rest & ((1u << bit) - 1u));
                    if (pos < kSmemStack) my_stk[pos * GPC] = refs[j];
                    else if (pos < kTravStack) my_gstk[pos] = refs[j];
                }
            }
            top += __popc(rest);
        }
        __syncwarp();
        if (live) {
            if (gm) {
                node = nxt;
                if (top > kTravStack) {  // cannot happen for fast trees (height <= 61)
                    if (h == 0) atomicAdd(&a.status->internal, 1ull);
                    ray = -1;
                    top = 0;
                }
            } else if (top == 0) {
                ray = -1;
            } else {
                --top;
                node = top < kSmemStack ? my_stk[top * GPC] : my_gstk[top];
            }
        } else {
            top = 0;
        }
    }
    __syncwarp();
    if (cn > 0) {
        unsigned long long base = 0;
        if (lane == 0) base = atomicAdd(&a.status->cand_count, (unsigned long long)cn);
        base = __shfl_sync(kFull, base, 0);
        for (int k = lane; k < cn; k += 32)
            if (base + k < (unsigned long long)a.cand_cap) a.cand[base + k] = my_cs[k];
    }
    if (STATS) {
        for (int o = 16; o; o >>= 1) visits += __shfl_xor_sync(kFull, visits, o);
        if (lane == 0) atomicAdd(&a.status->visits, visits);
    }
}

// Pairs, written branch-light: two lanes per segment, lane h tests slots 2h
// and 2h+1 of the 4-wide node (two 256-bit loads from one 128-B line).
// Candidate staging, stack pushes and the next-node choice are predicated
// stores / selects rather than branches.
__device__ __forceinline__ bool box_hit(const float f[8], float b0, float b1, float b2, float b3,
                                        float b4, float b5) {
    return (b0 <= f[1]) & (b1 >= f[0]) & (b2 <= f[3]) & (b3 >= f[2]) & (b4 <= f[5]) & (b5 >= f[4]);
}

template <bool STATS>
__global__ void __launch_bounds__(kTravThreads) k_trav_pair(TravArgs a) {
    constexpr int GPC = kTravThreads / 2;
    constexpr unsigned kGroupBits = 0x55555555u;
    __shared__ int stk[kPairStack][GPC];
    __shared__ float4 qs[kTravThreads / 32][32][2];
    __shared__ int2 cs[kTravThreads / 32][128];
    const int lane = threadIdx.x & 31;
    const int warp = threadIdx.x >> 5;
    const int h = lane & 1;
    const int gshift = lane & ~1;
    const unsigned lt = (1u << lane) - 1u;
    const unsigned below_me = (1u << (2 * h)) - 1u;  // group slot bits owned by lane 0 if h==1
    const int n_int = a.n_int;
    const int root = n_int > 0 ? __ldg(&a.hdr->root) : 0;
    const int gid = threadIdx.x >> 1;
    int2* const my_cs = cs[warp];
    const RsSlot* const slots = &a.nodes4[0].s[2 * h];

    int qhead = 0, qcount = 0;
    bool exhausted = false;
    int cn = 0;
    int ray = -1, node = root, top = 0;
    float b0 = 0.f, b1 = 0.f, b2 = 0.f, b3 = 0.f, b4 = 0.f, b5 = 0.f;
    unsigned long long visits = 0;

    for (;;) {
        const unsigned idle = __ballot_sync(kFull, ray < 0) & kGroupBits;
        if (idle) {
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
                        live |= (__float_as_int(f[6]) >= 0) & box_hit(f, bx[0], bx[1], bx[2], bx[3], bx[4], bx[5]);
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
            const int take = nidle < avail ? nidle : (avail > 0 ? avail : 0);
            const int rank = __popc(idle & ((1u << gshift) - 1u));
            if (ray < 0 && rank < take) {
                const float4 u = qs[warp][qhead + rank][0];
                const float4 v = qs[warp][qhead + rank][1];
                b0 = u.x; b1 = u.y; b2 = u.z; b3 = u.w; b4 = v.x; b5 = v.y;
                ray = __float_as_int(v.z);
                node = root;
                top = 0;
            }
            qhead += take;
            __syncwarp();
        }
        const bool live = ray >= 0;
        float fa[8], fb[8];
        ld_slot8(slots + 4 * node, fa);
        ld_slot8(slots + 4 * node + 1, fb);
        const int ra = __float_as_int(fa[6]), rb = __float_as_int(fb[6]);
        const bool ha = live & (ra >= 0) & box_hit(fa, b0, b1, b2, b3, b4, b5);
        const bool hb = live & (rb >= 0) & box_hit(fb, b0, b1, b2, b3, b4, b5);
        const bool la = ha & (ra >= n_int), lb = hb & (rb >= n_int);
        const bool ia = ha & (ra < n_int), ib = hb & (rb < n_int);
        if (STATS) visits += (h == 0) & live;
        // ---- candidates: predicated staging stores ----
        const unsigned ba = __ballot_sync(kFull, la), bb = __ballot_sync(kFull, lb);
        const int pa = cn + __popc(ba & lt) + __popc(bb & lt);
        if (la) my_cs[pa] = make_int2(ray, ra - n_int);
        if (lb) my_cs[pa + la] = make_int2(ray, rb - n_int);
        cn += __popc(ba) + __popc(bb);
        if (cn >= 32) {
            __syncwarp();
            unsigned long long base = 0;
            if (lane == 0) base = atomicAdd(&a.status->cand_count, 32ull);
            base = __shfl_sync(kFull, base, 0);
            const int2 c0 = my_cs[lane];
            const int2 c1 = my_cs[32 + lane];
            const int2 c2 = my_cs[64 + lane];
            if (base + lane < (unsigned long long)a.cand_cap) a.cand[base + lane] = c0;
            __syncwarp();
            cn -= 32;
            if (lane < cn) my_cs[lane] = c1;
            if (lane + 32 < cn) my_cs[32 + lane] = c2;
        }
        // ---- next node: first internal hit; push the others; else pop ----
        const unsigned mine = (unsigned)ia | ((unsigned)ib << 1);
        const unsigned other = __shfl_xor_sync(kFull, mine, 1);
        const unsigned gm = h ? (other | (mine << 2)) : (mine | (other << 2));
        const int first = __ffs(gm) - 1;  // -1 when gm == 0
        const int nxt = __shfl_sync(kFull, (first & 1) ? rb : ra, gshift + ((first >> 1) & 1));
        const unsigned rest = gm & (gm - 1u);
        const bool pa_ = (rest >> (2 * h)) & 1u, pb_ = (rest >> (2 * h + 1)) & 1u;
        const int qa = top + __popc(rest & below_me);
        const int qb = qa + pa_;
        if (pa_ & (qa < kPairStack)) stk[qa][gid] = ra;
        if (pb_ & (qb < kPairStack)) stk[qb][gid] = rb;
        top += __popc(rest);
        __syncwarp();
        const bool empty = gm == 0u;
        const int popped = stk[top > 0 ? top - 1 : 0][gid];
        const bool pop = live & empty & (top > 0);
        node = empty ? popped : nxt;
        top -= pop;
        // a deeper stack than kPairStack: flag it; the host re-runs the
        // query with the binary kernels (never seen on real trees)
        const bool ovf = live & (top > kPairStack);
        if (ovf & (h == 0)) atomicAdd(&a.status->internal, 1ull);
        const bool done = !live | (empty & !pop) | ovf;
        ray = done ? -1 : ray;
        top = done ? 0 : top;
        node = done ? root : node;  // idle groups keep loading a valid node
    }
    __syncwarp();
    if (cn > 0) {
        unsigned long long base = 0;
        if (lane == 0) base = atomicAdd(&a.status->cand_count, (unsigned long long)cn);
        base = __shfl_sync(kFull, base, 0);
        for (int k = lane; k < cn; k += 32)
            if (base + k < (unsigned long long)a.cand_cap) a.cand[base + k] = my_cs[k];
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
    // overflow detection: the append counter ran past the buffer, so some
    // candidates were dropped; the host re-launches with a buffer of the
    // claimed size (rs_capi.cu fast_query / host pipeline / graph fallback)
    if (blockIdx.x == 0 && threadIdx.x == 0 && *a.cand_count > (unsigned long long)a.cand_cap) *a.dropped = 1;
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

// Ordered barycentric compaction over segments (engine.py:206-215): each CTA
// owns a tile of kCompactItems x 256 segments, block-scans the hit flags,
// takes its tile's offset from the scanned per-tile counts, and writes its
// rows at their final ascending positions with point/distance computed from
// the winning t in reference op order (_core.pyx:330-348).
constexpr int kCompactThreads = 256;

// The winning hit's t: stored by the traversal (best_t), or recomputed from
// the winning triangle's leaf record with the same f64 test (identical
// operands and op order as the traversal's mt_hit_pre, so the same t).
__device__ __forceinline__ double win_t(const CompactArgs& a, long long i, int tri, double sx,
                                        double sy, double sz, double dx, double dy, double dz) {
    if (a.best_t) {
        const unsigned long long key = a.best_t[i];
        return key == 0ull ? 0.0 : __longlong_as_double((long long)key);
    }
    const RsLeaf* L = a.leaves + __ldg(a.leaf_of + tri);
    const float4 p0 = __ldg(&L->p0), p1 = __ldg(&L->p1), p2 = __ldg(&L->p2);
    double t = 0.0;
    mt_hit(p0.x, p0.y, p0.z, p0.w, p1.x, p1.y, p1.z, p1.w, p2.x, sx, sy, sz, dx, dy, dz, &t);
    return t;
}

__global__ void __launch_bounds__(256) k_leaf_inverse(const RsLeaf* __restrict__ leaves, int n,
                                                      int* __restrict__ leaf_of) {
    for (int k = blockIdx.x * 256 + threadIdx.x; k < n; k += gridDim.x * 256)
        leaf_of[__float_as_int(__ldg(&leaves[k].p2.y))] = k;
}

void launch_leaf_inverse(const RsLeaf* leaves, int n, int* leaf_of, cudaStream_t s) {
    if (n <= 0) return;
    count_launches(1);
    const int g = (n + 255) / 256;
    k_leaf_inverse<<<g < 2048 ? g : 2048, 256, 0, s>>>(leaves, n, leaf_of);
}
constexpr int kCompactItems = 16;
constexpr int kCompactTile = kCompactThreads * kCompactItems;

// ROWS: the compaction also forms each row's distance and point (t stored
// by the traversal); without ROWS it writes only ray index and triangle,
// and k_bary_rows recomputes t and the geometry one row per thread (at 110
// registers the fused recompute left the compaction at 24% occupancy).
// The tiles' offsets come from k_bary_tile_counts + k_bary_tile_scan (a
// decoupled look-back chain across the tiles held every CTA at its barrier:
// C3 50 -> 33 us for the three kernels).
template <bool ROWS>
__global__ void __launch_bounds__(kCompactThreads) k_bary_compact(CompactArgs a) {
    // Striped tile: in round k, thread t owns segment base + k*256 + t, so
    // every load and every output row of a round is coalesced across the
    // warp.  A segment's rank = hits in earlier rounds of the tile + hits of
    // lower threads in its round (ballots + a warp-sum scan per round).
    __shared__ unsigned s_round[kCompactItems][kCompactThreads / 32];
    __shared__ unsigned long long s_prefix;
    const long long tile = blockIdx.x;
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    const unsigned lt = (1u << l) - 1u;
    const long long base = tile * kCompactTile;
    int tri[kCompactItems];
    unsigned inwarp[kCompactItems];
#pragma unroll
    for (int k = 0; k < kCompactItems; ++k) {
        const long long i = base + k * kCompactThreads + threadIdx.x;
        tri[k] = i < a.n_r ? a.best_tri[i] : -1;
        const unsigned m = __ballot_sync(kFull, tri[k] >= 0);
        inwarp[k] = __popc(m & lt);
        if (l == 0) s_round[k][w] = __popc(m);
    }
    __syncthreads();
    // warp 0: exclusive offsets of every (round, warp) cell in tile order
    if (w == 0) {
        constexpr int kCells = kCompactItems * (kCompactThreads / 32);  // 128
        unsigned v[kCells / 32], run = 0;
#pragma unroll
        for (int j = 0; j < kCells / 32; ++j) {
            v[j] = (&s_round[0][0])[l * (kCells / 32) + j];
            run += v[j];
        }
        unsigned x = run;
        for (int o = 1; o < 32; o <<= 1) {
            const unsigned y = __shfl_up_sync(kFull, x, o);
            if (l >= o) x += y;
        }
        const unsigned agg = __shfl_sync(kFull, x, 31);
        unsigned off = x - run;
#pragma unroll
        for (int j = 0; j < kCells / 32; ++j) {
            const unsigned c = v[j];
            (&s_round[0][0])[l * (kCells / 32) + j] = off;
            off += c;
        }
        (void)agg;
        if (l == 0) s_prefix = a.tile_status[tile];  // exclusive prefix; k_bary_tile_scan wrote n_hits
    }
    __syncthreads();
    const unsigned long long tb = s_prefix + (a.row_base ? *a.row_base : 0ull);
#pragma unroll
    for (int k = 0; k < kCompactItems; ++k) {
        if (tri[k] < 0) continue;
        const long long i = base + k * kCompactThreads + threadIdx.x;
        const unsigned long long pos = tb + s_round[k][w] + inwarp[k];
        a.ray[pos] = (int)(i + a.ray_offset);
        a.tri[pos] = tri[k];
        if (!ROWS) continue;
        const float* s = a.starts + 3 * i;
        const float* e = a.ends + 3 * i;
        const double sx = s[0], sy = s[1], sz = s[2];
        const double dx = __dsub_rn((double)e[0], sx), dy = __dsub_rn((double)e[1], sy),
                     dz = __dsub_rn((double)e[2], sz);
        const double t = win_t(a, i, tri[k], sx, sy, sz, dx, dy, dz);
        float px, py, pz, d;
        hit_point(sx, sy, sz, dx, dy, dz, t, &px, &py, &pz, &d);
        a.dist[pos] = d;
        a.point[3 * pos] = px;
        a.point[3 * pos + 1] = py;
        a.point[3 * pos + 2] = pz;
    }
}

// Hits per compaction tile (the reduce pass of the scanned compaction).
__global__ void __launch_bounds__(kCompactThreads) k_bary_tile_counts(const int* __restrict__ best_tri,
                                                                      long long n_r, unsigned* counts) {
    __shared__ unsigned s_w[kCompactThreads / 32];
    const long long base = (long long)blockIdx.x * kCompactTile;
    unsigned c = 0;
#pragma unroll
    for (int k = 0; k < kCompactItems; ++k) {
        const long long i = base + k * kCompactThreads + threadIdx.x;
        c += (i < n_r && __ldg(best_tri + i) >= 0) ? 1u : 0u;
    }
    for (int o = 16; o; o >>= 1) c += __shfl_xor_sync(kFull, c, o);
    if ((threadIdx.x & 31) == 0) s_w[threadIdx.x >> 5] = c;
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned t = 0;
        for (int j = 0; j < kCompactThreads / 32; ++j) t += s_w[j];
        counts[blockIdx.x] = t;
    }
}

// Exclusive scan of the tile counts (one CTA): prefix[tile], and the total
// into *n_hits.
__global__ void __launch_bounds__(1024) k_bary_tile_scan(const unsigned* __restrict__ counts, long long tiles,
                                                         unsigned long long* prefix, unsigned long long* n_hits) {
    __shared__ unsigned long long s_w[32];
    const long long per = (tiles + 1023) / 1024;
    const long long lo = threadIdx.x * per, hi = lo + per < tiles ? lo + per : tiles;
    unsigned long long sum = 0;
    for (long long j = lo; j < hi; ++j) sum += counts[j];
    const int l = threadIdx.x & 31, w = threadIdx.x >> 5;
    unsigned long long x = sum;  // inclusive scan within the warp
    for (int o = 1; o < 32; o <<= 1) {
        const unsigned long long y = __shfl_up_sync(kFull, x, o);
        if (l >= o) x += y;
    }
    if (l == 31) s_w[w] = x;
    __syncthreads();
    if (w == 0) {
        const unsigned long long v = s_w[l];
        unsigned long long z = v;
        for (int o = 1; o < 32; o <<= 1) {
            const unsigned long long y = __shfl_up_sync(kFull, z, o);
            if (l >= o) z += y;
        }
        s_w[l] = z - v;  // exclusive over warps
        if (l == 31) *n_hits = z;
    }
    __syncthreads();
    unsigned long long run = s_w[w] + x - sum;
    for (long long j = lo; j < hi; ++j) {
        prefix[j] = run;
        run += counts[j];
    }
}

// The rows of one compaction (k_bary_compact<false>): t recomputed from the
// winning leaf, then distance and point, one row per thread.
__global__ void __launch_bounds__(256) k_bary_rows(CompactArgs a) {
    const unsigned long long base = a.row_base ? *a.row_base : 0ull;
    const unsigned long long hits = *a.n_hits;
    for (unsigned long long r = blockIdx.x * 256ull + threadIdx.x; r < hits; r += gridDim.x * 256ull) {
        const unsigned long long pos = base + r;
        const long long i = (long long)a.ray[pos] - a.ray_offset;
        const float* s = a.starts + 3 * i;
        const float* e = a.ends + 3 * i;
        const double sx = s[0], sy = s[1], sz = s[2];
        const double dx = __dsub_rn((double)e[0], sx), dy = __dsub_rn((double)e[1], sy),
                     dz = __dsub_rn((double)e[2], sz);
        const double t = win_t(a, i, a.tri[pos], sx, sy, sz, dx, dy, dz);
        float px, py, pz, d;
        hit_point(sx, sy, sz, dx, dy, dz, t, &px, &py, &pz, &d);
        a.dist[pos] = d;
        a.point[3 * pos] = px;
        a.point[3 * pos + 1] = py;
        a.point[3 * pos + 2] = pz;
    }
}

__global__ void __launch_bounds__(256) k_bary_dense(CompactArgs a, int* detected, int* tri_out,
                                                    float* dist, float* points) {
    const long long i = blockIdx.x * 256ll + threadIdx.x;
    if (i >= a.n_r) return;
    const int tri = a.best_tri[i];
    float px = 0.f, py = 0.f, pz = 0.f, d = 0.f;
    if (tri >= 0) {
        const float* s = a.starts + 3 * i;
        const float* e = a.ends + 3 * i;
        const double sx = s[0], sy = s[1], sz = s[2];
        const double dx = __dsub_rn((double)e[0], sx), dy = __dsub_rn((double)e[1], sy),
                     dz = __dsub_rn((double)e[2], sz);
        const double t = win_t(a, i, tri, sx, sy, sz, dx, dy, dz);
        hit_point(sx, sy, sz, dx, dy, dz, t, &px, &py, &pz, &d);
    }
    detected[i] = tri >= 0;
    tri_out[i] = tri;
    dist[i] = d;
    points[3 * i] = px;
    points[3 * i + 1] = py;
    points[3 * i + 2] = pz;
}

// ------------------------------------------------------------ host glue ---

static int sm_count() { return device_sms(); }

// persistent grid: at most 16 CTAs per SM of kTravThreads, <= kTravThreads/2 groups each
size_t trav_gstack_ints() { return (size_t)sm_count() * 16 * (kTravThreads / 2) * kTravStack; }

void launch_trav(const TravArgs& a, bool stats, cudaStream_t s) {
    if (a.n_r <= 0) return;
    count_launches(1);
    static const int lanes = [] {
        const char* e = getenv("RS_TRAV_LANES");
        return e && e[0] == '4' ? 4 : 2;
    }();
    auto k = lanes == 4 ? (stats ? k_trav_group<4, true> : k_trav_group<4, false>)
                        : (stats ? k_trav_pair<true> : k_trav_pair<false>);
    const int o = occupancy((const void*)k, kTravThreads);
    const long long want = (a.n_r + kTravThreads / lanes - 1) / (kTravThreads / lanes);
    const long long pg = (long long)sm_count() * (o > 0 ? (o < 16 ? o : 16) : 1);
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

// ---- sort_rays un-permutation on device (engine.py:191-198) ----------------
//
// Rows computed for Morton-sorted segments carry sorted slots; the caller
// wants original indices, ascending.  boolean/count: out[perm[k]] = in[k].
// barycentric: inv[perm[ray[r]]] = r over a dense n-array (-1 elsewhere), then
// an ordered compaction of inv gathers the rows in ascending original index.
__global__ void __launch_bounds__(256) k_unpermute_dense(const long long* __restrict__ perm, long long n,
                                                         const int* __restrict__ in, int* __restrict__ out) {
    for (long long k = blockIdx.x * 256ll + threadIdx.x; k < n; k += gridDim.x * 256ll) out[perm[k]] = in[k];
}

__global__ void __launch_bounds__(256) k_rows_inverse(const long long* __restrict__ perm,
                                                      const int* __restrict__ ray, long long k_rows,
                                                      int* __restrict__ inv) {
    for (long long r = blockIdx.x * 256ll + threadIdx.x; r < k_rows; r += gridDim.x * 256ll)
        inv[perm[ray[r]]] = (int)r;
}

struct GatherArgs {
    const int* inv;
    long long n;
    const float* dist;
    const int* tri;
    const float* pt;
    int* o_ray;
    float* o_dist;
    int* o_tri;
    float* o_pt;
    unsigned long long* tile_status;
    unsigned long long* tile_counter;
};

// Ordered compaction of inv >= 0 (striped tiles and decoupled look-back, as
// k_bary_compact), gathering row inv[i] to position rank(i).
__global__ void __launch_bounds__(kCompactThreads) k_gather_compact(GatherArgs a) {
    __shared__ unsigned s_round[kCompactItems][kCompactThreads / 32];
    __shared__ unsigned long long s_prefix;
    __shared__ int s_tile;
    if (threadIdx.x == 0) s_tile = (int)atomicAdd(a.tile_counter, 1ull);
    __syncthreads();
    const long long tile = s_tile;
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    const unsigned lt = (1u << l) - 1u;
    const long long base = tile * kCompactTile;
    int src[kCompactItems];
    unsigned inwarp[kCompactItems];
#pragma unroll
    for (int k = 0; k < kCompactItems; ++k) {
        const long long i = base + k * kCompactThreads + threadIdx.x;
        src[k] = i < a.n ? a.inv[i] : -1;
        const unsigned m = __ballot_sync(kFull, src[k] >= 0);
        inwarp[k] = __popc(m & lt);
        if (l == 0) s_round[k][w] = __popc(m);
    }
    __syncthreads();
    if (w == 0) {
        constexpr int kCells = kCompactItems * (kCompactThreads / 32);
        unsigned v[kCells / 32], run = 0;
#pragma unroll
        for (int j = 0; j < kCells / 32; ++j) {
            v[j] = (&s_round[0][0])[l * (kCells / 32) + j];
            run += v[j];
        }
        unsigned x = run;
        for (int o = 1; o < 32; o <<= 1) {
            const unsigned y = __shfl_up_sync(kFull, x, o);
            if (l >= o) x += y;
        }
        const unsigned agg = __shfl_sync(kFull, x, 31);
        unsigned off = x - run;
#pragma unroll
        for (int j = 0; j < kCells / 32; ++j) {
            const unsigned c = v[j];
            (&s_round[0][0])[l * (kCells / 32) + j] = off;
            off += c;
        }
        const unsigned long long excl = lookback_warp(a.tile_status, tile, agg);
        if (l == 0) s_prefix = excl;
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < kCompactItems; ++k) {
        if (src[k] < 0) continue;
        const long long i = base + k * kCompactThreads + threadIdx.x;
        const unsigned long long pos = s_prefix + s_round[k][w] + inwarp[k];
        const long long r = src[k];
        a.o_ray[pos] = (int)i;
        a.o_dist[pos] = a.dist[r];
        a.o_tri[pos] = a.tri[r];
        a.o_pt[3 * pos] = a.pt[3 * r];
        a.o_pt[3 * pos + 1] = a.pt[3 * r + 1];
        a.o_pt[3 * pos + 2] = a.pt[3 * r + 2];
    }
}

size_t unpermute_scratch_bytes(long long n) {
    // inv (n ints), tile status words, tile counter
    return ((4ull * n + 255) & ~255ull) + (size_t)((n + kCompactTile - 1) / kCompactTile) * 8 + 16;
}

void launch_unpermute_dense(const long long* perm, long long n, const int* in, int* out, cudaStream_t s) {
    if (n <= 0) return;
    count_launches(1);
    const long long g = (n + 255) / 256;
    k_unpermute_dense<<<(unsigned)(g < 4096 ? g : 4096), 256, 0, s>>>(perm, n, in, out);
}

void launch_unpermute_rows(const long long* perm, long long n, const int* ray, const float* dist,
                           const int* tri, const float* pt, long long k_rows, int* o_ray, float* o_dist,
                           int* o_tri, float* o_pt, void* scratch, cudaStream_t s) {
    if (n <= 0) return;
    int* inv = static_cast<int*>(scratch);
    unsigned long long* st = reinterpret_cast<unsigned long long*>(
        static_cast<char*>(scratch) + ((4ull * n + 255) & ~255ull));
    const long long tiles = (n + kCompactTile - 1) / kCompactTile;
    cudaMemsetAsync(inv, 0xFF, 4ull * n, s);
    cudaMemsetAsync(st, 0, (size_t)tiles * 8 + 16, s);
    count_launches(2);
    if (k_rows > 0) {
        const long long g = (k_rows + 255) / 256;
        k_rows_inverse<<<(unsigned)(g < 4096 ? g : 4096), 256, 0, s>>>(perm, ray, k_rows, inv);
    }
    GatherArgs a{inv, n, dist, tri, pt, o_ray, o_dist, o_tri, o_pt, st, st + tiles};
    k_gather_compact<<<(unsigned)tiles, kCompactThreads, 0, s>>>(a);
}

// [tile words (look-back status, or the scanned prefixes) x tiles]
// [tile counts, u32 x tiles, padded to 8 B][ticket counter]
size_t bary_compact_scratch(long long n_r) {
    const size_t tiles = (size_t)((n_r + kCompactTile - 1) / kCompactTile);
    return tiles * 8 + ((tiles * 4 + 7) & ~size_t(7)) + 8;
}


__global__ void k_advance_rows(unsigned long long* row_base, const unsigned long long* n_hits) {
    *row_base += *n_hits;
}

void launch_bary_compact(const CompactArgs& a, cudaStream_t s) {
    if (a.n_r <= 0) return;
    const unsigned tiles = (unsigned)((a.n_r + kCompactTile - 1) / kCompactTile);
    const bool rows = a.best_t || a.fused;
    unsigned* counts = reinterpret_cast<unsigned*>(a.tile_status + tiles);
    count_launches(3);
    k_bary_tile_counts<<<tiles, kCompactThreads, 0, s>>>(a.best_tri, a.n_r, counts);
    k_bary_tile_scan<<<1, 1024, 0, s>>>(counts, (long long)tiles, a.tile_status, a.n_hits);
    if (rows) {
        k_bary_compact<true><<<tiles, kCompactThreads, 0, s>>>(a);
    } else {
        k_bary_compact<false><<<tiles, kCompactThreads, 0, s>>>(a);
        const long long want = (a.n_r + 255) / 256, cap = (long long)device_sms() * 16;
        count_launches(1);
        k_bary_rows<<<(unsigned)(want < cap ? want : cap), 256, 0, s>>>(a);
    }
    if (a.row_base) {
        count_launches(1);
        k_advance_rows<<<1, 1, 0, s>>>(a.row_base, a.n_hits);
    }
}

void launch_bary_dense(const CompactArgs& a, int* detected, int* tri, float* dist, float* points,
                       cudaStream_t s) {
    if (a.n_r <= 0) return;
    count_launches(1);
    k_bary_dense<<<(unsigned)((a.n_r + 255) / 256), 256, 0, s>>>(a, detected, tri, dist, points);
}

}  // namespace rs
