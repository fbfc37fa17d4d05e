// rs_sorted.cu -- the fast-tree hot path: coherent per-segment traversal.
//
// Segments arrive in caller order, which for random inputs means neighbouring
// lanes walk unrelated parts of the tree and every node load is a scattered
// 128-B line (L1-wavefront bound).  So the query first reorders the segments
// spatially with a two-pass counting sort, fused with root culling:
//
//   k_bin_count    per segment: f32 AABB (engine.py:115-122), test against the
//                  root's children (a segment overlapping none of them has no
//                  candidates: its result is the pre-zeroed default and it is
//                  dropped here), 21-bit isotropic Morton key of the box centre
//                  over the root box, warp-aggregated histogram atomics.
//   k_tile_scan +  two-level exclusive scan of the 2M bins.
//   k_bin_scan
//   k_bin_scatter  same key; each live segment's record (start, id, end; 32 B)
//                  goes to its bin.
//   k_trav_sorted  one thread per record, in bin order: stack traversal of the
//                  4-wide BVH (four 256-bit slot loads per visit, exact f32
//                  box tests), f64 Moller-Trumbore at the leaves in reference
//                  op order, boolean early exit, result written to the
//                  segment's original row.  Lanes of a warp hold spatially
//                  adjacent segments, so their node loads coalesce.
//
// Results do not depend on the order: boolean = any, count = sum, barycentric
// = min over (t, triangle id) (_core.pyx:304-322).
#include "rs_common.cuh"
#include "rs_internal.h"

#include <cstdint>
#include <cstdlib>

namespace rs {

constexpr unsigned kFullMask = 0xffffffffu;
constexpr int kAxisBits = 7;                 // bins per axis = 128
constexpr int kBinBits = 3 * kAxisBits;
constexpr int kBins = 1 << kBinBits;
constexpr int kScanShift = 10;
constexpr int kScanTile = 1 << kScanShift;
constexpr int kScanTiles = kBins / kScanTile;
constexpr int kSortedThreads = 128;
constexpr int kSortedStack = 64;  // fast tree: <= 3 pending per 4-wide level; deeper -> fallback
#ifndef RS_SORTED_MIN_BLOCKS
#define RS_SORTED_MIN_BLOCKS 8
#endif
constexpr int kSortedMinBlocks = RS_SORTED_MIN_BLOCKS;  // 8 x 128 threads: <= 64 registers

__device__ __forceinline__ void ld_slot(const RsSlot* p, float f[8]) {
    asm("ld.global.nc.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
        : "=f"(f[0]), "=f"(f[1]), "=f"(f[2]), "=f"(f[3]), "=f"(f[4]), "=f"(f[5]), "=f"(f[6]),
          "=f"(f[7])
        : "l"(p));
}

__device__ __forceinline__ bool slot_hit(const float f[8], const float b[6]) {
    return (__float_as_int(f[6]) >= 0) & (b[0] <= f[1]) & (b[1] >= f[0]) & (b[2] <= f[3]) &
           (b[3] >= f[2]) & (b[4] <= f[5]) & (b[5] >= f[4]);
}

__device__ __forceinline__ unsigned spread_bits(unsigned v) {  // bit i -> bit 3i
    unsigned r = 0;
#pragma unroll
    for (int i = 0; i < kAxisBits; ++i) r |= ((v >> i) & 1u) << (3 * i);
    return r;
}

// Root box + culling helper shared by both binning passes.
struct RootInfo {
    float lo[3], hi[3], inv[3];
};

// The root box (union of all triangle boxes) comes from the build's k_prep,
// so the binning can run concurrently with the rest of the build.
__device__ __forceinline__ void root_info(const RsHeader* hdr, RootInfo& ri) {
    float hi[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        ri.lo[k] = from_ord32(~__ldg(&hdr->bmin[k]));
        hi[k] = from_ord32(__ldg(&hdr->bmax[k]));
    }
#pragma unroll
    for (int k = 0; k < 3; ++k) ri.hi[k] = hi[k];
    const float ext = fmaxf(fmaxf(hi[0] - ri.lo[0], hi[1] - ri.lo[1]), fmaxf(hi[2] - ri.lo[2], 1e-30f));
#pragma unroll
    for (int k = 0; k < 3; ++k) ri.inv[k] = ((float)(1 << kAxisBits) - 0.01f) / ext;
}

// Returns the bin of a live segment, or -1 when its box misses the root box
// (no leaf box can overlap it: its result is the pre-zeroed default).
__device__ __forceinline__ int seg_bin(const float s[3], const float e[3], const RootInfo& ri) {
    float b[6];
    b[0] = fminf(s[0], e[0]); b[1] = fmaxf(s[0], e[0]);
    b[2] = fminf(s[1], e[1]); b[3] = fmaxf(s[1], e[1]);
    b[4] = fminf(s[2], e[2]); b[5] = fmaxf(s[2], e[2]);
    const bool live = (b[0] <= ri.hi[0]) & (b[1] >= ri.lo[0]) & (b[2] <= ri.hi[1]) &
                      (b[3] >= ri.lo[1]) & (b[4] <= ri.hi[2]) & (b[5] >= ri.lo[2]);
    if (!live) return -1;
    unsigned key = 0;
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        const float c = 0.5f * (b[2 * k] + b[2 * k + 1]);
        const float q = fminf(fmaxf((c - ri.lo[k]) * ri.inv[k], 0.f), (float)((1 << kAxisBits) - 1));
        key |= spread_bits((unsigned)q) << k;
    }
    return (int)key;
}

// Four consecutive segments per thread: 3 x 16-B loads per endpoint array
// (the (N,3) f32 AoS rows of segments 4t..4t+3 are 48 contiguous bytes).
template <bool VEC>
__device__ __forceinline__ int load4(const float* __restrict__ S, const float* __restrict__ E,
                                     long long q, long long n, float s[4][3], float e[4][3]) {
    const long long i0 = 4 * q;
    const int cnt = n - i0 >= 4 ? 4 : (int)(n - i0);
    if (VEC && cnt == 4) {
        const float4* s4 = reinterpret_cast<const float4*>(S + 3 * i0);
        const float4* e4 = reinterpret_cast<const float4*>(E + 3 * i0);
        float fs[12], fe[12];
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            const float4 a = __ldg(s4 + k), c = __ldg(e4 + k);
            fs[4 * k] = a.x; fs[4 * k + 1] = a.y; fs[4 * k + 2] = a.z; fs[4 * k + 3] = a.w;
            fe[4 * k] = c.x; fe[4 * k + 1] = c.y; fe[4 * k + 2] = c.z; fe[4 * k + 3] = c.w;
        }
#pragma unroll
        for (int j = 0; j < 4; ++j)
#pragma unroll
            for (int k = 0; k < 3; ++k) {
                s[j][k] = fs[3 * j + k];
                e[j][k] = fe[3 * j + k];
            }
    } else {
#pragma unroll
        for (int j = 0; j < 4; ++j)
#pragma unroll
            for (int k = 0; k < 3; ++k) {
                s[j][k] = j < cnt ? __ldg(S + 3 * (i0 + j) + k) : 0.f;
                e[j][k] = j < cnt ? __ldg(E + 3 * (i0 + j) + k) : 0.f;
            }
    }
    return cnt;
}

template <bool VEC>
__global__ void __launch_bounds__(256) k_bin_count(SortedArgs a) {
    RootInfo ri;
    root_info(a.hdr, ri);
    const long long nq = (a.n_r + 3) / 4;
    for (long long q = blockIdx.x * 256ll + threadIdx.x; q < nq; q += gridDim.x * 256ll) {
        float s[4][3], e[4][3];
        const int cnt = load4<VEC>(a.starts, a.ends, q, a.n_r, s, e);
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int bin = j < cnt ? seg_bin(s[j], e[j], ri) : -1;
            const unsigned act = __activemask();
            const unsigned peers = __match_any_sync(act, bin);
            if (bin >= 0 && (__ffs(peers) - 1) == (int)(threadIdx.x & 31))
                atomicAdd(a.bins + bin, __popc(peers));
        }
    }
}

// Exclusive scan of the bin counters in two levels: k_tile_reduce sums each
// 1024-bin tile, k_tile_scan scans the tile sums in one CTA, then k_bin_scan
// scans each tile's bins from its tile offset.

__device__ __forceinline__ unsigned block_excl_scan_256(unsigned v, unsigned* wtot, unsigned* total) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    unsigned x = v;
    for (int o = 1; o < 32; o <<= 1) {
        const unsigned y = __shfl_up_sync(kFullMask, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) wtot[w] = x;
    __syncthreads();
    unsigned before = 0, all = 0;
    for (int k = 0; k < (int)(blockDim.x >> 5); ++k) {
        if (k < w) before += wtot[k];
        all += wtot[k];
    }
    if (total) *total = all;
    return before + x - v;
}

__global__ void __launch_bounds__(256) k_tile_reduce(SortedArgs a) {
    __shared__ unsigned wtot[8];
    const uint4 v = *reinterpret_cast<const uint4*>(a.bins + blockIdx.x * kScanTile + threadIdx.x * 4);
    unsigned total;
    block_excl_scan_256(v.x + v.y + v.z + v.w, wtot, &total);
    if (threadIdx.x == 0) a.tile_sum[blockIdx.x] = total;
}

__global__ void __launch_bounds__(256) k_tile_scan(SortedArgs a) {
    __shared__ unsigned wtot[8];
    constexpr int per = kScanTiles / 256;
    unsigned v[per], sum = 0;
#pragma unroll
    for (int k = 0; k < per; ++k) {
        v[k] = a.tile_sum[threadIdx.x * per + k];
        sum += v[k];
    }
    unsigned total;
    unsigned run = block_excl_scan_256(sum, wtot, &total);
#pragma unroll
    for (int k = 0; k < per; ++k) {
        a.tile_sum[threadIdx.x * per + k] = run;  // becomes the tile offset
        run += v[k];
    }
    if (threadIdx.x == 0) *a.n_live = total;
}

__global__ void __launch_bounds__(256) k_bin_scan(SortedArgs a) {
    __shared__ unsigned wtot[8];
    const int tile = blockIdx.x;
    const int base = tile * kScanTile + threadIdx.x * 4;
    const uint4 v = *reinterpret_cast<const uint4*>(a.bins + base);
    unsigned run = __ldg(a.tile_sum + tile) +
                   block_excl_scan_256(v.x + v.y + v.z + v.w, wtot, nullptr);
    uint4 o;
    o.x = run; run += v.x;
    o.y = run; run += v.y;
    o.z = run; run += v.z;
    o.w = run;
    *reinterpret_cast<uint4*>(a.cursor + base) = o;
}

template <bool VEC>
__global__ void __launch_bounds__(256) k_bin_scatter(SortedArgs a) {
    RootInfo ri;
    root_info(a.hdr, ri);
    const long long nq = (a.n_r + 3) / 4;
    const int lane = threadIdx.x & 31;
    for (long long q = blockIdx.x * 256ll + threadIdx.x; q < nq; q += gridDim.x * 256ll) {
        float s[4][3], e[4][3];
        const int cnt = load4<VEC>(a.starts, a.ends, q, a.n_r, s, e);
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int bin = j < cnt ? seg_bin(s[j], e[j], ri) : -1;
            const unsigned act = __activemask();
            const unsigned peers = __match_any_sync(act, bin);
            const int leader = __ffs(peers) - 1;
            unsigned pos = 0;
            if (bin >= 0 && leader == lane) pos = atomicAdd(a.cursor + bin, __popc(peers));
            pos = __shfl_sync(peers, pos, leader);
            if (bin < 0) continue;
            pos += __popc(peers & ((1u << lane) - 1u));
            const long long id = 4 * q + j;
            a.rec[2 * pos] = make_float4(s[j][0], s[j][1], s[j][2], __int_as_float((int)id));
            a.rec[2 * pos + 1] = make_float4(e[j][0], e[j][1], e[j][2], 0.f);
        }
    }
}

template <int MODE, bool STATS>
__global__ void __launch_bounds__(kSortedThreads) k_trav_sorted(SortedArgs a) {
    const unsigned n_live = *a.n_live;
    const int n_int = a.n_int;
    const int root = n_int > 0 ? __ldg(&a.hdr->root) : 0;
    unsigned long long visits = 0, mts = 0;
    int stack[kSortedStack];
    // each CTA walks one contiguous run of records (one spatial region), so
    // the subtree it touches stays resident in its SM's L1
    const unsigned per_cta = ((n_live + gridDim.x - 1) / gridDim.x + kSortedThreads - 1) /
                             kSortedThreads * kSortedThreads;
    const unsigned beg = blockIdx.x * per_cta;
    const unsigned end = beg + per_cta < n_live ? beg + per_cta : n_live;
    for (unsigned idx = beg + threadIdx.x; idx < end; idx += kSortedThreads) {
        const float4 r0 = a.rec[2 * idx], r1 = a.rec[2 * idx + 1];
        const int id = __float_as_int(r0.w);
        float b[6];
        b[0] = fminf(r0.x, r1.x); b[1] = fmaxf(r0.x, r1.x);
        b[2] = fminf(r0.y, r1.y); b[3] = fmaxf(r0.y, r1.y);
        b[4] = fminf(r0.z, r1.z); b[5] = fmaxf(r0.z, r1.z);
        const double sx = r0.x, sy = r0.y, sz = r0.z;
        const double dx = __dsub_rn((double)r1.x, sx), dy = __dsub_rn((double)r1.y, sy),
                     dz = __dsub_rn((double)r1.z, sz);
        int det = 0, nh = 0, btri = -1;
        double bt = 0.0;
        int top = 0, node = root;
        bool ovf = false;
        for (;;) {
            if (STATS) ++visits;
            int next = -1;
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                float f[8];
                ld_slot(&a.nodes4[node].s[j], f);
                if (!slot_hit(f, b)) continue;
                const int ref = __float_as_int(f[6]);
                if (ref >= n_int) {  // leaf: exact test (_core.pyx:304-320)
                    const RsLeaf* L = a.leaves + (ref - n_int);
                    const float4 p0 = __ldg(&L->p0), p1 = __ldg(&L->p1), p2 = __ldg(&L->p2);
                    double t;
                    if (STATS) ++mts;
                    if (mt_hit(p0.x, p0.y, p0.z, p0.w, p1.x, p1.y, p1.z, p1.w, p2.x, sx, sy, sz, dx,
                               dy, dz, &t)) {
                        const int tid = __float_as_int(p2.y);
                        det = 1;
                        ++nh;
                        if (MODE == kBarycentric &&
                            (btri < 0 || t < bt || (t == bt && tid < btri))) {
                            bt = t;
                            btri = tid;
                        }
                    }
                } else if (next < 0) {
                    next = ref;
                } else if (top < kSortedStack) {
                    stack[top++] = ref;
                } else {
                    ovf = true;
                }
            }
            if (MODE == kBoolean && det) break;
            if (next >= 0) {
                node = next;
            } else if (top > 0) {
                node = stack[--top];
            } else {
                break;
            }
        }
        if (ovf) atomicAdd(&a.status->internal, 1ull);
        if (MODE == kBoolean) {
            if (det) a.flags[id] = 1;
        } else if (MODE == kCount) {
            if (nh) a.flags[id] = nh;
        } else if (btri >= 0) {
            a.best_t[id] = bt == 0.0 ? 0ull : (unsigned long long)__double_as_longlong(bt);
            a.best_tri[id] = btri;
        }
    }
    if (STATS) {
        for (int o = 16; o; o >>= 1) {
            visits += __shfl_xor_sync(kFullMask, visits, o);
            mts += __shfl_xor_sync(kFullMask, mts, o);
        }
        if ((threadIdx.x & 31) == 0) {
            atomicAdd(&a.status->visits, visits);
            atomicAdd(&a.status->mts, mts);
        }
    }
}

// Exact test of one candidate leaf (inlined: an out-of-line call measured
// 12% slower on C2).
template <int MODE>
__device__ __forceinline__ void leaf_exact(const RsLeaf* __restrict__ leaves, int leaf, float4 r0,
                                        float4 r1, int& det, int& nh, int& btri, double& bt) {
    const double sx = r0.x, sy = r0.y, sz = r0.z;
    const double dx = __dsub_rn((double)r1.x, sx), dy = __dsub_rn((double)r1.y, sy),
                 dz = __dsub_rn((double)r1.z, sz);
    const RsLeaf* L = leaves + leaf;
    const float4 p0 = __ldg(&L->p0), p1 = __ldg(&L->p1), p2 = __ldg(&L->p2);
    double t;
    if (mt_hit(p0.x, p0.y, p0.z, p0.w, p1.x, p1.y, p1.z, p1.w, p2.x, sx, sy, sz, dx, dy, dz, &t)) {
        const int tid = __float_as_int(p2.y);
        det = 1;
        ++nh;
        if (MODE == kBarycentric && (btri < 0 || t < bt || (t == bt && tid < btri))) {
            bt = t;
            btri = tid;
        }
    }
}

// Binary-node traversal (default): the coherent record order over the 64-B
// RsNode records (two 256-bit loads per visit).
template <int MODE>
__global__ void __launch_bounds__(kSortedThreads, kSortedMinBlocks) k_trav_sorted_bin(SortedArgs a) {
    const unsigned n_live = *a.n_live;
    const int n_int = a.n_int;
    const int root = n_int > 0 ? __ldg(&a.hdr->root) : 0;
    const RsSlot* const nodes = reinterpret_cast<const RsSlot*>(a.nodes);
    const RsLeaf* const leaves = a.leaves;
    const float4* const rec = a.rec;
    int stack[kSortedStack];
    const unsigned per_cta = ((n_live + gridDim.x - 1) / gridDim.x + kSortedThreads - 1) /
                             kSortedThreads * kSortedThreads;
    const unsigned beg = blockIdx.x * per_cta;
    const unsigned end = beg + per_cta < n_live ? beg + per_cta : n_live;
    for (unsigned idx = beg + threadIdx.x; idx < end; idx += kSortedThreads) {
        const float4 r0 = rec[2 * idx], r1 = rec[2 * idx + 1];
        const int id = __float_as_int(r0.w);
        const float b0 = fminf(r0.x, r1.x), b1 = fmaxf(r0.x, r1.x);
        const float b2 = fminf(r0.y, r1.y), b3 = fmaxf(r0.y, r1.y);
        const float b4 = fminf(r0.z, r1.z), b5 = fmaxf(r0.z, r1.z);
        int det = 0, nh = 0, btri = -1;
        double bt = 0.0;
        int top = 0, node = root;
        bool ovf = false;
        if (n_int == 0) {  // single triangle: the leaf is the root (_core.pyx:260-267)
            const float4 p0 = __ldg(&leaves[0].p0), p1 = __ldg(&leaves[0].p1), p2 = __ldg(&leaves[0].p2);
            const bool o = (b0 <= fmaxf(fmaxf(p0.x, p0.w), p1.z)) & (b1 >= fminf(fminf(p0.x, p0.w), p1.z)) &
                           (b2 <= fmaxf(fmaxf(p0.y, p1.x), p1.w)) & (b3 >= fminf(fminf(p0.y, p1.x), p1.w)) &
                           (b4 <= fmaxf(fmaxf(p0.z, p1.y), p2.x)) & (b5 >= fminf(fminf(p0.z, p1.y), p2.x));
            if (o) leaf_exact<MODE>(leaves, 0, r0, r1, det, nh, btri, bt);
        } else {
            for (;;) {
                float f0[8], f1[8];
                ld_slot(nodes + 2 * node, f0);
                ld_slot(nodes + 2 * node + 1, f1);
                // RsNode: [l.x0 l.x1 l.y0 l.y1 l.z0 l.z1 r.x0 r.x1] [r.y0 r.y1 r.z0 r.z1 lref rref - -]
                const int ca = __float_as_int(f1[4]), cb = __float_as_int(f1[5]);
                const bool oa = (b0 <= f0[1]) & (b1 >= f0[0]) & (b2 <= f0[3]) & (b3 >= f0[2]) &
                                (b4 <= f0[5]) & (b5 >= f0[4]);
                const bool ob = (b0 <= f0[7]) & (b1 >= f0[6]) & (b2 <= f1[1]) & (b3 >= f1[0]) &
                                (b4 <= f1[3]) & (b5 >= f1[2]);
                const bool la = ca >= n_int, lb = cb >= n_int;
                if (oa & la) leaf_exact<MODE>(leaves, ca - n_int, r0, r1, det, nh, btri, bt);
                if (ob & lb) leaf_exact<MODE>(leaves, cb - n_int, r0, r1, det, nh, btri, bt);
                if (MODE == kBoolean && det) break;
                const bool ta = oa & !la, tb = ob & !lb;
                if (ta & tb) {
                    if (top < kSortedStack) stack[top++] = cb;
                    else ovf = true;
                }
                if (ta | tb) {
                    node = ta ? ca : cb;
                } else if (top > 0) {
                    node = stack[--top];
                } else {
                    break;
                }
            }
        }
        if (ovf) atomicAdd(&a.status->internal, 1ull);
        if (MODE == kBoolean) {
            if (det) a.flags[id] = 1;
        } else if (MODE == kCount) {
            if (nh) a.flags[id] = nh;
        } else if (btri >= 0) {
            a.best_t[id] = bt == 0.0 ? 0ull : (unsigned long long)__double_as_longlong(bt);
            a.best_tri[id] = btri;
        }
    }
}

// ------------------------------------------------------------ host glue ---

size_t sorted_bins() { return kBins; }

static int sm_total() {
    static int sms = 0;
    if (!sms) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    }
    return sms;
}

bool sorted_wide() {
    static const bool wide = [] {
        const char* e = getenv("RS_SORTED_WIDE");
        return e && e[0] == '1';
    }();
    return wide;
}

void launch_binning(const SortedArgs& a, cudaStream_t s) {
    if (a.n_r <= 0) return;
    count_launches(5);
    const int sms = sm_total();
    const bool vec = ((reinterpret_cast<uintptr_t>(a.starts) | reinterpret_cast<uintptr_t>(a.ends)) & 15) == 0;
    const long long want = (a.n_r + 1023) / 1024;
    const unsigned g = (unsigned)(want < sms * 16ll ? want : sms * 16ll);
    if (vec) k_bin_count<true><<<g, 256, 0, s>>>(a);
    else k_bin_count<false><<<g, 256, 0, s>>>(a);
    k_tile_reduce<<<kScanTiles, 256, 0, s>>>(a);
    k_tile_scan<<<1, 256, 0, s>>>(a);
    k_bin_scan<<<kScanTiles, 256, 0, s>>>(a);
    if (vec) k_bin_scatter<true><<<g, 256, 0, s>>>(a);
    else k_bin_scatter<false><<<g, 256, 0, s>>>(a);
}

void launch_sorted_trav(const SortedArgs& a, int mode, bool stats, cudaStream_t s) {
    if (a.n_r <= 0) return;
    count_launches(1);
    const int sms = sm_total();
    static int occ[3] = {0, 0, 0};
    int& o = occ[mode];
    if (!o) {
        const void* k = mode == kBoolean ? (const void*)k_trav_sorted<kBoolean, false>
                        : mode == kCount ? (const void*)k_trav_sorted<kCount, false>
                                         : (const void*)k_trav_sorted<kBarycentric, false>;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, k, kSortedThreads, 0);
        if (o < 1) o = 1;
    }
    const long long wt = (a.n_r + kSortedThreads - 1) / kSortedThreads;
    const unsigned gt = (unsigned)(wt < (long long)sms * o ? wt : (long long)sms * o);
    // binary nodes measured faster on coherent segments (C2: 0.64 vs 0.67 ms);
    // RS_SORTED_WIDE=1 selects the 4-wide per-thread traversal instead
    const bool bin_nodes = !sorted_wide();
    hot_kernel_mark(0, s);
    if (bin_nodes && !stats) {
        if (mode == kBoolean) k_trav_sorted_bin<kBoolean><<<gt, kSortedThreads, 0, s>>>(a);
        else if (mode == kCount) k_trav_sorted_bin<kCount><<<gt, kSortedThreads, 0, s>>>(a);
        else k_trav_sorted_bin<kBarycentric><<<gt, kSortedThreads, 0, s>>>(a);
        hot_kernel_mark(1, s);
        return;
    }
    if (mode == kBoolean) {
        if (stats) k_trav_sorted<kBoolean, true><<<gt, kSortedThreads, 0, s>>>(a);
        else k_trav_sorted<kBoolean, false><<<gt, kSortedThreads, 0, s>>>(a);
    } else if (mode == kCount) {
        if (stats) k_trav_sorted<kCount, true><<<gt, kSortedThreads, 0, s>>>(a);
        else k_trav_sorted<kCount, false><<<gt, kSortedThreads, 0, s>>>(a);
    } else {
        if (stats) k_trav_sorted<kBarycentric, true><<<gt, kSortedThreads, 0, s>>>(a);
        else k_trav_sorted<kBarycentric, false><<<gt, kSortedThreads, 0, s>>>(a);
    }
    hot_kernel_mark(1, s);
}

}  // namespace rs
