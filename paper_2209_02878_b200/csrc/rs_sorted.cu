// rs_sorted.cu -- the fast-tree hot path: coherent per-segment traversal.
//
// Segments arrive in caller order, which for random inputs means neighbouring
// lanes walk unrelated parts of the tree and every node load is a scattered
// 128-B line (L1-wavefront bound).  So the query first reorders the segments
// spatially with a two-pass counting sort, fused with root culling:
//
//   k_seg_sample     box statistics of 4096 sampled segments; its last CTA
//                    derives the bin geometry (bits per axis, key tables) once
//                    for the call (root box, sample, depth complexity).
//   k_bin_count_tma  per segment, streamed through shared memory by TMA bulk
//                    copies: f32 AABB (engine.py:115-122), root-box cull (a
//                    segment outside it has no candidates: its result is the
//                    pre-zeroed default and it is dropped), Morton key of the
//                    box centre (up to 2^19 bins), histogram reductions.
//   k_bin_scan1      single-pass exclusive scan of the active bins.
//   k_bin_scatter    same key; each live segment's record (start, id, end;
//                    32 B) goes to its bin's next slot.
//   k_trav_tile      tiles of consecutive records (a small region): the
//                    tile's candidate list from a Morton key range or a walk
//                    of the tree, filtered per warp and per lane, then the f64
//                    Moller-Trumbore test at the candidates in reference op
//                    order, results written to the segments' original rows.
//   k_trav_sorted_bin / k_trav_sorted: per-record stack walks (sparse batches,
//                    tiles whose lists overflow, statistics).
//
// Results do not depend on the order: boolean = any, count = sum, barycentric
// = min over (t, triangle id) (_core.pyx:304-322).
#include "rs_common.cuh"
#include "rs_internal.h"

#include <cstdint>
#include <cstdlib>
#include <cstring>

namespace rs {

constexpr unsigned kFullMask = 0xffffffffu;
// up to 512k spatial bins: the scatter's open output lines (one 128-B line
// per bin) stay within half of L2 (1B-segment C5: 2M bins took the scatter
// from 13 to 17 ms; C2-C4 use 2^18-2^19 bins anyway)
#ifndef RS_BIN_BITS
#define RS_BIN_BITS 19
#endif
constexpr int kBinBits = RS_BIN_BITS;
constexpr int kSampleCtas = 32;              // k_seg_sample grid
constexpr int kSampleThreads = 128;
constexpr int kBins = 1 << kBinBits;
constexpr int kScanShift = 10;
constexpr int kScanTile = 1 << kScanShift;
constexpr int kScanTiles = kBins / kScanTile;
// zeroed words in tile_sum after the look-back words: the scan's ticket, then
// k_seg_sample's completion counter
constexpr int kScanTicket = 2 * kScanTiles;
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

// One 32-B record (start, id, end) as a single 256-bit store: one full
// sector per record instead of two half-sector writes.
__device__ __forceinline__ void st_rec(float4* dst, const float s[3], int id, const float e[3]) {
    asm volatile("st.global.v8.f32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(dst), "f"(s[0]), "f"(s[1]),
                 "f"(s[2]), "f"(__int_as_float(id)), "f"(e[0]), "f"(e[1]), "f"(e[2]), "f"(0.f)
                 : "memory");
}

// Sorted-order segment access: the scatter wrote each live segment's 32-B
// record (start, id, end).  (Writing only 4-B segment ids and gathering the
// rows in the traversal measured 3.7x slower on C2: the gathered rows miss
// L1 and are re-read from DRAM.)
__device__ __forceinline__ void get_rec(const SortedArgs& a, unsigned idx, float4& r0, float4& r1) {
    r0 = a.rec[2ull * idx];
    r1 = a.rec[2ull * idx + 1];
}

// The record's last read (the tile kernel's processing pass): marked
// evict-first in L2, so the dead records stop displacing the outputs
// (flags / winning triangles / hit bits written at random by segment id).
__device__ __forceinline__ void get_rec_last(const SortedArgs& a, unsigned idx, float4& r0, float4& r1) {
#ifdef RS_NO_EVICT_HINT
    get_rec(a, idx, r0, r1);
#else
    unsigned long long pol;
    asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    const float4* p = a.rec + 2ull * idx;
    asm volatile("ld.global.L2::cache_hint.v4.f32 {%0,%1,%2,%3}, [%4], %5;"
                 : "=f"(r0.x), "=f"(r0.y), "=f"(r0.z), "=f"(r0.w) : "l"(p), "l"(pol));
    asm volatile("ld.global.L2::cache_hint.v4.f32 {%0,%1,%2,%3}, [%4], %5;"
                 : "=f"(r1.x), "=f"(r1.y), "=f"(r1.z), "=f"(r1.w) : "l"(p + 1), "l"(pol));
#endif
}

__device__ __forceinline__ void put_rec(const SortedArgs& a, unsigned pos, const float s[3], int id,
                                        const float e[3]) {
    st_rec(a.rec + 2ull * pos, s, id, e);
}

__device__ __forceinline__ unsigned spread3(unsigned v) {  // bit i -> bit 3i (i < 10)
    v &= 0x3ffu;
    v = (v | (v << 16)) & 0x030000ffu;
    v = (v | (v << 8)) & 0x0300f00fu;
    v = (v | (v << 4)) & 0x030c30c3u;
    v = (v | (v << 2)) & 0x09249249u;
    return v;
}
__device__ __forceinline__ unsigned spread2(unsigned v) {  // bit i -> bit 2i (i < 16)
    v &= 0xffffu;
    v = (v | (v << 8)) & 0x00ff00ffu;
    v = (v | (v << 4)) & 0x0f0f0f0fu;
    v = (v | (v << 2)) & 0x33333333u;
    v = (v | (v << 1)) & 0x55555555u;
    return v;
}

// Root box + bin geometry shared by both binning passes.  The 21 key bits
// are shared out so that cells are as close to cubes as the root box allows
// (greedy: the next bit halves the currently longest cell side): a flat
// terrain gets fine xy cells and few z cells instead of 128 per axis.
// Axes are ranked by bit count (A >= B >= C); the key interleaves all three
// over C's bits, then A and B, then A alone (a Morton order with unequal
// axis resolutions).
struct RootInfo {
    float lo[3], hi[3], scale[3];
    int qmax[3];
    int pa, pb, pc;  // axes by bit count, descending
    int bb, bc;      // bits of B and C
    int nbits;       // key bits: keys < 2^nbits
};

// The root box (union of all triangle boxes) comes from the build's k_prep,
// so the binning can run concurrently with the rest of the build.
__device__ __forceinline__ void root_info_compute(const RsHeader* hdr, const SortedArgs& a,
                                                  const float st[4], RootInfo& ri) {
    float e0, e1, e2;
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        ri.lo[k] = from_ord32(~__ldg(&hdr->bmin[k]));
        ri.hi[k] = from_ord32(__ldg(&hdr->bmax[k]));
    }
    e0 = fmaxf(ri.hi[0] - ri.lo[0], 0.f);
    e1 = fmaxf(ri.hi[1] - ri.lo[1], 0.f);
    e2 = fmaxf(ri.hi[2] - ri.lo[2], 0.f);
    // a cell side below the typical segment-box side along that axis buys
    // no coherence (neighbouring boxes overlap anyway): such an axis only
    // gets bits once every other axis is that fine too
    const float f0 = st[3] > 0.f ? st[0] / st[3] : 0.f;
    const float f1 = st[3] > 0.f ? st[1] / st[3] : 0.f;
    const float f2 = st[3] > 0.f ? st[2] / st[3] : 0.f;
    // total bits: about a.bin_occupancy live segments per bin, so the bins'
    // open output lines stay L2-resident during the scatter
    const double live = (double)a.n_r * (st[3] / (float)(kSampleCtas * kSampleThreads));
    // stacked surfaces (depth complexity, projected triangle-box area over
    // the root box's, above 6): proportionally finer bins, since a tile's
    // candidate list holds every layer under its records (C4, depth 12.8:
    // 1.79 -> 1.54 ms; the single terrains C2/C5 sit at 3.2-3.4)
    const float ra = e0 * e1 + e1 * e2 + e2 * e0;
    const float depth = ra > 0.f ? __ldg(&hdr->parea) / ra : 0.f;
    const double occ = depth > 6.f ? fmax(1.0, (double)a.bin_occupancy * 6.0 / depth) : (double)a.bin_occupancy;
    int nbits = 0;
    while (nbits < kBinBits && (double)(1u << (nbits + 1)) * occ <= live) ++nbits;
    nbits = nbits < 8 ? 8 : nbits;
    ri.nbits = nbits;
    float c0 = e0, c1 = e1, c2 = e2;
    int b0 = 0, b1 = 0, b2 = 0;
    for (int i = 0; i < nbits; ++i) {
        const float g0 = c0 > f0 ? c0 : 0.f, g1 = c1 > f1 ? c1 : 0.f, g2 = c2 > f2 ? c2 : 0.f;
        const bool any = (g0 > 0.f) | (g1 > 0.f) | (g2 > 0.f);
        const float h0 = any ? g0 : c0, h1 = any ? g1 : c1, h2 = any ? g2 : c2;
        if (h0 >= h1 && h0 >= h2) { ++b0; c0 *= 0.5f; }
        else if (h1 >= h2) { ++b1; c1 *= 0.5f; }
        else { ++b2; c2 *= 0.5f; }
    }
    ri.qmax[0] = (1 << b0) - 1; ri.qmax[1] = (1 << b1) - 1; ri.qmax[2] = (1 << b2) - 1;
    ri.scale[0] = e0 > 0.f ? (float)(1 << b0) / e0 : 0.f;
    ri.scale[1] = e1 > 0.f ? (float)(1 << b1) / e1 : 0.f;
    ri.scale[2] = e2 > 0.f ? (float)(1 << b2) / e2 : 0.f;
    // rank the axes by bit count (ties: lower axis first)
    const int pa = (b0 >= b1 && b0 >= b2) ? 0 : (b1 >= b2 ? 1 : 2);
    int pc;
    if (pa == 0) pc = b2 < b1 ? 2 : 1;
    else if (pa == 1) pc = b2 < b0 ? 2 : 0;
    else pc = b1 < b0 ? 1 : 0;
    ri.pa = pa;
    ri.pc = pc;
    ri.pb = 3 - pa - pc;
    const int bits[3] = {b0, b1, b2};
    ri.bb = bits[ri.pb];
    ri.bc = bits[pc];
}

// Key bit position of axis bit i for an axis of role r (0 = A, 1 = B, 2 = C;
// see RootInfo): all three axes interleave over C's bits, then A and B,
// then A alone.
__device__ __forceinline__ int key_pos(int role, int i, int bb, int bc) {
    if (i < bc) return 3 * i + role;
    if (i < bb) return 3 * bc + 2 * (i - bc) + role;
    return 2 * bb + bc + (i - bb);
}

// The bin geometry is derived once per call, by the last CTA of
// k_seg_sample (bin_geom_fill), into global memory: the RootInfo and
// per-axis deposit tables (the key is the OR over axes of
// T[axis][chunk][7-bit chunk of q], 9 table lookups instead of ~80 ALU ops of
// axis ranking and bit spreading per key).  Every binning CTA copies it to
// shared memory instead of re-deriving it serially on one thread.
struct alignas(16) BinLut {
    unsigned t[3][3][128];
};
struct BinGeom {
    RootInfo ri;
    BinLut lut;
};
size_t bin_geom_bytes() { return sizeof(BinGeom); }

// the 3x3x128 deposit tables of a bin geometry (all threads of the CTA)
__device__ __forceinline__ void lut_fill(const RootInfo& ri, unsigned (*t)[3][128]) {
    for (int e = threadIdx.x; e < 3 * 3 * 128; e += blockDim.x) {
        const int axis = e / 384, chunk = (e / 128) % 3, v = e % 128;
        const int role = axis == ri.pa ? 0 : (axis == ri.pb ? 1 : 2);
        const int nb = axis == ri.pa ? (ri.nbits - ri.bb - ri.bc) : (axis == ri.pb ? ri.bb : ri.bc);
        unsigned out = 0;
        for (int j = 0; j < 7; ++j) {
            const int i = 7 * chunk + j;
            if (((v >> j) & 1) && i < nb) out |= 1u << key_pos(role, i, ri.bb, ri.bc);
        }
        t[axis][chunk][v] = out;
    }
}

// the sample CTAs' partials (one thread, fixed order)
__device__ __forceinline__ void stats_serial(const SortedArgs& a, float st[4]) {
    st[0] = st[1] = st[2] = st[3] = 0.f;
    for (int c = 0; c < kSampleCtas; ++c)
#pragma unroll
        for (int k = 0; k < 4; ++k) st[k] += a.seg_stats[4 * c + k];
}

__device__ __forceinline__ void bin_geom_fill(const SortedArgs& a) {
    __shared__ RootInfo s_ri;
    BinGeom* g = reinterpret_cast<BinGeom*>(a.geom);
    static_assert(kSampleCtas == 32, "one lane per sample CTA");
    if (threadIdx.x < 32) {
        // the sample CTAs' partials, summed in a fixed shuffle tree (deterministic)
        float st[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            float v = __ldcg(a.seg_stats + 4 * threadIdx.x + k);
            for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(kFullMask, v, o);
            st[k] = v;
        }
        if (threadIdx.x == 0) {
            root_info_compute(a.hdr, a, st, s_ri);
            g->ri = s_ri;
        }
    }
    __syncthreads();
    lut_fill(s_ri, g->lut.t);
}

// geom_mode 1: copy the precomputed geometry; 0 (A/B): thread 0 derives it
// and the CTA fills the tables itself
__device__ __forceinline__ void root_info(const SortedArgs& a, RootInfo& ri, const BinLut*& lut) {
    __shared__ RootInfo s_ri;
    __shared__ BinLut s_lut;
    if (a.geom_mode) {
        const BinGeom* g = reinterpret_cast<const BinGeom*>(a.geom);
        constexpr int kRiWords = sizeof(RootInfo) / 4;
        static_assert(sizeof(RootInfo) % 4 == 0, "RootInfo is copied as words");
        if (threadIdx.x < kRiWords)
            reinterpret_cast<unsigned*>(&s_ri)[threadIdx.x] = __ldg(reinterpret_cast<const unsigned*>(&g->ri) + threadIdx.x);
        const uint4* src = reinterpret_cast<const uint4*>(&g->lut);
        uint4* dst = reinterpret_cast<uint4*>(&s_lut);
        for (int e = threadIdx.x; e < (int)(sizeof(BinLut) / 16); e += blockDim.x) dst[e] = __ldg(src + e);
        __syncthreads();
    } else {
        if (threadIdx.x == 0) {
            float st[4];
            stats_serial(a, st);
            root_info_compute(a.hdr, a, st, s_ri);
        }
        __syncthreads();
        lut_fill(s_ri, s_lut.t);
        __syncthreads();
    }
    ri = s_ri;
    lut = &s_lut;
}

// Returns the bin of a live segment, or -1 when its box misses the root box
// (no leaf box can overlap it: its result is the pre-zeroed default).
__device__ __forceinline__ int seg_bin(const float s[3], const float e[3], const RootInfo& ri,
                                       const BinLut* lut) {
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
        const float f = fminf(fmaxf((c - ri.lo[k]) * ri.scale[k], 0.f), (float)ri.qmax[k]);
        const unsigned q = (unsigned)f;
        key |= lut->t[k][0][q & 127u] | lut->t[k][1][(q >> 7) & 127u] | lut->t[k][2][q >> 14];
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

// Sample statistics over a fixed strided sample of kSampleCtas x 128
// segments: per CTA, the summed box sides of the sampled segments that
// overlap the root box and their count.  root_info_compute sums the CTA
// partials in a fixed order (deterministic) and derives the bin geometry.
__global__ void __launch_bounds__(kSampleThreads) k_seg_sample(SortedArgs a) {
    __shared__ float red[4][kSampleThreads / 32];
    float lo[3], hi[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        lo[k] = from_ord32(~__ldg(&a.hdr->bmin[k]));
        hi[k] = from_ord32(__ldg(&a.hdr->bmax[k]));
    }
    float acc[4] = {0.f, 0.f, 0.f, 0.f};
    const long long n_s = (long long)kSampleCtas * kSampleThreads;
    const long long stride = a.n_r / n_s > 0 ? a.n_r / n_s : 1;
    const long long i = ((long long)blockIdx.x * kSampleThreads + threadIdx.x) * stride;
    if (i < a.n_r) {
        float b[6];
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            const float p = __ldg(a.starts + 3 * i + k), q = __ldg(a.ends + 3 * i + k);
            b[2 * k] = fminf(p, q);
            b[2 * k + 1] = fmaxf(p, q);
        }
        const bool live = (b[0] <= hi[0]) & (b[1] >= lo[0]) & (b[2] <= hi[1]) & (b[3] >= lo[1]) &
                          (b[4] <= hi[2]) & (b[5] >= lo[2]);
        if (live) {
            acc[0] = b[1] - b[0];
            acc[1] = b[3] - b[2];
            acc[2] = b[5] - b[4];
            acc[3] = 1.f;
        }
    }
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        float v = acc[k];
        for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(kFullMask, v, o);
        if (lane == 0) red[k][w] = v;
    }
    __syncthreads();
    if (threadIdx.x < 4) {
        float v = 0.f;
        for (int j = 0; j < kSampleThreads / 32; ++j) v += red[threadIdx.x][j];
        a.seg_stats[4 * blockIdx.x + threadIdx.x] = v;
        __threadfence();
    }
    // the last CTA to finish derives the bin geometry for the binning passes
    __shared__ bool s_last;
    __syncthreads();
    if (threadIdx.x == 0) s_last = atomicAdd(a.tile_sum + kScanTicket + 1, 1u) == kSampleCtas - 1;
    __syncthreads();
    if (!s_last || !a.geom_mode) return;
    __threadfence();
    bin_geom_fill(a);
}

// Histogram pass.  Inputs arrive in caller order, so a warp's bins rarely
// coincide: plain fire-and-forget reductions, with warp aggregation only
// when neighbouring lanes share a bin (pre-sorted inputs).
template <bool VEC>
__global__ void __launch_bounds__(256) k_bin_count(SortedArgs a) {
    RootInfo ri;
    const BinLut* lut;
    root_info(a, ri, lut);
    const long long nq = (a.n_r + 3) / 4;
    const int lane = threadIdx.x & 31;
    for (long long q = blockIdx.x * 256ll + threadIdx.x; q < nq; q += gridDim.x * 256ll) {
        float s[4][3], e[4][3];
        const int cnt = load4<VEC>(a.starts, a.ends, q, a.n_r, s, e);
        int bin[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) bin[j] = j < cnt ? seg_bin(s[j], e[j], ri, lut) : -1;
        const unsigned act = __activemask();
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int up = __shfl_up_sync(act, bin[j], 1);
            if (__any_sync(act, lane > 0 && bin[j] >= 0 && up == bin[j])) {
                const unsigned peers = __match_any_sync(act, bin[j]);
                if (bin[j] >= 0 && (__ffs(peers) - 1) == lane) atomicAdd(a.bins + bin[j], __popc(peers));
            } else if (bin[j] >= 0) {
                atomicAdd(a.bins + bin[j], 1u);
            }
        }
    }
}

// Block-wide exclusive scan of 256 per-thread values (k_bin_scan1).
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

// Scatter pass: the same bins; each live segment's 32-B record goes to its
// bin's next slot.  The four cursor claims of a thread are issued together
// (their round trips overlap) before any record is written.
// Single-pass exclusive scan of the active bins (keys < 2^nbits): one CTA
// per 1024-bin tile in ticket order, decoupled look-back across tiles; the
// last active tile publishes the live count.  Tiles beyond the active range
// exit at once.
__global__ void __launch_bounds__(256) k_bin_scan1(SortedArgs a) {
    __shared__ unsigned wtot[8];
    __shared__ int s_tile, s_active;
    __shared__ unsigned s_excl;
    if (threadIdx.x == 0) {
        int nbits;
        if (a.geom_mode) {
            nbits = (int)__ldg(&reinterpret_cast<const BinGeom*>(a.geom)->ri.nbits);
        } else {
            float st[4];
            RootInfo ri;
            stats_serial(a, st);
            root_info_compute(a.hdr, a, st, ri);
            nbits = ri.nbits;
        }
        const int active = (1 << nbits) > kScanTile ? (1 << nbits) / kScanTile : 1;
        s_active = active;
        s_tile = (int)atomicAdd(a.tile_sum + kScanTicket, 1u);
    }
    __syncthreads();
    const int tile = s_tile;
    if (tile >= s_active) return;
    const int base = tile * kScanTile + threadIdx.x * 4;
    const uint4 v = *reinterpret_cast<const uint4*>(a.bins + base);
    unsigned total;
    const unsigned local = block_excl_scan_256(v.x + v.y + v.z + v.w, wtot, &total);
    if (threadIdx.x < 32) {
        const unsigned long long excl =
            lookback_warp(reinterpret_cast<unsigned long long*>(a.tile_sum), tile, total);
        if (threadIdx.x == 0) {
            s_excl = (unsigned)excl;
            if (tile == s_active - 1) *a.n_live = (unsigned)(excl + total);
        }
    }
    __syncthreads();
    unsigned run = s_excl + local;
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
    const BinLut* lut;
    root_info(a, ri, lut);
    const long long nq = (a.n_r + 3) / 4;
    const int lane = threadIdx.x & 31;
    for (long long q = blockIdx.x * 256ll + threadIdx.x; q < nq; q += gridDim.x * 256ll) {
        float s[4][3], e[4][3];
        const int cnt = load4<VEC>(a.starts, a.ends, q, a.n_r, s, e);
        int bin[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) bin[j] = j < cnt ? seg_bin(s[j], e[j], ri, lut) : -1;
        const unsigned act = __activemask();
        bool dup = false;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int up = __shfl_up_sync(act, bin[j], 1);
            dup |= lane > 0 && bin[j] >= 0 && up == bin[j];
        }
        unsigned pos[4];
        if (__any_sync(act, dup)) {
            // neighbouring lanes share bins: one claim per distinct bin
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const unsigned peers = __match_any_sync(act, bin[j]);
                const int leader = __ffs(peers) - 1;
                unsigned p = 0;
                if (bin[j] >= 0 && leader == lane) p = atomicAdd(a.cursor + bin[j], __popc(peers));
                pos[j] = __shfl_sync(peers, p, leader) + __popc(peers & ((1u << lane) - 1u));
            }
        } else {
#pragma unroll
            for (int j = 0; j < 4; ++j) pos[j] = bin[j] >= 0 ? atomicAdd(a.cursor + bin[j], 1u) : 0u;
        }
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            if (bin[j] < 0) continue;
            put_rec(a, pos[j], s[j], (int)(4 * q + j), e[j]);
        }
    }
}

// ---- binning passes over TMA bulk copies ------------------------------------
//
// The two binning passes stream 24 B per segment and do ~100 instructions of
// key arithmetic per segment.  With plain loads a thread's loads sit idle
// while it computes, so the passes reached about half of HBM bandwidth.  Here
// each CTA keeps two 1024-segment stages in shared memory, filled by the TMA
// engine (cp.async.bulk global->shared, completion on an mbarrier) one chunk
// ahead of the compute, so the DRAM stream never waits for the key math.
#ifndef RS_STREAM_THREADS
#define RS_STREAM_THREADS 128  // x 9 CTAs per SM, 7 resident (A/B vs 256 x 4: C3 -7 us, C2 -1.5, C4 +3;
                                // 7 CTAs or plain reductions without the duplicate check: no gain)
#endif
#ifndef RS_STREAM_CTAS
#define RS_STREAM_CTAS 9
#endif
constexpr int kStreamThreads = RS_STREAM_THREADS;
constexpr int kStreamSegs = 4 * kStreamThreads;  // four segments per thread per stage
constexpr unsigned kStreamStageBytes = 2u * kStreamSegs * 12u;  // starts + ends
constexpr size_t kStreamSmem = 2 * kStreamStageBytes + 64;

__device__ __forceinline__ unsigned smem_u32(const void* p) {
    return (unsigned)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned parity) {
    asm volatile(
        "{\n .reg .pred p;\n"
        "RS_MBAR_WAIT%=:\n"
        " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        " @!p bra RS_MBAR_WAIT%=;\n}\n" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes,
                                         unsigned long long* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}

// Calls body(s, e, cnt, q) for every group of four consecutive segments
// (q = group index), with the full 1024-segment chunks streamed through
// shared memory and the ragged tail read directly.
template <class Body>
__device__ __forceinline__ void stream_segments(const SortedArgs& a, Body&& body) {
    extern __shared__ __align__(128) unsigned char stream_smem[];
    unsigned long long* bar = reinterpret_cast<unsigned long long*>(stream_smem + 2 * kStreamStageBytes);
    const long long nfull = a.n_r / kStreamSegs;
    const long long first = blockIdx.x;
    const long long step = gridDim.x;
    auto stage = [&](int st) { return reinterpret_cast<float*>(stream_smem + st * kStreamStageBytes); };
    auto issue = [&](long long c, int st) {
        const size_t off = (size_t)c * kStreamSegs * 3;
        mbar_expect_tx(&bar[st], kStreamStageBytes);
        bulk_g2s(stage(st), a.starts + off, kStreamSegs * 12u, &bar[st]);
        bulk_g2s(stage(st) + kStreamSegs * 3, a.ends + off, kStreamSegs * 12u, &bar[st]);
    };
    if (threadIdx.x == 0) {
        mbar_init(&bar[0], 1);
        mbar_init(&bar[1], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        if (first < nfull) issue(first, 0);
        if (first + step < nfull) issue(first + step, 1);
    }
    int it = 0;
    for (long long c = first; c < nfull; c += step, ++it) {
        const int st = it & 1;
        mbar_wait(&bar[st], (unsigned)((it >> 1) & 1));
        const float* S = stage(st);
        const float* E = stage(st) + kStreamSegs * 3;
        const int t = threadIdx.x;
        float s[4][3], e[4][3];
        const float4* s4 = reinterpret_cast<const float4*>(S + 12 * t);
        const float4* e4 = reinterpret_cast<const float4*>(E + 12 * t);
        float fs[12], fe[12];
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            const float4 x = s4[k], y = e4[k];
            fs[4 * k] = x.x; fs[4 * k + 1] = x.y; fs[4 * k + 2] = x.z; fs[4 * k + 3] = x.w;
            fe[4 * k] = y.x; fe[4 * k + 1] = y.y; fe[4 * k + 2] = y.z; fe[4 * k + 3] = y.w;
        }
#pragma unroll
        for (int j = 0; j < 4; ++j)
#pragma unroll
            for (int k = 0; k < 3; ++k) {
                s[j][k] = fs[3 * j + k];
                e[j][k] = fe[3 * j + k];
            }
        __syncthreads();  // every thread has its data in registers: the stage may refill
        if (threadIdx.x == 0 && c + 2 * step < nfull) {
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            issue(c + 2 * step, st);
        }
        body(s, e, 4, c * (kStreamSegs / 4) + t);
    }
    // ragged tail (< one chunk): the last CTA reads it directly
    if (blockIdx.x == gridDim.x - 1) {
        const long long nq = (a.n_r + 3) / 4;
        for (long long q = nfull * (kStreamSegs / 4) + threadIdx.x; q < nq; q += kStreamThreads) {
            float s[4][3], e[4][3];
            const int cnt = load4<false>(a.starts, a.ends, q, a.n_r, s, e);
            body(s, e, cnt, q);
        }
    }
}

__global__ void __launch_bounds__(kStreamThreads) k_bin_count_tma(SortedArgs a) {
    RootInfo ri;
    const BinLut* lut;
    root_info(a, ri, lut);
    const int lane = threadIdx.x & 31;
    stream_segments(a, [&](float (&s)[4][3], float (&e)[4][3], int cnt, long long q) {
        if (a.zero_flags) {  // the boolean/count outputs' zero preset, fused
            if (cnt == 4) {
                *reinterpret_cast<int4*>(a.flags + 4 * q) = make_int4(0, 0, 0, 0);
            } else {
                for (int j = 0; j < cnt; ++j) a.flags[4 * q + j] = 0;
            }
        }
        int bin[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) bin[j] = j < cnt ? seg_bin(s[j], e[j], ri, lut) : -1;
        const unsigned act = __activemask();
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int up = __shfl_up_sync(act, bin[j], 1);
            if (__any_sync(act, lane > 0 && bin[j] >= 0 && up == bin[j])) {
                const unsigned peers = __match_any_sync(act, bin[j]);
                if (bin[j] >= 0 && (__ffs(peers) - 1) == lane) atomicAdd(a.bins + bin[j], __popc(peers));
            } else if (bin[j] >= 0) {
                atomicAdd(a.bins + bin[j], 1u);
            }
        }
    });
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
        float4 r0, r1;
        get_rec(a, idx, r0, r1);
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
            if (det) {
                if (a.hitbits) atomicOr(a.hitbits + (id >> 5), 1u << (id & 31));
                else a.flags[id] = 1;
            }
        } else if (MODE == kCount) {
            if (nh) a.flags[id] = nh;
        } else if (btri >= 0) {
            if (a.best_t) a.best_t[id] = bt == 0.0 ? 0ull : (unsigned long long)__double_as_longlong(bt);
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

// One segment's stack traversal of the binary tree (RsNode records, two
// 256-bit loads per visit) with the exact test at the leaves
// (_core.pyx:255-322 semantics, order-free accumulation).
template <int MODE>
__device__ __forceinline__ void trav_one(const RsSlot* __restrict__ nodes,
                                         const RsLeaf* __restrict__ leaves, int n_int, int root,
                                         float4 r0, float4 r1, int& det, int& nh, int& btri,
                                         double& bt, bool& ovf) {
    int stack[kSortedStack];
    const float b0 = fminf(r0.x, r1.x), b1 = fmaxf(r0.x, r1.x);
    const float b2 = fminf(r0.y, r1.y), b3 = fmaxf(r0.y, r1.y);
    const float b4 = fminf(r0.z, r1.z), b5 = fmaxf(r0.z, r1.z);
    if (n_int == 0) {  // single triangle: the leaf is the root (_core.pyx:260-267)
        const float4 p0 = __ldg(&leaves[0].p0), p1 = __ldg(&leaves[0].p1), p2 = __ldg(&leaves[0].p2);
        const bool o = (b0 <= fmaxf(fmaxf(p0.x, p0.w), p1.z)) & (b1 >= fminf(fminf(p0.x, p0.w), p1.z)) &
                       (b2 <= fmaxf(fmaxf(p0.y, p1.x), p1.w)) & (b3 >= fminf(fminf(p0.y, p1.x), p1.w)) &
                       (b4 <= fmaxf(fmaxf(p0.z, p1.y), p2.x)) & (b5 >= fminf(fminf(p0.z, p1.y), p2.x));
        if (o) leaf_exact<MODE>(leaves, 0, r0, r1, det, nh, btri, bt);
        return;
    }
    int top = 0, node = root;
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

template <int MODE>
__device__ __forceinline__ void write_result(const SortedArgs& a, int id, int det, int nh,
                                             int btri, double bt) {
    if (MODE == kBoolean) {
        if (det) {
            if (a.hitbits) atomicOr(a.hitbits + (id >> 5), 1u << (id & 31));
            else a.flags[id] = 1;
        }
    } else if (MODE == kCount) {
        if (nh) a.flags[id] = nh;
    } else if (btri >= 0) {
        if (a.best_t) a.best_t[id] = bt == 0.0 ? 0ull : (unsigned long long)__double_as_longlong(bt);
        a.best_tri[id] = btri;
    }
}

// Binary-node traversal, one thread per record in the coherent record order.
template <int MODE>
__global__ void __launch_bounds__(kSortedThreads, kSortedMinBlocks) k_trav_sorted_bin(SortedArgs a) {
    const unsigned n_live = *a.n_live;
    const int n_int = a.n_int;
    const int root = n_int > 0 ? __ldg(&a.hdr->root) : 0;
    const RsSlot* const nodes = reinterpret_cast<const RsSlot*>(a.nodes);
    const unsigned per_cta = ((n_live + gridDim.x - 1) / gridDim.x + kSortedThreads - 1) /
                             kSortedThreads * kSortedThreads;
    const unsigned beg = blockIdx.x * per_cta;
    const unsigned end = beg + per_cta < n_live ? beg + per_cta : n_live;
    for (unsigned idx = beg + threadIdx.x; idx < end; idx += kSortedThreads) {
        float4 r0, r1;
        get_rec(a, idx, r0, r1);
        int det = 0, nh = 0, btri = -1;
        double bt = 0.0;
        bool ovf = false;
        trav_one<MODE>(nodes, a.leaves, n_int, root, r0, r1, det, nh, btri, bt, ovf);
        if (ovf) atomicAdd(&a.status->internal, 1ull);
        write_result<MODE>(a, __float_as_int(r0.w), det, nh, btri, bt);
    }
}

// ---- tile traversal (default) ---------------------------------------------
//
// The records are in spatial-bin order, so a contiguous run of them (a tile)
// covers a small region.  One CTA per tile:
//   1. union box U of the tile's segment boxes (block reduction);
//   2. cooperative breadth-first walk of the tree with U: every leaf whose
//      exact box overlaps U goes to a shared-memory candidate list L.  Any
//      leaf overlapping a segment's box overlaps U (the segment box is inside
//      U and every internal box contains its subtree's boxes), so L holds
//      every candidate of every segment of the tile;
//   3. per warp of 32 records: the warp's union box W filters L (one ballot
//      per 32 entries); each lane then runs the exact f32 box test of its own
//      segment against the surviving entries (broadcast shared-memory reads)
//      and the f64 Moller-Trumbore test on its overlaps.
// The top of the tree is walked once per tile instead of once per segment,
// and the per-segment loop has no stack and no dependent global loads.
// A tile whose walk exceeds the shared-memory capacities (huge segments,
// random soups) falls back to trav_one for its records.
constexpr int kTileThreads = 128;
#ifndef RS_TILE_MIN_BLOCKS
#define RS_TILE_MIN_BLOCKS 8
#endif
constexpr int kTileMinBlocks = RS_TILE_MIN_BLOCKS;
#ifndef RS_TILE_LCAP
#define RS_TILE_LCAP 256
#endif
constexpr int kTileLCap = RS_TILE_LCAP;  // leaf candidates per tile (256: smaller shared footprint leaves more L1; C2 -5%)
constexpr int kTileFCap = 256;  // walk frontier per level
#ifndef RS_CUT_DEPTH
#define RS_CUT_DEPTH 6
#endif
constexpr int kCutDepth = RS_CUT_DEPTH;  // the walk starts from the depth-6 cut (7, 8 measured slower: smem vs occupancy)
constexpr int kCutCap = 1 << kCutDepth;
// a tile's walk seeds its leaf list and first frontier from the cut without
// capacity checks: at most kCutCap entries each
static_assert(kCutCap <= kTileLCap && kCutCap <= kTileFCap, "cut larger than the tile lists");
#ifndef RS_WCAP
#define RS_WCAP 16
#endif
constexpr int kWCap = RS_WCAP;  // warp candidates prepared per round

// One warp's prepared candidates: the triangle's first vertex and edges in
// f64 (formed once per warp instead of once per exact test), its exact box
// and original id.
struct WarpCand {
    double a[3][kWCap], e1[3][kWCap], e2[3][kWCap];
    float4 xy[kWCap];
    float2 z[kWCap];
    int tid[kWCap];
};

struct TileSmem {
    float4 lxy[kTileLCap];  // leaf box x0 x1 y0 y1
    float2 lz[kTileLCap];   // z0 z1
    int lid[kTileLCap];     // leaf index (Morton order)
    int front[2][kTileFCap];
    float4 cxy[kCutCap];    // the cut: entry boxes and refs (built once per CTA)
    float2 cz[kCutCap];
    int cref[kCutCap];
    WarpCand wc[kTileThreads / 32];
    unsigned char slot[kTileThreads / 32][kWCap][32];  // per-lane candidate lists
    float part[kTileThreads / 32][6];
    int nf[3];
    int nl;
    int ovf;
    int ncut;
    unsigned tile;
    unsigned long long rk[8][2];  // Morton-range sub-boxes: key bounds
    int rr[8][2];                 // and their leaf intervals [i0, i1)
    int nr;
};

__device__ __forceinline__ float wred_min(float v) {
    float r;
    asm volatile("redux.sync.min.f32 %0, %1, 0xffffffff;" : "=f"(r) : "f"(v));
    return r;
}
__device__ __forceinline__ float wred_max(float v) {
    float r;
    asm volatile("redux.sync.max.f32 %0, %1, 0xffffffff;" : "=f"(r) : "f"(v));
    return r;
}

__device__ __forceinline__ bool box_ov(const float q[6], float4 xy, float2 z) {
    return (q[0] <= xy.y) & (q[1] >= xy.x) & (q[2] <= xy.w) & (q[3] >= xy.z) & (q[4] <= z.y) &
           (q[5] >= z.x);
}

// One warp's 32 records (r0, r1 per lane) against a candidate list L
// (lxy/lz/lid, nl entries) that holds every leaf any of them can overlap:
// L filtered by the warp's union box W; each round prepares up to kWCap of
// the survivors (one lane each: f64 vertex and edges into shared memory),
// then every lane keeps the ones its own box overlaps and the exact tests
// run in passes over the per-lane lists, so the warp executes each pass once.
template <int MODE>
__device__ __forceinline__ void process_chunk(const SortedArgs& a, float4 r0, float4 r1, bool valid,
                                              const float4* lxy, const float2* lz, const int* lid,
                                              int nl, WarpCand& wc, unsigned char (*slots)[32],
                                              int& det, int& nh, int& btri, double& bt) {
    const int lane = threadIdx.x & 31;
    float b[6];
    b[0] = fminf(r0.x, r1.x); b[1] = fmaxf(r0.x, r1.x);
    b[2] = fminf(r0.y, r1.y); b[3] = fmaxf(r0.y, r1.y);
    b[4] = fminf(r0.z, r1.z); b[5] = fmaxf(r0.z, r1.z);
    float w[6];
#pragma unroll
    for (int k = 0; k < 6; k += 2) {
        w[k] = wred_min(valid ? b[k] : INFINITY);
        w[k + 1] = wred_max(valid ? b[k + 1] : -INFINITY);
    }
    bool live = valid;
    for (int cb = 0; cb < nl; cb += 32) {
        const int j = cb + lane;
        const bool hit = j < nl && box_ov(w, lxy[j], lz[j]);
        const unsigned m = __ballot_sync(kFullMask, hit);
        const int nm = __popc(m);
        const int rank = __popc(m & ((1u << lane) - 1u));
        for (int base = 0; base < nm; base += kWCap) {
            const int nw = nm - base < kWCap ? nm - base : kWCap;
            if (hit && rank >= base && rank < base + kWCap) {
                const int e = rank - base;
                const RsLeaf* L = a.leaves + lid[j];
                const float4 p0 = __ldg(&L->p0), p1 = __ldg(&L->p1), p2 = __ldg(&L->p2);
                const double ax = p0.x, ay = p0.y, az = p0.z;
                wc.a[0][e] = ax;
                wc.a[1][e] = ay;
                wc.a[2][e] = az;
                wc.e1[0][e] = __dsub_rn((double)p0.w, ax);
                wc.e1[1][e] = __dsub_rn((double)p1.x, ay);
                wc.e1[2][e] = __dsub_rn((double)p1.y, az);
                wc.e2[0][e] = __dsub_rn((double)p1.z, ax);
                wc.e2[1][e] = __dsub_rn((double)p1.w, ay);
                wc.e2[2][e] = __dsub_rn((double)p2.x, az);
                wc.xy[e] = lxy[j];
                wc.z[e] = lz[j];
                wc.tid[e] = __float_as_int(p2.y);
            }
            __syncwarp();
            int nc = 0;
            if (live)
                for (int i = 0; i < nw; ++i)
                    if (box_ov(b, wc.xy[i], wc.z[i])) slots[nc++][lane] = (unsigned char)i;
            const int most = __reduce_max_sync(kFullMask, nc);
            for (int i = 0; i < most; ++i) {
                if (i < nc && live) {
                    const int e = slots[i][lane];
                    const double sx = r0.x, sy = r0.y, sz = r0.z;
                    const double dx = __dsub_rn((double)r1.x, sx),
                                 dy = __dsub_rn((double)r1.y, sy),
                                 dz = __dsub_rn((double)r1.z, sz);
                    double t;
                    if (mt_hit_pre(wc.a[0][e], wc.a[1][e], wc.a[2][e], wc.e1[0][e],
                                   wc.e1[1][e], wc.e1[2][e], wc.e2[0][e], wc.e2[1][e],
                                   wc.e2[2][e], sx, sy, sz, dx, dy, dz, &t)) {
                        const int tid = wc.tid[e];
                        det = 1;
                        ++nh;
                        if (MODE == kBarycentric &&
                            (btri < 0 || t < bt || (t == bt && tid < btri))) {
                            bt = t;
                            btri = tid;
                        }
                        if (MODE == kBoolean) live = false;
                    }
                }
            }
            __syncwarp();
        }
        if (MODE == kBoolean && !__any_sync(kFullMask, live)) break;
    }
}

// Out-of-line fallback (keeps the tile loop's registers free).
template <int MODE, bool WIDE>
__device__ __noinline__ void trav_one_call(const SortedArgs& a, const RsSlot* nodes, int root,
                                           float4 r0, float4 r1, int& det, int& nh, int& btri,
                                           double& bt) {
    bool ovf = false;
    trav_one<MODE>(nodes, a.leaves, a.n_int, root, r0, r1, det, nh, btri, bt, ovf);
    if (ovf) atomicAdd(&a.status->internal, 1ull);
}

// The depth-kCutDepth cut of the tree (every node at that depth, plus the
// leaves above it), with each entry's exact box taken from its parent's
// record.  Warp 0 builds it once per CTA; every tile's walk starts from it.
template <class SM>
__device__ __forceinline__ void build_cut(SM& sm, const RsSlot* nodes, int n_int, int root) {
    if (threadIdx.x >= 32) return;
    const int lane = threadIdx.x;
    // level 0: the root's two children
    int n = 0;
    if (lane == 0) {
        float f0[8], f1[8];
        ld_slot(nodes + 2 * root, f0);
        ld_slot(nodes + 2 * root + 1, f1);
        sm.cxy[0] = make_float4(f0[0], f0[1], f0[2], f0[3]);
        sm.cz[0] = make_float2(f0[4], f0[5]);
        sm.cref[0] = __float_as_int(f1[4]);
        sm.cxy[1] = make_float4(f0[6], f0[7], f1[0], f1[1]);
        sm.cz[1] = make_float2(f1[2], f1[3]);
        sm.cref[1] = __float_as_int(f1[5]);
    }
    n = 2;
    __syncwarp();
    for (int d = 1; d < kCutDepth; ++d) {
        // expand every internal entry into its two children (in place: entry
        // i's children go to slots i and n + (rank of i among internals)),
        // 32 entries per step; all reads of a step precede its writes
        const int n0 = n;
        int added = 0;
        for (int c0i = 0; c0i < n0; c0i += 32) {
            const int i = c0i + lane;
            float4 xy[2];
            float2 z[2];
            int c0 = -1, c1 = -1;
            bool internal = false;
            if (i < n0) {
                const int ref = sm.cref[i];
                internal = ref < n_int;
                if (internal) {
                    float f0[8], f1[8];
                    ld_slot(nodes + 2 * ref, f0);
                    ld_slot(nodes + 2 * ref + 1, f1);
                    xy[0] = make_float4(f0[0], f0[1], f0[2], f0[3]);
                    z[0] = make_float2(f0[4], f0[5]);
                    c0 = __float_as_int(f1[4]);
                    xy[1] = make_float4(f0[6], f0[7], f1[0], f1[1]);
                    z[1] = make_float2(f1[2], f1[3]);
                    c1 = __float_as_int(f1[5]);
                }
            }
            const unsigned m = __ballot_sync(kFullMask, internal);
            __syncwarp();
            if (internal) {
                const int extra = n0 + added + __popc(m & ((1u << lane) - 1u));
                sm.cxy[i] = xy[0]; sm.cz[i] = z[0]; sm.cref[i] = c0;
                sm.cxy[extra] = xy[1]; sm.cz[extra] = z[1]; sm.cref[extra] = c1;
            }
            added += __popc(m);
            __syncwarp();
        }
        n = n0 + added;
    }
    if (lane == 0) sm.ncut = n;
}

// ---- Morton-range candidate lists ------------------------------------------
#ifndef RS_RANGE_SPLIT
#define RS_RANGE_SPLIT 0
#endif
// Triangle t's centroid lies in its box, so a box overlapping U has its
// centroid inside U grown by the largest triangle side per axis, S.  Morton
// order is monotone in every coordinate, so every such centroid's key lies
// in [key(U.lo - S), key(U.hi + S)]: a contiguous run of the sorted leaves.
// Scanning that run (exact box test against U) yields exactly the walk's
// candidate list when the run is short; long runs (boxes straddling a coarse
// Morton boundary) fall back to the walk.
// Quantised key coordinates of a point, exactly as k_keys forms them.
__device__ __forceinline__ void range_q(const SortedArgs& a, const double p[3], unsigned q[3]) {
    double lo[3], ext[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        lo[k] = from_ord(~__ldg(&a.hdr->smin[k]));
        ext[k] = __dsub_rn(from_ord(__ldg(&a.hdr->smax[k])), lo[k]);
    }
    if (a.key_mode == 0) {
        const double e = fmax(fmax(ext[0], ext[1]), ext[2]);
        ext[0] = ext[1] = ext[2] = e;
    }
    const double gmax = (double)((1u << kIsoBits) - 1u);
#pragma unroll
    for (int k = 0; k < 3; ++k) q[k] = ext[k] > 0.0 ? quant1(p[k], lo[k], ext[k], gmax) : 0u;
}

__device__ __forceinline__ unsigned long long code_of(const unsigned q[3]) {
    return split21(q[0]) | (split21(q[1]) << 1) | (split21(q[2]) << 2);
}

// Split the key box [ql, qh] at the highest key bit where its corner keys
// differ (that bit is one axis's bit l: the halves lie below / above the
// axis value with bit l set), up to three times: at most 8 sub-boxes whose
// key ranges are disjoint and together hold every key of the box, far
// tighter than the box's single range.  Returns the count; writes the
// corner keys.
__device__ __forceinline__ int range_split(const unsigned ql[3], const unsigned qh[3],
                                           unsigned long long (*rk)[2]) {
    unsigned lo[8][3], hi[8][3];
    int n = 1;
#pragma unroll
    for (int k = 0; k < 3; ++k) { lo[0][k] = ql[k]; hi[0][k] = qh[k]; }
    for (int d = 0; d < RS_RANGE_SPLIT; ++d) {
        const int m = n;
        for (int b = 0; b < m; ++b) {
            const unsigned long long x = code_of(lo[b]) ^ code_of(hi[b]);
            if (!x) continue;
            const int p = 63 - __clzll((long long)x), ax = p % 3, l = p / 3;
            const unsigned bnd = (hi[b][ax] >> l) << l;
#pragma unroll
            for (int k = 0; k < 3; ++k) { lo[n][k] = lo[b][k]; hi[n][k] = hi[b][k]; }
            hi[b][ax] = bnd - 1;  // box b keeps the lower half
            lo[n][ax] = bnd;      // box n takes the upper half
            ++n;
        }
    }
    for (int b = 0; b < n; ++b) {
        rk[b][0] = code_of(lo[b]);
        rk[b][1] = code_of(hi[b]);
    }
    return n;
}

__device__ __forceinline__ unsigned long long range_key(const SortedArgs& a, const double p[3]) {
    double lo[3], ext[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        lo[k] = from_ord(~__ldg(&a.hdr->smin[k]));
        ext[k] = __dsub_rn(from_ord(__ldg(&a.hdr->smax[k])), lo[k]);
    }
    if (a.key_mode == 0) {
        const double e = fmax(fmax(ext[0], ext[1]), ext[2]);
        ext[0] = ext[1] = ext[2] = e;
    }
    const double gmax = (double)((1u << kIsoBits) - 1u);
    unsigned long long code = 0;
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        const unsigned q = ext[k] > 0.0 ? quant1(p[k], lo[k], ext[k], gmax) : 0u;
        code |= split21(q) << k;
    }
    return code;
}

// First index i with codes[i] > key (upper) or >= key (lower), by warp 0:
// two rounds over the sample table, then the stride window.
__device__ __forceinline__ int warp_bound(const SortedArgs& a, unsigned long long key, bool upper) {
    const int lane = threadIdx.x & 31;
    const int n = a.n_int + 1, m = a.n_samples, st = a.sample_stride;
    auto before = [&](unsigned long long c) { return upper ? c <= key : c < key; };
    // sample index of the last sample "before" key (-1 if none)
    const int step = (m + 31) / 32;
    int j = lane * step;
    bool b = j < m && before(__ldg(a.code_samples + j));
    unsigned mk = __ballot_sync(kFullMask, b);
    int s0 = mk ? (31 - __clz(mk)) * step : -1;
    if (s0 >= 0) {
        j = s0 + lane;
        b = lane < step && j < m && before(__ldg(a.code_samples + j));
        mk = __ballot_sync(kFullMask, b);
        s0 += 31 - __clz(mk);
    }
    // window of codes after sample s0 (codes[s0*st] is "before" key)
    int base = s0 < 0 ? 0 : s0 * st;
    const int lim = s0 < 0 ? 0 : ((s0 + 1) * st < n ? (s0 + 1) * st : n);
    for (; base < lim; base += 32) {
        j = base + lane;
        b = j < lim && before(__ldg(a.codes + j));
        mk = __ballot_sync(kFullMask, b);
        if (mk != kFullMask) return base + __popc(mk);
    }
    return lim;
}

template <int MODE, bool WIDE>
__global__ void __launch_bounds__(kTileThreads, kTileMinBlocks) k_trav_tile(SortedArgs a) {
    __shared__ TileSmem sm;
    const unsigned n_live = *a.n_live;
    const int n_int = a.n_int;
    const int root = __ldg(&a.hdr->root);
    const RsSlot* const nodes = reinterpret_cast<const RsSlot*>(a.nodes);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    // tile size: about a.tile_area triangles' worth of records, but at least
    // a.tile_balance tiles per CTA; a multiple of the CTA size
    unsigned T = (unsigned)((unsigned long long)a.tile_area * n_live / (unsigned)(n_int + 1));
    const unsigned per = a.tile_balance * gridDim.x;
    const unsigned bal = (n_live + per - 1) / per;
    T = T < bal ? T : bal;
    if (a.tile_depth) {
        // stacked surfaces: the candidate lists grow with the depth
        // complexity (projected triangle-box area over the root box's), so
        // the tile shrinks with it
        float r[3];
#pragma unroll
        for (int k = 0; k < 3; ++k)
            r[k] = from_ord32(__ldg(&a.hdr->bmax[k])) - from_ord32(~__ldg(&a.hdr->bmin[k]));
        const float ra = r[0] * r[1] + r[1] * r[2] + r[2] * r[0];
        const float depth = ra > 0.f ? __ldg(&a.hdr->parea) / ra : 0.f;
        if (depth > 1.f) {
            // cap = tile_depth / depth^1.5 (sweeps: C4, depth 12.8, best at
            // 256-record tiles; C5, depth 3.4, at ~2048; C2's 512 uncapped)
            const float cap = (float)a.tile_depth / (depth * sqrtf(depth));
            T = (float)T < cap ? T : (unsigned)cap;
        }
    }
    T = (T + kTileThreads - 1) / kTileThreads * kTileThreads;
    T = T < kTileThreads ? kTileThreads : (T > 16384 ? 16384 : T);
    const unsigned n_tiles = (n_live + T - 1) / T;
    build_cut(sm, nodes, n_int, root);
    if (tid == 0) sm.tile = atomicAdd(reinterpret_cast<unsigned*>(&a.status->tile_counter), 1u);
    __syncthreads();
    const int ncut = sm.ncut;
    for (;;) {
        const unsigned tile = sm.tile;
        if (tile >= n_tiles) break;
        const unsigned beg = tile * T;
        const unsigned end = beg + T < n_live ? beg + T : n_live;
        // 1. union box U of the tile's segment boxes
        float u[6] = {INFINITY, -INFINITY, INFINITY, -INFINITY, INFINITY, -INFINITY};
        for (unsigned idx = beg + tid; idx < end; idx += kTileThreads) {
            float4 r0, r1;
        get_rec(a, idx, r0, r1);
            u[0] = fminf(u[0], fminf(r0.x, r1.x)); u[1] = fmaxf(u[1], fmaxf(r0.x, r1.x));
            u[2] = fminf(u[2], fminf(r0.y, r1.y)); u[3] = fmaxf(u[3], fmaxf(r0.y, r1.y));
            u[4] = fminf(u[4], fminf(r0.z, r1.z)); u[5] = fmaxf(u[5], fmaxf(r0.z, r1.z));
        }
#pragma unroll
        for (int k = 0; k < 6; k += 2) {
            u[k] = wred_min(u[k]);
            u[k + 1] = wred_max(u[k + 1]);
        }
        if (lane == 0) {
#pragma unroll
            for (int k = 0; k < 6; ++k) sm.part[warp][k] = u[k];
        }
        if (tid == 0) {
            sm.nf[0] = 0; sm.nf[1] = 0; sm.nf[2] = 0;
            sm.nl = 0;
            sm.ovf = 0;
        }
        __syncthreads();
#pragma unroll
        for (int w = 0; w < kTileThreads / 32; ++w)
#pragma unroll
            for (int k = 0; k < 6; k += 2) {
                if (w == 0) { u[k] = sm.part[0][k]; u[k + 1] = sm.part[0][k + 1]; }
                else { u[k] = fminf(u[k], sm.part[w][k]); u[k + 1] = fmaxf(u[k + 1], sm.part[w][k + 1]); }
            }
        // 2a. the Morton-range list when the runs of candidate keys are short
        bool ranged = false;
        if (a.codes) {
            if (tid == 0) {
                double plo[3], phi[3];
#pragma unroll
                for (int k = 0; k < 3; ++k) {
                    const double sz = (double)__uint_as_float(__ldg(&a.hdr->tsize[k]));
                    const double l = (double)u[2 * k], h = (double)u[2 * k + 1];
                    plo[k] = l - sz - 1e-9 * (fabs(l) + sz + 1.0);
                    phi[k] = h + sz + 1e-9 * (fabs(h) + sz + 1.0);
                }
                unsigned ql[3], qh[3];
                range_q(a, plo, ql);
                range_q(a, phi, qh);
                sm.nr = range_split(ql, qh, sm.rk);
            }
            __syncthreads();
            const int nr = sm.nr;
            // one bound per warp: 2 * nr searches over the four warps
            for (int t = warp; t < 2 * nr; t += kTileThreads / 32) {
                const int r = t >> 1, hi = t & 1;
                const int i = warp_bound(a, sm.rk[r][hi], hi != 0);
                if (lane == 0) sm.rr[r][hi] = i;
            }
            __syncthreads();
            int total = 0;
            for (int r = 0; r < nr; ++r) total += sm.rr[r][1] - sm.rr[r][0];
            if (total <= (int)a.range_max) {
                ranged = true;
                for (int r = 0; r < nr; ++r) {
                    const int i0 = sm.rr[r][0], i1 = sm.rr[r][1];
                    for (int i = i0 + tid; i < i1; i += kTileThreads) {
                        const float2* lb = reinterpret_cast<const float2*>(a.leaf_boxes + 6ll * i);
                        const float2 x = __ldg(lb), y = __ldg(lb + 1), z = __ldg(lb + 2);
                        const float4 xy = make_float4(x.x, x.y, y.x, y.y);
                        if (box_ov(u, xy, z)) {
                            const int k = atomicAdd(&sm.nl, 1);
                            if (k < kTileLCap) {
                                sm.lxy[k] = xy;
                                sm.lz[k] = z;
                                sm.lid[k] = i;
                            } else {
                                sm.ovf = 1;
                            }
                        }
                    }
                }
                __syncthreads();
            }
        }
        // 2b. otherwise the breadth-first walk with U, from the cut
        if (!ranged) {
        for (int ci = tid; ci < ncut; ci += kTileThreads) {
            const int ref = sm.cref[ci];
            if (box_ov(u, sm.cxy[ci], sm.cz[ci])) {
                if (ref >= n_int) {
                    const int k = atomicAdd(&sm.nl, 1);
                    sm.lxy[k] = sm.cxy[ci];
                    sm.lz[k] = sm.cz[ci];
                    sm.lid[k] = ref - n_int;
                } else {
                    sm.front[0][atomicAdd(&sm.nf[0], 1)] = ref;
                }
            }
        }
        __syncthreads();
        for (int level = 0;; ++level) {
            const int n = sm.nf[level % 3];
            if (n == 0 || sm.ovf) break;
            const int* cur = sm.front[level & 1];
            int* nxt = sm.front[(level + 1) & 1];
            int* nnf = &sm.nf[(level + 1) % 3];
            if (tid == 0) sm.nf[(level + 2) % 3] = 0;
            // a child overlapping U: leaves join L, internal nodes the next level
            auto take = [&](float x0, float x1, float y0, float y1, float z0, float z1, int ref) {
                if (ref >= n_int) {
                    const int k = atomicAdd(&sm.nl, 1);
                    if (k < kTileLCap) {
                        sm.lxy[k] = make_float4(x0, x1, y0, y1);
                        sm.lz[k] = make_float2(z0, z1);
                        sm.lid[k] = ref - n_int;
                    } else {
                        sm.ovf = 1;
                    }
                } else {
                    const int k = atomicAdd(nnf, 1);
                    if (k < kTileFCap) nxt[k] = ref;
                    else sm.ovf = 1;
                }
            };
            for (int i = tid; i < n; i += kTileThreads) {
                const int node = cur[i];
                if (WIDE) {  // collapsed 4-wide node: one 32-B slot per child
                    const float4* slot = reinterpret_cast<const float4*>(a.nodes4 + node);
#pragma unroll
                    for (int j = 0; j < 4; ++j) {
                        const float4 p = __ldg(slot + 2 * j), q = __ldg(slot + 2 * j + 1);
                        const int ref = __float_as_int(q.z);
                        if ((ref >= 0) & (u[0] <= p.y) & (u[1] >= p.x) & (u[2] <= p.w) & (u[3] >= p.z) &
                            (u[4] <= q.y) & (u[5] >= q.x))
                            take(p.x, p.y, p.z, p.w, q.x, q.y, ref);
                    }
                } else {
                    float f0[8], f1[8];
                    ld_slot(nodes + 2 * node, f0);
                    ld_slot(nodes + 2 * node + 1, f1);
                    const int ca = __float_as_int(f1[4]), cb = __float_as_int(f1[5]);
                    if ((u[0] <= f0[1]) & (u[1] >= f0[0]) & (u[2] <= f0[3]) & (u[3] >= f0[2]) &
                        (u[4] <= f0[5]) & (u[5] >= f0[4]))
                        take(f0[0], f0[1], f0[2], f0[3], f0[4], f0[5], ca);
                    if ((u[0] <= f0[7]) & (u[1] >= f0[6]) & (u[2] <= f1[1]) & (u[3] >= f1[0]) &
                        (u[4] <= f1[3]) & (u[5] >= f1[2]))
                        take(f0[6], f0[7], f1[0], f1[1], f1[2], f1[3], cb);
                }
            }
            __syncthreads();
        }
        }
        const bool fallback = sm.ovf != 0;
        const int nl = sm.nl;
#ifdef RS_TILE_STATS
        if (tid == 0) {
            atomicAdd(&a.status->visits, (unsigned long long)nl);
            if (fallback) atomicAdd(&a.status->cand_count, 1ull);
        }
#endif
        // 3. segments, one warp per 32 consecutive records
        for (unsigned base = beg + warp * 32; base < end; base += kTileThreads) {
            const unsigned idx = base + lane;
            const bool valid = idx < end;
            float4 r0 = make_float4(0.f, 0.f, 0.f, 0.f), r1 = r0;
            if (valid) get_rec_last(a, idx, r0, r1);
            int det = 0, nh = 0, btri = -1;
            double bt = 0.0;
            if (fallback) {
                if (valid) trav_one_call<MODE, WIDE>(a, nodes, root, r0, r1, det, nh, btri, bt);
            } else {
                process_chunk<MODE>(a, r0, r1, valid, sm.lxy, sm.lz, sm.lid, nl, sm.wc[warp], sm.slot[warp],
                                    det, nh, btri, bt);
            }
            if (valid) write_result<MODE>(a, __float_as_int(r0.w), det, nh, btri, bt);
        }
        __syncthreads();  // the next tile reuses the shared lists
        if (tid == 0) sm.tile = atomicAdd(reinterpret_cast<unsigned*>(&a.status->tile_counter), 1u);
        __syncthreads();
    }
}

// ------------------------------------------------------------ host glue ---

size_t sorted_bins() { return kBins; }

static int sm_total() { return device_sms(); }

bool sorted_wide() {
    static const bool wide = [] {
        const char* e = getenv("RS_SORTED_WIDE");
        return e && e[0] == '1';
    }();
    return wide;
}

// Tuning knobs of the sorted path (rs_set_option; initial values from the
// environment).  trav: 0 auto (tile when dense enough), 1 per-thread binary,
// 2 per-thread 4-wide, 3 tile always.
struct SortedOpts {
    int trav = 0;
    unsigned tile_density = 16;  // auto: tiles when segments >= this x triangles
    unsigned tile_balance = 8;   // at least this many tiles per CTA
    unsigned tile_area = 48;     // about this many triangles' worth of records per tile
    unsigned tile_depth = 11000; // and at most this / depth-complexity^1.5 records (0: off)
    unsigned bin_occ = 16;       // target live segments per spatial bin
    int bin_tma = 1;             // binning passes stream through TMA bulk copies
    int tile_wide = 0;           // tile walk over the collapsed 4-wide nodes (A/B: no gain on C2)
    int fast_keys = 0;           // fast-tree key grid: 0 isotropic, 1 per-axis, 2 auto
    unsigned range_max = 4096;   // tile lists from a Morton key range of at most this many leaves (0: walk only)
    int geom = 1;                // 1: bin geometry derived once by k_seg_sample (A/B round 2: C2 -9 us, C3 -2.5 us)
    int fast_path = 0;           // 0 binned tiles, 1 collision buffer (rs_trav.cu)
    long long cand_cap = 0;      // collision buffer: initial capacity (0: 2 x segments + 4096)
};
static SortedOpts& opts() {
    static SortedOpts o = [] {
        SortedOpts d;
        auto num = [](const char* name, long long def) {
            const char* e = getenv(name);
            return e && *e ? atoll(e) : def;
        };
        const char* t = getenv("RS_TRAV");
        if (t && t[0] == 'b') d.trav = 1;
        else if ((t && t[0] == 'w') || sorted_wide()) d.trav = 2;
        else if (t && t[0] == 't') d.trav = 3;
        d.tile_density = (unsigned)num("RS_TILE_DENSITY", d.tile_density);
        d.tile_balance = (unsigned)num("RS_TILE_BALANCE", d.tile_balance);
        d.tile_area = (unsigned)num("RS_TILE_AREA", d.tile_area);
        d.tile_depth = (unsigned)num("RS_TILE_DEPTH", d.tile_depth);
        d.bin_occ = (unsigned)num("RS_BIN_OCC", d.bin_occ);
        d.bin_tma = (int)num("RS_BIN_TMA", d.bin_tma);
        d.tile_wide = (int)num("RS_TILE_WIDE", d.tile_wide);
        d.fast_keys = (int)num("RS_FAST_KEYS", d.fast_keys);
        d.range_max = (unsigned)num("RS_RANGE_MAX", d.range_max);
        d.geom = (int)num("RS_GEOM", d.geom);
        const char* fp = getenv("RS_FAST_PATH");
        if (fp && fp[0] == 'b') d.fast_path = 1;
        d.cand_cap = num("RS_CAND_CAP", d.cand_cap);
        return d;
    }();
    return o;
}

int sorted_option(const char* name, long long value, long long* old) {
    SortedOpts& o = opts();
    long long prev;
    if (!strcmp(name, "trav")) { prev = o.trav; if (value >= 0) o.trav = (int)value; }
    else if (!strcmp(name, "tile_density")) { prev = o.tile_density; if (value >= 0) o.tile_density = (unsigned)value; }
    else if (!strcmp(name, "tile_balance")) { prev = o.tile_balance; if (value > 0) o.tile_balance = (unsigned)value; }
    else if (!strcmp(name, "tile_area")) { prev = o.tile_area; if (value > 0) o.tile_area = (unsigned)value; }
    else if (!strcmp(name, "tile_depth")) { prev = o.tile_depth; if (value >= 0) o.tile_depth = (unsigned)value; }
    else if (!strcmp(name, "bin_occupancy")) { prev = o.bin_occ; if (value > 0) o.bin_occ = (unsigned)value; }
    else if (!strcmp(name, "bin_tma")) { prev = o.bin_tma; if (value >= 0) o.bin_tma = (int)value; }
    else if (!strcmp(name, "tile_wide")) { prev = o.tile_wide; if (value >= 0) o.tile_wide = (int)value; }
    else if (!strcmp(name, "range_max")) { prev = o.range_max; if (value >= 0) o.range_max = (unsigned)value; }
    else if (!strcmp(name, "fast_keys")) { prev = o.fast_keys; if (value >= 0 && value <= 2) o.fast_keys = (int)value; }
    else if (!strcmp(name, "geom")) { prev = o.geom; if (value >= 0) o.geom = value ? 1 : 0; }
    else if (!strcmp(name, "fast_path")) { prev = o.fast_path; if (value >= 0 && value <= 1) o.fast_path = (int)value; }
    else if (!strcmp(name, "cand_cap")) { prev = o.cand_cap; if (value >= 0) o.cand_cap = value; }
    else return -1;
    if (old) *old = prev;
    return 0;
}

static int trav_variant() { return opts().trav; }
int fast_key_mode() { return opts().fast_keys; }
int fast_path() { return opts().fast_path; }
long long cand_cap_override() { return opts().cand_cap; }
static unsigned tile_min_density() { return opts().tile_density; }
static unsigned tile_balance() { return opts().tile_balance; }
static unsigned bin_occupancy() { return opts().bin_occ; }
static unsigned tile_area() { return opts().tile_area; }

bool binning_zeroes_flags(const float* starts, const float* ends, long long n_r, const int* flags) {
    const uintptr_t al = reinterpret_cast<uintptr_t>(starts) | reinterpret_cast<uintptr_t>(ends) |
                         reinterpret_cast<uintptr_t>(flags);
    return flags && (al & 15) == 0 && opts().bin_tma && n_r >= kStreamSegs;
}

__global__ void __launch_bounds__(256) k_expand_bits(int* __restrict__ flags, const unsigned* __restrict__ bits,
                                                    long long n) {
    // one thread per 4 flags (one 16-B store; consecutive threads write
    // consecutive 16 B), 8 threads share a bitmap word
    const long long n4 = n / 4;
    const bool vec = (reinterpret_cast<uintptr_t>(flags) & 15) == 0;
    for (long long j = blockIdx.x * 256ll + threadIdx.x; j < n4; j += gridDim.x * 256ll) {
        const unsigned b = __ldg(bits + (j >> 3)) >> (4 * (j & 7));
        const int4 v = make_int4(b & 1, (b >> 1) & 1, (b >> 2) & 1, (b >> 3) & 1);
        if (vec) {
            reinterpret_cast<int4*>(flags)[j] = v;
        } else {
            flags[4 * j] = v.x; flags[4 * j + 1] = v.y; flags[4 * j + 2] = v.z; flags[4 * j + 3] = v.w;
        }
    }
    if (blockIdx.x == 0 && threadIdx.x < (unsigned)(n - 4 * n4)) {
        const long long i = 4 * n4 + threadIdx.x;
        flags[i] = (__ldg(bits + (i >> 5)) >> (i & 31)) & 1;
    }
}

// bits[w] bit j = (flags[32 w + j] != 0): one ballot per warp over 32
// consecutive flags (128 coalesced bytes in, 4 out)
__global__ void __launch_bounds__(256) k_pack_flags(const int* __restrict__ flags, long long n,
                                                   unsigned* __restrict__ bits) {
    const long long words = (n + 31) / 32;
    const int lane = threadIdx.x & 31;
    for (long long w = (blockIdx.x * 256ll + threadIdx.x) >> 5; w < words; w += (gridDim.x * 256ll) >> 5) {
        const long long i = 32 * w + lane;
        const unsigned b = __ballot_sync(kFullMask, i < n && __ldg(flags + i) != 0);
        if (lane == 0) bits[w] = b;
    }
}

void launch_pack_flags(const int* flags, long long n, unsigned* bits, cudaStream_t s) {
    if (n <= 0) return;
    const long long want = ((n + 31) / 32 * 32 + 255) / 256;
    const long long cap = (long long)sm_total() * 8;
    count_launches(1);
    k_pack_flags<<<(unsigned)(want < cap ? want : cap), 256, 0, s>>>(flags, n, bits);
}

void launch_expand_bits(int* flags, const unsigned* hitbits, long long n, cudaStream_t s) {
    if (n <= 0) return;
    const long long want = (n / 4 + 255) / 256 + 1;
    const long long cap = (long long)sm_total() * 8;
    count_launches(1);
    k_expand_bits<<<(unsigned)(want < cap ? want : cap), 256, 0, s>>>(flags, hitbits, n);
}

void launch_binning(const SortedArgs& a0, cudaStream_t s, bool zero_flags) {
    SortedArgs a = a0;
    a.zero_flags = zero_flags && !a.hitbits && binning_zeroes_flags(a.starts, a.ends, a.n_r, a.flags);
    a.geom_mode = opts().geom;
    a.bin_occupancy = bin_occupancy();
    if (a.n_r <= 0) return;
    count_launches(4);
    const int sms = sm_total();
    k_seg_sample<<<kSampleCtas, kSampleThreads, 0, s>>>(a);
    const bool vec = ((reinterpret_cast<uintptr_t>(a.starts) | reinterpret_cast<uintptr_t>(a.ends)) & 15) == 0;
    if (vec && opts().bin_tma && a.n_r >= kStreamSegs) {
        // histogram over TMA-streamed segments; the scatter with plain
        // loads and twice the warps (its cursor claims need the parallelism)
        ensure_dynamic_smem((const void*)k_bin_count_tma, (int)kStreamSmem);
        const long long chunks = a.n_r / kStreamSegs;
        const unsigned g = (unsigned)(chunks < sms * (long long)RS_STREAM_CTAS ? chunks : sms * (long long)RS_STREAM_CTAS);
        stage_mark(5, s);
        k_bin_count_tma<<<g, kStreamThreads, kStreamSmem, s>>>(a);
        stage_mark(6, s);
        k_bin_scan1<<<kScanTiles, 256, 0, s>>>(a);
        stage_mark(7, s);
        const long long want = (a.n_r + 1023) / 1024;
        const unsigned g2 = (unsigned)(want < sms * 16ll ? want : sms * 16ll);
        k_bin_scatter<true><<<g2, 256, 0, s>>>(a);
        stage_mark(8, s);
        return;
    }
    const long long want = (a.n_r + 1023) / 1024;
    const unsigned g = (unsigned)(want < sms * 16ll ? want : sms * 16ll);
    stage_mark(5, s);
    if (vec) k_bin_count<true><<<g, 256, 0, s>>>(a);
    else k_bin_count<false><<<g, 256, 0, s>>>(a);
    stage_mark(6, s);
    k_bin_scan1<<<kScanTiles, 256, 0, s>>>(a);
    stage_mark(7, s);
    if (vec) k_bin_scatter<true><<<g, 256, 0, s>>>(a);
    else k_bin_scatter<false><<<g, 256, 0, s>>>(a);
    stage_mark(8, s);
}

template <int MODE>
static void launch_tile(const SortedArgs& a, int sms, cudaStream_t s) {
    const bool wide = a.nodes4 != nullptr && opts().tile_wide;
    const int o = occupancy(wide ? (const void*)k_trav_tile<MODE, true> : (const void*)k_trav_tile<MODE, false>,
                            kTileThreads);
    if (wide) k_trav_tile<MODE, true><<<sms * o, kTileThreads, 0, s>>>(a);
    else k_trav_tile<MODE, false><<<sms * o, kTileThreads, 0, s>>>(a);
}

static const char* g_hot_name = "";
const char* hot_kernel_name() { return g_hot_name; }

static thread_local long long g_batch_rays = 0;
void set_batch_rays(long long n) { g_batch_rays = n; }

void launch_sorted_trav(const SortedArgs& a0, int mode, bool stats, cudaStream_t s) {
    if (a0.n_r <= 0) return;
    SortedArgs a = a0;
    a.tile_area = tile_area();
    a.tile_depth = opts().tile_depth;
    a.range_max = opts().range_max;
    if (!a.range_max) a.codes = nullptr;
    a.tile_min_density = tile_min_density();
    a.tile_balance = tile_balance();
    count_launches(1);
    const int sms = sm_total();
    int variant = trav_variant();
    // tiles pay off only with many segments per triangle (a tile's walk is
    // amortised over its records); a single triangle has no tree to walk
    // (a chunk of a streamed batch decides by the whole batch's density: the
    // same scene must not switch to the per-record walk because it arrives
    // in pieces)
    const long long n_density = a.n_r > g_batch_rays ? a.n_r : g_batch_rays;
    if (variant == 0)
        variant = n_density < (long long)a.tile_min_density * (a.n_int + 1) ? 1 : 3;
    if (a.n_int == 0) variant = 1;
    hot_kernel_mark(0, s);
    g_hot_name = variant == 3 ? "k_trav_tile" : variant == 1 ? "k_trav_sorted_bin" : "k_trav_sorted";
    if (variant == 3 && !stats) {
        if (mode == kBoolean) launch_tile<kBoolean>(a, sms, s);
        else if (mode == kCount) launch_tile<kCount>(a, sms, s);
        else launch_tile<kBarycentric>(a, sms, s);
        hot_kernel_mark(1, s);
        return;
    }
    const int o = occupancy(mode == kBoolean ? (const void*)k_trav_sorted<kBoolean, false>
                            : mode == kCount ? (const void*)k_trav_sorted<kCount, false>
                                             : (const void*)k_trav_sorted<kBarycentric, false>,
                            kSortedThreads);
    const long long wt = (a.n_r + kSortedThreads - 1) / kSortedThreads;
    const unsigned gt = (unsigned)(wt < (long long)sms * o ? wt : (long long)sms * o);
    if (variant == 1 && !stats) {
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
