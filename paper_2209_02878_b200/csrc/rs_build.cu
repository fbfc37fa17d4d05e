// rs_build.cu -- device BVH construction for sm_100a.
//
//   k_prep      per triangle: f64 centroid (morton.py:34-37), grid-wide
//               support min/max (morton.py:40-45) via ordered-u64 atomics after
//               a block reduction, the root box (union of triangle boxes, for
//               the query's binning), and the reference's _reset_tree of
//               internal slot j (lbvh.py:175-195).
//   k_keys      per triangle: quantise (morton.py:48-63 or the isotropic fast
//               grid) and interleave (morton.py:117-128) -> (code, index).
//   onesweep    stable LSD radix sort, 8-bit digits, one kernel per pass with
//               decoupled look-back (== np.lexsort((idx, code)), morton.py:131-146).
//   k_climb     Apetrei single-pass climb (lbvh.py:198-233, _core.pyx:148-184):
//               write child/range, release fence, acq_rel visit counter; the
//               second arriver unions the children and also emits the packed
//               64-B RsNode the traversal reads.  k_climb_lean: the same climb
//               for query-only fast trees, writing only the RsNode records.
#include <cuda/atomic>

#include "rs_common.cuh"
#include "rs_internal.h"

namespace rs {

// ------------------------------------------------------------------ prep ---

__device__ __forceinline__ double warp_min(double v) {
    for (int o = 16; o; o >>= 1) v = fmin(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}
__device__ __forceinline__ double warp_max(double v) {
    for (int o = 16; o; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}

__global__ void __launch_bounds__(256) k_prep(const float* __restrict__ V,
                                              const int* __restrict__ T, int n, double* cent,
                                              RsHeader* hdr, TreeArrays ta, int do_centroids,
                                              int lean) {
    __shared__ double red[8][6];
    __shared__ float fred[8][6];
    __shared__ float sred[8][3];
    double lo[3] = {INFINITY, INFINITY, INFINITY}, hi[3] = {-INFINITY, -INFINITY, -INFINITY};
    float blo[3] = {INFINITY, INFINITY, INFINITY}, bhi[3] = {-INFINITY, -INFINITY, -INFINITY};
    float tsz[3] = {0.f, 0.f, 0.f};
    float parea = 0.f;  // depth complexity numerator (tile sizing only; order-free use)
    for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < n; j += gridDim.x * blockDim.x) {
        // _reset_tree (lbvh.py:181-189) for internal slot j; a lean build
        // (query-only tree, never downloaded) keeps just the visit counters
        if (!lean) {
            reinterpret_cast<float2*>(ta.int_bounds + 6ll * j)[0] = make_float2(0.f, 0.f);
            reinterpret_cast<float2*>(ta.int_bounds + 6ll * j)[1] = make_float2(0.f, 0.f);
            reinterpret_cast<float2*>(ta.int_bounds + 6ll * j)[2] = make_float2(0.f, 0.f);
            ta.child_l[j] = kEmpty;
            ta.child_r[j] = kEmpty;
            ta.range_l[j] = -1;
            ta.range_r[j] = -1;
            ta.int_tri[j] = -1;
        }
        ta.visit[j] = 0;
        const int ia = T[3ll * j], ib = T[3ll * j + 1], ic = T[3ll * j + 2];
        float dside[3];
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            const float fa = V[3ll * ia + k], fb = V[3ll * ib + k], fc = V[3ll * ic + k];
            const float tl = fminf(fminf(fa, fb), fc), th = fmaxf(fmaxf(fa, fb), fc);
            blo[k] = fminf(blo[k], tl);  // root box = union of triangle boxes
            bhi[k] = fmaxf(bhi[k], th);
            tsz[k] = fmaxf(tsz[k], th - tl);
            dside[k] = th - tl;
            if (do_centroids) {
                const double m = __ddiv_rn(__dadd_rn(__dadd_rn((double)fa, (double)fb), (double)fc), 3.0);
                cent[3ll * j + k] = m;
                lo[k] = fmin(lo[k], m);
                hi[k] = fmax(hi[k], m);
            }
        }
        parea += dside[0] * dside[1] + dside[1] * dside[2] + dside[2] * dside[0];
    }
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    for (int o = 16; o; o >>= 1) parea += __shfl_xor_sync(0xffffffffu, parea, o);
    __shared__ float pred[32];
    if (l == 0) pred[w] = parea;
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        lo[k] = warp_min(lo[k]);
        hi[k] = warp_max(hi[k]);
        for (int o = 16; o; o >>= 1) {
            blo[k] = fminf(blo[k], __shfl_xor_sync(0xffffffffu, blo[k], o));
            bhi[k] = fmaxf(bhi[k], __shfl_xor_sync(0xffffffffu, bhi[k], o));
            tsz[k] = fmaxf(tsz[k], __shfl_xor_sync(0xffffffffu, tsz[k], o));
        }
    }
    if (l == 0)
        for (int k = 0; k < 3; ++k) {
            red[w][k] = lo[k];
            red[w][3 + k] = hi[k];
            fred[w][k] = blo[k];
            fred[w][3 + k] = bhi[k];
            sred[w][k] = tsz[k];
        }
    __syncthreads();
    if (threadIdx.x < 3) {
        float v = 0.f;
        for (int i = 0; i < (int)(blockDim.x >> 5); ++i) v = fmaxf(v, sred[i][threadIdx.x]);
        if (v > 0.f) atomicMax(&hdr->tsize[threadIdx.x], __float_as_uint(v));
    }
    if (threadIdx.x == 32) {  // one float atomic per CTA (tile sizing only: order-free)
        float v = 0.f;
        for (int i = 0; i < (int)(blockDim.x >> 5); ++i) v += pred[i];
        if (v > 0.f) atomicAdd(&hdr->parea, v);
    }
    if (threadIdx.x < 6) {
        const int k = threadIdx.x;
        double v = red[0][k];
        float fv = fred[0][k];
        for (int i = 1; i < (int)(blockDim.x >> 5); ++i) {
            v = k < 3 ? fmin(v, red[i][k]) : fmax(v, red[i][k]);
            fv = k < 3 ? fminf(fv, fred[i][k]) : fmaxf(fv, fred[i][k]);
        }
        if (do_centroids && isfinite(v)) {
            if (k < 3)
                atomicMax(&hdr->smin[k], ~ord_of(v));
            else
                atomicMax(&hdr->smax[k - 3], ord_of(v));
        }
        if (isfinite(fv)) {
            if (k < 3)
                atomicMax(&hdr->bmin[k], ~ord32(fv));
            else
                atomicMax(&hdr->bmax[k - 3], ord32(fv));
        }
    }
}

// ------------------------------------------------------------------ keys ---

__global__ void __launch_bounds__(256) k_keys(const double* __restrict__ cent, int n,
                                              const RsHeader* __restrict__ hdr, int kind,
                                              unsigned long long* keys, int* vals, int fast_mode) {
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= n) return;
    double lo[3], ext[3], gmax;
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        lo[k] = from_ord(~hdr->smin[k]);
        ext[k] = __dsub_rn(from_ord(hdr->smax[k]), lo[k]);
    }
    if (kind == kTreeFast) {
        // 30-bit keys.  Isotropic grid (one extent for every axis) for flat
        // meshes: a thin terrain's z splits would come early and prune
        // nothing for segments crossing it.  Per-axis grid (fast_mode 1, or
        // auto when the thinnest centroid extent is at least a fifth of the
        // widest): stacked surfaces separate near the root, so segments in
        // the empty space between them are culled in a few levels.
        const double emax = fmax(fmax(ext[0], ext[1]), ext[2]);
        const double emin = fmin(fmin(ext[0], ext[1]), ext[2]);
        const bool per_axis = fast_mode == 1 || (fast_mode == 2 && emin >= 0.2 * emax);
        if (!per_axis) ext[0] = ext[1] = ext[2] = emax;
        gmax = (double)((1u << kIsoBits) - 1u);
    } else {
        gmax = kGridMax21;
    }
    unsigned long long code = 0;
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        const unsigned q = ext[k] > 0.0 ? quant1(cent[3ll * j + k], lo[k], ext[k], gmax) : 0u;
        code |= split21(q) << k;
    }
    keys[j] = code;
    vals[j] = j;
}

// -------------------------------------------------- segment Morton order ---
// sort_segments_by_morton (engine.py:125-147): f64 midpoints (s + e) / 2,
// their support, the reference's per-axis 21-bit quantisation and 63-bit
// interleave (k_keys, reference kind), a stable sort by (code, index).

__global__ void __launch_bounds__(256) k_mid_prep(const float* __restrict__ S,
                                                  const float* __restrict__ E, int n, double* mid,
                                                  RsHeader* hdr) {
    __shared__ double red[8][6];
    double lo[3] = {INFINITY, INFINITY, INFINITY}, hi[3] = {-INFINITY, -INFINITY, -INFINITY};
    for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < n; j += gridDim.x * blockDim.x) {
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            const double m = __ddiv_rn(__dadd_rn((double)S[3ll * j + k], (double)E[3ll * j + k]), 2.0);
            mid[3ll * j + k] = m;
            lo[k] = fmin(lo[k], m);
            hi[k] = fmax(hi[k], m);
        }
    }
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        lo[k] = warp_min(lo[k]);
        hi[k] = warp_max(hi[k]);
    }
    if (l == 0)
        for (int k = 0; k < 3; ++k) {
            red[w][k] = lo[k];
            red[w][3 + k] = hi[k];
        }
    __syncthreads();
    if (threadIdx.x < 6) {
        const int k = threadIdx.x;
        double v = red[0][k];
        for (int i = 1; i < (int)(blockDim.x >> 5); ++i) v = k < 3 ? fmin(v, red[i][k]) : fmax(v, red[i][k]);
        if (isfinite(v)) {
            if (k < 3) atomicMax(&hdr->smin[k], ~ord_of(v));
            else atomicMax(&hdr->smax[k - 3], ord_of(v));
        }
    }
}

__global__ void __launch_bounds__(256) k_gather_segments(const int* __restrict__ order,
                                                         const float* __restrict__ S,
                                                         const float* __restrict__ E, int n,
                                                         float* So, float* Eo, long long* perm) {
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= n) return;
    const int i = order[j];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        So[3ll * j + k] = S[3ll * i + k];
        Eo[3ll * j + k] = E[3ll * i + k];
    }
    perm[j] = i;
}

// ------------------------------------------------------------ radix sort ---

constexpr int kSortThreads = 256;
constexpr int kSortItems = 8;
constexpr int kSortTile = kSortThreads * kSortItems;  // 2048 keys per tile
constexpr int kSortWarps = kSortThreads / 32;

__global__ void __launch_bounds__(256) k_sort_hist(const unsigned long long* __restrict__ keys,
                                                   int n, int passes, unsigned* ghist) {
    __shared__ unsigned h[8][256];
    for (int i = threadIdx.x; i < 8 * 256; i += blockDim.x) (&h[0][0])[i] = 0;
    __syncthreads();
    for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < n; j += gridDim.x * blockDim.x) {
        const unsigned long long k = keys[j];
        for (int p = 0; p < passes; ++p) atomicAdd(&h[p][(k >> (8 * p)) & 255u], 1u);
    }
    __syncthreads();
    for (int i = threadIdx.x; i < passes * 256; i += blockDim.x) {
        const unsigned v = (&h[0][0])[i];
        if (v) atomicAdd(&ghist[i], v);
    }
}

// Onesweep pass: status words are (flag << 62 | count), flag 1 = tile
// aggregate, 2 = inclusive prefix over tiles <= this one.
__global__ void __launch_bounds__(kSortThreads) k_onesweep(
    const unsigned long long* __restrict__ kin, const int* __restrict__ vin,
    unsigned long long* __restrict__ kout, int* __restrict__ vout, int n, int shift,
    const unsigned* __restrict__ ghist, unsigned long long* status, unsigned* tile_counter) {
    __shared__ unsigned warp_cnt[kSortWarps][256];
    __shared__ unsigned long long gbase[256];
    __shared__ unsigned wsum[kSortWarps];
    __shared__ int s_tile;
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    // exclusive scan of this pass's global digit histogram (digit = thread)
    unsigned dig_excl;
    {
        const unsigned hv = ghist[threadIdx.x];
        unsigned x = hv;
        for (int o = 1; o < 32; o <<= 1) {
            const unsigned y = __shfl_up_sync(0xffffffffu, x, o);
            if (l >= o) x += y;
        }
        if (l == 31) wsum[w] = x;
        __syncthreads();
        unsigned before = 0;
        for (int i = 0; i < w; ++i) before += wsum[i];
        dig_excl = before + x - hv;
    }
    for (int i = threadIdx.x; i < kSortWarps * 256; i += blockDim.x) (&warp_cnt[0][0])[i] = 0;
    if (threadIdx.x == 0) s_tile = (int)atomicAdd(tile_counter, 1u);
    __syncthreads();
    const int tile = s_tile;
    const long long base = (long long)tile * kSortTile + (long long)w * 32 * kSortItems;

    unsigned long long key[kSortItems];
    int val[kSortItems];
    unsigned rank[kSortItems];
    int dig[kSortItems];
#pragma unroll
    for (int k = 0; k < kSortItems; ++k) {
        const long long idx = base + k * 32 + l;
        const bool ok = idx < n;
        key[k] = ok ? kin[idx] : 0ull;
        val[k] = ok ? vin[idx] : 0;
        dig[k] = ok ? (int)((key[k] >> shift) & 255u) : -1;
    }
    const unsigned lt = (1u << l) - 1u;
#pragma unroll
    for (int k = 0; k < kSortItems; ++k) {
        const int d = dig[k];
        const unsigned peers = __match_any_sync(0xffffffffu, d);
        unsigned r = 0;
        if (d >= 0) r = warp_cnt[w][d] + __popc(peers & lt);
        __syncwarp();
        if (d >= 0 && (peers & lt) == 0) warp_cnt[w][d] += __popc(peers);
        __syncwarp();
        rank[k] = r;
    }
    __syncthreads();
    // per digit: scan across warps, publish tile count, look back.
    const int d = threadIdx.x;  // kSortThreads == 256 == radix
    unsigned tot = 0;
#pragma unroll
    for (int i = 0; i < kSortWarps; ++i) {
        const unsigned c = warp_cnt[i][d];
        warp_cnt[i][d] = tot;
        tot += c;
    }
    {
        cuda::atomic_ref<unsigned long long, cuda::thread_scope_device> me(
            status[(long long)tile * 256 + d]);
        unsigned long long excl = 0;
        if (tile == 0) {
            me.store((2ull << 62) | tot, cuda::memory_order_release);
        } else {
            me.store((1ull << 62) | tot, cuda::memory_order_release);
            // look back 8 predecessors per round (independent loads in
            // flight), summing aggregates until an inclusive prefix
            constexpr int kLB = 8;
            for (int j = tile - 1; j >= 0;) {
                unsigned long long v[kLB];
#pragma unroll
                for (int k = 0; k < kLB; ++k)
                    v[k] = j - k >= 0 ? reinterpret_cast<volatile unsigned long long*>(status)[(long long)(j - k) * 256 + d]
                                      : (2ull << 62);
                int k = 0;
                bool done = false;
                for (; k < kLB; ++k) {
                    const unsigned flag = (unsigned)(v[k] >> 62);
                    if (flag == 0) break;  // not published yet: re-read from here
                    excl += v[k] & ((1ull << 62) - 1);
                    if (flag == 2) { done = true; break; }
                }
                if (done) break;
                j -= k;
            }
            __threadfence();
            me.store((2ull << 62) | (excl + tot), cuda::memory_order_release);
        }
        // exclusive global digit base: keys with smaller digits + tiles before us
        gbase[d] = (unsigned long long)dig_excl + excl;
    }
    // local reorder: stage the tile's keys in digit order in shared memory,
    // then write each digit's run out contiguously (coalesced stores instead
    // of one scattered 8-B + 4-B store per key)
    __shared__ unsigned dig_local[256];
    __shared__ unsigned long long s_key[kSortTile];
    __shared__ int s_val[kSortTile];
    {
        // exclusive scan over digits of the tile's per-digit totals
        unsigned x = tot;
        for (int o = 1; o < 32; o <<= 1) {
            const unsigned y = __shfl_up_sync(0xffffffffu, x, o);
            if (l >= o) x += y;
        }
        if (l == 31) wsum[w] = x;
        __syncthreads();
        unsigned before = 0;
        for (int i = 0; i < w; ++i) before += wsum[i];
        dig_local[d] = before + x - tot;
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < kSortItems; ++k) {
        const int dd = dig[k];
        if (dd < 0) continue;
        const unsigned lp = dig_local[dd] + warp_cnt[w][dd] + rank[k];
        s_key[lp] = key[k];
        s_val[lp] = val[k];
    }
    __syncthreads();
    const long long tile_base = (long long)tile * kSortTile;
    const int cnt = n - tile_base < kSortTile ? (int)(n - tile_base) : kSortTile;
    for (int j = threadIdx.x; j < cnt; j += kSortThreads) {
        const unsigned long long kk = s_key[j];
        const int dd = (int)((kk >> shift) & 255u);
        const unsigned long long pos = gbase[dd] + (unsigned long long)(j - (int)dig_local[dd]);
        kout[pos] = kk;
        vout[pos] = s_val[j];
    }
}

// ----------------------------------------------------------------- climb ---

// lbvh.py:130-145 / _core.pyx:52-64: strict order on split positions a, b.
__device__ __forceinline__ bool delta_less(const unsigned long long* __restrict__ c,
                                           const int* __restrict__ id, int a, int b) {
    const unsigned long long xa = c[a] ^ c[a + 1], xb = c[b] ^ c[b + 1];
    if (xa != xb) return xa < xb;
    const int ia = id[a] ^ id[a + 1], ib = id[b] ^ id[b + 1];
    if (ia != ib) return ia < ib;
    return a < b;
}

__device__ __forceinline__ void load_box_cg(const float* p, float b[6]) {
    const float2 x = __ldcg(reinterpret_cast<const float2*>(p));
    const float2 y = __ldcg(reinterpret_cast<const float2*>(p) + 1);
    const float2 z = __ldcg(reinterpret_cast<const float2*>(p) + 2);
    b[0] = x.x; b[1] = x.y; b[2] = y.x; b[3] = y.y; b[4] = z.x; b[5] = z.y;
}

__global__ void __launch_bounds__(256) k_climb(const float* __restrict__ V,
                                               const int* __restrict__ T, int n,
                                               const unsigned long long* __restrict__ codes,
                                               const int* __restrict__ ids, TreeArrays ta,
                                               RsNode* nodes, RsLeaf* leaves, RsHeader* hdr) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int n_int = n - 1;
    // leaf init (lbvh.py:190-194) + the packed leaf record for the exact test
    const int tid = ids[i];
    const int ia = T[3ll * tid], ib = T[3ll * tid + 1], ic = T[3ll * tid + 2];
    float a[3], b[3], c[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        a[k] = V[3ll * ia + k];
        b[k] = V[3ll * ib + k];
        c[k] = V[3ll * ic + k];
    }
    float box[6];
#pragma unroll
    for (int k = 0; k < 3; ++k) {  // mesh.py:74-75
        box[2 * k] = fminf(fminf(a[k], b[k]), c[k]);
        box[2 * k + 1] = fmaxf(fmaxf(a[k], b[k]), c[k]);
    }
    float* lb_out = ta.leaf_bounds + 6ll * i;
    reinterpret_cast<float2*>(lb_out)[0] = make_float2(box[0], box[1]);
    reinterpret_cast<float2*>(lb_out)[1] = make_float2(box[2], box[3]);
    reinterpret_cast<float2*>(lb_out)[2] = make_float2(box[4], box[5]);
    ta.leaf_tri[i] = tid;
    ta.leaf_range_l[i] = i;
    ta.leaf_range_r[i] = i;
    ta.sorted_ids[i] = tid;
    RsLeaf lf;
    lf.p0 = make_float4(a[0], a[1], a[2], b[0]);
    lf.p1 = make_float4(b[1], b[2], c[0], c[1]);
    lf.p2 = make_float4(c[2], __int_as_float(tid), 0.f, 0.f);
    leaves[i] = lf;
    if (n == 1) {  // lbvh.py:163-166: the single leaf is the root
        ta.child_l[0] = n_int;
        hdr->root = n_int;
        hdr->height = 0;
        return;
    }
    int left = i, right = i, node = n_int + i, height = 0;
    for (;;) {
        if (left == 0 && right == n - 1) {  // root reached (lbvh.py:210-214)
            ta.parent[node] = -1;
            ta.child_l[n - 1] = node;
            if (node < n_int) ta.int_tri[node] = -2;
            hdr->root = node;
            hdr->height = height;
            return;
        }
        int parent;
        if (left == 0 || (right != n - 1 && delta_less(codes, ids, right, left - 1))) {
            parent = right;
            ta.child_l[parent] = node;
            ta.range_l[parent] = left;
        } else {
            parent = left - 1;
            ta.child_r[parent] = node;
            ta.range_r[parent] = right;
        }
        ta.height[node] = height;  // ref-indexed: internal 0..n-2, leaves n-1..2n-2
        ta.parent[node] = parent;
        cuda::atomic_ref<int, cuda::thread_scope_device> vis(ta.visit[parent]);
        if (vis.fetch_add(1, cuda::memory_order_acq_rel) == 0) return;  // first arriver stops
        left = __ldcg(ta.range_l + parent);
        right = __ldcg(ta.range_r + parent);
        const int cl = __ldcg(ta.child_l + parent), cr = __ldcg(ta.child_r + parent);
        float l6[6], r6[6];
        load_box_cg(cl < n_int ? ta.int_bounds + 6ll * cl : ta.leaf_bounds + 6ll * (cl - n_int), l6);
        load_box_cg(cr < n_int ? ta.int_bounds + 6ll * cr : ta.leaf_bounds + 6ll * (cr - n_int), r6);
        const int hl = __ldcg(ta.height + cl), hr = __ldcg(ta.height + cr);
        height = 1 + (hl > hr ? hl : hr);
#pragma unroll
        for (int k = 0; k < 3; ++k) {  // _core.pyx:181-183 (_fmin/_fmax)
            box[2 * k] = l6[2 * k] < r6[2 * k] ? l6[2 * k] : r6[2 * k];
            box[2 * k + 1] = l6[2 * k + 1] > r6[2 * k + 1] ? l6[2 * k + 1] : r6[2 * k + 1];
        }
        float* pb = ta.int_bounds + 6ll * parent;
        reinterpret_cast<float2*>(pb)[0] = make_float2(box[0], box[1]);
        reinterpret_cast<float2*>(pb)[1] = make_float2(box[2], box[3]);
        reinterpret_cast<float2*>(pb)[2] = make_float2(box[4], box[5]);
        RsNode nd;
        nd.a = make_float4(l6[0], l6[1], l6[2], l6[3]);
        nd.b = make_float4(l6[4], l6[5], r6[0], r6[1]);
        nd.c = make_float4(r6[2], r6[3], r6[4], r6[5]);
        nd.d = make_int4(cl, cr, 0, 0);
        nodes[parent] = nd;
        node = parent;
    }
}

// -------------------------------------------------------------- collapse ---

__device__ __forceinline__ RsSlot make_slot(float x0, float x1, float y0, float y1, float z0,
                                            float z1, int ref) {
    RsSlot t;
    t.lo_x = x0; t.hi_x = x1; t.lo_y = y0; t.hi_y = y1; t.lo_z = z0; t.hi_z = z1;
    t.ref = ref;
    t.pad = 0;
    return t;
}

__device__ __forceinline__ RsSlot empty_slot() {
    return make_slot(INFINITY, -INFINITY, INFINITY, -INFINITY, INFINITY, -INFINITY, kEmpty);
}

__global__ void __launch_bounds__(256) k_collapse(int n, TreeArrays ta, const RsNode* __restrict__ nodes,
                                                  RsNode4* __restrict__ nodes4,
                                                  const RsHeader* __restrict__ hdr) {
    const int p = blockIdx.x * blockDim.x + threadIdx.x;
    const int n_int = n - 1;
    if (n == 1) {  // single leaf: a root node holding it
        if (p == 0) {
            const float* b = ta.leaf_bounds;
            RsNode4 q;
            q.s[0] = make_slot(b[0], b[1], b[2], b[3], b[4], b[5], 0);
            q.s[1] = q.s[2] = q.s[3] = empty_slot();
            nodes4[0] = q;
        }
        return;
    }
    if (p >= n_int) return;
    int depth = 0;
    for (int x = __ldg(ta.parent + p); x >= 0; x = __ldg(ta.parent + x)) ++depth;
    if (depth & 1) return;  // absorbed into its parent's 4-wide node
    const RsNode nd = nodes[p];
    RsSlot out[4];
    int k = 0;
    const int ca = nd.d.x, cb = nd.d.y;
    if (ca >= n_int) {
        out[k++] = make_slot(nd.a.x, nd.a.y, nd.a.z, nd.a.w, nd.b.x, nd.b.y, ca);
    } else {
        const RsNode c = nodes[ca];
        out[k++] = make_slot(c.a.x, c.a.y, c.a.z, c.a.w, c.b.x, c.b.y, c.d.x);
        out[k++] = make_slot(c.b.z, c.b.w, c.c.x, c.c.y, c.c.z, c.c.w, c.d.y);
    }
    if (cb >= n_int) {
        out[k++] = make_slot(nd.b.z, nd.b.w, nd.c.x, nd.c.y, nd.c.z, nd.c.w, cb);
    } else {
        const RsNode c = nodes[cb];
        out[k++] = make_slot(c.a.x, c.a.y, c.a.z, c.a.w, c.b.x, c.b.y, c.d.x);
        out[k++] = make_slot(c.b.z, c.b.w, c.c.x, c.c.y, c.c.z, c.c.w, c.d.y);
    }
    while (k < 4) out[k++] = empty_slot();
    RsNode4* q = nodes4 + p;
#pragma unroll
    for (int j = 0; j < 4; ++j) q->s[j] = out[j];
}

// ------------------------------------------------------------ host glue ---

static int grid_for(long long n, int block, int cap) {
    long long g = (n + block - 1) / block;
    if (g < 1) g = 1;
    return (int)(g < cap ? g : cap);
}

void launch_prep(const float* V, const int* T, int n, double* cent, RsHeader* hdr,
                 const TreeArrays& ta, bool centroids, cudaStream_t s, bool lean) {
    count_launches(1);
    k_prep<<<grid_for(n, 256, 148 * 8), 256, 0, s>>>(V, T, n, cent, hdr, ta, centroids ? 1 : 0,
                                                     lean ? 1 : 0);
}

void launch_keys(const double* cent, int n, const RsHeader* hdr, int kind,
                 unsigned long long* keys, int* vals, cudaStream_t s) {
    count_launches(1);
    k_keys<<<grid_for(n, 256, 1 << 30), 256, 0, s>>>(cent, n, hdr, kind, keys, vals, fast_key_mode());
}

void launch_collapse(int n, const TreeArrays& ta, const RsNode* nodes, RsNode4* nodes4,
                     const RsHeader* hdr, cudaStream_t s) {
    count_launches(1);
    k_collapse<<<grid_for(n, 256, 1 << 30), 256, 0, s>>>(n, ta, nodes, nodes4, hdr);
}

size_t sort_scratch_bytes(int n, int passes) {
    const long long tiles = (n + kSortTile - 1) / kSortTile;
    return (size_t)passes * 256 * 4 + 64 + (size_t)passes * tiles * 256 * 8;
}

// Sorts (keys, vals) by the low 8*passes bits of the key; returns via
// (keys, vals) when passes is even, else (keys_alt, vals_alt).  scratch must
// hold sort_scratch_bytes(n, passes) bytes.
void launch_sort(unsigned long long* keys, int* vals, unsigned long long* keys_alt,
                 int* vals_alt, int n, int passes, void* scratch, cudaStream_t s) {
    const long long tiles = (n + kSortTile - 1) / kSortTile;
    unsigned* ghist = reinterpret_cast<unsigned*>(scratch);
    unsigned* counters = ghist + passes * 256;
    unsigned long long* status =
        reinterpret_cast<unsigned long long*>(reinterpret_cast<char*>(scratch) + passes * 256 * 4 + 64);
    cudaMemsetAsync(scratch, 0, sort_scratch_bytes(n, passes), s);
    count_launches(1 + passes);
    k_sort_hist<<<grid_for(n, 256, 148 * 4), 256, 0, s>>>(keys, n, passes, ghist);
    unsigned long long *ki = keys, *ko = keys_alt;
    int *vi = vals, *vo = vals_alt;
    for (int p = 0; p < passes; ++p) {
        k_onesweep<<<(unsigned)tiles, kSortThreads, 0, s>>>(ki, vi, ko, vo, n, 8 * p,
                                                            ghist + 256 * p, status + p * tiles * 256,
                                                            counters + p);
        unsigned long long* tk = ki; ki = ko; ko = tk;
        int* tv = vi; vi = vo; vo = tv;
    }
}

void launch_sort_segments(const float* S, const float* E, int n, float* So, float* Eo,
                          long long* perm, void* scratch, cudaStream_t s) {
    char* p = reinterpret_cast<char*>(scratch);
    auto take = [&](size_t bytes) { char* r = p; p += (bytes + 255) & ~size_t(255); return r; };
    RsHeader* hdr = reinterpret_cast<RsHeader*>(take(sizeof(RsHeader)));
    double* mid = reinterpret_cast<double*>(take(24ull * n));
    unsigned long long* keys = reinterpret_cast<unsigned long long*>(take(8ull * n));
    unsigned long long* keys2 = reinterpret_cast<unsigned long long*>(take(8ull * n));
    int* vals = reinterpret_cast<int*>(take(4ull * n));
    int* vals2 = reinterpret_cast<int*>(take(4ull * n));
    void* sort_scratch = take(sort_scratch_bytes(n, 8));
    cudaMemsetAsync(hdr, 0, sizeof(RsHeader), s);
    count_launches(3);
    k_mid_prep<<<grid_for(n, 256, 148 * 8), 256, 0, s>>>(S, E, n, mid, hdr);
    k_keys<<<grid_for(n, 256, 1 << 30), 256, 0, s>>>(mid, n, hdr, kTreeReference, keys, vals, 0);
    launch_sort(keys, vals, keys2, vals2, n, 8, sort_scratch, s);  // 8 passes: result in (keys, vals)
    k_gather_segments<<<grid_for(n, 256, 1 << 30), 256, 0, s>>>(vals, S, E, n, So, Eo, perm);
}

size_t sort_segments_scratch_bytes(int n) {
    auto r = [](size_t b) { return (b + 255) & ~size_t(255); };
    return r(sizeof(RsHeader)) + r(24ull * n) + 2 * r(8ull * n) + 2 * r(4ull * n) + r(sort_scratch_bytes(n, 8));
}

void launch_climb(const float* V, const int* T, int n, const unsigned long long* codes,
                  const int* ids, const TreeArrays& ta, RsNode* nodes, RsLeaf* leaves,
                  RsHeader* hdr, cudaStream_t s) {
    count_launches(1);
    k_climb<<<grid_for(n, 256, 1 << 30), 256, 0, s>>>(V, T, n, codes, ids, ta, nodes, leaves, hdr);
}

// ------------------------------------------------------------ lean climb ---
// The same Apetrei climb (same parent choice, so the same tree) for trees
// that are only queried: each arriving child writes its half of the
// parent's 64-B RsNode (its exact box, its ref, its end of the parent's
// range in d.z / d.w) before the acq_rel visit counter; the second arriver
// reads the whole record back.  No reference SoA arrays, heights or parent
// links: about half the climb's memory traffic.
__global__ void __launch_bounds__(256) k_climb_lean(const float* __restrict__ V,
                                                    const int* __restrict__ T, int n,
                                                    const unsigned long long* __restrict__ codes,
                                                    const int* __restrict__ ids, int* visit,
                                                    RsNode* nodes, RsLeaf* leaves, RsHeader* hdr,
                                                    float* leaf_boxes) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int n_int = n - 1;
    const int tid = ids[i];
    const int ia = T[3ll * tid], ib = T[3ll * tid + 1], ic = T[3ll * tid + 2];
    float a[3], b[3], c[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        a[k] = V[3ll * ia + k];
        b[k] = V[3ll * ib + k];
        c[k] = V[3ll * ic + k];
    }
    float box[6];
#pragma unroll
    for (int k = 0; k < 3; ++k) {  // mesh.py:74-75
        box[2 * k] = fminf(fminf(a[k], b[k]), c[k]);
        box[2 * k + 1] = fmaxf(fmaxf(a[k], b[k]), c[k]);
    }
    RsLeaf lf;
    lf.p0 = make_float4(a[0], a[1], a[2], b[0]);
    lf.p1 = make_float4(b[1], b[2], c[0], c[1]);
    lf.p2 = make_float4(c[2], __int_as_float(tid), 0.f, 0.f);
    leaves[i] = lf;
    float2* lb = reinterpret_cast<float2*>(leaf_boxes + 6ll * i);  // for the Morton-range lists
    lb[0] = make_float2(box[0], box[1]);
    lb[1] = make_float2(box[2], box[3]);
    lb[2] = make_float2(box[4], box[5]);
    if (n == 1) {
        hdr->root = n_int;
        return;
    }
    int left = i, right = i, node = n_int + i;
    for (;;) {
        if (left == 0 && right == n - 1) {
            hdr->root = node;
            return;
        }
        int parent;
        float* rec;
        if (left == 0 || (right != n - 1 && delta_less(codes, ids, right, left - 1))) {
            parent = right;  // we are the left child
            rec = reinterpret_cast<float*>(nodes + parent);
            reinterpret_cast<float4*>(rec)[0] = make_float4(box[0], box[1], box[2], box[3]);
            reinterpret_cast<float2*>(rec)[2] = make_float2(box[4], box[5]);
            reinterpret_cast<int*>(rec)[12] = node;
            reinterpret_cast<int*>(rec)[14] = left;
        } else {
            parent = left - 1;  // we are the right child
            rec = reinterpret_cast<float*>(nodes + parent);
            reinterpret_cast<float2*>(rec)[3] = make_float2(box[0], box[1]);
            reinterpret_cast<float4*>(rec)[2] = make_float4(box[2], box[3], box[4], box[5]);
            reinterpret_cast<int*>(rec)[13] = node;
            reinterpret_cast<int*>(rec)[15] = right;
        }
        cuda::atomic_ref<int, cuda::thread_scope_device> vis(visit[parent]);
        if (vis.fetch_add(1, cuda::memory_order_acq_rel) == 0) return;  // first arriver stops
        const float4 q0 = __ldcg(reinterpret_cast<const float4*>(rec));
        const float4 q1 = __ldcg(reinterpret_cast<const float4*>(rec) + 1);
        const float4 q2 = __ldcg(reinterpret_cast<const float4*>(rec) + 2);
        const int4 q3 = __ldcg(reinterpret_cast<const int4*>(rec) + 3);
        // _core.pyx:181-183: parent box = (min, max) of the children's
        box[0] = q0.x < q1.z ? q0.x : q1.z;
        box[1] = q0.y > q1.w ? q0.y : q1.w;
        box[2] = q0.z < q2.x ? q0.z : q2.x;
        box[3] = q0.w > q2.y ? q0.w : q2.y;
        box[4] = q1.x < q2.z ? q1.x : q2.z;
        box[5] = q1.y > q2.w ? q1.y : q2.w;
        left = q3.z;
        right = q3.w;
        node = parent;
    }
}

void launch_climb_lean(const float* V, const int* T, int n, const unsigned long long* codes,
                       const int* ids, int* visit, RsNode* nodes, RsLeaf* leaves, RsHeader* hdr,
                       float* leaf_boxes, cudaStream_t s) {
    count_launches(1);
    k_climb_lean<<<grid_for(n, 256, 1 << 30), 256, 0, s>>>(V, T, n, codes, ids, visit, nodes, leaves,
                                                           hdr, leaf_boxes);
}

// Every stride-th sorted key (the first level of the traversal's key search).
__global__ void k_code_samples(const unsigned long long* __restrict__ codes, int n, int stride,
                               unsigned long long* samples, int m) {
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k < m) samples[k] = codes[(long long)k * stride];
}

void launch_code_samples(const unsigned long long* codes, int n, int stride,
                         unsigned long long* samples, int m, cudaStream_t s) {
    count_launches(1);
    k_code_samples<<<(m + 255) / 256, 256, 0, s>>>(codes, n, stride, samples, m);
}

// The build's kernels (captured graphs give them the highest node priority,
// rs_capi.cu capture_graph).
bool is_build_kernel(const void* f) {
    return f == (const void*)k_prep || f == (const void*)k_keys || f == (const void*)k_sort_hist ||
           f == (const void*)k_onesweep || f == (const void*)k_climb_lean || f == (const void*)k_climb ||
           f == (const void*)k_code_samples;
}

}  // namespace rs
