// rs_query.cu -- per-segment BVH traversal + exact test (the hot path) and the
// all-pairs baseline, sm_100a.
//
// Semantics follow _core.pyx:195-352 (batch_query) / lbvh.py:244-359:
//   * candidate set = leaves whose f32 triangle AABB overlaps the segment
//     AABB (touching counts); each candidate gets the f64 Moller-Trumbore test;
//   * boolean: any hit; count: number of hits; barycentric: min over (t, tid).
// The reference buffers candidates (max_collisions) and tests them in batches.
// Every mode's OUTPUT is independent of the batching (any / sum / min over a
// total order), so this kernel tests each candidate the moment it is found and
// keeps no buffer.  The one observable the batching does change is the
// boolean-mode stack-overflow error: the reference stops at the first flush
// that holds a hit.  With ref_semantics the kernel counts candidates since the
// last flush and applies the same early exit at the same points, and checks
// `top >= max_stack` at the same push, so the reported overflowing segment is
// identical (tests/test_gpu_parity.py::test_overflow_index).
#include <cuda/atomic>

#include <cstdlib>

#include "rs_common.cuh"
#include "rs_internal.h"

namespace rs {

constexpr int kQueryThreads = 128;

// A/B tuning switches: RS_BINARY_FAST=1 traverses fast trees with the
// binary kernels; RS_SIMPLE_QUERY=1 picks one-segment-per-thread over the
// persistent binary kernel.
static bool env_flag(const char* k) {
    const char* e = getenv(k);
    return e && e[0] == '1';
}
static const bool g_simple_query = env_flag("RS_SIMPLE_QUERY");
static const bool g_binary_fast = env_flag("RS_BINARY_FAST");

struct Ray {
    float box[6];
    double sx, sy, sz, dx, dy, dz;
};

__device__ __forceinline__ void load_ray(const float* __restrict__ s, const float* __restrict__ e,
                                         long long i, Ray& r) {
    const float s0 = __ldg(s + 3 * i), s1 = __ldg(s + 3 * i + 1), s2 = __ldg(s + 3 * i + 2);
    const float e0 = __ldg(e + 3 * i), e1 = __ldg(e + 3 * i + 1), e2 = __ldg(e + 3 * i + 2);
    // engine.py:115-122
    r.box[0] = fminf(s0, e0); r.box[1] = fmaxf(s0, e0);
    r.box[2] = fminf(s1, e1); r.box[3] = fmaxf(s1, e1);
    r.box[4] = fminf(s2, e2); r.box[5] = fmaxf(s2, e2);
    r.sx = s0; r.sy = s1; r.sz = s2;
    // _core.pyx:81-83: d = (double)e - s
    r.dx = __dsub_rn((double)e0, r.sx);
    r.dy = __dsub_rn((double)e1, r.sy);
    r.dz = __dsub_rn((double)e2, r.sz);
}

struct Hit {
    int det;
    int n_hits;
    int best_tri;
    double best_t;
};

template <int MODE>
__device__ __forceinline__ void test_leaf(const RsLeaf* __restrict__ leaves, int leaf,
                                          const Ray& r, Hit& h, unsigned long long& mts) {
    const float4 p0 = __ldg(&leaves[leaf].p0);
    const float4 p1 = __ldg(&leaves[leaf].p1);
    const float4 p2 = __ldg(&leaves[leaf].p2);
    double t;
    ++mts;
    if (mt_hit(p0.x, p0.y, p0.z, p0.w, p1.x, p1.y, p1.z, p1.w, p2.x, r.sx, r.sy, r.sz, r.dx,
               r.dy, r.dz, &t)) {
        const int tid = __float_as_int(p2.y);
        h.det = 1;
        h.n_hits += 1;
        if (MODE == kBarycentric) {  // _core.pyx:317-320
            if (h.best_tri < 0 || t < h.best_t || (t == h.best_t && tid < h.best_tri)) {
                h.best_t = t;
                h.best_tri = tid;
            }
        }
    }
}

// Returns false on a max_stack overflow (reference semantics).
template <int MODE, bool REF, int KSTACK>
__device__ __forceinline__ bool trace(const QueryArgs& a, const Ray& r, Hit& h,
                                      unsigned long long& visits, unsigned long long& mts,
                                      bool& internal_ovf) {
    const int n_int = a.n_int;
    h.det = 0;
    h.n_hits = 0;
    h.best_tri = -1;
    h.best_t = 0.0;
    int node = __ldg(&a.hdr->root);
    if (node >= n_int) {  // single-triangle tree: leaf root (_core.pyx:260-267)
        const float4 p0 = __ldg(&a.leaves[0].p0), p1 = __ldg(&a.leaves[0].p1),
                     p2 = __ldg(&a.leaves[0].p2);
        const float x0 = fminf(fminf(p0.x, p0.w), p1.z), x1 = fmaxf(fmaxf(p0.x, p0.w), p1.z);
        const float y0 = fminf(fminf(p0.y, p1.x), p1.w), y1 = fmaxf(fmaxf(p0.y, p1.x), p1.w);
        const float z0 = fminf(fminf(p0.z, p1.y), p2.x), z1 = fmaxf(fmaxf(p0.z, p1.y), p2.x);
        if (overlap6(r.box, x0, x1, y0, y1, z0, z1)) test_leaf<MODE>(a.leaves, 0, r, h, mts);
        return true;
    }
    int stack[KSTACK];
    int top = 0;  // stack[-1] is the reference's EMPTY sentinel (lbvh.py:107)
    int count = 0;  // candidates since the last flush (REF boolean only)
    const int cap = REF ? (a.max_stack - 1 < KSTACK ? a.max_stack - 1 : KSTACK) : KSTACK;
    for (;;) {
        ++visits;
        const float4* np = reinterpret_cast<const float4*>(a.nodes + node);
        const float4 n0 = __ldg(np), n1 = __ldg(np + 1), n2 = __ldg(np + 2);
        const int4 nd = __ldg(reinterpret_cast<const int4*>(np + 3));
        const bool oa = overlap6(r.box, n0.x, n0.y, n0.z, n0.w, n1.x, n1.y);
        const bool ob = overlap6(r.box, n1.z, n1.w, n2.x, n2.y, n2.z, n2.w);
        const int ca = nd.x, cb = nd.y;
        const bool la = ca >= n_int, lb = cb >= n_int;
        if (oa && la) {
            test_leaf<MODE>(a.leaves, ca - n_int, r, h, mts);
            ++count;
        }
        if (ob && lb) {
            test_leaf<MODE>(a.leaves, cb - n_int, r, h, mts);
            ++count;
        }
        const bool ta = oa && !la, tb = ob && !lb;
        if (!ta && !tb) {
            if (top == 0) break;  // popped the sentinel: traversal complete
            node = stack[--top];
        } else {
            node = ta ? ca : cb;
            if (ta && tb) {
                // reference: `if top >= max_stack` with top counting the sentinel
                if (top >= cap) {
                    if (REF && top + 1 >= a.max_stack) return false;
                    internal_ovf = true;
                    return true;
                }
                stack[top++] = cb;
            }
        }
        if (MODE == kBoolean) {
            if (REF) {  // flush point: buffer "full" at max_collisions - 1
                if (count >= a.max_coll - 1) {
                    if (h.det) return true;
                    count = 0;
                }
            } else if (h.det) {
                return true;
            }
        }
    }
    return true;
}

template <int MODE>
__device__ __forceinline__ void write_dense(const QueryArgs& a, long long i, const Ray& r,
                                            const Hit& h) {
    if (MODE == kBoolean) {
        a.detected[i] = h.det;
    } else if (MODE == kCount) {
        a.counts[i] = h.n_hits;
    } else {
        a.detected[i] = h.best_tri >= 0;
        a.tri[i] = h.best_tri;
        float px = 0.f, py = 0.f, pz = 0.f, d = 0.f;
        if (h.best_tri >= 0) hit_point(r.sx, r.sy, r.sz, r.dx, r.dy, r.dz, h.best_t, &px, &py, &pz, &d);
        a.dist[i] = d;
        a.points[3 * i] = px;
        a.points[3 * i + 1] = py;
        a.points[3 * i + 2] = pz;
    }
}

__device__ __forceinline__ void flush_stats(const QueryArgs& a, unsigned long long visits,
                                            unsigned long long mts) {
    for (int o = 16; o; o >>= 1) {
        visits += __shfl_xor_sync(0xffffffffu, visits, o);
        mts += __shfl_xor_sync(0xffffffffu, mts, o);
    }
    if ((threadIdx.x & 31) == 0) {
        atomicAdd(&a.status->visits, visits);
        atomicAdd(&a.status->mts, mts);
    }
}

template <int MODE, bool REF, int KSTACK, bool STATS>
__global__ void __launch_bounds__(kQueryThreads) k_query_dense(QueryArgs a) {
    const long long i = (long long)blockIdx.x * kQueryThreads + threadIdx.x;
    unsigned long long visits = 0, mts = 0;
    if (i < a.n_r) {
        Ray r;
        load_ray(a.starts, a.ends, i, r);
        Hit h;
        bool iovf = false;
        if (!trace<MODE, REF, KSTACK>(a, r, h, visits, mts, iovf)) {
            atomicMax(&a.status->bad, ~(unsigned long long)(i + a.ray_offset));
        } else {
            if (iovf) atomicAdd(&a.status->internal, 1ull);
            write_dense<MODE>(a, i, r, h);
        }
    }
    if (STATS) flush_stats(a, visits, mts);
}

// ---------------------------------------------------- persistent warps ---
//
// One traversal step = one internal-node visit.  Returns 0 (continue),
// 1 (ray finished), 2 (reference max_stack overflow), 3 (internal capacity).
struct Trav {
    int node;
    int top;
    int count;
};

template <int MODE, bool REF, int KSTACK>
__device__ __forceinline__ int trav_step(const QueryArgs& a, const Ray& r, Hit& h, Trav& t,
                                         int* stack, int cap, unsigned long long& visits,
                                         unsigned long long& mts) {
    const int n_int = a.n_int;
    const int node = t.node;
    if (node >= n_int) {  // single-triangle tree: leaf root (_core.pyx:260-267)
        const float4 p0 = __ldg(&a.leaves[0].p0), p1 = __ldg(&a.leaves[0].p1),
                     p2 = __ldg(&a.leaves[0].p2);
        const float x0 = fminf(fminf(p0.x, p0.w), p1.z), x1 = fmaxf(fmaxf(p0.x, p0.w), p1.z);
        const float y0 = fminf(fminf(p0.y, p1.x), p1.w), y1 = fmaxf(fmaxf(p0.y, p1.x), p1.w);
        const float z0 = fminf(fminf(p0.z, p1.y), p2.x), z1 = fmaxf(fmaxf(p0.z, p1.y), p2.x);
        if (overlap6(r.box, x0, x1, y0, y1, z0, z1)) test_leaf<MODE>(a.leaves, 0, r, h, mts);
        return 1;
    }
    ++visits;
    const float4* np = reinterpret_cast<const float4*>(a.nodes + node);
    const float4 n0 = __ldg(np), n1 = __ldg(np + 1), n2 = __ldg(np + 2);
    const int4 nd = __ldg(reinterpret_cast<const int4*>(np + 3));
    const bool oa = overlap6(r.box, n0.x, n0.y, n0.z, n0.w, n1.x, n1.y);
    const bool ob = overlap6(r.box, n1.z, n1.w, n2.x, n2.y, n2.z, n2.w);
    const int ca = nd.x, cb = nd.y;
    const bool la = ca >= n_int, lb = cb >= n_int;
    if (oa && la) {
        test_leaf<MODE>(a.leaves, ca - n_int, r, h, mts);
        ++t.count;
    }
    if (ob && lb) {
        test_leaf<MODE>(a.leaves, cb - n_int, r, h, mts);
        ++t.count;
    }
    const bool ta = oa && !la, tb = ob && !lb;
    if (!ta && !tb) {
        if (t.top == 0) return 1;
        t.node = stack[--t.top];
    } else {
        t.node = ta ? ca : cb;
        if (ta && tb) {
            if (t.top >= cap) return (REF && t.top + 1 >= a.max_stack) ? 2 : 3;
            stack[t.top++] = cb;
        }
    }
    if (MODE == kBoolean) {
        if (REF) {
            if (t.count >= a.max_coll - 1) {
                if (h.det) return 1;
                t.count = 0;
            }
        } else if (h.det) {
            return 1;
        }
    }
    return 0;
}

// Persistent warps with dynamic ray fetch: a lane whose segment is finished
// goes idle; once kRefill lanes of the warp are idle the warp claims that
// many new segments with one atomicAdd on a global counter (contiguous ids ->
// coalesced endpoint loads).  Keeps SIMD lanes busy although half of the
// segments leave the tree at the root and the rest need 10-40 node visits.
constexpr int kPersistThreads = 128;
constexpr int kRefill = 8;

template <int MODE, bool REF, int KSTACK, bool STATS>
__global__ void __launch_bounds__(kPersistThreads) k_query_persistent(QueryArgs a) {
    const unsigned kFull = 0xffffffffu;
    const int lane = threadIdx.x & 31;
    const unsigned lt = (1u << lane) - 1u;
    int stack[KSTACK];
    const int root = __ldg(&a.hdr->root);
    const int cap = REF ? (a.max_stack - 1 < KSTACK ? a.max_stack - 1 : KSTACK) : KSTACK;
    long long ray = -1;
    Ray r;
    Hit h;
    Trav t;
    bool exhausted = false;
    unsigned long long visits = 0, mts = 0;
    for (;;) {
        const unsigned idle = __ballot_sync(kFull, ray < 0);
        if (!exhausted && __popc(idle) >= kRefill) {
            const int k = __popc(idle);
            const int leader = __ffs(idle) - 1;
            unsigned long long base = 0;
            if (lane == leader) base = atomicAdd(&a.status->tile_counter, (unsigned long long)k);
            base = __shfl_sync(kFull, base, leader);
            if (base + k >= (unsigned long long)a.n_r) exhausted = true;
            if (ray < 0) {
                const long long mine = (long long)base + __popc(idle & lt);
                if (mine < a.n_r) {
                    ray = mine;
                    load_ray(a.starts, a.ends, ray, r);
                    h.det = 0;
                    h.n_hits = 0;
                    h.best_tri = -1;
                    h.best_t = 0.0;
                    t.node = root;
                    t.top = 0;
                    t.count = 0;
                }
            }
        } else if (idle == kFull) {
            break;
        }
        if (ray >= 0) {
            const int st = trav_step<MODE, REF, KSTACK>(a, r, h, t, stack, cap, visits, mts);
            if (st != 0) {
                if (st == 1) write_dense<MODE>(a, ray, r, h);
                else if (st == 2) atomicMax(&a.status->bad, ~(unsigned long long)(ray + a.ray_offset));
                else atomicAdd(&a.status->internal, 1ull);
                ray = -1;
            }
        }
    }
    if (STATS) flush_stats(a, visits, mts);
}

// ------------------------------------------------ 4-lane quad traversal ---
//
// Fast trees are traversed as a 4-wide BVH by groups of 4 lanes: one segment
// per group, one child slot per lane.  A node visit is one 256-bit load per
// lane, i.e. the group reads exactly one 128-B line, so the 8 groups of a warp
// touch 8 lines per step instead of the 32+ scattered lines of a
// thread-per-segment binary traversal (which is L1-wavefront bound).  Leaf
// children are exact-tested by the lane that found them, internal hits are
// pushed in parallel onto the group's shared-memory stack.
constexpr int kQuadThreads = 128;
constexpr int kQuadGroups = kQuadThreads / 4;
constexpr int kQuadStack = 96;  // 4-wide depth <= 31 (binary height <= 61) x 3 pushes
constexpr int kQuadRefill = 2;  // refill when >= 2 groups of the warp are idle

__device__ __forceinline__ void ld_slot(const RsSlot* p, float f[8]) {
    asm volatile("ld.global.nc.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=f"(f[0]), "=f"(f[1]), "=f"(f[2]), "=f"(f[3]), "=f"(f[4]), "=f"(f[5]),
                   "=f"(f[6]), "=f"(f[7])
                 : "l"(p));
}

template <int MODE, bool STATS>
__global__ void __launch_bounds__(kQuadThreads) k_query_quad(QueryArgs a) {
    __shared__ int stk[kQuadStack][kQuadGroups];
    const unsigned kFull = 0xffffffffu;
    const int lane = threadIdx.x & 31;
    const int q = lane & 3;
    const int gshift = lane & ~3;
    const int gid = threadIdx.x >> 2;
    const int n_int = a.n_int;
    const int root = n_int > 0 ? __ldg(&a.hdr->root) : 0;
    long long ray = -1;
    Ray r;
    int node = 0, top = 0;
    Hit h;
    h.det = 0; h.n_hits = 0; h.best_tri = -1; h.best_t = 0.0;
    bool exhausted = false;
    unsigned long long visits = 0, mts = 0;
    for (;;) {
        const unsigned idle = __ballot_sync(kFull, ray < 0);
        const int idle_groups = __popc(idle) >> 2;
        if (!exhausted && idle_groups >= kQuadRefill) {
            const int leader = __ffs(idle) - 1;
            unsigned long long base = 0;
            if (lane == leader)
                base = atomicAdd(&a.status->tile_counter, (unsigned long long)idle_groups);
            base = __shfl_sync(kFull, base, leader);
            if (base + idle_groups >= (unsigned long long)a.n_r) exhausted = true;
            if (ray < 0) {
                const long long mine =
                    (long long)base + (__popc(idle & ((1u << gshift) - 1u)) >> 2);
                if (mine < a.n_r) {
                    ray = mine;
                    load_ray(a.starts, a.ends, ray, r);
                    node = root;
                    top = 0;
                    h.det = 0; h.n_hits = 0; h.best_tri = -1; h.best_t = 0.0;
                }
            }
        } else if (idle == kFull) {
            break;
        }
        const bool active = ray >= 0;
        bool ihit = false;
        int ref = kEmpty;
        if (active) {
            float f[8];
            ld_slot(&a.nodes4[node].s[q], f);
            ref = __float_as_int(f[6]);
            const bool hit = ref >= 0 && overlap6(r.box, f[0], f[1], f[2], f[3], f[4], f[5]);
            if (STATS && q == 0) ++visits;
            if (hit && ref >= n_int) test_leaf<MODE>(a.leaves, ref - n_int, r, h, mts);
            ihit = hit && ref < n_int;
        }
        const unsigned gmask = (__ballot_sync(kFull, ihit) >> gshift) & 0xFu;
        bool finish = false;
        if (MODE == kBoolean) finish = ((__ballot_sync(kFull, h.det != 0) >> gshift) & 0xFu) != 0;
        bool ovf = false;
        if (active && !finish) {
            const int k = __popc(gmask);
            if (top + k > kQuadStack) {
                ovf = finish = true;
            } else {
                if (ihit) stk[top + __popc(gmask & ((1u << q) - 1u))][gid] = ref;
                top += k;
                if (top == 0) finish = true;
            }
        }
        __syncwarp();
        if (active && !finish) node = stk[--top][gid];
        if (__any_sync(kFull, active && finish)) {
            // reduce the group's per-lane partial results (lanes of other
            // groups shuffle within their own group; results are ignored)
            Hit g = h;
#pragma unroll
            for (int o = 1; o <= 2; o <<= 1) {
                const int od = __shfl_xor_sync(kFull, g.det, o);
                const int on = __shfl_xor_sync(kFull, g.n_hits, o);
                const int ot = __shfl_xor_sync(kFull, g.best_tri, o);
                const double obt = __shfl_xor_sync(kFull, g.best_t, o);
                g.det |= od;
                g.n_hits += on;
                if (ot >= 0 && (g.best_tri < 0 || obt < g.best_t || (obt == g.best_t && ot < g.best_tri))) {
                    g.best_t = obt;
                    g.best_tri = ot;
                }
            }
            if (active && finish) {
                h = g;
                if (q == 0) {
                    if (ovf) atomicAdd(&a.status->internal, 1ull);
                    else write_dense<MODE>(a, ray, r, h);
                }
                ray = -1;
            }
        }
        __syncwarp();
    }
    if (STATS) flush_stats(a, visits, mts);
}

// Barycentric with fused ordered compaction (engine.py:206-215): each CTA
// takes a dynamic tile id, traces its rays, block-scans the hit flags and
// chains a decoupled look-back over the tile prefixes, then writes its hits at
// their final ascending positions.  One pass, no dense intermediate arrays.
template <bool REF, int KSTACK, bool STATS>
__global__ void __launch_bounds__(kQueryThreads) k_query_compact(QueryArgs a) {
    __shared__ int s_tile;
    __shared__ unsigned s_warp[kQueryThreads / 32];
    __shared__ unsigned long long s_prefix;
    if (threadIdx.x == 0) s_tile = (int)atomicAdd(&a.status->tile_counter, 1ull);
    __syncthreads();
    const int tile = s_tile;
    const long long i = (long long)tile * kQueryThreads + threadIdx.x;
    unsigned long long visits = 0, mts = 0;
    Ray r;
    Hit h;
    h.best_tri = -1;
    bool ok = true;
    if (i < a.n_r) {
        load_ray(a.starts, a.ends, i, r);
        bool iovf = false;
        ok = trace<kBarycentric, REF, KSTACK>(a, r, h, visits, mts, iovf);
        if (!ok) atomicMax(&a.status->bad, ~(unsigned long long)(i + a.ray_offset));
        if (iovf) atomicAdd(&a.status->internal, 1ull);
    }
    const bool hit = ok && i < a.n_r && h.best_tri >= 0;
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    const unsigned ball = __ballot_sync(0xffffffffu, hit);
    if (l == 0) s_warp[w] = __popc(ball);
    __syncthreads();
    if (w == 0) {
        unsigned agg = 0, mine = 0;
        for (int k = 0; k < kQueryThreads / 32; ++k) {
            if (k == l) mine = agg;
            agg += s_warp[k];
        }
        __syncwarp();
        if (l < kQueryThreads / 32) s_warp[l] = mine;
        const unsigned long long excl = lookback_warp(a.tile_status, tile, agg);
        if (l == 0) {
            s_prefix = excl;
            if ((long long)(tile + 1) * kQueryThreads >= a.n_r) atomicMax(&a.status->hits, excl + agg);
        }
    }
    __syncthreads();
    if (hit) {
        const unsigned long long pos =
            s_prefix + s_warp[w] + __popc(ball & ((1u << l) - 1u));
        float px, py, pz, d;
        hit_point(r.sx, r.sy, r.sz, r.dx, r.dy, r.dz, h.best_t, &px, &py, &pz, &d);
        a.c_ray[pos] = (int)(i + a.ray_offset);
        a.c_dist[pos] = d;
        a.c_tri[pos] = h.best_tri;
        a.c_point[3 * pos] = px;
        a.c_point[3 * pos + 1] = py;
        a.c_point[3 * pos + 2] = pz;
    }
    if (STATS) flush_stats(a, visits, mts);
}

size_t compact_scratch_bytes(long long n_r) {
    return (size_t)((n_r + kQueryThreads - 1) / kQueryThreads) * 8;
}

template <int MODE, bool REF, int KS>
static void go(const QueryArgs& a, bool compact, bool stats, cudaStream_t s) {
    const unsigned grid = (unsigned)((a.n_r + kQueryThreads - 1) / kQueryThreads);
    if (compact) {
        if constexpr (MODE == kBarycentric) {
            if (stats) k_query_compact<REF, KS, true><<<grid, kQueryThreads, 0, s>>>(a);
            else k_query_compact<REF, KS, false><<<grid, kQueryThreads, 0, s>>>(a);
        }
        return;
    }
    if (!REF && a.nodes4 && !g_binary_fast) {
        auto kq = stats ? k_query_quad<MODE, true> : k_query_quad<MODE, false>;
        const int oq = occupancy((const void*)kq, kQuadThreads);
        const int sms = device_sms();
        long long want = (a.n_r + kQuadGroups - 1) / kQuadGroups;
        long long pg = (long long)sms * (oq > 0 ? oq : 1);
        kq<<<(unsigned)(want < pg ? want : pg), kQuadThreads, 0, s>>>(a);
        return;
    }
    if (g_simple_query) {
        if (stats) k_query_dense<MODE, REF, KS, true><<<grid, kQueryThreads, 0, s>>>(a);
        else k_query_dense<MODE, REF, KS, false><<<grid, kQueryThreads, 0, s>>>(a);
        return;
    }
    auto kern = stats ? k_query_persistent<MODE, REF, KS, true> : k_query_persistent<MODE, REF, KS, false>;
    const int occ = occupancy((const void*)kern, kPersistThreads);
    const int sms = device_sms();
    long long want = (a.n_r + kPersistThreads - 1) / kPersistThreads;
    long long pg = (long long)sms * (occ > 0 ? occ : 1);
    kern<<<(unsigned)(want < pg ? want : pg), kPersistThreads, 0, s>>>(a);
}

template <int MODE, bool REF>
static int go_ks(const QueryArgs& a, bool compact, int kstack, bool stats, cudaStream_t s) {
    if (kstack <= 32) go<MODE, REF, 32>(a, compact, stats, s);
    else if (kstack <= 64) go<MODE, REF, 64>(a, compact, stats, s);
    else if (kstack <= 128) go<MODE, REF, 128>(a, compact, stats, s);
    else if (kstack <= 256) go<MODE, REF, 256>(a, compact, stats, s);
    else return -1;
    return 0;
}

int launch_query(const QueryArgs& a, int mode, bool ref, bool compact, int kstack, bool stats,
                 cudaStream_t s) {
    if (a.n_r <= 0) return 0;
    count_launches(1);
    switch (mode) {
        case kBoolean:
            return ref ? go_ks<kBoolean, true>(a, false, kstack, stats, s)
                       : go_ks<kBoolean, false>(a, false, kstack, stats, s);
        case kCount:
            return ref ? go_ks<kCount, true>(a, false, kstack, stats, s)
                       : go_ks<kCount, false>(a, false, kstack, stats, s);
        case kBarycentric:
            return ref ? go_ks<kBarycentric, true>(a, compact, kstack, stats, s)
                       : go_ks<kBarycentric, false>(a, compact, kstack, stats, s);
    }
    return -1;
}

// ------------------------------------------------------------ all-pairs ---

// _core.pyx:355-433: every (segment, triangle) pair, AABB prescreen then the
// exact test, triangles in ascending id.  Triangles are staged through shared
// memory in tiles; one segment per thread.
constexpr int kBaseThreads = 128;
constexpr int kBaseTile = 256;

template <int MODE>
__global__ void __launch_bounds__(kBaseThreads) k_baseline(BaselineArgs a) {
    __shared__ float sv[kBaseTile][9];
    const long long i = (long long)blockIdx.x * kBaseThreads + threadIdx.x;
    Ray r;
    const bool live = i < a.n_r;
    if (live) load_ray(a.starts, a.ends, i, r);
    Hit h{0, 0, -1, 0.0};
    bool done = !live;
    for (int j0 = 0; j0 < a.n_t; j0 += kBaseTile) {
        if (__syncthreads_and(done)) break;
        for (int k = threadIdx.x; k < kBaseTile; k += kBaseThreads) {
            const int j = j0 + k;
            if (j < a.n_t) {
                const int ia = a.T[3ll * j], ib = a.T[3ll * j + 1], ic = a.T[3ll * j + 2];
#pragma unroll
                for (int c = 0; c < 3; ++c) {
                    sv[k][c] = a.V[3ll * ia + c];
                    sv[k][3 + c] = a.V[3ll * ib + c];
                    sv[k][6 + c] = a.V[3ll * ic + c];
                }
            }
        }
        __syncthreads();
        const int jn = a.n_t - j0 < kBaseTile ? a.n_t - j0 : kBaseTile;
        for (int k = 0; k < jn && !done; ++k) {
            const float* v = sv[k];
            const float x0 = fminf(fminf(v[0], v[3]), v[6]), x1 = fmaxf(fmaxf(v[0], v[3]), v[6]);
            const float y0 = fminf(fminf(v[1], v[4]), v[7]), y1 = fmaxf(fmaxf(v[1], v[4]), v[7]);
            const float z0 = fminf(fminf(v[2], v[5]), v[8]), z1 = fmaxf(fmaxf(v[2], v[5]), v[8]);
            if (!overlap6(r.box, x0, x1, y0, y1, z0, z1)) continue;
            double t;
            if (!mt_hit(v[0], v[1], v[2], v[3], v[4], v[5], v[6], v[7], v[8], r.sx, r.sy, r.sz,
                        r.dx, r.dy, r.dz, &t))
                continue;
            h.det = 1;
            h.n_hits += 1;
            if (MODE == kBoolean) { done = true; break; }
            if (h.best_tri < 0 || t < h.best_t) {  // ascending j: ties keep the lower id
                h.best_t = t;
                h.best_tri = j0 + k;
            }
        }
        __syncthreads();
    }
    if (!live) return;
    if (MODE == kBoolean) {
        a.detected[i] = h.det;
    } else if (MODE == kCount) {
        a.counts[i] = h.n_hits;
    } else if (a.best_tri) {
        a.best_tri[i] = h.best_tri;
        a.best_t[i] = h.best_tri >= 0 && h.best_t != 0.0 ? (unsigned long long)__double_as_longlong(h.best_t) : 0ull;
    } else {
        a.detected[i] = h.best_tri >= 0;
        a.tri[i] = h.best_tri;
        float px = 0.f, py = 0.f, pz = 0.f, d = 0.f;
        if (h.best_tri >= 0) hit_point(r.sx, r.sy, r.sz, r.dx, r.dy, r.dz, h.best_t, &px, &py, &pz, &d);
        a.dist[i] = d;
        a.points[3 * i] = px;
        a.points[3 * i + 1] = py;
        a.points[3 * i + 2] = pz;
    }
}

// oracle_intersect (oracle.py:30-158): the reference's independent
// verification oracle -- every (segment, triangle) pair, no box prescreen,
// plane intersection then three edge sign tests, f64 -- a formulation
// algebraically independent of Moller-Trumbore (SPEC.md "oracle uses a
// formulation algebraically independent of Moller-Trumbore").  Its results
// agree with the engine's except for grazing pairs; the reference compares
// them at 1e-4 on the floats.
__device__ __forceinline__ double dot3(double ax, double ay, double az, double bx, double by, double bz) {
    return ax * bx + ay * by + az * bz;
}

template <int MODE>
__global__ void __launch_bounds__(kBaseThreads) k_sign_oracle(BaselineArgs a) {
    __shared__ float sv[kBaseTile][9];
    const long long i = (long long)blockIdx.x * kBaseThreads + threadIdx.x;
    Ray r;
    const bool live = i < a.n_r;
    if (live) load_ray(a.starts, a.ends, i, r);
    Hit h{0, 0, -1, 0.0};
    bool done = !live;
    for (int j0 = 0; j0 < a.n_t; j0 += kBaseTile) {
        if (__syncthreads_and(done)) break;
        for (int k = threadIdx.x; k < kBaseTile; k += kBaseThreads) {
            const int j = j0 + k;
            if (j < a.n_t) {
                const int ia = a.T[3ll * j], ib = a.T[3ll * j + 1], ic = a.T[3ll * j + 2];
#pragma unroll
                for (int c = 0; c < 3; ++c) {
                    sv[k][c] = a.V[3ll * ia + c];
                    sv[k][3 + c] = a.V[3ll * ib + c];
                    sv[k][6 + c] = a.V[3ll * ic + c];
                }
            }
        }
        __syncthreads();
        const int jn = a.n_t - j0 < kBaseTile ? a.n_t - j0 : kBaseTile;
        for (int k = 0; k < jn && !done; ++k) {
            const float* v = sv[k];
            const double ax = v[0], ay = v[1], az = v[2], bx = v[3], by = v[4], bz = v[5];
            const double cx = v[6], cy = v[7], cz = v[8];
            const double e1x = bx - ax, e1y = by - ay, e1z = bz - az;
            const double e2x = cx - ax, e2y = cy - ay, e2z = cz - az;
            const double nx = e1y * e2z - e1z * e2y, ny = e1z * e2x - e1x * e2z, nz = e1x * e2y - e1y * e2x;
            const double denom = dot3(r.dx, r.dy, r.dz, nx, ny, nz);
            if (fabs(denom) < kDetEps) continue;
            const double t = (dot3(nx, ny, nz, ax, ay, az) - dot3(r.sx, r.sy, r.sz, nx, ny, nz)) / denom;
            if (!(t >= 0.0 && t <= 1.0)) continue;
            const double px = r.sx + t * r.dx, py = r.sy + t * r.dy, pz = r.sz + t * r.dz;
            bool in = true;
            // edges (b - a, a), (c - b, b), (a - c, c): n . (e x (p - v)) >= 0
            const double ex[3] = {e1x, cx - bx, ax - cx}, ey[3] = {e1y, cy - by, ay - cy},
                         ez[3] = {e1z, cz - bz, az - cz};
            const double vx[3] = {ax, bx, cx}, vy[3] = {ay, by, cy}, vz[3] = {az, bz, cz};
#pragma unroll
            for (int q = 0; q < 3; ++q) {
                const double rx = px - vx[q], ry = py - vy[q], rz = pz - vz[q];
                const double qx = ey[q] * rz - ez[q] * ry, qy = ez[q] * rx - ex[q] * rz, qz = ex[q] * ry - ey[q] * rx;
                in = in && (qx * nx + qy * ny + qz * nz >= 0.0);
            }
            if (!in) continue;
            h.det = 1;
            h.n_hits += 1;
            if (MODE == kBoolean) { done = true; break; }
            if (h.best_tri < 0 || t < h.best_t) {  // ascending j: argmin keeps the lowest id
                h.best_t = t;
                h.best_tri = j0 + k;
            }
        }
        __syncthreads();
    }
    if (!live) return;
    if (MODE == kBoolean) {
        a.detected[i] = h.det;
    } else if (MODE == kCount) {
        a.counts[i] = h.n_hits;
    } else {
        a.best_tri[i] = h.best_tri;
        a.best_t[i] = h.best_tri >= 0 && h.best_t != 0.0 ? (unsigned long long)__double_as_longlong(h.best_t) : 0ull;
    }
}

void launch_sign_oracle(const BaselineArgs& a, int mode, cudaStream_t s) {
    if (a.n_r <= 0) return;
    count_launches(1);
    const unsigned grid = (unsigned)((a.n_r + kBaseThreads - 1) / kBaseThreads);
    if (mode == kBoolean) k_sign_oracle<kBoolean><<<grid, kBaseThreads, 0, s>>>(a);
    else if (mode == kCount) k_sign_oracle<kCount><<<grid, kBaseThreads, 0, s>>>(a);
    else k_sign_oracle<kBarycentric><<<grid, kBaseThreads, 0, s>>>(a);
}

void launch_baseline(const BaselineArgs& a, int mode, cudaStream_t s) {
    if (a.n_r <= 0) return;
    count_launches(1);
    const unsigned grid = (unsigned)((a.n_r + kBaseThreads - 1) / kBaseThreads);
    if (mode == kBoolean) k_baseline<kBoolean><<<grid, kBaseThreads, 0, s>>>(a);
    else if (mode == kCount) k_baseline<kCount><<<grid, kBaseThreads, 0, s>>>(a);
    else k_baseline<kBarycentric><<<grid, kBaseThreads, 0, s>>>(a);
}

}  // namespace rs
