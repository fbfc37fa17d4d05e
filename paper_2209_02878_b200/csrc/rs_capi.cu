// rs_capi.cu -- the extern "C" boundary (include/raysurf_b200.h) and the
// native host runtime behind it: stream-ordered device memory (cudaMallocAsync
// pool), tree lifetime, status read-back, and the chunked H2D / query / D2H
// pipeline of rs_run_batch_host.
#include <atomic>
#include <chrono>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <map>
#include <tuple>
#include <memory>
#include <set>
#include <vector>
#include <condition_variable>
#include <mutex>
#include <thread>
#include <string>

#include "../../include/raysurf_b200.h"
#include "rs_common.cuh"
#include "rs_internal.h"

using namespace rs;

namespace rs {
void hot_kernel_mark(int which, cudaStream_t s);
static std::atomic<long long> g_launches{0};
void count_launches(long long k) { g_launches.fetch_add(k, std::memory_order_relaxed); }

// Per-device launch facts, safe for concurrent callers and for processes
// that drive several GPUs: the SM count, occupancy per (kernel, block,
// dynamic smem) and the max-dynamic-shared-memory opt-in (a per-device,
// per-function attribute) are cached per device under one mutex.
static std::mutex g_dev_mu;
static std::map<std::tuple<int, const void*, int, size_t>, int> g_occ;
static std::set<std::pair<int, const void*>> g_smem_attr;
static std::map<int, int> g_sms;

int current_device() {
    int dev = 0;
    cudaGetDevice(&dev);
    return dev;
}

int device_sms() {
    const int dev = current_device();
    std::lock_guard<std::mutex> lk(g_dev_mu);
    auto it = g_sms.find(dev);
    if (it != g_sms.end()) return it->second;
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (sms < 1) sms = 1;
    g_sms[dev] = sms;
    return sms;
}

int occupancy(const void* kernel, int threads, size_t smem) {
    const auto key = std::make_tuple(current_device(), kernel, threads, smem);
    std::lock_guard<std::mutex> lk(g_dev_mu);
    auto it = g_occ.find(key);
    if (it != g_occ.end()) return it->second;
    int o = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, kernel, threads, smem);
    cudaGetLastError();
    if (o < 1) o = 1;
    g_occ[key] = o;
    return o;
}

void ensure_dynamic_smem(const void* kernel, int bytes) {
    const auto key = std::make_pair(current_device(), kernel);
    std::lock_guard<std::mutex> lk(g_dev_mu);
    if (g_smem_attr.count(key)) return;
    cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
    g_smem_attr.insert(key);
}
}  // namespace rs

struct rs_tree {
    int64_t n;
    int kind;
    char* block;
    RsHeader* hdr;
    RsNode* nodes;
    RsLeaf* leaves;
    RsNode4* nodes4;  // fast trees only
    TreeArrays ta;
    // lean fast trees keep their sorted keys (+ a sample of every stride-th)
    // for the traversal's Morton-range candidate lists; freed with the tree
    char* scratch = nullptr;
    const unsigned long long* codes = nullptr;
    unsigned long long* code_samples = nullptr;
    int sample_stride = 0, n_samples = 0, key_mode = 0;
    // leaf index by triangle id (the barycentric compaction's t recompute;
    // part of the tree block, rewritten by every barycentric fast query --
    // concurrent queries on one tree write identical values)
    int* leaf_of = nullptr;
};

namespace {

thread_local std::string g_err;

// RS_BINARY_FAST=1: traverse fast trees with the binary kernels (A/B tuning).
const bool g_binary_fast = [] {
    const char* e = getenv("RS_BINARY_FAST");
    return e && e[0] == '1';
}();

// ---- device timing marks ---------------------------------------------------
//
// The reference fills ResultSet.timings with per-phase seconds
// (engine.py:238-288: "ray sort", "ray boxes", "quantization", "encoding",
// "sorting", "reset", "construct", "query").  Here the phases run on the
// device (two streams), so they are timed with CUDA events: every call
// records (tag, event) marks in enqueue order, and a phase is the summed
// elapsed time over its (start tag, next end tag) pairs, which also covers
// the host pipeline's per-chunk binning and traversal.  Tags: 0 call start,
// 1/2 query start/end, 3/4 traversal kernel start/end, 5 + k stage k (0 prep
// done, 1 sort done, 2 climb done, 4 binning start, 8 binning done, 13 keys
// done, others diagnostic).
//
// Levels (rs_set_timing): 0 off, 1 the reference's phases (+ traversal
// kernel), 2 the traversal kernel only (bench's timed region), 3 every stage.
// Inside a captured graph each mark hangs off a side branch (forked from
// its stream, joined only at the graph's end): in the kernel chain every
// event-record node added ~6 us of latency per call.
int default_timing() {  // RS_TIMING overrides the default level (1) of a new thread
    const char* e = getenv("RS_TIMING");
    return e && e[0] >= '0' && e[0] <= '3' ? e[0] - '0' : 1;
}
thread_local int g_timing = default_timing();
constexpr int kStageEvents = 16;
constexpr int kTagStage = 5;
constexpr int kTagCount = kTagStage + kStageEvents;
struct Mark {
    int tag;
    cudaEvent_t ev;
};
thread_local std::vector<cudaEvent_t> g_pool;  // timing events, reused across calls
thread_local size_t g_pool_used = 0;
thread_local std::vector<Mark> g_marks;        // the current call's marks
thread_local std::vector<cudaEvent_t> g_fj;    // capture-time fork/join events
thread_local size_t g_fj_used = 0;
thread_local std::vector<cudaEvent_t> g_joins;
thread_local cudaStream_t g_tstream = nullptr;
thread_local float g_host_ms[2] = {};

// the last call's results, computed from its marks (eagerly after a graph
// replay, whose events belong to the graph; lazily otherwise)
constexpr int kPhaseCount = 7;  // ray boxes, quantization, encoding, sorting, reset, construct, query
struct TimingResult {
    bool valid = false;
    float phase[kPhaseCount];
    float build, query, hot;
    float stage[kStageEvents];
};
thread_local TimingResult g_tres;
thread_local bool g_have_marks = false;

// hot-kernel mark mask: bit 0 records the start event, bit 1 the end event
// (a batch traversed in two parts marks the first part's start and the
// second part's end)
thread_local int g_hot_mark_mask = 3;

bool mark_enabled(int tag) {
    switch (g_timing) {
        case 1:
            return tag <= 4 || tag == kTagStage + 0 || tag == kTagStage + 1 || tag == kTagStage + 2 ||
                   tag == kTagStage + 4 || tag == kTagStage + 8 || tag == kTagStage + 13;
        case 2: return tag == 3 || tag == 4;
        case 3: return true;
        default: return false;
    }
}

cudaEvent_t take_event(std::vector<cudaEvent_t>& pool, size_t& used, unsigned flags) {
    if (used == pool.size()) {
        cudaEvent_t e = nullptr;
        cudaEventCreateWithFlags(&e, flags);
        pool.push_back(e);
    }
    return pool[used++];
}

// A new top-level call: forget the previous call's marks.
void marks_reset() {
    g_pool_used = 0;
    g_marks.clear();
    g_tres.valid = false;
    g_have_marks = false;
}

void mark(int tag, cudaStream_t s) {
    if (!mark_enabled(tag)) return;
    cudaEvent_t ev = take_event(g_pool, g_pool_used, cudaEventDefault);
    g_marks.push_back({tag, ev});
    g_have_marks = true;
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    cudaStreamIsCapturing(s, &cs);
    if (cs != cudaStreamCaptureStatusActive) {
        cudaEventRecord(ev, s);
        return;
    }
    if (!g_tstream) cudaStreamCreateWithFlags(&g_tstream, cudaStreamNonBlocking);
    cudaEvent_t fork = take_event(g_fj, g_fj_used, cudaEventDisableTiming);
    cudaEvent_t join = take_event(g_fj, g_fj_used, cudaEventDisableTiming);
    cudaEventRecord(fork, s);
    cudaStreamWaitEvent(g_tstream, fork, 0);
    cudaEventRecordWithFlags(ev, g_tstream, cudaEventRecordExternal);  // a timing node of the graph
    cudaEventRecord(join, g_tstream);
    g_joins.push_back(join);
}

void ev_record(int k, cudaStream_t s) { mark(k, s); }

// joins the side branches back into s (before a capture ends)
void timing_join(cudaStream_t s) {
    for (cudaEvent_t j : g_joins) cudaStreamWaitEvent(s, j, 0);
    g_joins.clear();
    g_fj_used = 0;
}

// Summed elapsed ms over (a, next b) pairs of `m`; -1 when no pair exists.
float pair_sum(const std::vector<Mark>& m, int a, int b) {
    float total = 0.f;
    bool any = false;
    for (size_t i = 0; i < m.size(); ++i) {
        if (m[i].tag != a) continue;
        for (size_t j = i + 1; j < m.size(); ++j) {
            if (m[j].tag != b) continue;
            float ms = 0.f;
            cudaEventSynchronize(m[j].ev);
            if (cudaEventElapsedTime(&ms, m[i].ev, m[j].ev) == cudaSuccess) {
                total += ms;
                any = true;
            }
            break;
        }
    }
    cudaGetLastError();
    return any ? total : -1.f;
}

TimingResult compute_timings(const std::vector<Mark>& m) {
    TimingResult r;
    const int S = kTagStage;
    r.phase[0] = pair_sum(m, S + 4, S + 8);   // ray boxes: segment boxes + spatial binning
    r.phase[1] = pair_sum(m, S + 0, S + 13);  // quantization (+ encoding, one fused kernel)
    r.phase[2] = r.phase[1] >= 0.f ? 0.f : -1.f;
    r.phase[3] = pair_sum(m, S + 13, S + 1);  // sorting
    r.phase[4] = pair_sum(m, 0, S + 0);       // reset (+ triangle boxes, centroids, support)
    r.phase[5] = pair_sum(m, S + 1, S + 2);   // construct (climb)
    if (r.phase[5] < 0.f) r.phase[5] = pair_sum(m, S + 0, S + 2);  // from caller-sorted keys
    r.phase[6] = pair_sum(m, 1, 2);           // query (traversal + compaction)
    r.build = pair_sum(m, 0, S + 2);
    r.query = r.phase[6];
    r.hot = pair_sum(m, 3, 4);
    for (int k = 0; k < kStageEvents; ++k) r.stage[k] = pair_sum(m, 0, S + k);
    r.stage[11] = g_host_ms[0];
    r.stage[12] = g_host_ms[1];
    r.stage[14] = pair_sum(m, 0, 3);
    r.stage[15] = pair_sum(m, 0, 4);
    r.valid = true;
    return r;
}

const TimingResult* last_timings() {
    if (!g_tres.valid && g_have_marks) g_tres = compute_timings(g_marks);
    return g_tres.valid ? &g_tres : nullptr;
}

int fail(int code, const char* fmt, ...) __attribute__((format(printf, 2, 3)));
int fail(int code, const char* fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    g_err = buf;
    return code;
}

#define CK(expr)                                                                          \
    do {                                                                                  \
        cudaError_t e_ = (expr);                                                          \
        if (e_ != cudaSuccess)                                                            \
            return fail(RS_CUDA_ERROR, "%s failed: %s (%s:%d)", #expr, cudaGetErrorString(e_), \
                        __FILE__, __LINE__);                                              \
    } while (0)

inline cudaStream_t S(void* s) { return reinterpret_cast<cudaStream_t>(s); }

inline size_t align256(size_t x) { return (x + 255) & ~size_t(255); }

// Carves consecutive 256-B aligned sub-buffers out of one allocation.
struct Carver {
    char* base;
    size_t off = 0;
    template <class T>
    T* take(size_t count) {
        T* p = reinterpret_cast<T*>(base + off);
        off += align256(count * sizeof(T));
        return p;
    }
};

size_t tree_bytes(int64_t n) {
    size_t b = align256(sizeof(RsHeader));
    b += align256(sizeof(RsNode) * (size_t)(n > 1 ? n - 1 : 1));
    b += align256(sizeof(RsLeaf) * (size_t)n);
    b += 2 * align256(sizeof(float) * 6 * (size_t)n);
    b += 11 * align256(sizeof(int) * (size_t)n);
    b += 2 * align256(sizeof(int) * 2 * (size_t)n);
    b += align256(sizeof(RsNode4) * (size_t)(n > 1 ? n - 1 : 1));
    return b;
}

void carve_tree(rs_tree* t) {
    Carver c{t->block};
    const size_t n = (size_t)t->n;
    t->hdr = c.take<RsHeader>(1);
    t->nodes = c.take<RsNode>(n > 1 ? n - 1 : 1);
    t->leaves = c.take<RsLeaf>(n);
    t->ta.int_bounds = c.take<float>(6 * n);
    t->ta.leaf_bounds = c.take<float>(6 * n);
    t->ta.child_l = c.take<int>(n);
    t->ta.child_r = c.take<int>(n);
    t->ta.range_l = c.take<int>(n);
    t->ta.range_r = c.take<int>(n);
    t->ta.int_tri = c.take<int>(n);
    t->ta.visit = c.take<int>(n);
    t->ta.leaf_tri = c.take<int>(n);
    t->ta.leaf_range_l = c.take<int>(n);
    t->ta.leaf_range_r = c.take<int>(n);
    t->ta.sorted_ids = c.take<int>(n);
    t->ta.height = c.take<int>(2 * n);
    t->ta.parent = c.take<int>(2 * n);
    t->nodes4 = c.take<RsNode4>(n > 1 ? n - 1 : 1);
    t->leaf_of = c.take<int>(n);
}

std::mutex g_pool_mu;
std::set<int> g_pool_configured;  // devices whose default pool keeps freed blocks

int configure_pool() {
    int dev = 0;
    CK(cudaGetDevice(&dev));
    std::lock_guard<std::mutex> lk(g_pool_mu);
    if (g_pool_configured.count(dev)) return RS_OK;
    cudaMemPool_t pool;
    CK(cudaDeviceGetDefaultMemPool(&pool, dev));
    unsigned long long thr = ~0ull;  // keep freed blocks cached in the pool
    CK(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr));
    g_pool_configured.insert(dev);
    return RS_OK;
}

int check_mesh(int64_t n_v, int64_t n_t) {
    if (n_t < 1) return fail(RS_INVALID_ARG, "cannot build a BVH over an empty mesh");
    if (n_t > 2147483647ll)
        return fail(RS_INVALID_ARG, "triangle count %lld exceeds capacity 2147483647", (long long)n_t);
    if (n_v < 3 || n_v > 2147483647ll)
        return fail(RS_INVALID_ARG, "vertex count %lld out of range", (long long)n_v);
    return RS_OK;
}

// Device memory of a captured graph.  A graph replayed every call keeps its
// scratch in one arena it owns (one cudaMalloc at capture time) instead of
// stream-ordered allocation and free nodes: the capture runs twice, once to
// size the arena (mode 1: allocations pass through and are summed), once to
// bump-allocate from it (mode 2: frees inside it are no-ops).
struct Arena {
    char* base = nullptr;
    size_t cap = 0, off = 0;
    int mode = 0;  // 0 off, 1 sizing, 2 bump
};
static thread_local Arena g_arena;

static cudaError_t dmalloc(void** p, size_t bytes, cudaStream_t s) {
    const size_t need = align256(bytes > 0 ? bytes : 1);
    if (g_arena.mode == 2) {
        if (g_arena.off + need > g_arena.cap) return cudaErrorMemoryAllocation;
        *p = g_arena.base + g_arena.off;
        g_arena.off += need;
        return cudaSuccess;
    }
    if (g_arena.mode == 1) g_arena.off += need;
    return cudaMallocAsync(p, bytes, s);
}
static cudaError_t dfree(void* p, cudaStream_t s) {
    if (g_arena.mode == 2 && static_cast<char*>(p) >= g_arena.base &&
        static_cast<char*>(p) < g_arena.base + g_arena.cap)
        return cudaSuccess;
    return cudaFreeAsync(p, s);
}

int alloc_tree(int64_t n, int kind, cudaStream_t s, rs_tree** out) {
    int rc = configure_pool();
    if (rc) return rc;
    rs_tree* t = new rs_tree();
    t->n = n;
    t->kind = kind;
    cudaError_t e = dmalloc(reinterpret_cast<void**>(&t->block), tree_bytes(n), s);
    if (e != cudaSuccess) {
        delete t;
        return fail(RS_CUDA_ERROR, "device allocation of %zu bytes failed: %s", tree_bytes(n),
                    cudaGetErrorString(e));
    }
    carve_tree(t);
    *out = t;
    return RS_OK;
}

// nodes4 (the 4-wide collapse) is read by the collision-buffer path and the
// A/B traversal variants
bool need_nodes4() {
    const bool buffer = rs::fast_path() == 1;
    long long trav = 0, wide = 0;
    rs::sorted_option("trav", -1, &trav);
    rs::sorted_option("tile_wide", -1, &wide);
    return buffer || trav == 2 || (wide && trav != 1);
}

// RS_ZERO_COPY=1: the compaction writes barycentric rows straight into mapped
// pinned host outputs (A/B: 3% slower than the lagged per-chunk copies).
static const bool g_zero_copy = [] {
    const char* e = getenv("RS_ZERO_COPY");
    return e && e[0] == '1';
}();

// RS_LEAN_BUILD=0: query-only fast trees keep the full reference SoA (A/B).
static const bool g_lean_build = [] {
    const char* e = getenv("RS_LEAN_BUILD");
    return !(e && e[0] == '0');
}();

// after_prep (optional) runs on the host right after k_prep is enqueued on
// `s`: the fast query forks its binning onto a second stream there, since it
// needs only the root box k_prep computes.
int build_impl(const float* V, int64_t n_v, const int* T, int64_t n_t, int kind,
               const uint64_t* sorted_codes, const int* sorted_ids, cudaStream_t s,
               rs_tree** out, const std::function<int(rs_tree*)>& after_prep = nullptr,
               bool lean = false) {
    int rc = check_mesh(n_v, n_t);
    if (rc) return rc;
    if (kind != kTreeReference && kind != kTreeFast)
        return fail(RS_INVALID_ARG, "unknown tree kind %d", kind);
    rs_tree* t = nullptr;
    rc = alloc_tree(n_t, kind, s, &t);
    if (rc) return rc;
    const int n = (int)n_t;
    CK(cudaMemsetAsync(t->hdr, 0, sizeof(RsHeader), s));
    if (sorted_codes) {
        launch_prep(V, T, n, nullptr, t->hdr, t->ta, false, s);
        stage_mark(0, s);
        launch_climb(V, T, n, reinterpret_cast<const unsigned long long*>(sorted_codes),
                     sorted_ids, t->ta, t->nodes, t->leaves, t->hdr, s);
        stage_mark(2, s);
    } else {
        const int passes = kind == kTreeFast ? 4 : 8;  // 30-bit vs 63-bit keys
        const size_t sb = sort_scratch_bytes(n, passes);
        constexpr int kMaxSamples = 1024;
        const size_t bytes = align256(24ull * n) + 2 * align256(8ull * n) + 2 * align256(4ull * n) +
                             align256(sb) + align256(8ull * kMaxSamples);
        char* scratch = nullptr;
        CK(dmalloc(reinterpret_cast<void**>(&scratch), bytes, s));
        Carver c{scratch};
        double* cent = c.take<double>(3ull * n);
        unsigned long long* keys = c.take<unsigned long long>(n);
        unsigned long long* keys2 = c.take<unsigned long long>(n);
        int* vals = c.take<int>(n);
        int* vals2 = c.take<int>(n);
        void* sort_scratch = c.take<char>(sb);
        unsigned long long* samples = c.take<unsigned long long>(kMaxSamples);
        // lean: a fast tree only this call queries (never downloaded, no
        // 4-wide collapse): records only
        lean = lean && kind == kTreeFast && !need_nodes4() && g_lean_build;
        launch_prep(V, T, n, cent, t->hdr, t->ta, true, s, lean);
        if (after_prep) {
            rc = after_prep(t);
            if (rc) return rc;
        }
        stage_mark(0, s);
        launch_keys(cent, n, t->hdr, kind, keys, vals, s);
        stage_mark(13, s);
        launch_sort(keys, vals, keys2, vals2, n, passes, sort_scratch, s);
        stage_mark(1, s);
        if (lean) launch_climb_lean(V, T, n, keys, vals, t->ta.visit, t->nodes, t->leaves, t->hdr,
                                    t->ta.leaf_bounds, s);
        else launch_climb(V, T, n, keys, vals, t->ta, t->nodes, t->leaves, t->hdr, s);
        if (kind == kTreeFast && need_nodes4()) launch_collapse(n, t->ta, t->nodes, t->nodes4, t->hdr, s);
        stage_mark(2, s);
        if (lean) {  // sorted keys stay with the tree (4 passes: the result is in `keys`)
            t->sample_stride = (n + kMaxSamples - 1) / kMaxSamples;
            t->n_samples = (n + t->sample_stride - 1) / t->sample_stride;
            launch_code_samples(keys, n, t->sample_stride, samples, t->n_samples, s);
            t->scratch = scratch;
            t->codes = keys;
            t->code_samples = samples;
            t->key_mode = fast_key_mode() == 1 ? 1 : 0;
        } else {
            CK(dfree(scratch, s));
        }
    }
    CK(cudaGetLastError());
    *out = t;
    return RS_OK;
}

int check_query(int mode, int max_coll, int max_stack) {
    if (mode < 0 || mode > 2) return fail(RS_INVALID_ARG, "unknown mode %d", mode);
    if (max_coll < 2) return fail(RS_INVALID_ARG, "collision buffer needs capacity >= 2");
    if (max_stack < 1) return fail(RS_INVALID_ARG, "traversal stack needs capacity >= 1");
    return RS_OK;
}

int kstack_for(bool ref, int max_stack) {
    if (!ref) return 64;  // fast tree height <= 61 (30 code bits + 31 id bits)
    return max_stack < 128 ? max_stack : 128;  // reference tree height <= 94
}

QueryArgs make_args(const rs_tree* t, const float* s, const float* e, int64_t n_r, int max_coll,
                    int max_stack, RsStatus* st) {
    QueryArgs a{};
    a.nodes = t->nodes;
    a.nodes4 = t->kind == kTreeFast ? t->nodes4 : nullptr;
    a.leaves = t->leaves;
    a.hdr = t->hdr;
    a.n_int = (int)(t->n - 1);
    a.starts = s;
    a.ends = e;
    a.n_r = n_r;
    a.max_coll = max_coll;
    a.max_stack = max_stack;
    a.status = st;
    return a;
}

int read_status(RsStatus* d_st, cudaStream_t s, RsStatus* h) {
    CK(cudaMemcpyAsync(h, d_st, sizeof(RsStatus), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    return RS_OK;
}

int status_code(const RsStatus& h, int64_t* bad_segment) {
    if (bad_segment) *bad_segment = h.bad ? (int64_t)~h.bad : -1;
    if (h.bad) return fail(RS_STACK_OVERFLOW, "traversal stack overflow");
    if (h.internal) return fail(RS_INTERNAL, "internal traversal capacity exceeded");
    return RS_OK;
}

// Per-thread cached pipeline resources for rs_run_batch_host.
struct Pipe {
    int device = -1;
    cudaStream_t copy = nullptr, copy2 = nullptr;  // H2D (both endpoint arrays) / D2H
    cudaEvent_t ev_in[2], ev_in2[2], ev_q[2], ev_out[2], ev_blk;
    RsStatus* hst = nullptr;  // pinned per-chunk statuses (barycentric row counts)
    int64_t hst_cap = 0;
    char* stg = nullptr;      // pinned staging for pageable inputs (2 chunk slots + mesh)
    size_t stg_cap = 0;
    unsigned* hbits = nullptr;  // pinned landing area of the packed boolean flags
    size_t hbits_cap = 0;       // words
};
thread_local Pipe g_pipe;

// Pageable host inputs are staged through pinned buffers: cudaMemcpyAsync
// from pageable memory runs at ~11 GB/s (the driver's own staging, CPU and
// DMA serialised), while several threads copying into pinned memory reach
// ~45 GB/s and the DMA of chunk k overlaps the copy of chunk k+1.  A small
// persistent pool (the caller takes one share of every copy).
class CopyPool {
  public:
    static CopyPool& get() {
        static CopyPool* p = new CopyPool();  // never destroyed: workers live for the process
        return *p;
    }
    void copy(void* dst, const void* src, size_t bytes) {
        if (bytes < (1u << 20) || workers_ == 0) {
            std::memcpy(dst, src, bytes);
            return;
        }
        char* d = static_cast<char*>(dst);
        const char* sp = static_cast<const char*>(src);
        parallel([=](int k, int parts) {
            const size_t per = ((bytes + parts - 1) / parts + 63) & ~size_t(63);
            const size_t lo = per * (size_t)k;
            if (lo < bytes) std::memcpy(d + lo, sp + lo, std::min(per, bytes - lo));
        });
    }
    // job(k, parts) for k = 0..parts-1, one part on the caller
    void parallel(const std::function<void(int, int)>& job) {
        if (workers_ == 0) {
            job(0, 1);
            return;
        }
        std::lock_guard<std::mutex> one(call_mu_);  // one parallel job at a time
        const int parts = workers_ + 1;
        {
            std::lock_guard<std::mutex> lk(mu_);
            job_ = &job;
            parts_ = parts;
            pending_ = workers_;
            ++gen_;
        }
        cv_.notify_all();
        job(0, parts);
        std::unique_lock<std::mutex> lk(mu_);
        done_cv_.wait(lk, [&] { return pending_ == 0; });
        job_ = nullptr;
    }
    int parts() const { return workers_ + 1; }

  private:
    CopyPool() {
        const unsigned hw = std::thread::hardware_concurrency();
        const char* e = getenv("RS_COPY_THREADS");
        // B200 box (16 host threads): 2 copiers 11.2 ms, 4 9.1 ms, 8 7.0 ms
        // per pageable 10M-segment C2 call
        workers_ = e && *e ? atoi(e) : (int)(hw >= 16 ? 8 : (hw > 1 ? hw / 2 : 0));
        for (int w = 0; w < workers_; ++w) std::thread([this, w] { loop(w + 1); }).detach();
    }
    void loop(int k) {
        unsigned long long seen = 0;
        for (;;) {
            const std::function<void(int, int)>* job;
            int parts;
            {
                std::unique_lock<std::mutex> lk(mu_);
                cv_.wait(lk, [&] { return gen_ != seen; });
                seen = gen_;
                job = job_;
                parts = parts_;
            }
            (*job)(k, parts);
            {
                std::lock_guard<std::mutex> lk(mu_);
                if (--pending_ == 0) done_cv_.notify_one();
            }
        }
    }
    int workers_ = 0;
    std::mutex call_mu_, mu_;
    std::condition_variable cv_, done_cv_;
    const std::function<void(int, int)>* job_ = nullptr;
    int parts_ = 1, pending_ = 0;
    unsigned long long gen_ = 0;
};

// dst[i] = bit i of bits, i < n (the packed boolean flags, expanded on the
// host threads)
static void expand_bits_host(const unsigned* bits, int64_t n, int32_t* dst) {
    const int64_t words = (n + 31) / 32;
    auto run = [&](int64_t w0, int64_t w1) {
        for (int64_t w = w0; w < w1; ++w) {
            const unsigned b = bits[w];
            int32_t* d = dst + 32 * w;
            const int m = (int)std::min<int64_t>(32, n - 32 * w);
            if (m == 32) {
                for (int j = 0; j < 32; ++j) d[j] = (int32_t)((b >> j) & 1u);
            } else {
                for (int j = 0; j < m; ++j) d[j] = (int32_t)((b >> j) & 1u);
            }
        }
    };
    if (words < 4096) {
        run(0, words);
        return;
    }
    CopyPool::get().parallel([&](int k, int parts) {
        const int64_t per = (words + parts - 1) / parts;
        const int64_t w0 = per * k, w1 = std::min(words, w0 + per);
        if (w0 < w1) run(w0, w1);
    });
}
// RS_PACK_FLAGS=0: boolean flags come back as int32 (A/B)
static const bool g_pack_flags = [] {
    const char* e = getenv("RS_PACK_FLAGS");
    return !(e && e[0] == '0');
}();

bool is_pageable(const void* p) {
    cudaPointerAttributes at{};
    if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
        cudaGetLastError();
        return true;
    }
    return at.type == cudaMemoryTypeUnregistered;
}

// per thread and per device: a thread that drives several GPUs keeps each
// device's streams, events and pinned buffers (g_pipe is the current one)
thread_local std::map<int, Pipe> g_pipes;

int pipe_init() {
    int dev;
    CK(cudaGetDevice(&dev));
    if (g_pipe.device == dev) return RS_OK;
    if (g_pipe.device >= 0) g_pipes[g_pipe.device] = g_pipe;  // park the previous device's set
    auto it = g_pipes.find(dev);
    if (it != g_pipes.end()) {
        g_pipe = it->second;
        return RS_OK;
    }
    g_pipe = Pipe{};
    CK(cudaStreamCreateWithFlags(&g_pipe.copy, cudaStreamNonBlocking));
    CK(cudaStreamCreateWithFlags(&g_pipe.copy2, cudaStreamNonBlocking));
    for (int k = 0; k < 2; ++k) {
        CK(cudaEventCreateWithFlags(&g_pipe.ev_in[k], cudaEventDisableTiming));
        CK(cudaEventCreateWithFlags(&g_pipe.ev_in2[k], cudaEventDisableTiming));
        CK(cudaEventCreateWithFlags(&g_pipe.ev_q[k], cudaEventDisableTiming));
        CK(cudaEventCreateWithFlags(&g_pipe.ev_out[k], cudaEventDisableTiming));
    }
    CK(cudaEventCreateWithFlags(&g_pipe.ev_blk, cudaEventDisableTiming));
    g_pipe.device = dev;
    return RS_OK;
}

}  // namespace

// ===================================================================== ABI ==

extern "C" {

int rs_abi_version(void) { return 1; }

const char* rs_last_error(void) { return g_err.c_str(); }

int rs_build(const float* d_verts, int64_t n_v, const int32_t* d_tris, int64_t n_t,
             int tree_kind, void* stream, rs_tree** out) {
    marks_reset();
    if (!out) return fail(RS_INVALID_ARG, "null output handle");
    mark(0, S(stream));
    return build_impl(d_verts, n_v, d_tris, n_t, tree_kind, nullptr, nullptr, S(stream), out);
}

int rs_build_from_sorted(const float* d_verts, int64_t n_v, const int32_t* d_tris, int64_t n_t,
                         const uint64_t* d_sorted_codes, const int32_t* d_sorted_ids,
                         void* stream, rs_tree** out) {
    marks_reset();
    if (!out || !d_sorted_codes || !d_sorted_ids) return fail(RS_INVALID_ARG, "null argument");
    mark(0, S(stream));
    return build_impl(d_verts, n_v, d_tris, n_t, kTreeReference, d_sorted_codes, d_sorted_ids,
                      S(stream), out);
}

int rs_tree_info(const rs_tree* t, int64_t* n_tri, int32_t* root, int32_t* height,
                 int32_t* kind, void* stream) {
    if (!t) return fail(RS_INVALID_ARG, "null tree");
    RsHeader h;
    CK(cudaMemcpyAsync(&h, t->hdr, sizeof h, cudaMemcpyDeviceToHost, S(stream)));
    CK(cudaStreamSynchronize(S(stream)));
    if (n_tri) *n_tri = t->n;
    if (root) *root = h.root;
    if (height) *height = h.height;
    if (kind) *kind = t->kind;
    return RS_OK;
}

int rs_tree_download(const rs_tree* t, float* ib, int32_t* cl, int32_t* cr, int32_t* rl,
                     int32_t* rr, int32_t* it, int32_t* vi, float* lb, int32_t* lt, int32_t* lrl,
                     int32_t* lrr, int32_t* si, void* stream) {
    if (!t) return fail(RS_INVALID_ARG, "null tree");
    const size_t n = (size_t)t->n;
    cudaStream_t s = S(stream);
    struct { void* h; const void* d; size_t b; } cp[] = {
        {ib, t->ta.int_bounds, 24 * n}, {cl, t->ta.child_l, 4 * n}, {cr, t->ta.child_r, 4 * n},
        {rl, t->ta.range_l, 4 * n}, {rr, t->ta.range_r, 4 * n}, {it, t->ta.int_tri, 4 * n},
        {vi, t->ta.visit, 4 * n}, {lb, t->ta.leaf_bounds, 24 * n}, {lt, t->ta.leaf_tri, 4 * n},
        {lrl, t->ta.leaf_range_l, 4 * n}, {lrr, t->ta.leaf_range_r, 4 * n},
        {si, t->ta.sorted_ids, 4 * n}};
    for (auto& c : cp)
        if (c.h) CK(cudaMemcpyAsync(c.h, c.d, c.b, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    return RS_OK;
}

int rs_free(rs_tree* t, void* stream) {
    if (!t) return RS_OK;
    if (t->scratch) dfree(t->scratch, S(stream));
    cudaError_t e = dfree(t->block, S(stream));
    delete t;
    if (e != cudaSuccess) return fail(RS_CUDA_ERROR, "cudaFreeAsync: %s", cudaGetErrorString(e));
    return RS_OK;
}

// Fast-tree query: 4-lane traversal -> collision buffer -> exact tests (->
// barycentric compaction).  Outputs: boolean/count -> flags (dense); bary ->
// compact rows (c_*) or dense rows (det/tri/dist/pts).  The collision buffer
// starts at 2 x n_r entries; if the traversal claimed more, everything is
// re-launched once with a buffer of exactly the claimed size.
struct FastOut {
    int32_t* flags = nullptr;
    int32_t *det = nullptr, *tri = nullptr;
    float *dist = nullptr, *pts = nullptr;
    int32_t *c_ray = nullptr, *c_tri = nullptr;
    float *c_dist = nullptr, *c_pt = nullptr;
    long long ray_offset = 0;
    unsigned long long* row_base = nullptr;  // compact rows: running row count across chunks
    bool mapped = false;  // compact rows go to host-mapped memory
};

struct FastScratch {
    char* blk = nullptr;
    RsStatus* st = nullptr;
    int2* cand = nullptr;
    int* chunk_fill = nullptr;
    unsigned long long *best_t = nullptr, *cand_t = nullptr, *tiles = nullptr, *tile_ctr = nullptr;
    int* best_tri = nullptr;
    long long cap = 0;
    size_t tiles_bytes = 0;
    int* gstack = nullptr;
    unsigned *bins = nullptr, *cursor = nullptr, *n_live = nullptr;
    float4* rec = nullptr;
    void* geom = nullptr;
    unsigned* hitbits = nullptr;  // large boolean batches: hit bitmap (see SortedArgs::hitbits)
    bool leaf_of_ready = false;   // barycentric: the tree's leaf_of inverse already built
};

// Boolean batches from this many segments on set hit bits instead of
// writing int32 flags at random (RS_HITBITS_MIN; C5 1B: the flags' partial
// sectors were half the traversal's 65 GB of DRAM traffic).
static std::atomic<long long> g_hitbits_min{[] {
    const char* e = getenv("RS_HITBITS_MIN");
    return e && *e ? atoll(e) : (1ll << 25);
}()};

// fast_path option 1 (or RS_FAST_PATH=buffer): pair traversal -> collision
// buffer -> exact pass; default 0: the binned tile traversal.
static bool buffer_path() { return rs::fast_path() == 1; }

// `sized`: a re-launch with the capacity the overflowing launch claimed (the
// cand_cap test override applies to first launches only).
static int fast_alloc(FastScratch& f, int64_t n_r, int mode, long long cap, cudaStream_t s,
                      bool sized = false) {
    if (!buffer_path()) cap = kCandChunk;  // the sorted path has no collision buffer
    else if (rs::cand_cap_override() > 0 && !sized) cap = rs::cand_cap_override();
    cap = ((cap + kCandChunk - 1) / kCandChunk) * kCandChunk;
    const bool bary = mode == kBarycentric;
    size_t total = 256;
    total += align256(sizeof(RsStatus));
    total += align256(8ull * cap) + align256(4ull * (cap / kCandChunk + 1));
    // barycentric: the sorted path keeps only the winning triangle per
    // segment (the compaction recomputes t); the collision-buffer path's
    // atomicMin needs the t keys
    const bool keys = bary && buffer_path();
    if (bary)
        total += (keys ? align256(8ull * n_r) : 0) + align256(4ull * n_r) + align256(8ull * cap) +
                 align256(bary_compact_scratch(n_r));
    if (buffer_path()) total += align256(4 * trav_gstack_ints());
    const bool bits = mode == kBoolean && !buffer_path() && n_r >= g_hitbits_min.load();
    total += 3 * align256(4 * sorted_bins()) + align256(4 * (64 + 4 * 32)) + align256(32ull * n_r) +
             align256(bin_geom_bytes()) +
             (bits ? align256(4ull * ((n_r + 31) / 32)) : 0);
    CK(dmalloc(reinterpret_cast<void**>(&f.blk), total, s));
    Carver c{f.blk};
    f.st = c.take<RsStatus>(1);
    f.cand = c.take<int2>(cap);
    f.chunk_fill = c.take<int>(cap / kCandChunk + 1);
    if (bary) {
        f.best_t = keys ? c.take<unsigned long long>(n_r) : nullptr;
        f.best_tri = c.take<int>(n_r);
        f.cand_t = c.take<unsigned long long>(cap);
        f.tiles = c.take<unsigned long long>(bary_compact_scratch(n_r) / 8);
        f.tile_ctr = f.tiles + (bary_compact_scratch(n_r) / 8 - 1);
        f.tiles_bytes = bary_compact_scratch(n_r);
    }
    if (buffer_path()) f.gstack = c.take<int>(trav_gstack_ints());
    f.bins = c.take<unsigned>(2 * sorted_bins());  // counters + look-back words (zeroed together)
    f.cursor = c.take<unsigned>(sorted_bins());
    f.n_live = c.take<unsigned>(64 + 4 * 32);
    f.rec = c.take<float4>(2ull * n_r);
    f.geom = c.take<char>(bin_geom_bytes());
    f.hitbits = bits ? c.take<unsigned>((n_r + 31) / 32) : nullptr;
    f.cap = cap;
    return RS_OK;
}

static SortedArgs sorted_args(const rs_tree* t, const float* d_s, const float* d_e, int64_t n_r,
                              const FastOut& o, FastScratch& f) {
    SortedArgs a{t->nodes4, t->nodes, t->leaves, t->hdr, (int)(t->n - 1), d_s, d_e, n_r,
                      f.bins, f.cursor, f.n_live, reinterpret_cast<float*>(f.n_live + 64), f.bins + sorted_bins(), f.rec, o.flags,
                      f.best_t, f.best_tri, f.st};
    a.codes = t->codes;
    a.code_samples = t->code_samples;
    a.sample_stride = t->sample_stride;
    a.n_samples = t->n_samples;
    a.leaf_boxes = t->ta.leaf_bounds;
    a.key_mode = t->key_mode;
    a.geom = f.geom;
    a.hitbits = f.hitbits;
    return a;
}

// Phase 1 of the sorted fast path: output presets + spatial binning.  Needs
// only the tree header's root box, so it may run concurrently with the rest
// of the build on another stream.
static int fast_presets(const float* d_s, const float* d_e, int64_t n_r, int mode, const FastOut& o,
                        FastScratch& f, cudaStream_t s) {
    const bool bary = mode == kBarycentric;
    CK(cudaMemsetAsync(f.st, 0, sizeof(RsStatus), s));
    // boolean/count outputs start at 0: zeroed by the histogram pass when it
    // can; with a hit bitmap the bitmap starts at 0 and k_expand_bits writes
    // every flag
    if (f.hitbits) CK(cudaMemsetAsync(f.hitbits, 0, 4ull * ((n_r + 31) / 32), s));
    else if (!bary && !binning_zeroes_flags(d_s, d_e, n_r, o.flags)) CK(cudaMemsetAsync(o.flags, 0, 4ull * n_r, s));
    if (bary) {
        if (f.best_t) CK(cudaMemsetAsync(f.best_t, 0xFF, 8ull * n_r, s));
        CK(cudaMemsetAsync(f.best_tri, 0xFF, 4ull * n_r, s));
        CK(cudaMemsetAsync(f.tiles, 0, f.tiles_bytes, s));
    }
    CK(cudaMemsetAsync(f.bins, 0, 4 * sorted_bins() + 4 * (2 * (sorted_bins() / 1024) + 64), s));  // counters, look-back words, ticket
    stage_mark(4, s);
    return RS_OK;
}

static int fast_bin(const rs_tree* t, const float* d_s, const float* d_e, int64_t n_r, int mode,
                    const FastOut& o, FastScratch& f, cudaStream_t s, bool presets = true) {
    if (presets) {
        const int rc = fast_presets(d_s, d_e, n_r, mode, o, f, s);
        if (rc) return rc;
    }
    launch_binning(sorted_args(t, d_s, d_e, n_r, o, f), s, mode != kBarycentric);
    return RS_OK;
}

// Phase 2: traversal (+ barycentric compaction).
static int fast_trav(const rs_tree* t, const float* d_s, const float* d_e, int64_t n_r, int mode,
                     const FastOut& o, FastScratch& f, bool stats, cudaStream_t s,
                     bool first = true, bool last = true) {
    if (first) ev_record(1, s);
    launch_sorted_trav(sorted_args(t, d_s, d_e, n_r, o, f), mode, stats, s);
    if (f.hitbits) launch_expand_bits(o.flags, f.hitbits, n_r, s);
    if (mode == kBarycentric) {
        if (!f.best_t && !f.leaf_of_ready)  // the compaction recomputes t from the winning leaf
            launch_leaf_inverse(t->leaves, (int)t->n, t->leaf_of, s);
        CompactArgs ca{n_r, f.best_t, f.best_tri, d_s, d_e, o.c_ray, o.c_dist, o.c_tri, o.c_pt,
                       f.tiles, f.tile_ctr, &f.st->hits, o.ray_offset, o.row_base, t->leaves, t->leaf_of,
                       o.mapped};
        if (o.c_ray) launch_bary_compact(ca, s);
        else launch_bary_dense(ca, o.det, o.tri, o.dist, o.pts, s);
    }
    CK(cudaGetLastError());
    if (last) ev_record(2, s);
    return RS_OK;
}

static int fast_launch(const rs_tree* t, const float* d_s, const float* d_e, int64_t n_r, int mode,
                       const FastOut& o, FastScratch& f, bool stats, cudaStream_t s) {
    const bool bary = mode == kBarycentric;
    if (!buffer_path()) {
        int rc = fast_bin(t, d_s, d_e, n_r, mode, o, f, s);
        if (rc) return rc;
        return fast_trav(t, d_s, d_e, n_r, mode, o, f, stats, s);
    }
    CK(cudaMemsetAsync(f.st, 0, sizeof(RsStatus), s));
    if (!bary) CK(cudaMemsetAsync(o.flags, 0, 4ull * n_r, s));
    if (bary) {
        CK(cudaMemsetAsync(f.best_t, 0xFF, 8ull * n_r, s));
        CK(cudaMemsetAsync(f.best_tri, 0xFF, 4ull * n_r, s));
        CK(cudaMemsetAsync(f.tiles, 0, f.tiles_bytes, s));
    }
    ev_record(1, s);
    TravArgs ta{t->nodes4, t->hdr, (int)(t->n - 1), d_s, d_e, n_r, f.cand, f.cap, f.chunk_fill,
                f.st, f.gstack};
    launch_trav(ta, stats, s);
    ExactArgs ea{f.cand, &f.st->cand_count, f.cap, f.chunk_fill, d_s, d_e, t->leaves,
                 o.flags, f.best_t, f.best_tri, f.cand_t, &f.st->mts, &f.st->dropped};
    launch_exact(ea, mode, stats, s);
    if (bary) {
        CompactArgs ca{n_r, f.best_t, f.best_tri, d_s, d_e, o.c_ray, o.c_dist, o.c_tri, o.c_pt,
                       f.tiles, f.tile_ctr, &f.st->hits, o.ray_offset, o.row_base};
        if (o.c_ray) launch_bary_compact(ca, s);
        else launch_bary_dense(ca, o.det, o.tri, o.dist, o.pts, s);
    }
    CK(cudaGetLastError());
    ev_record(2, s);
    return RS_OK;
}

static int fast_query(const rs_tree* t, const float* d_s, const float* d_e, int64_t n_r, int mode,
                      const FastOut& o, bool stats, RsStatus* h, cudaStream_t s) {
    FastScratch f;
    long long cap = 2ll * n_r + 4096;
    for (int attempt = 0; attempt < 2; ++attempt) {
        int rc = fast_alloc(f, n_r, mode, cap, s, attempt > 0);
        if (rc) return rc;
        rc = fast_launch(t, d_s, d_e, n_r, mode, o, f, stats, s);
        if (!rc) rc = read_status(f.st, s, h);
        CK(dfree(f.blk, s));
        if (rc) return rc;
        if ((long long)h->cand_count <= f.cap) return RS_OK;
        cap = (long long)h->cand_count;  // collision buffer overflow: re-launch once, sized
    }
    return fail(RS_INTERNAL, "collision buffer overflow after re-launch");
}

// The pair traversal keeps a bounded shared-memory stack; a tree deep enough
// to exceed it (pathological inputs only) is re-queried with the binary
// kernels, whose stack covers the fast tree's full height.
static int binary_query(const rs_tree* t, const float* d_s, const float* d_e, int64_t n_r,
                        int mode, const FastOut& o, RsStatus* h, cudaStream_t s);

static int query_impl(const rs_tree* t, const float* d_s, const float* d_e, int64_t n_r, int mode,
                      int max_coll, int max_stack, int ref, int32_t* det, int32_t* cnt,
                      int32_t* tri, float* dist, float* pts, int32_t* c_ray, float* c_dist,
                      int32_t* c_tri, float* c_pt, int64_t* n_hits, int64_t* bad, bool stats,
                      int64_t* visits, int64_t* mts, cudaStream_t s) {
    if (!t) return fail(RS_INVALID_ARG, "null tree");
    int rc = check_query(mode, max_coll, max_stack);
    if (rc) return rc;
    if (n_r < 0) return fail(RS_INVALID_ARG, "negative segment count");
    if (n_r > 2147483647ll) return fail(RS_INVALID_ARG, "segment count exceeds int32 indexing");
    // statistics (rs_query_stats) come from the per-segment binary walk, the
    // unit SURVEY 8(d)'s V_int / N_mt count, on either tree kind
    if (t->kind == kTreeFast && n_r > 0 && !g_binary_fast && !stats) {
        FastOut o;
        o.flags = mode == kCount ? cnt : det;
        o.det = det; o.tri = tri; o.dist = dist; o.pts = pts;
        o.c_ray = c_ray; o.c_dist = c_dist; o.c_tri = c_tri; o.c_pt = c_pt;
        RsStatus h{};
        rc = fast_query(t, d_s, d_e, n_r, mode, o, stats, &h, s);
        if (rc) return rc;
        if (h.internal) {
            rc = binary_query(t, d_s, d_e, n_r, mode, o, &h, s);
            if (rc) return rc;
        }
        if (n_hits) *n_hits = (int64_t)h.hits;
        if (visits) *visits = (int64_t)h.visits;
        if (mts) *mts = (int64_t)h.mts;
        return status_code(h, bad);
    }
    const bool compact = c_ray != nullptr;
    const size_t cs = compact ? compact_scratch_bytes(n_r) : 0;
    char* blk = nullptr;
    CK(dmalloc(reinterpret_cast<void**>(&blk), align256(sizeof(RsStatus)) + cs + 256, s));
    RsStatus* st = reinterpret_cast<RsStatus*>(blk);
    CK(cudaMemsetAsync(blk, 0, align256(sizeof(RsStatus)) + cs, s));
    QueryArgs a = make_args(t, d_s, d_e, n_r, max_coll, max_stack, st);
    if (t->kind == kTreeFast) a.nodes4 = nullptr;  // binary kernels over the fast tree's records
    a.detected = det; a.counts = cnt; a.tri = tri; a.dist = dist; a.points = pts;
    a.c_ray = c_ray; a.c_dist = c_dist; a.c_tri = c_tri; a.c_point = c_pt;
    a.tile_status = reinterpret_cast<unsigned long long*>(blk + align256(sizeof(RsStatus)));
    ev_record(1, s);
    if (launch_query(a, mode, ref != 0, compact, kstack_for(ref != 0, max_stack), stats, s))
        return fail(RS_INVALID_ARG, "no kernel variant for this configuration");
    CK(cudaGetLastError());
    ev_record(2, s);
    RsStatus h;
    rc = read_status(st, s, &h);
    CK(dfree(blk, s));
    if (rc) return rc;
    if (n_hits) *n_hits = (int64_t)h.hits;
    if (visits) *visits = (int64_t)h.visits;
    if (mts) *mts = (int64_t)h.mts;
    return status_code(h, bad);
}

static int binary_query(const rs_tree* t, const float* d_s, const float* d_e, int64_t n_r,
                        int mode, const FastOut& o, RsStatus* h, cudaStream_t s) {
    const bool compact = o.c_ray != nullptr;
    char* blk = nullptr;
    const size_t cs = compact ? compact_scratch_bytes(n_r) : 0;
    CK(dmalloc(reinterpret_cast<void**>(&blk), align256(sizeof(RsStatus)) + cs + 256, s));
    CK(cudaMemsetAsync(blk, 0, align256(sizeof(RsStatus)) + cs, s));
    RsStatus* st = reinterpret_cast<RsStatus*>(blk);
    QueryArgs a = make_args(t, d_s, d_e, n_r, 32, 1 << 30, st);
    a.detected = mode == kCount ? nullptr : (mode == kBarycentric ? o.det : o.flags);
    a.counts = o.flags;
    a.tri = o.tri; a.dist = o.dist; a.points = o.pts;
    a.c_ray = o.c_ray; a.c_dist = o.c_dist; a.c_tri = o.c_tri; a.c_point = o.c_pt;
    a.ray_offset = o.ray_offset;
    a.tile_status = reinterpret_cast<unsigned long long*>(blk + align256(sizeof(RsStatus)));
    a.nodes4 = nullptr;  // binary kernels
    if (launch_query(a, mode, false, compact, 64, false, s))
        return fail(RS_INTERNAL, "no binary kernel variant");
    CK(cudaGetLastError());
    int rc = read_status(st, s, h);
    CK(dfree(blk, s));
    return rc;
}

int rs_query(const rs_tree* t, const float* d_starts, const float* d_ends, int64_t n_r, int mode,
             int max_coll, int max_stack, int ref, int32_t* d_detected, int32_t* d_counts,
             int32_t* d_tri, float* d_dist, float* d_points, int64_t* bad, void* stream) {
    marks_reset();
    if (mode == kBoolean && !d_detected) return fail(RS_INVALID_ARG, "boolean needs d_detected");
    if (mode == kCount && !d_counts) return fail(RS_INVALID_ARG, "count needs d_counts");
    if (mode == kBarycentric && !(d_detected && d_tri && d_dist && d_points))
        return fail(RS_INVALID_ARG, "barycentric needs detected/tri/dist/points");
    return query_impl(t, d_starts, d_ends, n_r, mode, max_coll, max_stack, ref, d_detected,
                      d_counts, d_tri, d_dist, d_points, nullptr, nullptr, nullptr, nullptr,
                      nullptr, bad, false, nullptr, nullptr, S(stream));
}

int rs_query_compact(const rs_tree* t, const float* d_starts, const float* d_ends, int64_t n_r,
                     int max_coll, int max_stack, int ref, int32_t* d_ray, float* d_dist,
                     int32_t* d_tri, float* d_pt, int64_t* n_hits, int64_t* bad, void* stream) {
    marks_reset();
    if (!(d_ray && d_dist && d_tri && d_pt)) return fail(RS_INVALID_ARG, "null output");
    if (n_hits) *n_hits = 0;
    return query_impl(t, d_starts, d_ends, n_r, kBarycentric, max_coll, max_stack, ref, nullptr,
                      nullptr, nullptr, nullptr, nullptr, d_ray, d_dist, d_tri, d_pt, n_hits, bad,
                      false, nullptr, nullptr, S(stream));
}

int rs_query_stats(const rs_tree* t, const float* d_starts, const float* d_ends, int64_t n_r,
                   int mode, int max_coll, int max_stack, int ref, int64_t* visits, int64_t* mts,
                   void* stream) {
    marks_reset();
    cudaStream_t s = S(stream);
    // outputs go to a scratch block: stats runs are diagnostics
    char* blk = nullptr;
    CK(dmalloc(reinterpret_cast<void**>(&blk), align256(28ull * (n_r > 0 ? n_r : 1)), s));
    int32_t* i0 = reinterpret_cast<int32_t*>(blk);
    float* f1 = reinterpret_cast<float*>(blk + 8ull * n_r);
    float* f3 = reinterpret_cast<float*>(blk + 16ull * n_r);
    int32_t* i2 = reinterpret_cast<int32_t*>(blk + 12ull * n_r);
    int64_t bad;
    int rc = query_impl(t, d_starts, d_ends, n_r, mode, max_coll, max_stack, ref, i0, i0, i2, f1,
                        f3, nullptr, nullptr, nullptr, nullptr, nullptr, &bad, true, visits, mts, s);
    dfree(blk, s);
    return rc;
}

int rs_sort_segments(const float* d_starts, const float* d_ends, int64_t n, float* d_out_starts,
                     float* d_out_ends, int64_t* d_perm, void* stream) {
    marks_reset();
    if (n < 0 || n > 2147483647ll) return fail(RS_INVALID_ARG, "bad segment count");
    if (n == 0) return RS_OK;
    if (!(d_starts && d_ends && d_out_starts && d_out_ends && d_perm)) return fail(RS_INVALID_ARG, "null pointer");
    cudaStream_t s = S(stream);
    char* blk = nullptr;
    CK(dmalloc(reinterpret_cast<void**>(&blk), sort_segments_scratch_bytes((int)n), s));
    launch_sort_segments(d_starts, d_ends, (int)n, d_out_starts, d_out_ends,
                         reinterpret_cast<long long*>(d_perm), blk, s);
    CK(cudaGetLastError());
    CK(dfree(blk, s));
    return RS_OK;
}

int rs_baseline(const float* d_verts, int64_t n_v, const int32_t* d_tris, int64_t n_t,
                const float* d_starts, const float* d_ends, int64_t n_r, int mode,
                int32_t* d_detected, int32_t* d_counts, int32_t* d_tri, float* d_dist,
                float* d_points, void* stream) {
    marks_reset();
    if (mode < 0 || mode > 2) return fail(RS_INVALID_ARG, "unknown mode %d", mode);
    if (n_t < 0 || n_r < 0 || n_t > 2147483647ll || n_r > 2147483647ll)
        return fail(RS_INVALID_ARG, "bad sizes");
    (void)n_v;
    BaselineArgs a{d_verts, d_tris, (int)n_t, d_starts, d_ends, n_r, d_detected, d_counts,
                   d_tri, d_dist, d_points, nullptr, nullptr};
    cudaStream_t s = S(stream);
    if (n_t > 0) launch_baseline(a, mode, s);
    CK(cudaGetLastError());
    CK(cudaStreamSynchronize(s));
    return RS_OK;
}

int rs_baseline_compact(const float* d_verts, int64_t n_v, const int32_t* d_tris, int64_t n_t,
                        const float* d_starts, const float* d_ends, int64_t n_r, int32_t* d_ray,
                        float* d_dist, int32_t* d_tri, float* d_pt, int64_t* n_hits, void* stream) {
    marks_reset();
    if (n_hits) *n_hits = 0;
    if (n_t < 0 || n_r < 0 || n_t > 2147483647ll || n_r > 2147483647ll)
        return fail(RS_INVALID_ARG, "bad sizes");
    if (!(d_ray && d_dist && d_tri && d_pt) && n_r > 0) return fail(RS_INVALID_ARG, "null output");
    (void)n_v;
    if (n_r == 0 || n_t == 0) return RS_OK;
    cudaStream_t s = S(stream);
    const size_t cs = bary_compact_scratch(n_r);
    char* blk = nullptr;
    const size_t total = align256(sizeof(RsStatus)) + align256(8ull * n_r) + align256(4ull * n_r) + align256(cs);
    CK(dmalloc(reinterpret_cast<void**>(&blk), total, s));
    Carver c{blk};
    RsStatus* st = c.take<RsStatus>(1);
    unsigned long long* best_t = c.take<unsigned long long>(n_r);
    int* best_tri = c.take<int>(n_r);
    unsigned long long* tiles = c.take<unsigned long long>(cs / 8);
    CK(cudaMemsetAsync(st, 0, sizeof(RsStatus), s));
    CK(cudaMemsetAsync(tiles, 0, cs, s));
    BaselineArgs a{d_verts, d_tris, (int)n_t, d_starts, d_ends, n_r, nullptr, nullptr,
                   nullptr, nullptr, nullptr, best_t, best_tri};
    launch_baseline(a, kBarycentric, s);
    CompactArgs ca{n_r, best_t, best_tri, d_starts, d_ends, d_ray, d_dist, d_tri, d_pt,
                   tiles, tiles + (cs / 8 - 1), &st->hits, 0, nullptr};
    launch_bary_compact(ca, s);
    CK(cudaGetLastError());
    RsStatus h;
    int rc = read_status(st, s, &h);
    CK(dfree(blk, s));
    if (rc) return rc;
    if (n_hits) *n_hits = (int64_t)h.hits;
    return RS_OK;
}

int rs_oracle_intersect(const float* d_verts, int64_t n_v, const int32_t* d_tris, int64_t n_t,
                        const float* d_starts, const float* d_ends, int64_t n_r, int mode,
                        int32_t* d_flags, int32_t* d_ray, float* d_dist, int32_t* d_tri, float* d_pt,
                        int64_t* n_hits, void* stream) {
    marks_reset();
    if (n_hits) *n_hits = 0;
    if (mode < 0 || mode > 2) return fail(RS_INVALID_ARG, "unknown mode %d", mode);
    if (n_t < 0 || n_r < 0 || n_t > 2147483647ll || n_r > 2147483647ll) return fail(RS_INVALID_ARG, "bad sizes");
    (void)n_v;
    cudaStream_t s = S(stream);
    if (mode != kBarycentric) {
        if (n_r && !d_flags) return fail(RS_INVALID_ARG, "null output");
        if (n_r) CK(cudaMemsetAsync(d_flags, 0, 4ull * n_r, s));
        BaselineArgs a{d_verts, d_tris, (int)n_t, d_starts, d_ends, n_r, d_flags, d_flags,
                       nullptr, nullptr, nullptr, nullptr, nullptr};
        if (n_t > 0) launch_sign_oracle(a, mode, s);
        CK(cudaGetLastError());
        CK(cudaStreamSynchronize(s));
        return RS_OK;
    }
    if (!(d_ray && d_dist && d_tri && d_pt) && n_r > 0) return fail(RS_INVALID_ARG, "null output");
    if (n_r == 0 || n_t == 0) return RS_OK;
    const size_t cs = bary_compact_scratch(n_r);
    char* blk = nullptr;
    const size_t total = align256(sizeof(RsStatus)) + align256(8ull * n_r) + align256(4ull * n_r) + align256(cs);
    CK(dmalloc(reinterpret_cast<void**>(&blk), total, s));
    Carver c{blk};
    RsStatus* st = c.take<RsStatus>(1);
    unsigned long long* best_t = c.take<unsigned long long>(n_r);
    int* best_tri = c.take<int>(n_r);
    unsigned long long* tiles = c.take<unsigned long long>(cs / 8);
    CK(cudaMemsetAsync(st, 0, sizeof(RsStatus), s));
    CK(cudaMemsetAsync(tiles, 0, cs, s));
    BaselineArgs a{d_verts, d_tris, (int)n_t, d_starts, d_ends, n_r, nullptr, nullptr,
                   nullptr, nullptr, nullptr, best_t, best_tri};
    launch_sign_oracle(a, kBarycentric, s);
    CompactArgs ca{n_r, best_t, best_tri, d_starts, d_ends, d_ray, d_dist, d_tri, d_pt,
                   tiles, tiles + (cs / 8 - 1), &st->hits, 0, nullptr};
    launch_bary_compact(ca, s);
    CK(cudaGetLastError());
    RsStatus h;
    int rc = read_status(st, s, &h);
    CK(dfree(blk, s));
    if (rc) return rc;
    if (n_hits) *n_hits = (int64_t)h.hits;
    return RS_OK;
}

int rs_segment_boxes(const float* d_starts, const float* d_ends, int64_t n, float* d_boxes,
                     void* stream) {
    if (n < 0) return fail(RS_INVALID_ARG, "negative count");
    if (n && !(d_starts && d_ends && d_boxes)) return fail(RS_INVALID_ARG, "null array");
    launch_segment_boxes(d_starts, d_ends, n, d_boxes, S(stream));
    CK(cudaGetLastError());
    return RS_OK;
}

int rs_unpermute_dense(const int64_t* d_perm, int64_t n, const int32_t* d_in, int32_t* d_out,
                       void* stream) {
    if (n < 0) return fail(RS_INVALID_ARG, "negative count");
    if (n && !(d_perm && d_in && d_out)) return fail(RS_INVALID_ARG, "null array");
    launch_unpermute_dense(reinterpret_cast<const long long*>(d_perm), n, d_in, d_out, S(stream));
    CK(cudaGetLastError());
    return RS_OK;
}

int rs_unpermute_rows(const int64_t* d_perm, int64_t n, const int32_t* d_ray, const float* d_dist,
                      const int32_t* d_tri, const float* d_pt, int64_t k, int32_t* o_ray,
                      float* o_dist, int32_t* o_tri, float* o_pt, void* stream) {
    if (n < 0 || k < 0 || k > n) return fail(RS_INVALID_ARG, "bad sizes");
    if (n == 0) return RS_OK;
    cudaStream_t s = S(stream);
    void* scratch = nullptr;
    CK(dmalloc(&scratch, unpermute_scratch_bytes(n), s));
    launch_unpermute_rows(reinterpret_cast<const long long*>(d_perm), n, d_ray, d_dist, d_tri, d_pt, k,
                          o_ray, o_dist, o_tri, o_pt, scratch, s);
    CK(cudaGetLastError());
    CK(dfree(scratch, s));
    return RS_OK;
}

struct Fork {
    cudaStream_t aux = nullptr;  // binning (default priority)
    cudaStream_t hp = nullptr;   // the build, at the highest stream priority
    cudaEvent_t prep = nullptr, bin = nullptr, bin2 = nullptr, start = nullptr, built = nullptr;
};
// per thread and per device (streams and events belong to one device)
static thread_local std::map<int, Fork> g_forks;
static thread_local Fork g_fork;

static int fork_init() {
    int dev = 0;
    CK(cudaGetDevice(&dev));
    Fork& f = g_forks[dev];
    if (!f.aux) {
        CK(cudaStreamCreateWithFlags(&f.aux, cudaStreamNonBlocking));
        CK(cudaEventCreateWithFlags(&f.prep, cudaEventDisableTiming));
        CK(cudaEventCreateWithFlags(&f.bin, cudaEventDisableTiming));
        CK(cudaEventCreateWithFlags(&f.bin2, cudaEventDisableTiming));
        CK(cudaEventCreateWithFlags(&f.start, cudaEventDisableTiming));
        CK(cudaEventCreateWithFlags(&f.built, cudaEventDisableTiming));
        int lo = 0, hi = 0;
        CK(cudaDeviceGetStreamPriorityRange(&lo, &hi));
        CK(cudaStreamCreateWithPriority(&f.hp, cudaStreamNonBlocking, hi));
    }
    g_fork = f;  // the current device's set
    return RS_OK;
}

// The build runs on a high-priority stream beside the binning: its small,
// latency-bound kernels (keys, 4 sort passes, climb) otherwise queue behind
// the bandwidth-bound binning CTAs for SM slots (RS_BUILD_PRIO=0: A/B).
static const bool g_build_prio = [] {
    const char* e = getenv("RS_BUILD_PRIO");
    return !(e && e[0] == '0');
}();

// RS_PIPELINE_PARTS=2: large batches are binned and traversed in two halves,
// so the second half's binning (memory-bound) overlaps the first half's
// traversal (latency-bound).
static int pipeline_parts() {
    static const int v = [] {
        const char* e = getenv("RS_PIPELINE_PARTS");
        return e && e[0] == '2' ? 2 : 1;
    }();
    return v;
}

__global__ void k_merge_status(RsStatus* dst, const RsStatus* src) {
    dst->hits += src->hits;
    dst->internal |= src->internal;
}

// Fast-tree run_batch with the binning forked onto a second stream right
// after k_prep: binning (two passes over the segments) overlaps keys, sort
// and climb.  Leaves the status in f.st (device); the caller frees f.blk.
// critical-path experiments (RS_DEBUG_DELAY_BUILD_US / _BIN_US): a
// one-thread spin of that many microseconds at the end of the build /
// binning stream
__global__ void k_debug_spin(long long ns) {
    long long t0;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    for (;;) {
        long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        if (t - t0 >= ns) break;
    }
}
static long long debug_delay_ns(const char* name) {
    const char* e = getenv(name);
    return e && *e ? atoll(e) * 1000ll : 0;
}

static int enqueue_fast_forked(const float* d_verts, int64_t n_v, const int32_t* d_tris,
                               int64_t n_t, const float* d_starts, const float* d_ends,
                               int64_t n_r, int mode, const FastOut& o, FastScratch& f,
                               cudaStream_t s, rs_tree** tree_out) {
    int rc = fork_init();
    if (rc) return rc;
    cudaStream_t aux = g_fork.aux;
    const bool two = pipeline_parts() == 2 && n_r >= (2ll << 20) && !o.det;
    const int64_t n1 = two ? ((n_r / 2 + 1023) / 1024) * 1024 : n_r, n2 = n_r - n1;
    FastOut o1 = o, o2 = o;
    FastScratch f2;
    cudaStream_t bs = s;  // the build's stream
    CK(cudaEventRecord(g_fork.start, s));
    if (g_build_prio) {
        bs = g_fork.hp;
        CK(cudaStreamWaitEvent(bs, g_fork.start, 0));
    }
    // the binning stream's presets (status, zeroed bins and outputs) need
    // nothing from the build: they run beside k_prep, off the critical path
    CK(cudaStreamWaitEvent(aux, g_fork.start, 0));
    rc = fast_alloc(f, n1, mode, 2ll * n1 + 4096, aux);
    if (rc) return rc;
    rc = fast_presets(d_starts, d_ends, n1, mode, o1, f, aux);
    if (rc) return rc;
    auto fork = [&](rs_tree* t) -> int {
        CK(cudaEventRecord(g_fork.prep, bs));
        CK(cudaStreamWaitEvent(aux, g_fork.prep, 0));
        int r = RS_OK;
        if (two) {
            r = fast_alloc(f2, n2, mode, 2ll * n2 + 4096, aux);
            if (r) return r;
            if (o.flags) o2.flags = o.flags + n1;
            o2.ray_offset = o.ray_offset + n1;
            if (mode == kBarycentric) {  // both halves compact into the same rows, in order
                unsigned long long* rows = reinterpret_cast<unsigned long long*>(f.n_live + 8);
                CK(cudaMemsetAsync(rows, 0, sizeof(unsigned long long), aux));
                o1.row_base = rows;
                o2.row_base = rows;
            }
        }
        r = fast_bin(t, d_starts, d_ends, n1, mode, o1, f, aux, false);
        if (r) return r;
        if (const long long ns = debug_delay_ns("RS_DEBUG_DELAY_BIN_US")) k_debug_spin<<<1, 1, 0, aux>>>(ns);
        CK(cudaEventRecord(g_fork.bin, aux));
        if (two) {
            r = fast_bin(t, d_starts + 3 * n1, d_ends + 3 * n1, n2, mode, o2, f2, aux);
            if (r) return r;
            CK(cudaEventRecord(g_fork.bin2, aux));
        }
        return RS_OK;
    };
    rs_tree* t = nullptr;
    rc = build_impl(d_verts, n_v, d_tris, n_t, kTreeFast, nullptr, nullptr, bs, &t, fork, true);
    if (rc) return rc;
    if (const long long ns = debug_delay_ns("RS_DEBUG_DELAY_BUILD_US")) k_debug_spin<<<1, 1, 0, bs>>>(ns);
    if (mode == kBarycentric && !f.best_t) {  // off the traversal's stream: beside the binning
        launch_leaf_inverse(t->leaves, (int)t->n, t->leaf_of, bs);
        f.leaf_of_ready = true;
        if (two) f2.leaf_of_ready = true;
    }
    if (bs != s) {
        CK(cudaEventRecord(g_fork.built, bs));
        CK(cudaStreamWaitEvent(s, g_fork.built, 0));
    }
    CK(cudaStreamWaitEvent(s, g_fork.bin, 0));
    if (!two) {
        rc = fast_trav(t, d_starts, d_ends, n_r, mode, o1, f, false, s);
    } else {
        g_hot_mark_mask = 1;
        rc = fast_trav(t, d_starts, d_ends, n1, mode, o1, f, false, s, true, false);
        g_hot_mark_mask = 2;
        CK(cudaStreamWaitEvent(s, g_fork.bin2, 0));
        if (!rc) rc = fast_trav(t, d_starts + 3 * n1, d_ends + 3 * n1, n2, mode, o2, f2, false, s, false, true);
        g_hot_mark_mask = 3;
        count_launches(1);
        k_merge_status<<<1, 1, 0, s>>>(f.st, f2.st);
        CK(dfree(f2.blk, s));
    }
    *tree_out = t;
    return rc;
}

static int run_device_direct(const float* d_verts, int64_t n_v, const int32_t* d_tris,
                             int64_t n_t, const float* d_starts, const float* d_ends, int64_t n_r,
                             int mode, int tree_kind, int max_coll, int max_stack, int32_t* d_flags,
                             int32_t* d_ray, float* d_dist, int32_t* d_tri, float* d_pt,
                             int64_t* n_hits, int64_t* bad, cudaStream_t s) {
    rs_tree* t = nullptr;
    if (tree_kind == kTreeFast && !buffer_path() && !g_binary_fast) {
        FastOut o;
        o.flags = d_flags;
        o.c_ray = d_ray; o.c_dist = d_dist; o.c_tri = d_tri; o.c_pt = d_pt;
        FastScratch f;
        int rc = enqueue_fast_forked(d_verts, n_v, d_tris, n_t, d_starts, d_ends, n_r, mode, o, f,
                                     s, &t);
        RsStatus h{};
        if (!rc) rc = read_status(f.st, s, &h);
        if (f.blk) dfree(f.blk, s);
        if (!rc && h.internal) rc = binary_query(t, d_starts, d_ends, n_r, mode, o, &h, s);
        if (!rc) {
            if (n_hits) *n_hits = (int64_t)h.hits;
            rc = status_code(h, bad);
        }
        const int rc2 = t ? rs_free(t, s) : RS_OK;
        return rc ? rc : rc2;
    }
    int rc = build_impl(d_verts, n_v, d_tris, n_t, tree_kind, nullptr, nullptr, s, &t, nullptr, true);
    if (rc) return rc;
    const int ref = tree_kind == kTreeReference;
    if (mode == kBarycentric)
        rc = query_impl(t, d_starts, d_ends, n_r, mode, max_coll, max_stack, ref, nullptr, nullptr,
                        nullptr, nullptr, nullptr, d_ray, d_dist, d_tri, d_pt, n_hits, bad, false,
                        nullptr, nullptr, s);
    else
        rc = query_impl(t, d_starts, d_ends, n_r, mode, max_coll, max_stack, ref, d_flags, d_flags,
                        nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, bad,
                        false, nullptr, nullptr, s);
    const int rc2 = rs_free(t, s);
    return rc ? rc : rc2;
}

// Batches above kDeviceChunk segments (BASELINE configs[4]: 1B segments per
// job, up to 1B / n_gpus per rank) are processed as one build and a loop of
// chunk queries on the caller's stream: the scratch (32-B records, keys,
// bins) is sized for one chunk and reused, each chunk leaves its status in
// its own slot, the barycentric rows of consecutive chunks compact through
// one device row counter (ascending ray index across the whole batch), and
// every chunk chooses its traversal kernel by the whole batch's density
// (set_batch_rays).  One synchronisation at the end.
// Option "device_chunk" (multiple of 1024) lowers it for tests.
static std::atomic<long long> g_device_chunk{[] {
    const char* e = getenv("RS_DEVICE_CHUNK");
    const long long v = e && *e ? atoll(e) : 0;
    return v > 0 ? ((v + 1023) / 1024) * 1024 : (1ll << 30);
}()};

static int run_device_chunked(const float* d_verts, int64_t n_v, const int32_t* d_tris,
                              int64_t n_t, const float* d_starts, const float* d_ends, int64_t n_r,
                              int mode, int32_t* d_flags, int32_t* d_ray, float* d_dist,
                              int32_t* d_tri, float* d_pt, int64_t* n_hits, int64_t* bad,
                              cudaStream_t s) {
    const int64_t kDeviceChunk = g_device_chunk.load();
    const int64_t nchunks = (n_r + kDeviceChunk - 1) / kDeviceChunk;
    const bool bary = mode == kBarycentric;
    rs_tree* t = nullptr;
    int rc = build_impl(d_verts, n_v, d_tris, n_t, kTreeFast, nullptr, nullptr, s, &t, nullptr, true);
    if (rc) return rc;
    struct Guard {
        rs_tree* t;
        char* blk = nullptr;
        FastScratch f;
        cudaStream_t s;
        ~Guard() {
            if (f.blk) dfree(f.blk, s);
            if (blk) dfree(blk, s);
            if (t) rs_free(t, s);
        }
    } g{t, nullptr, {}, s};
    const size_t st_bytes = align256(sizeof(RsStatus) * nchunks);
    CK(dmalloc(reinterpret_cast<void**>(&g.blk), st_bytes + 256, s));
    CK(cudaMemsetAsync(g.blk, 0, st_bytes + 256, s));
    RsStatus* st = reinterpret_cast<RsStatus*>(g.blk);
    unsigned long long* rows = reinterpret_cast<unsigned long long*>(g.blk + st_bytes);
    rc = fast_alloc(g.f, std::min(n_r, kDeviceChunk), mode, 2 * kDeviceChunk + 4096, s);
    if (rc) return rc;
    rs::set_batch_rays(n_r);
    ev_record(1, s);
    for (int64_t k = 0; k < nchunks && !rc; ++k) {
        const int64_t lo = k * kDeviceChunk, cnt = std::min(kDeviceChunk, n_r - lo);
        g.f.st = st + k;
        FastOut o;
        o.ray_offset = lo;
        if (bary) {
            o.c_ray = d_ray; o.c_dist = d_dist; o.c_tri = d_tri; o.c_pt = d_pt;
            o.row_base = rows;
        } else {
            o.flags = d_flags + lo;
        }
        rc = fast_bin(t, d_starts + 3 * lo, d_ends + 3 * lo, cnt, mode, o, g.f, s);
        if (!rc) rc = fast_trav(t, d_starts + 3 * lo, d_ends + 3 * lo, cnt, mode, o, g.f, false, s,
                                false, false);
    }
    ev_record(2, s);
    rs::set_batch_rays(0);
    if (rc) return rc;
    std::vector<RsStatus> h((size_t)nchunks);
    CK(cudaMemcpyAsync(h.data(), st, sizeof(RsStatus) * nchunks, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    unsigned long long hits = 0, internal = 0;
    for (const RsStatus& x : h) {
        hits += x.hits;
        internal |= x.internal;
    }
    if (internal) {
        // a fast-path walk exceeded its capacity (never expected): the whole
        // batch again with the binary kernels, chunk by chunk
        hits = 0;
        CK(cudaMemsetAsync(rows, 0, sizeof(unsigned long long), s));
        for (int64_t k = 0; k < nchunks; ++k) {
            const int64_t lo = k * kDeviceChunk, cnt = std::min(kDeviceChunk, n_r - lo);
            FastOut o;
            o.ray_offset = lo;
            if (bary) {
                o.c_ray = d_ray + hits; o.c_dist = d_dist + hits; o.c_tri = d_tri + hits;
                o.c_pt = d_pt + 3 * hits;
            } else {
                o.flags = d_flags + lo;
            }
            RsStatus hb{};
            rc = binary_query(t, d_starts + 3 * lo, d_ends + 3 * lo, cnt, mode, o, &hb, s);
            if (rc) return rc;
            if (hb.internal) return fail(RS_INTERNAL, "internal traversal capacity exceeded");
            hits += hb.hits;
        }
    }
    if (n_hits) *n_hits = (int64_t)hits;
    if (bad) *bad = -1;
    return RS_OK;
}

// The status words go to mapped pinned host memory from a one-warp kernel:
// a D2H copy node at the end of the graph cost ~11 us of copy-engine latency
// per call, the kernel's PCIe writes ~2 us.
__global__ void k_status_out(RsStatus* dst, const RsStatus* src) {
    constexpr int kWords = sizeof(RsStatus) / 8;
    static_assert(sizeof(RsStatus) % 8 == 0 && kWords <= 32, "status is copied as 8-B words");
    if (threadIdx.x < kWords)
        reinterpret_cast<volatile unsigned long long*>(dst)[threadIdx.x] =
            reinterpret_cast<const volatile unsigned long long*>(src)[threadIdx.x];
    __threadfence_system();
}
static const bool g_status_copy = [] {  // RS_STATUS_COPY=1: D2H copy node instead (A/B)
    const char* e = getenv("RS_STATUS_COPY");
    return e && e[0] == '1';
}();
struct StatusDst {
    RsStatus* host;  // pinned, mapped
    RsStatus* dev;   // its device alias
};
static int status_out(const StatusDst& d, const RsStatus* st, cudaStream_t s) {
    if (g_status_copy) {
        CK(cudaMemcpyAsync(d.host, st, sizeof(RsStatus), cudaMemcpyDeviceToHost, s));
        return RS_OK;
    }
    count_launches(1);
    k_status_out<<<1, 32, 0, s>>>(d.dev, st);
    CK(cudaGetLastError());
    return RS_OK;
}

// Everything rs_run_batch_device does, enqueued without a host sync so it can
// be captured into one CUDA graph: build, query, status -> pinned host.
static int enqueue_device_batch_body(const float* d_verts, int64_t n_v, const int32_t* d_tris,
                                int64_t n_t, const float* d_starts, const float* d_ends,
                                int64_t n_r, int mode, int tree_kind, int max_coll, int max_stack,
                                int32_t* d_flags, int32_t* d_ray, float* d_dist, int32_t* d_tri,
                                float* d_pt, const StatusDst& h_status, cudaStream_t s) {
    rs_tree* t = nullptr;
    if (tree_kind == kTreeFast && !buffer_path() && !g_binary_fast) {
        FastOut o;
        o.flags = d_flags;
        o.c_ray = d_ray; o.c_dist = d_dist; o.c_tri = d_tri; o.c_pt = d_pt;
        FastScratch f;
        int rc = enqueue_fast_forked(d_verts, n_v, d_tris, n_t, d_starts, d_ends, n_r, mode, o, f,
                                     s, &t);
        if (rc) return rc;
        rc = status_out(h_status, f.st, s);
        if (rc) return rc;
        stage_mark(9, s);
        CK(dfree(f.blk, s));
        rc = rs_free(t, s);
        stage_mark(10, s);
        return rc;
    }
    int rc = build_impl(d_verts, n_v, d_tris, n_t, tree_kind, nullptr, nullptr, s, &t, nullptr, true);
    if (rc) return rc;
    if (tree_kind == kTreeFast && !g_binary_fast) {
        FastOut o;
        o.flags = d_flags;
        o.c_ray = d_ray; o.c_dist = d_dist; o.c_tri = d_tri; o.c_pt = d_pt;
        FastScratch f;
        rc = fast_alloc(f, n_r, mode, 2ll * n_r + 4096, s);
        if (rc) return rc;
        rc = fast_launch(t, d_starts, d_ends, n_r, mode, o, f, false, s);
        if (rc) return rc;
        rc = status_out(h_status, f.st, s);
        if (rc) return rc;
        CK(dfree(f.blk, s));
    } else {
        const bool compact = mode == kBarycentric;
        const size_t cs = compact ? compact_scratch_bytes(n_r) : 0;
        char* blk = nullptr;
        CK(dmalloc(reinterpret_cast<void**>(&blk), align256(sizeof(RsStatus)) + cs + 256, s));
        CK(cudaMemsetAsync(blk, 0, align256(sizeof(RsStatus)) + cs, s));
        RsStatus* st = reinterpret_cast<RsStatus*>(blk);
        const int ref = tree_kind == kTreeReference;
        QueryArgs a = make_args(t, d_starts, d_ends, n_r, max_coll, max_stack, st);
        a.detected = d_flags; a.counts = d_flags;
        a.c_ray = d_ray; a.c_dist = d_dist; a.c_tri = d_tri; a.c_point = d_pt;
        a.tile_status = reinterpret_cast<unsigned long long*>(blk + align256(sizeof(RsStatus)));
        ev_record(1, s);
        if (launch_query(a, mode, ref != 0, compact, kstack_for(ref != 0, max_stack), false, s))
            return fail(RS_INVALID_ARG, "no kernel variant for this configuration");
        ev_record(2, s);
        rc = status_out(h_status, st, s);
        if (rc) return rc;
        CK(dfree(blk, s));
    }
    return rs_free(t, s);
}

static int enqueue_device_batch(const float* d_verts, int64_t n_v, const int32_t* d_tris,
                                int64_t n_t, const float* d_starts, const float* d_ends,
                                int64_t n_r, int mode, int tree_kind, int max_coll, int max_stack,
                                int32_t* d_flags, int32_t* d_ray, float* d_dist, int32_t* d_tri,
                                float* d_pt, const StatusDst& h_status, cudaStream_t s) {
    mark(0, s);
    const int rc = enqueue_device_batch_body(d_verts, n_v, d_tris, n_t, d_starts, d_ends, n_r, mode,
                                             tree_kind, max_coll, max_stack, d_flags, d_ray, d_dist,
                                             d_tri, d_pt, h_status, s);
    timing_join(s);  // the timing branches end the graph
    return rc;
}

struct GraphKey {
    const void* p[9];
    int64_t n_v, n_t, n_r;
    int mode, kind, mc, ms, timing, opt_gen, device;
    bool operator<(const GraphKey& o) const { return std::memcmp(this, &o, sizeof *this) < 0; }
};
// One captured run_batch.  Entries are shared: a caller holds a reference
// for the whole launch + wait + status read, so an eviction by another
// thread only drops the cache's reference and the resources go with the
// last user.  `run` serialises calls on the same entry (they share its
// status word and scratch arena; identical keys also share outputs).
struct GraphEntry {
    cudaGraphExec_t exec = nullptr;
    RsStatus* h_status = nullptr;  // pinned, mapped
    RsStatus* d_status = nullptr;  // its device alias
    char* arena = nullptr;         // the graph's scratch (see Arena)
    unsigned long long stamp = 0;  // LRU clock (under g_graph_mu)
    long long kernels = 0;         // kernel nodes in the graph (for rs_kernel_launches)
    std::vector<Mark> marks;       // timing nodes baked into the graph (events owned here)
    std::mutex run;
    ~GraphEntry() {
        if (exec) cudaGraphExecDestroy(exec);
        if (h_status) cudaFreeHost(h_status);
        if (arena) cudaFree(arena);
        for (auto& m : marks) cudaEventDestroy(m.ev);
    }
};
static thread_local RsStatus g_last_status{};
static std::atomic<int> g_opt_gen{0};  // bumped by rs_set_option: captured graphs bake the options in
static std::mutex g_graph_mu;
static std::map<GraphKey, std::shared_ptr<GraphEntry>> g_graphs;
static std::set<GraphKey> g_seen;  // argument sets called once (captured on the next call)
static unsigned long long g_graph_clock = 0;
static const bool g_use_arena = [] {  // RS_GRAPH_ARENA=0: allocation nodes in the graph (A/B)
    const char* e = getenv("RS_GRAPH_ARENA");
    return !(e && e[0] == '0');
}();
static const bool g_use_graphs = [] {
    const char* e = getenv("RS_NO_GRAPH");
    return !(e && e[0] == '1');
}();

// Capture one argument set into a new entry (two passes: the first sizes the
// scratch arena, the second captures from it).  Returns null on failure
// (the caller then runs the direct launches).
static std::shared_ptr<GraphEntry> capture_graph(const float* d_verts, int64_t n_v, const int32_t* d_tris,
                                                 int64_t n_t, const float* d_starts, const float* d_ends,
                                                 int64_t n_r, int mode, int tree_kind, int max_coll,
                                                 int max_stack, int32_t* d_flags, int32_t* d_ray,
                                                 float* d_dist, int32_t* d_tri, float* d_pt) {
    auto e = std::make_shared<GraphEntry>();
    if (cudaHostAlloc(reinterpret_cast<void**>(&e->h_status), sizeof(RsStatus), cudaHostAllocMapped) != cudaSuccess ||
        cudaHostGetDevicePointer(reinterpret_cast<void**>(&e->d_status), e->h_status, 0) != cudaSuccess) {
        cudaGetLastError();
        return nullptr;
    }
    // capture on a private stream (the caller's may be the legacy default
    // stream, which cannot be captured); replay on the caller's
    static thread_local cudaStream_t cap = nullptr;
    if (!cap && cudaStreamCreateWithFlags(&cap, cudaStreamNonBlocking) != cudaSuccess) return nullptr;
    cudaGraph_t g = nullptr;
    const long long k0 = rs::g_launches.load();
    auto capture_once = [&](cudaGraph_t* out) -> int {
        marks_reset();
        if (cudaStreamBeginCapture(cap, cudaStreamCaptureModeThreadLocal) != cudaSuccess) return RS_CUDA_ERROR;
        const int r = enqueue_device_batch(d_verts, n_v, d_tris, n_t, d_starts, d_ends, n_r, mode,
                                           tree_kind, max_coll, max_stack, d_flags, d_ray, d_dist,
                                           d_tri, d_pt, StatusDst{e->h_status, e->d_status}, cap);
        const cudaError_t ce = cudaStreamEndCapture(cap, out);
        return r != RS_OK ? r : (ce == cudaSuccess && *out ? RS_OK : RS_CUDA_ERROR);
    };
    g_arena = Arena{nullptr, 0, 0, 1};
    int erc = capture_once(&g);
    const size_t arena_bytes = g_arena.off;
    g_arena = Arena{};
    if (g) cudaGraphDestroy(g);
    g = nullptr;
    if (erc == RS_OK && g_use_arena &&
        cudaMalloc(reinterpret_cast<void**>(&e->arena), arena_bytes) == cudaSuccess) {
        g_arena = Arena{e->arena, arena_bytes, 0, 2};
        erc = capture_once(&g);
        g_arena = Arena{};
    } else if (erc == RS_OK) {
        cudaGetLastError();
        e->arena = nullptr;
        erc = capture_once(&g);  // stream-ordered allocation nodes instead
    }
    e->kernels = rs::g_launches.load() - k0;
    rs::g_launches.store(k0);  // counted when replayed
    // the timing events recorded by the graph's nodes now belong to it
    e->marks = g_marks;
    g_pool.erase(g_pool.begin(), g_pool.begin() + (ptrdiff_t)g_pool_used);
    marks_reset();
    // the build's kernel nodes at the highest priority: the binning's CTAs
    // otherwise hold the SMs the latency-bound build kernels need (the
    // graph runs with per-node priorities)
    if (erc == RS_OK && g && g_build_prio) {
        int lo = 0, hi = 0;
        cudaDeviceGetStreamPriorityRange(&lo, &hi);
        size_t nn = 0;
        cudaGraphGetNodes(g, nullptr, &nn);
        std::vector<cudaGraphNode_t> nodes(nn);
        cudaGraphGetNodes(g, nodes.data(), &nn);
        for (cudaGraphNode_t nd : nodes) {
            cudaGraphNodeType ty;
            if (cudaGraphNodeGetType(nd, &ty) != cudaSuccess || ty != cudaGraphNodeTypeKernel) continue;
            cudaKernelNodeParams kp{};
            if (cudaGraphKernelNodeGetParams(nd, &kp) != cudaSuccess || !rs::is_build_kernel(kp.func)) continue;
            cudaKernelNodeAttrValue v{};
            v.priority = hi;
            cudaGraphKernelNodeSetAttribute(nd, cudaLaunchAttributePriority, &v);
        }
        cudaGetLastError();
    }
    const bool ok = erc == RS_OK && g &&
                    cudaGraphInstantiate(&e->exec, g, g_build_prio ? cudaGraphInstantiateFlagUseNodePriority : 0) ==
                        cudaSuccess;
    if (g) cudaGraphDestroy(g);
    if (!ok) {
        const cudaError_t ce = cudaGetLastError();
        if (getenv("RS_DEBUG_GRAPH"))
            fprintf(stderr, "[rs] graph capture failed: rc %d, %s\n", erc, cudaGetErrorString(ce));
        return nullptr;
    }
    return e;
}

int rs_run_batch_device(const float* d_verts, int64_t n_v, const int32_t* d_tris, int64_t n_t,
                        const float* d_starts, const float* d_ends, int64_t n_r, int mode,
                        int tree_kind, int max_coll, int max_stack, int32_t* d_flags,
                        int32_t* d_ray, float* d_dist, int32_t* d_tri, float* d_pt,
                        int64_t* n_hits, int64_t* bad, void* stream) {
    marks_reset();
    g_last_status = RsStatus{};  // zeros unless this call runs a graph
    int rc = check_query(mode, max_coll, max_stack);
    if (rc) return rc;
    if (bad) *bad = -1;
    if (n_hits) *n_hits = 0;
    if (n_r == 0 || n_t == 0) return RS_OK;  // engine.py:233-234 (caller pre-zeroes d_flags)
    rc = check_mesh(n_v, n_t);
    if (rc) return rc;
    if (n_r > 2147483647ll) return fail(RS_INVALID_ARG, "segment count exceeds int32 indexing");
    if (tree_kind != kTreeReference && tree_kind != kTreeFast)
        return fail(RS_INVALID_ARG, "unknown tree kind %d", tree_kind);
    cudaStream_t s = S(stream);
    if (n_r > g_device_chunk.load() && tree_kind == kTreeFast && !buffer_path() && !g_binary_fast)
        return run_device_chunked(d_verts, n_v, d_tris, n_t, d_starts, d_ends, n_r, mode, d_flags,
                                  d_ray, d_dist, d_tri, d_pt, n_hits, bad, s);
    bool done = false;
    if (g_use_graphs) {
        // The whole step (about 20 launches, memsets and stream-ordered
        // allocations) is captured once per argument set and replayed as one
        // CUDA graph launch.
        rc = configure_pool();
        if (rc) return rc;
        GraphKey key{};
        const void* ptrs[9] = {d_verts, d_tris, d_starts, d_ends, d_flags, d_ray, d_dist, d_tri, d_pt};
        std::memcpy(key.p, ptrs, sizeof ptrs);
        key.n_v = n_v; key.n_t = n_t; key.n_r = n_r;
        key.mode = mode; key.kind = tree_kind; key.mc = max_coll; key.ms = max_stack;
        key.timing = g_timing;
        key.opt_gen = g_opt_gen.load();
        CK(cudaGetDevice(&key.device));
        std::shared_ptr<GraphEntry> ge;
        bool capture = true;
        {
            std::lock_guard<std::mutex> lk(g_graph_mu);
            auto it = g_graphs.find(key);
            if (it != g_graphs.end()) {
                ge = it->second;
                ge->stamp = ++g_graph_clock;
            } else {
                // capture only on an argument set's second call: a one-off
                // call (fresh buffers every time) runs the direct launches
                // instead of paying for capture + instantiation
                capture = g_seen.count(key) != 0;
                if (!capture) {
                    if (g_seen.size() >= 64) g_seen.clear();
                    g_seen.insert(key);
                }
            }
        }
        if (!ge && capture) {
            ge = capture_graph(d_verts, n_v, d_tris, n_t, d_starts, d_ends, n_r, mode, tree_kind,
                               max_coll, max_stack, d_flags, d_ray, d_dist, d_tri, d_pt);
            if (ge) {
                std::lock_guard<std::mutex> lk(g_graph_mu);
                auto it = g_graphs.find(key);
                if (it != g_graphs.end()) {
                    ge = it->second;  // another thread captured it meanwhile
                } else {
                    if (g_graphs.size() >= 8) {  // bounded cache: drop the least recently used
                        auto victim = g_graphs.begin();
                        for (auto v = g_graphs.begin(); v != g_graphs.end(); ++v)
                            if (v->second->stamp < victim->second->stamp) victim = v;
                        g_graphs.erase(victim);  // freed when its last user returns
                    }
                    g_graphs[key] = ge;
                }
                ge->stamp = ++g_graph_clock;
            }
        }
        if (ge) {
            std::lock_guard<std::mutex> run(ge->run);
            using clk = std::chrono::steady_clock;
            const auto h0 = clk::now();
            CK(cudaGraphLaunch(ge->exec, s));
            const auto h1 = clk::now();
            rs::g_launches.fetch_add(ge->kernels);
            CK(cudaStreamSynchronize(s));
            g_host_ms[0] = std::chrono::duration<float, std::milli>(h1 - h0).count();
            g_host_ms[1] = std::chrono::duration<float, std::milli>(clk::now() - h1).count();
            const RsStatus h = *ge->h_status;  // written by k_status_out before the sync returned
            g_last_status = h;
            if (!ge->marks.empty()) {
                g_tres = compute_timings(ge->marks);  // eagerly: the events belong to the graph
                g_have_marks = true;
            }
            if (!h.internal && !h.dropped) {
                if (n_hits) *n_hits = (int64_t)h.hits;
                rc = status_code(h, bad);
                done = true;
            }
            // internal capacity flag: fall through to the direct path, which
            // re-queries with the binary kernels; a collision-buffer overflow
            // (candidates dropped): the direct path re-launches with a buffer
            // of the claimed size
        }
    }
    if (!done) {
        marks_reset();
        mark(0, s);
        rc = run_device_direct(d_verts, n_v, d_tris, n_t, d_starts, d_ends, n_r, mode, tree_kind,
                               max_coll, max_stack, d_flags, d_ray, d_dist, d_tri, d_pt, n_hits, bad,
                               s);
    }
    return rc;
}

RS_API int rs_generate_segments(const float* d_verts, const int32_t* d_tris, int64_t n_t,
                                double z_lo, double z_hi, double x_hi, double y_hi,
                                double frac, uint64_t seed, int64_t first, int64_t n,
                                float* d_starts, float* d_ends, uint8_t* d_flags, void* stream) {
    if (n < 0 || first < 0 || n_t < 1 || !(frac >= 0.0 && frac <= 1.0))
        return fail(RS_INVALID_ARG, "invalid generator arguments");
    if (n && (!d_verts || !d_tris || !d_starts || !d_ends)) return fail(RS_INVALID_ARG, "null array");
    launch_generate(d_verts, d_tris, n_t, z_lo, z_hi, x_hi, y_hi, frac, seed, first, n, d_starts,
                    d_ends, d_flags, S(stream));
    CK(cudaGetLastError());
    return RS_OK;
}

RS_API int rs_set_timing(int enable) {
    g_timing = enable >= 0 && enable <= 3 ? enable : 1;
    marks_reset();
    return RS_OK;
}

RS_API int rs_last_timings(float* build_ms, float* query_ms, float* hot_ms) {
    const TimingResult* r = last_timings();
    if (!r) return fail(RS_INVALID_ARG, "no timed call yet (rs_set_timing)");
    if (build_ms) *build_ms = r->build;
    if (query_ms) *query_ms = r->query;
    if (hot_ms) *hot_ms = r->hot;
    return RS_OK;
}

RS_API int rs_last_phases(float* ms, int n) {
    const TimingResult* r = last_timings();
    if (!r) return fail(RS_INVALID_ARG, "no timed call yet (rs_set_timing)");
    for (int k = 0; k < n && k < kPhaseCount; ++k) ms[k] = r->phase[k];
    return RS_OK;
}

RS_API int rs_stage_times(float* ms, int n) {
    const TimingResult* r = last_timings();
    if (!r || g_timing != 3) return fail(RS_INVALID_ARG, "no stage-timed call yet (rs_set_timing(3))");
    for (int k = 0; k < n && k < kStageEvents; ++k) ms[k] = r->stage[k];
    return RS_OK;
}

RS_API long long rs_kernel_launches(void) { return g_launches.load(); }

RS_API int rs_set_option(const char* name, long long value, long long* old_value) {
    if (!name) return fail(RS_INVALID_ARG, "null option name");
    if (!strcmp(name, "hitbits_min")) {  // tests: the bitmap path on small batches
        if (old_value) *old_value = g_hitbits_min.load();
        if (value >= 0) g_hitbits_min.store(value);
        g_opt_gen.fetch_add(1);
        return RS_OK;
    }
    if (!strcmp(name, "device_chunk")) {
        if (old_value) *old_value = g_device_chunk.load();
        if (value > 0) g_device_chunk.store(((value + 1023) / 1024) * 1024);
        return RS_OK;
    }
    if (rs::sorted_option(name, value, old_value)) return fail(RS_INVALID_ARG, "unknown option %s", name);
    g_opt_gen.fetch_add(1);
    return RS_OK;
}

RS_API const char* rs_hot_kernel(void) { return rs::hot_kernel_name(); }

// Diagnostics: the device status words of the calling thread's last
// graph-replayed rs_run_batch_device (bad, internal, hits, tile_counter,
// visits, mts, cand_count, pad); builds with -DRS_TILE_STATS fill the
// traversal counters.
RS_API int rs_last_status(unsigned long long* out8) {
    std::memcpy(out8, &g_last_status, sizeof(RsStatus));
    return RS_OK;
}

}  // extern "C"

void rs::stage_mark(int k, cudaStream_t s) {
    if (k >= 0 && k < kStageEvents) mark(kTagStage + k, s);
}

void rs::hot_kernel_mark(int which, cudaStream_t s) {
    if (g_hot_mark_mask & (1 << which)) mark(3 + which, s);
}

// chunks of a large pageable batch (RS_STAGE_PARTS): the first chunk's
// host copy is exposed, so staged batches use finer chunks
static const int64_t g_stage_parts = [] {
    const char* e = getenv("RS_STAGE_PARTS");
    return (int64_t)(e && *e ? atoi(e) : 16);
}();

// set while the host pipeline re-runs a batch with the binary kernels
static thread_local bool g_force_binary = false;

extern "C" {

static int run_batch_host_impl(const float* h_verts, int64_t n_v, const int32_t* h_tris, int64_t n_t,
                               const float* h_starts, const float* h_ends, int64_t n_r, int mode,
                               int tree_kind, int max_coll, int max_stack, int64_t chunk_rays,
                               int32_t* h_flags, int32_t* h_ray, float* h_dist, int32_t* h_tri,
                               float* h_pt, int64_t* n_hits, int64_t* bad, void* stream) {
    int rc = check_query(mode, max_coll, max_stack);
    if (rc) return rc;
    if (bad) *bad = -1;
    if (n_hits) *n_hits = 0;
    if (n_r == 0 || n_t == 0) {
        if (h_flags && n_r > 0) memset(h_flags, 0, sizeof(int32_t) * (size_t)n_r);
        return RS_OK;
    }
    if (n_r > 2147483647ll) return fail(RS_INVALID_ARG, "segment count exceeds int32 indexing");
    rc = check_mesh(n_v, n_t);
    if (rc) return rc;
    rc = configure_pool();
    if (rc) return rc;
    rc = pipe_init();
    if (rc) return rc;
    cudaStream_t s = S(stream);
    cudaStream_t cp = g_pipe.copy;
    const bool auto_chunks = chunk_rays <= 0;
    // large batches: 8 chunks (12 for barycentric, whose per-chunk row copies
    // trail the device; C3 e2e 5.70 -> 5.51 ms)
    const int64_t big_parts = mode == kBarycentric ? 12 : (is_pageable(h_starts) ? g_stage_parts : 8);
    if (auto_chunks)
        chunk_rays = n_r > (8ll << 20) ? (n_r + big_parts - 1) / big_parts
                                       : (n_r > (1 << 20) ? (n_r + 3) / 4 : n_r);
    chunk_rays = ((chunk_rays + 127) / 128) * 128;
    // chunk boundaries: uniform; with automatic sizing the last chunk is
    // split 3:1 so the work left after the final upload (its query and flag
    // copy) is a quarter chunk
    std::vector<int64_t> bounds;
    for (int64_t lo = 0; lo < n_r; lo += chunk_rays) bounds.push_back(lo);
    if (auto_chunks && bounds.size() > 1) {
        const int64_t last = bounds.back(), rem = n_r - last;
        const int64_t cut = ((rem * 3 / 4 + 127) / 128) * 128;  // (7:1 and 15:1 measured slower)
        if (cut > 0 && cut < rem) bounds.push_back(last + cut);
    }
    bounds.push_back(n_r);
    const int64_t nchunks = (int64_t)bounds.size() - 1;
    auto chunk_lo = [&](int64_t k) { return bounds[k]; };
    auto chunk_cnt = [&](int64_t k) { return bounds[k + 1] - bounds[k]; };
    const bool bary = mode == kBarycentric;
    const bool fast_tree = tree_kind == kTreeFast && !g_binary_fast;
    const bool fast = fast_tree && !g_force_binary;
    // Barycentric rows into pinned host outputs: each chunk's compaction
    // writes its rows straight into the caller's (mapped) host arrays at the
    // running row count, so the D2H overlaps the remaining uploads instead
    // of one copy after the last chunk.  Pageable outputs: device rows + copy.
    int32_t *zray = nullptr, *ztri = nullptr;
    float *zdist = nullptr, *zpt = nullptr;
    bool zc = false;
    if (bary && fast && g_zero_copy && !buffer_path()) {
        void *a = nullptr, *b = nullptr, *cc = nullptr, *d = nullptr;
        zc = cudaHostGetDevicePointer(&a, h_ray, 0) == cudaSuccess &&
             cudaHostGetDevicePointer(&b, h_dist, 0) == cudaSuccess &&
             cudaHostGetDevicePointer(&cc, h_tri, 0) == cudaSuccess &&
             cudaHostGetDevicePointer(&d, h_pt, 0) == cudaSuccess;
        cudaGetLastError();
        zray = static_cast<int32_t*>(a); zdist = static_cast<float*>(b);
        ztri = static_cast<int32_t*>(cc); zpt = static_cast<float*>(d);
    }

    // one device block: mesh, 2x chunk inputs, outputs, status, tile status
    const size_t mesh_b = align256(12ull * n_v) + align256(12ull * n_t);
    const size_t in_b = 2 * 2 * align256(12ull * chunk_rays);
    // boolean flags return as bits (the PCIe D2H of 4-B flags ran beside the
    // uploads and slowed them by ~10%); the host threads expand them
    const bool pack = mode == kBoolean && g_pack_flags;
    const size_t bits_b = pack ? align256(4ull * (chunk_rays / 32 + 1)) : 0;
    const size_t out_b = bary ? (zc ? 256 : 4 * align256(12ull * n_r)) : 2 * align256(4ull * chunk_rays) + 2 * bits_b;
    const size_t tiles_b = align256(compact_scratch_bytes(chunk_rays)) * (size_t)nchunks;
    const size_t st_b = align256(sizeof(RsStatus) * (size_t)nchunks);
    // every exit (errors included) drains the pipeline's streams and
    // releases the device block, the tree and the per-buffer scratch
    struct Cleanup {
        cudaStream_t s;
        char* blk = nullptr;
        rs_tree* t = nullptr;
        FastScratch fs[2];
        ~Cleanup() {
            cudaStreamSynchronize(g_pipe.copy);
            cudaStreamSynchronize(g_pipe.copy2);
            cudaStreamSynchronize(s);
            for (auto& f : fs)
                if (f.blk) dfree(f.blk, s);
            if (t) rs_free(t, s);
            if (blk) dfree(blk, s);
            cudaStreamSynchronize(s);
        }
    } guard{s};
    FastScratch* fs = guard.fs;
    CK(dmalloc(reinterpret_cast<void**>(&guard.blk), mesh_b + in_b + out_b + tiles_b + st_b, s));
    char* blk = guard.blk;
    Carver c{blk};
    float* dV = c.take<float>(3ull * n_v);
    int* dT = c.take<int>(3ull * n_t);
    float* din[2][2];
    for (int k = 0; k < 2; ++k) {
        din[k][0] = c.take<float>(3ull * chunk_rays);
        din[k][1] = c.take<float>(3ull * chunk_rays);
    }
    int32_t* dflag[2] = {nullptr, nullptr};
    int32_t *dray = nullptr, *dtri = nullptr;
    float *ddist = nullptr, *dpt = nullptr;
    unsigned long long* d_rows = nullptr;
    if (bary && zc) {
        d_rows = c.take<unsigned long long>(1);
    } else if (bary) {
        dray = c.take<int32_t>(n_r);
        ddist = c.take<float>(n_r);
        dtri = c.take<int32_t>(n_r);
        dpt = c.take<float>(3ull * n_r);
    } else {
        dflag[0] = c.take<int32_t>(chunk_rays);
        dflag[1] = c.take<int32_t>(chunk_rays);
    }
    unsigned* dbits[2] = {nullptr, nullptr};
    if (pack) {
        dbits[0] = c.take<unsigned>(chunk_rays / 32 + 1);
        dbits[1] = c.take<unsigned>(chunk_rays / 32 + 1);
        const size_t words = (size_t)(n_r / 32) + (size_t)nchunks + 1;
        if (g_pipe.hbits_cap < words) {
            if (g_pipe.hbits) {
                CK(cudaStreamSynchronize(g_pipe.copy2));  // a previous call's copies may still land
                cudaFreeHost(g_pipe.hbits);
            }
            g_pipe.hbits = nullptr;
            g_pipe.hbits_cap = 0;
            CK(cudaHostAlloc(reinterpret_cast<void**>(&g_pipe.hbits), 4 * words, cudaHostAllocDefault));
            g_pipe.hbits_cap = words;
        }
    }
    // chunk boundaries are multiples of 128 rows: chunk k's bits start at word lo / 32
    auto expand_chunk = [&](int64_t k) -> int {
        CK(cudaEventSynchronize(g_pipe.ev_out[k & 1]));
        expand_bits_host(g_pipe.hbits + chunk_lo(k) / 32, chunk_cnt(k), h_flags + chunk_lo(k));
        return RS_OK;
    };
    char* tiles = reinterpret_cast<char*>(c.take<char>(align256(compact_scratch_bytes(chunk_rays)) * nchunks));
    RsStatus* st = c.take<RsStatus>(nchunks);
    // Streams: s computes (build, then one query per chunk), h2d = g_pipe.copy
    // uploads the chunks (PCIe H2D is the bound of this path: the inputs are
    // 24 B per segment), d2h = g_pipe.copy2 returns each chunk's flags as soon
    // as its query ends.  The uploads start right after the allocation, so
    // the mesh upload and the build overlap chunk 0's transfer.
    cudaStream_t h2d = cp, d2h = g_pipe.copy2;
    CK(cudaMemsetAsync(tiles, 0, tiles_b + st_b, s));
    if (d_rows) CK(cudaMemsetAsync(d_rows, 0, sizeof(unsigned long long), s));
    CK(cudaEventRecord(g_pipe.ev_blk, s));
    CK(cudaStreamWaitEvent(h2d, g_pipe.ev_blk, 0));
    CK(cudaStreamWaitEvent(d2h, g_pipe.ev_blk, 0));
    // pageable inputs: two pinned chunk slots (starts, ends) + the mesh
    const bool stage_in = is_pageable(h_starts) || is_pageable(h_ends);
    const bool stage_mesh = is_pageable(h_verts) || is_pageable(h_tris);
    const size_t slot_b = align256(24ull * chunk_rays);
    const size_t mesh_hb = align256(12ull * n_v) + align256(12ull * n_t);
    float* stg_in[2] = {nullptr, nullptr};
    if (stage_in || stage_mesh) {
        const size_t need = (stage_in ? 2 * slot_b : 0) + (stage_mesh ? mesh_hb : 0);
        if (g_pipe.stg_cap < need) {
            CK(cudaStreamSynchronize(h2d));  // the old slots may still feed a copy
            if (g_pipe.stg) cudaFreeHost(g_pipe.stg);
            g_pipe.stg = nullptr;
            g_pipe.stg_cap = 0;
            CK(cudaHostAlloc(reinterpret_cast<void**>(&g_pipe.stg), need, cudaHostAllocDefault));
            g_pipe.stg_cap = need;
        }
        if (stage_in) {
            stg_in[0] = reinterpret_cast<float*>(g_pipe.stg);
            stg_in[1] = reinterpret_cast<float*>(g_pipe.stg + slot_b);
        }
    }
    const float* mesh_v = h_verts;
    const int32_t* mesh_t = h_tris;
    if (stage_mesh) {
        char* m = g_pipe.stg + (stage_in ? 2 * slot_b : 0);
        CopyPool::get().copy(m, h_verts, 12ull * n_v);
        CopyPool::get().copy(m + align256(12ull * n_v), h_tris, 12ull * n_t);
        mesh_v = reinterpret_cast<const float*>(m);
        mesh_t = reinterpret_cast<const int32_t*>(m + align256(12ull * n_v));
    }
    // chunk k's rows into slot k & 1 (its previous upload must have landed)
    auto stage_chunk = [&](int64_t k) -> int {
        const int b = (int)(k & 1);
        if (k >= 2) CK(cudaEventSynchronize(g_pipe.ev_in[b]));
        const int64_t lo = chunk_lo(k), cnt = chunk_cnt(k);
        CopyPool::get().copy(stg_in[b], h_starts + 3 * lo, 12ull * cnt);
        CopyPool::get().copy(stg_in[b] + 3 * chunk_rays, h_ends + 3 * lo, 12ull * cnt);
        return RS_OK;
    };
    if (stage_in && (rc = stage_chunk(0))) return rc;
    CK(cudaMemcpyAsync(dV, mesh_v, 12ull * n_v, cudaMemcpyHostToDevice, s));
    CK(cudaMemcpyAsync(dT, mesh_t, 12ull * n_t, cudaMemcpyHostToDevice, s));
    mark(0, s);
    rc = build_impl(dV, n_v, dT, n_t, tree_kind, nullptr, nullptr, s, &guard.t, nullptr, true);
    if (rc) return rc;
    rs_tree* const t = guard.t;
    const int ref = tree_kind == kTreeReference;
    if (fast_tree && g_force_binary) max_stack = 1 << 30;  // the binary walk of a fast tree: no overflow rule
    if (fast)
        for (int b = 0; b < 2; ++b) {
            rc = fast_alloc(fs[b], chunk_rays, mode, 2 * chunk_rays + 4096, s);
            if (rc) return rc;
        }
    unsigned long long running = 0;  // barycentric rows already placed
    // Barycentric rows (device-compacted per chunk) come back one chunk
    // behind: once chunk j's status has landed in pinned memory the host
    // knows its row count and queues the row copies at the running offset,
    // while the device already works on chunk j+1.
    const bool lagged = bary && !zc && !buffer_path();
    if (lagged && g_pipe.hst_cap < nchunks) {
        if (g_pipe.hst) cudaFreeHost(g_pipe.hst);
        CK(cudaHostAlloc(reinterpret_cast<void**>(&g_pipe.hst), sizeof(RsStatus) * nchunks,
                         cudaHostAllocDefault));
        g_pipe.hst_cap = nchunks;
    }
    auto retire = [&](int64_t j) -> int {
        CK(cudaEventSynchronize(g_pipe.ev_out[j & 1]));
        const size_t m = (size_t)g_pipe.hst[j].hits;
        const int64_t lo = chunk_lo(j);
        if (m && !g_pipe.hst[j].bad && !g_pipe.hst[j].internal) {
            CK(cudaMemcpyAsync(h_ray + running, dray + lo, 4 * m, cudaMemcpyDeviceToHost, d2h));
            CK(cudaMemcpyAsync(h_dist + running, ddist + lo, 4 * m, cudaMemcpyDeviceToHost, d2h));
            CK(cudaMemcpyAsync(h_tri + running, dtri + lo, 4 * m, cudaMemcpyDeviceToHost, d2h));
            CK(cudaMemcpyAsync(h_pt + 3 * running, dpt + 3 * lo, 12 * m, cudaMemcpyDeviceToHost, d2h));
        }
        running += m;
        return RS_OK;
    };
    for (int64_t k = 0; k < nchunks; ++k) {
        const int b = (int)(k & 1);
        const int64_t lo = chunk_lo(k);
        const int64_t cnt = chunk_cnt(k);
        if (k >= 2) CK(cudaStreamWaitEvent(h2d, g_pipe.ev_q[b], 0));  // input buffer b free again
        const float* src_s = stage_in ? stg_in[b] : h_starts + 3 * lo;
        const float* src_e = stage_in ? stg_in[b] + 3 * chunk_rays : h_ends + 3 * lo;
        CK(cudaMemcpyAsync(din[b][0], src_s, 12ull * cnt, cudaMemcpyHostToDevice, h2d));
        CK(cudaMemcpyAsync(din[b][1], src_e, 12ull * cnt, cudaMemcpyHostToDevice, h2d));
        CK(cudaEventRecord(g_pipe.ev_in[b], h2d));
        CK(cudaStreamWaitEvent(s, g_pipe.ev_in[b], 0));
        if (k >= 2 && !bary) CK(cudaStreamWaitEvent(s, g_pipe.ev_out[b], 0));  // flags b read back
        if (fast) {
            fs[b].st = st + k;
            FastOut o;
            o.ray_offset = lo;
            if (bary && zc) {
                o.c_ray = zray; o.c_dist = zdist; o.c_tri = ztri; o.c_pt = zpt;
                o.row_base = d_rows;
                o.mapped = true;
            } else if (bary) {
                o.c_ray = dray + lo; o.c_dist = ddist + lo; o.c_tri = dtri + lo; o.c_pt = dpt + 3 * lo;
            } else {
                o.flags = dflag[b];
            }
            rc = fast_launch(t, din[b][0], din[b][1], cnt, mode, o, fs[b], false, s);
            if (rc) return rc;
        } else {
            QueryArgs a = make_args(t, din[b][0], din[b][1], cnt, max_coll, max_stack, st + k);
            if (fast_tree) a.nodes4 = nullptr;  // binary kernels over the fast tree's records
            a.ray_offset = lo;
            if (bary) {
                // each chunk compacts into its own region; rows are concatenated on the host
                a.c_ray = dray + lo;
                a.c_dist = ddist + lo;
                a.c_tri = dtri + lo;
                a.c_point = dpt + 3 * lo;
                a.tile_status = reinterpret_cast<unsigned long long*>(
                    tiles + align256(compact_scratch_bytes(chunk_rays)) * k);
            } else {
                a.detected = dflag[b];
                a.counts = dflag[b];
            }
            mark(1, s);
            const int lq = launch_query(a, mode, ref != 0, bary, kstack_for(ref != 0, max_stack), false, s);
            mark(2, s);
            if (lq) return fail(RS_INVALID_ARG, "no kernel variant for this configuration");
            CK(cudaGetLastError());
        }
        if (pack) launch_pack_flags(dflag[b], cnt, dbits[b], s);
        CK(cudaEventRecord(g_pipe.ev_q[b], s));
        if (pack) {
            CK(cudaStreamWaitEvent(d2h, g_pipe.ev_q[b], 0));
            CK(cudaMemcpyAsync(g_pipe.hbits + lo / 32, dbits[b], 4ull * ((cnt + 31) / 32), cudaMemcpyDeviceToHost, d2h));
            CK(cudaEventRecord(g_pipe.ev_out[b], d2h));
        } else if (!bary) {
            CK(cudaStreamWaitEvent(d2h, g_pipe.ev_q[b], 0));
            CK(cudaMemcpyAsync(h_flags + lo, dflag[b], 4ull * cnt, cudaMemcpyDeviceToHost, d2h));
            CK(cudaEventRecord(g_pipe.ev_out[b], d2h));
        } else if (lagged) {
            CK(cudaStreamWaitEvent(d2h, g_pipe.ev_q[b], 0));
            CK(cudaMemcpyAsync(g_pipe.hst + k, st + k, sizeof(RsStatus), cudaMemcpyDeviceToHost, d2h));
            CK(cudaEventRecord(g_pipe.ev_out[b], d2h));
            if (k >= 1 && (rc = retire(k - 1))) return rc;
        }
        // the next chunk's rows into the other pinned slot while this one uploads
        if (stage_in && k + 1 < nchunks && (rc = stage_chunk(k + 1))) return rc;
        // the previous chunk's flags, expanded while this chunk uploads
        if (pack && k >= 1 && (rc = expand_chunk(k - 1))) return rc;
    }
    if (pack && (rc = expand_chunk(nchunks - 1))) return rc;
    if (lagged && (rc = retire(nchunks - 1))) return rc;
    cp = d2h;
    // statuses of every chunk; barycentric row counts come back with them
    std::vector<RsStatus> hst_v((size_t)nchunks);
    RsStatus* hst = hst_v.data();
    CK(cudaStreamWaitEvent(cp, g_pipe.ev_q[(nchunks - 1) & 1], 0));
    CK(cudaMemcpyAsync(hst, st, sizeof(RsStatus) * nchunks, cudaMemcpyDeviceToHost, cp));
    CK(cudaStreamSynchronize(cp));
    if (fast) {
        for (int b = 0; b < 2; ++b) {
            CK(dfree(fs[b].blk, s));
            fs[b].blk = nullptr;
        }
        // collision-buffer overflow in a chunk: redo that chunk with a buffer
        // sized to what its traversal claimed
        for (int64_t k = 0; k < nchunks; ++k) {
            if ((long long)hst[k].cand_count <= fs[0].cap) continue;
            const int64_t lo = chunk_lo(k);
            const int64_t cnt = chunk_cnt(k);
            CK(cudaStreamSynchronize(cp));
            CK(cudaMemcpyAsync(din[0][0], h_starts + 3 * lo, 12ull * cnt, cudaMemcpyHostToDevice, s));
            CK(cudaMemcpyAsync(din[0][1], h_ends + 3 * lo, 12ull * cnt, cudaMemcpyHostToDevice, s));
            FastOut o;
            o.ray_offset = lo;
            if (bary) {
                o.c_ray = dray + lo; o.c_dist = ddist + lo; o.c_tri = dtri + lo; o.c_pt = dpt + 3 * lo;
            } else {
                o.flags = dflag[0];
            }
            rc = fast_query(t, din[0][0], din[0][1], cnt, mode, o, false, hst + k, s);
            if (rc) return rc;
            if (!bary) {
                CK(cudaMemcpyAsync(h_flags + lo, dflag[0], 4ull * cnt, cudaMemcpyDeviceToHost, s));
                CK(cudaStreamSynchronize(s));
            }
        }
    }
    unsigned long long badv = 0, internal = 0;
    for (int64_t k = 0; k < nchunks; ++k) {
        if (hst[k].bad && (!badv || ~hst[k].bad < ~badv)) badv = hst[k].bad;
        internal |= hst[k].internal;
    }
    if (fast && internal) {
        // a fast-path walk exceeded its capacity (never expected: fast trees
        // are at most 61 deep): redo the batch with the binary kernels, as
        // the device path does (binary_query)
        guard.~Cleanup();
        new (&guard) Cleanup{s};
        g_force_binary = true;
        rc = run_batch_host_impl(h_verts, n_v, h_tris, n_t, h_starts, h_ends, n_r, mode, tree_kind,
                                 max_coll, max_stack, chunk_rays, h_flags, h_ray, h_dist, h_tri, h_pt,
                                 n_hits, bad, stream);
        g_force_binary = false;
        return rc;
    }
    if (bary && zc) {
        for (int64_t k = 0; k < nchunks; ++k) running += hst[k].hits;  // rows already in place
    } else if (bary && lagged) {
        CK(cudaStreamSynchronize(cp));  // rows already queued chunk by chunk
    } else if (bary && !badv && !internal) {
        for (int64_t k = 0; k < nchunks; ++k) {
            const int64_t lo = chunk_lo(k);
            const size_t m = (size_t)hst[k].hits;
            if (m) {
                CK(cudaMemcpyAsync(h_ray + running, dray + lo, 4 * m, cudaMemcpyDeviceToHost, cp));
                CK(cudaMemcpyAsync(h_dist + running, ddist + lo, 4 * m, cudaMemcpyDeviceToHost, cp));
                CK(cudaMemcpyAsync(h_tri + running, dtri + lo, 4 * m, cudaMemcpyDeviceToHost, cp));
                CK(cudaMemcpyAsync(h_pt + 3 * running, dpt + 3 * lo, 12 * m, cudaMemcpyDeviceToHost, cp));
            }
            running += m;
        }
        CK(cudaStreamSynchronize(cp));
    }
    if (n_hits) *n_hits = (int64_t)running;
    RsStatus agg{};
    agg.bad = badv;
    agg.internal = internal;
    return status_code(agg, bad);
}

int rs_run_batch_host(const float* h_verts, int64_t n_v, const int32_t* h_tris, int64_t n_t,
                      const float* h_starts, const float* h_ends, int64_t n_r, int mode,
                      int tree_kind, int max_coll, int max_stack, int64_t chunk_rays,
                      int32_t* h_flags, int32_t* h_ray, float* h_dist, int32_t* h_tri,
                      float* h_pt, int64_t* n_hits, int64_t* bad, void* stream) {
    marks_reset();
    rs::set_batch_rays(n_r);  // chunks choose their traversal by the whole batch's density
    const int rc = run_batch_host_impl(h_verts, n_v, h_tris, n_t, h_starts, h_ends, n_r, mode, tree_kind,
                                       max_coll, max_stack, chunk_rays, h_flags, h_ray, h_dist, h_tri,
                                       h_pt, n_hits, bad, stream);
    rs::set_batch_rays(0);
    return rc;
}

}  // extern "C"
