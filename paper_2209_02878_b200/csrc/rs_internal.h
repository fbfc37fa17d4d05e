// rs_internal.h -- host-side declarations shared by the .cu translation units.
#pragma once

#include <cuda_runtime.h>

#include "rs_common.cuh"

namespace rs {

// Number of kernels this library has launched (bench.py's gpu_launches).
void count_launches(long long k);
// Per-device launch facts (cached per device, thread-safe; rs_capi.cu).
int device_sms();
int occupancy(const void* kernel, int threads, size_t dynamic_smem = 0);
void ensure_dynamic_smem(const void* kernel, int bytes);
// Device timing of the dominant kernel (bench.py roofline): 0 before, 1 after.
void hot_kernel_mark(int which, cudaStream_t s);
void stage_mark(int k, cudaStream_t s);  // rs_set_timing(3) diagnostics

// The reference BvhTree SoA fields (lbvh.py:39-55) plus climb scratch.
struct TreeArrays {
    float* int_bounds;   // (n,6)
    int* child_l;        // (n,)  slot n-1: root ref
    int* child_r;
    int* range_l;
    int* range_r;
    int* int_tri;        // -1 internal, -2 root
    int* visit;
    float* leaf_bounds;  // (n,6)
    int* leaf_tri;
    int* leaf_range_l;
    int* leaf_range_r;
    int* sorted_ids;
    int* height;         // (2n,) subtree height by node ref
    int* parent;         // (2n,) parent internal node by node ref (root: -1)
};

bool is_build_kernel(const void* f);

void launch_prep(const float* V, const int* T, int n, double* cent, RsHeader* hdr,
                 const TreeArrays& ta, bool centroids, cudaStream_t s, bool lean = false);
// Query-only climb: RsNode/RsLeaf records and the root, no SoA fields.
void launch_climb_lean(const float* V, const int* T, int n, const unsigned long long* codes,
                       const int* ids, int* visit, RsNode* nodes, RsLeaf* leaves, RsHeader* hdr,
                       float* leaf_boxes, cudaStream_t s);
void launch_code_samples(const unsigned long long* codes, int n, int stride,
                         unsigned long long* samples, int m, cudaStream_t s);
void launch_keys(const double* cent, int n, const RsHeader* hdr, int kind,
                 unsigned long long* keys, int* vals, cudaStream_t s);
size_t sort_scratch_bytes(int n, int passes);
void launch_sort(unsigned long long* keys, int* vals, unsigned long long* keys_alt,
                 int* vals_alt, int n, int passes, void* scratch, cudaStream_t s);
// sort_segments_by_morton on device (engine.py:125-147): So/Eo = the
// segments in Z-order of their f64 midpoints, perm[k] = original index.
size_t sort_segments_scratch_bytes(int n);
void launch_sort_segments(const float* S, const float* E, int n, float* So, float* Eo,
                          long long* perm, void* scratch, cudaStream_t s);
void launch_climb(const float* V, const int* T, int n, const unsigned long long* codes,
                  const int* ids, const TreeArrays& ta, RsNode* nodes, RsLeaf* leaves,
                  RsHeader* hdr, cudaStream_t s);

// Collapse the binary LBVH into the 4-wide BVH the fast traversal reads:
// internal nodes at even depth are kept, each takes its grandchildren (or a
// leaf child itself) as its <= 4 children.  Node4 slots are indexed by the
// binary node id (sparse), so no allocation pass is needed.
void launch_collapse(int n, const TreeArrays& ta, const RsNode* nodes, RsNode4* nodes4,
                     const RsHeader* hdr, cudaStream_t s);

// Query-side launch parameters.
struct QueryArgs {
    const RsNode* nodes;
    const RsNode4* nodes4;  // fast trees: 4-wide nodes (null for reference trees)
    const RsLeaf* leaves;
    const RsHeader* hdr;  // root ref is read on device (no host sync after a build)
    int n_int;
    const float* starts;  // (n_r,3) f32 AoS
    const float* ends;
    long long n_r;
    int max_coll;
    int max_stack;
    // dense outputs (rows [0, n_r) of the caller's arrays), any may be null
    int* detected;
    int* counts;
    int* tri;
    float* dist;
    float* points;
    // compact barycentric outputs
    int* c_ray;
    float* c_dist;
    int* c_tri;
    float* c_point;
    unsigned long long* tile_status;
    long long ray_offset;  // added to compacted ray indices
    RsStatus* status;
};

// kstack: traversal stack capacity.  Fast trees (30-bit codes + 31-bit ids)
// have height <= 61, so 64 always suffices; reference trees use
// min(max_stack, 128) (height <= 94).
// ref_semantics: emulate the reference's collision-buffer flush points and
// max_stack overflow exactly (reference tree); compact: barycentric rows.
int launch_query(const QueryArgs& a, int mode, bool ref_semantics, bool compact, int kstack,
                 bool stats, cudaStream_t s);
size_t compact_scratch_bytes(long long n_r);

// Fast-tree path (rs_trav.cu): traversal -> collision buffer -> exact tests.
struct TravArgs {
    const RsNode4* nodes4;
    const RsHeader* hdr;
    int n_int;
    const float* starts;
    const float* ends;
    long long n_r;
    int2* cand;            // collision buffer (segment, leaf)
    long long cand_cap;    // multiple of kCandChunk
    int* chunk_fill;       // entries used per chunk
    RsStatus* status;
    int* gstack;           // per-group traversal stack overflow (trav_gstack_ints())
};
size_t trav_gstack_ints();
struct ExactArgs {
    const int2* cand;
    const unsigned long long* cand_count;
    long long cand_cap;
    const int* chunk_fill;
    const float* starts;
    const float* ends;
    const RsLeaf* leaves;
    int* flags;                  // boolean: crossing (pre-zeroed); count: counts (pre-zeroed)
    unsigned long long* best_t;  // barycentric: min t key per segment (pre-set to ~0)
    int* best_tri;               // barycentric: winning triangle (pre-set to -1)
    unsigned long long* cand_t;  // barycentric: t key per candidate
    unsigned long long* mts;
    unsigned long long* dropped; // set when the buffer overflowed (results incomplete)
};
struct CompactArgs {
    long long n_r;
    const unsigned long long* best_t;
    const int* best_tri;
    const float* starts;
    const float* ends;
    int* ray;
    float* dist;
    int* tri;
    float* point;
    unsigned long long* tile_status;
    unsigned long long* tile_counter;
    unsigned long long* n_hits;
    long long ray_offset;
    unsigned long long* row_base;  // optional: rows land at *row_base + rank, then *row_base += hits
    // best_t == null (sorted fast path): t is recomputed for each hit row
    // from its winning triangle -- leaves[leaf_of[tri]] -- with the same f64
    // test, instead of being stored per segment by the traversal
    const RsLeaf* leaves;
    const int* leaf_of;
    // rows land in host-mapped memory: form them in one kernel (a second
    // pass would read ray/triangle back over PCIe)
    bool fused;
};
// leaf_of[leaves[k].id] = k for the n leaves (the compaction's t recompute).
void launch_leaf_inverse(const RsLeaf* leaves, int n, int* leaf_of, cudaStream_t s);
void launch_trav(const TravArgs& a, bool stats, cudaStream_t s);

// Coherent fast path (rs_sorted.cu): root cull + counting sort into spatial
// bins, then one thread per segment in bin order.
struct SortedArgs {
    const RsNode4* nodes4;
    const RsNode* nodes;
    const RsLeaf* leaves;
    const RsHeader* hdr;
    int n_int;
    const float* starts;
    const float* ends;
    long long n_r;
    unsigned* bins;      // sorted_bins() counters (zeroed)
    unsigned* cursor;    // sorted_bins() scatter cursors
    unsigned* n_live;    // live segment count (written by the scan)
    float* seg_stats;    // k_seg_sample: per-CTA (sum of box sides x/y/z, live count)
    unsigned* tile_sum;  // sorted_bins()/1024 per-tile counts (zeroed) -> tile offsets
    float4* rec;         // n_r x 32-B records (start, id, end)
    int* flags;                  // boolean / count output (pre-zeroed)
    unsigned long long* best_t;  // barycentric (pre-set ~0)
    int* best_tri;               // barycentric (pre-set -1)
    RsStatus* status;
    unsigned bin_occupancy;  // binning: target live segments per bin (set at launch)
    unsigned tile_area;  // tile traversal: target triangles' worth of records per tile (set at launch)
    unsigned tile_depth; // tile traversal: records per tile <= tile_depth / depth complexity (0: off)
    // Morton-range candidate lists (fast lean trees; codes == nullptr disables)
    const unsigned long long* codes;         // sorted 30-bit keys, leaf order
    const unsigned long long* code_samples;  // codes[k * sample_stride]
    int sample_stride;
    int n_samples;
    const float* leaf_boxes;                 // (n, 6) exact leaf boxes, leaf order
    unsigned range_max;                      // scan at most this many leaves, else walk
    int key_mode;                            // keys' grid: 0 isotropic, 1 per-axis
    unsigned tile_balance;      // tile traversal: at least this many tiles per CTA
    unsigned tile_min_density;  // tile traversal only above this many records per triangle
    int zero_flags;             // the histogram pass zeroes flags (instead of a preset memset)
    void* geom;                 // bin_geom_bytes(): bin geometry, written by k_seg_sample
    int geom_mode;              // 1: binning CTAs copy geom; 0: each derives it
    // boolean batches too large for their flags to stay in L2: hits set bits
    // here (n_r / 32 words, L2-resident) and k_expand_bits writes the int32
    // flags afterwards in one coalesced pass, instead of one partial-sector
    // DRAM read-modify-write per hit (null: flags written directly)
    unsigned* hitbits;
};
// Writes flags[i] = bit i of hitbits for i < n (every row: no zero preset needed).
void launch_expand_bits(int* flags, const unsigned* hitbits, long long n, cudaStream_t s);
// bits[w] bit j = (flags[32 w + j] != 0), (n + 31) / 32 words (the host
// pipeline returns boolean flags as bits: 32x fewer D2H bytes)
void launch_pack_flags(const int* flags, long long n, unsigned* bits, cudaStream_t s);
size_t sorted_bins();
size_t bin_geom_bytes();
bool sorted_wide();  // RS_SORTED_WIDE=1: 4-wide per-thread traversal (needs nodes4)
// binning needs only the header's root box (available right after k_prep)
void launch_binning(const SortedArgs& a, cudaStream_t s, bool zero_flags = false);
// whether launch_binning(..., zero_flags=true) can zero `flags` in its
// histogram pass (TMA path, 16-B aligned rows and flags)
bool binning_zeroes_flags(const float* starts, const float* ends, long long n_r, const int* flags);
void launch_sorted_trav(const SortedArgs& a, int mode, bool stats, cudaStream_t s);
// the whole batch's segment count while its chunks are traversed (0: none)
void set_batch_rays(long long n);
// Tuning knob by name (trav, tile_density, tile_balance, tile_area,
// bin_occupancy); value < 0 (or 0 for counts) only reads.  -1: unknown name.
int sorted_option(const char* name, long long value, long long* old);
// Fast-tree key grid: 0 isotropic, 1 per-axis, 2 auto (option "fast_keys").
int fast_key_mode();
// Fast-tree query path (option "fast_path"): 0 binned tile traversal
// (default), 1 collision buffer (pair traversal -> warp-aggregated append ->
// exact pass, re-launched with a sized buffer on overflow).
int fast_path();
// Initial collision-buffer capacity in entries (option "cand_cap"; 0: 2 x segments + 4096).
long long cand_cap_override();
// Name of the traversal kernel the last launch_sorted_trav chose.
const char* hot_kernel_name();
void launch_exact(const ExactArgs& a, int mode, bool stats, cudaStream_t s);
size_t bary_compact_scratch(long long n_r);
void launch_bary_compact(const CompactArgs& a, cudaStream_t s);  // also advances a.row_base
void launch_bary_dense(const CompactArgs& a, int* detected, int* tri, float* dist, float* points,
                       cudaStream_t s);

// Synthetic terrain segments on device (rs_gen.cu): the reference
// generator's distribution (oracle.py:228-271) from a counter-based RNG.
void launch_generate(const float* V, const int* T, long long n_t, double z_lo, double z_hi,
                     double x_hi, double y_hi, double frac, unsigned long long seed,
                     long long first, long long n, float* S, float* E, unsigned char* flags,
                     cudaStream_t s);

// sort_rays un-permutation (rs_trav.cu): dense rows out[perm[k]] = in[k];
// barycentric rows re-ordered ascending by original index perm[ray[r]].
void launch_unpermute_dense(const long long* perm, long long n, const int* in, int* out, cudaStream_t s);
size_t unpermute_scratch_bytes(long long n);
void launch_unpermute_rows(const long long* perm, long long n, const int* ray, const float* dist,
                           const int* tri, const float* pt, long long k_rows, int* o_ray, float* o_dist,
                           int* o_tri, float* o_pt, void* scratch, cudaStream_t s);

void launch_segment_boxes(const float* S, const float* E, long long n, float* B, cudaStream_t s);

struct BaselineArgs {
    const float* V;
    const int* T;
    int n_t;
    const float* starts;
    const float* ends;
    long long n_r;
    int* detected;
    int* counts;
    int* tri;
    float* dist;
    float* points;
    // barycentric into per-segment (t key, triangle) for k_bary_compact
    // instead of dense rows (null: dense)
    unsigned long long* best_t;
    int* best_tri;
};
void launch_baseline(const BaselineArgs& a, int mode, cudaStream_t s);
// oracle_intersect's plane + sign-test all-pairs (barycentric: best_t/best_tri)
void launch_sign_oracle(const BaselineArgs& a, int mode, cudaStream_t s);

}  // namespace rs
