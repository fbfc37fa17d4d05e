// rs_gen.cu -- on-device synthetic segments for the terrain scenes.
//
// BASELINE configs[4] needs 1B segments: 24 GB of
// input that cannot come from the reference's numpy generator
// (raysurf/oracle.py:167-274) through PCIe in reasonable time.  This kernel
// restates that generator's DISTRIBUTION with a counter-based RNG keyed by
// (seed, global segment index), so any shard [first, first + n) of a batch
// is generated on the GPU that queries it, identically for every sharding:
//
//   flag     crossing with probability `crossing_fraction`      (oracle.py:219-222)
//   crossers vertical through a barycentric-interior point of a random
//            triangle, margin 0.05, from below or above the surface's z range
//            (oracle.py:228-249): ground truth = exactly one crossing
//   misses   kind 0 above / 1 below (xy within the domain +-1), 2 beside
//            (x in [-6,-1]) (oracle.py:251-271): ground truth = none
//
// Every f64 operation is explicitly rounded (no FMA contraction), so the
// numpy restatement in oracle/gen_oracle.py reproduces the output bit for bit.
#include "rs_internal.h"

namespace rs {

namespace {

__device__ __forceinline__ uint4 philox4x32_10(uint4 c, uint2 k) {
    constexpr unsigned M0 = 0xD2511F53u, M1 = 0xCD9E8D57u, W0 = 0x9E3779B9u, W1 = 0xBB67AE85u;
#pragma unroll
    for (int r = 0; r < 10; ++r) {
        const unsigned hi0 = __umulhi(M0, c.x), lo0 = M0 * c.x;
        const unsigned hi1 = __umulhi(M1, c.z), lo1 = M1 * c.z;
        c = make_uint4(hi1 ^ c.y ^ k.x, lo1, hi0 ^ c.w ^ k.y, lo0);
        k.x += W0;
        k.y += W1;
    }
    return c;
}

// numpy's 53-bit double from two 32-bit words: ((a >> 5) * 2^26 + (b >> 6)) / 2^53
__device__ __forceinline__ double u53(unsigned a, unsigned b) {
    return (double)((unsigned long long)(a >> 5) * 67108864ull + (b >> 6)) * (1.0 / 9007199254740992.0);
}

// a + (b - a) * u, rounded step by step (numpy's uniform)
__device__ __forceinline__ double uni(double a, double b, double u) {
    return __dadd_rn(a, __dmul_rn(__dsub_rn(b, a), u));
}

struct GenArgs {
    const float* V;
    const int* T;
    long long n_t;
    double z_lo, z_hi, z_pad, x_hi, y_hi, frac;
    unsigned long long seed;
    long long first;
    long long n;
    float* S;
    float* E;
    unsigned char* flags;
};

__global__ void __launch_bounds__(256) k_generate(GenArgs a) {
    const uint2 key = make_uint2((unsigned)a.seed, (unsigned)(a.seed >> 32) ^ 0x5EEDu);
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < a.n;
         i += (long long)gridDim.x * blockDim.x) {
        const unsigned long long g = (unsigned long long)(a.first + i);
        // 16 words: counters (g_lo, g_hi, 0..3, 0)
        unsigned w[16];
#pragma unroll
        for (int c = 0; c < 4; ++c) {
            const uint4 r = philox4x32_10(make_uint4((unsigned)g, (unsigned)(g >> 32), (unsigned)c, 0u), key);
            w[4 * c] = r.x; w[4 * c + 1] = r.y; w[4 * c + 2] = r.z; w[4 * c + 3] = r.w;
        }
        double u[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) u[k] = u53(w[2 * k], w[2 * k + 1]);
        const bool cross = u[0] < a.frac;
        double s0, s1, s2, e0, e1, e2;
        if (cross) {
            long long t = (long long)(u[1] * (double)a.n_t);  // exact: n_t < 2^53
            if (t >= a.n_t) t = a.n_t - 1;
            double w0 = u[2], w1 = u[3];
            if (__dadd_rn(w0, w1) > 1.0) { w0 = __dsub_rn(1.0, w0); w1 = __dsub_rn(1.0, w1); }
            const double m = 0.05, scale = __dsub_rn(1.0, __dmul_rn(3.0, m));
            const double b0 = __dadd_rn(m, __dmul_rn(scale, __dsub_rn(1.0, __dadd_rn(w0, w1))));
            const double b1 = __dadd_rn(m, __dmul_rn(scale, w0));
            const double b2 = __dadd_rn(m, __dmul_rn(scale, w1));
            const int* tri = a.T + 3 * t;
            const float* c0 = a.V + 3ll * tri[0];
            const float* c1 = a.V + 3ll * tri[1];
            const float* c2 = a.V + 3ll * tri[2];
            const double px = __dadd_rn(__dadd_rn(__dmul_rn(b0, (double)c0[0]), __dmul_rn(b1, (double)c1[0])),
                                        __dmul_rn(b2, (double)c2[0]));
            const double py = __dadd_rn(__dadd_rn(__dmul_rn(b0, (double)c0[1]), __dmul_rn(b1, (double)c1[1])),
                                        __dmul_rn(b2, (double)c2[1]));
            const double below = __dsub_rn(a.z_lo, __dmul_rn(a.z_pad, __dadd_rn(1.0, u[4])));
            const double above = __dadd_rn(a.z_hi, __dmul_rn(a.z_pad, __dadd_rn(1.0, u[5])));
            const bool up = u[6] < 0.5;
            s0 = e0 = px;
            s1 = e1 = py;
            s2 = up ? below : above;
            e2 = up ? above : below;
        } else {
            const int kind = (int)(u[1] * 3.0);
            s1 = uni(-1.0, a.y_hi, u[4]);
            e1 = uni(-1.0, a.y_hi, u[5]);
            if (kind == 2) {
                s0 = uni(-6.0, -1.0, u[2]);
                e0 = uni(-6.0, -1.0, u[3]);
                const double lo = __dsub_rn(a.z_lo, a.z_pad), hi = __dadd_rn(a.z_hi, a.z_pad);
                s2 = uni(lo, hi, u[6]);
                e2 = uni(lo, hi, u[7]);
            } else {
                s0 = uni(-1.0, a.x_hi, u[2]);
                e0 = uni(-1.0, a.x_hi, u[3]);
                const double span = __dmul_rn(2.0, a.z_pad);
                if (kind == 0) {
                    const double base = __dadd_rn(a.z_hi, a.z_pad);
                    s2 = __dadd_rn(base, uni(0.0, span, u[6]));
                    e2 = __dadd_rn(base, uni(0.0, span, u[7]));
                } else {
                    const double base = __dsub_rn(a.z_lo, a.z_pad);
                    s2 = __dsub_rn(base, uni(0.0, span, u[6]));
                    e2 = __dsub_rn(base, uni(0.0, span, u[7]));
                }
            }
        }
        float* sp = a.S + 3 * i;
        float* ep = a.E + 3 * i;
        sp[0] = __double2float_rn(s0); sp[1] = __double2float_rn(s1); sp[2] = __double2float_rn(s2);
        ep[0] = __double2float_rn(e0); ep[1] = __double2float_rn(e1); ep[2] = __double2float_rn(e2);
        if (a.flags) a.flags[i] = cross ? 1 : 0;
    }
}

}  // namespace

void launch_generate(const float* V, const int* T, long long n_t, double z_lo, double z_hi,
                     double x_hi, double y_hi, double frac, unsigned long long seed,
                     long long first, long long n, float* S, float* E, unsigned char* flags,
                     cudaStream_t s) {
    if (n <= 0) return;
    GenArgs a{V, T, n_t, z_lo, z_hi, 0.5 + 0.1 * (z_hi - z_lo), x_hi, y_hi, frac, seed, first, n,
              S, E, flags};
    const long long blocks_needed = (n + 255) / 256;
    const long long cap = (long long)device_sms() * 8;
    k_generate<<<(unsigned)(blocks_needed < cap ? blocks_needed : cap), 256, 0, s>>>(a);
    count_launches(1);
}

// compute_segment_boxes (engine.py:115-122): (n,6) f32 [xmin,xmax,ymin,ymax,zmin,zmax].
__global__ void __launch_bounds__(256) k_segment_boxes(const float* __restrict__ S, const float* __restrict__ E,
                                                       long long n, float* __restrict__ B) {
    for (long long i = blockIdx.x * 256ll + threadIdx.x; i < n; i += gridDim.x * 256ll) {
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            const float p = __ldg(S + 3 * i + k), q = __ldg(E + 3 * i + k);
            B[6 * i + 2 * k] = fminf(p, q);
            B[6 * i + 2 * k + 1] = fmaxf(p, q);
        }
    }
}

void launch_segment_boxes(const float* S, const float* E, long long n, float* B, cudaStream_t s) {
    if (n <= 0) return;
    const long long want = (n + 255) / 256, cap = (long long)device_sms() * 8;
    k_segment_boxes<<<(unsigned)(want < cap ? want : cap), 256, 0, s>>>(S, E, n, B);
    count_launches(1);
}

}  // namespace rs
