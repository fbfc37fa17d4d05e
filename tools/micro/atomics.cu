// L2 atomic / scattered-store throughput probe (diagnostics for the binning
// scatter): 16M random indices over 512k u32 counters.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k_red(unsigned* c, const unsigned* idx, int n) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) atomicAdd(c + idx[i], 1u);
}
__global__ void k_atom(unsigned* c, const unsigned* idx, int n, unsigned* out) {
    for (int i = (blockIdx.x * blockDim.x + threadIdx.x) * 4; i < n; i += gridDim.x * blockDim.x * 4) {
        unsigned p[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) p[j] = atomicAdd(c + idx[i + j], 1u);
#pragma unroll
        for (int j = 0; j < 4; ++j) out[i + j] = p[j];
    }
}
__global__ void k_atom_st(unsigned* c, const unsigned* idx, int n, float4* rec, unsigned cap) {
    for (int i = (blockIdx.x * blockDim.x + threadIdx.x) * 4; i < n; i += gridDim.x * blockDim.x * 4) {
        unsigned p[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) p[j] = atomicAdd(c + idx[i + j], 1u);
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const unsigned q = (idx[i + j] * 32u + (p[j] & 31u)) % cap;
            rec[2ull * q] = make_float4(1, 2, 3, 4);
            rec[2ull * q + 1] = make_float4(5, 6, 7, 8);
        }
    }
}
__global__ void k_st(const unsigned* idx, int n, float4* rec, unsigned cap) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const unsigned q = (idx[i] * 32u + (i & 31)) % cap;
        rec[2ull * q] = make_float4(1, 2, 3, 4);
        rec[2ull * q + 1] = make_float4(5, 6, 7, 8);
    }
}
int main() {
    const int n = 16 << 20, bins = 512 << 10;
    const unsigned cap = 16u << 20;
    unsigned *c, *idx, *out;
    float4* rec;
    cudaMalloc(&c, 4ull * bins); cudaMalloc(&idx, 4ull * n); cudaMalloc(&out, 4ull * n);
    cudaMalloc(&rec, 32ull * cap);
    unsigned* h = new unsigned[n];
    unsigned long long x = 88172645463325252ull;
    for (int i = 0; i < n; ++i) { x ^= x << 13; x ^= x >> 7; x ^= x << 17; h[i] = (unsigned)(x % bins); }
    cudaMemcpy(idx, h, 4ull * n, cudaMemcpyHostToDevice);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    for (int grid_mul : {4, 8, 16}) {
        const int grid = sms * grid_mul;
        float ms;
        for (int rep = 0; rep < 2; ++rep) {
            cudaMemset(c, 0, 4ull * bins);
            cudaEventRecord(a); k_red<<<grid, 256>>>(c, idx, n); cudaEventRecord(b); cudaEventSynchronize(b);
            cudaEventElapsedTime(&ms, a, b);
            if (rep) printf("grid %d x256  RED      %.1f us  %.1f Gop/s\n", grid, ms * 1e3, n / ms / 1e6);
            cudaEventRecord(a); k_atom<<<grid, 256>>>(c, idx, n, out); cudaEventRecord(b); cudaEventSynchronize(b);
            cudaEventElapsedTime(&ms, a, b);
            if (rep) printf("grid %d x256  ATOM x4  %.1f us  %.1f Gop/s\n", grid, ms * 1e3, n / ms / 1e6);
            cudaEventRecord(a); k_atom_st<<<grid, 256>>>(c, idx, n, rec, cap); cudaEventRecord(b); cudaEventSynchronize(b);
            cudaEventElapsedTime(&ms, a, b);
            if (rep) printf("grid %d x256  ATOM+ST  %.1f us  %.1f Gop/s\n", grid, ms * 1e3, n / ms / 1e6);
            cudaEventRecord(a); k_st<<<grid, 256>>>(idx, n, rec, cap); cudaEventRecord(b); cudaEventSynchronize(b);
            cudaEventElapsedTime(&ms, a, b);
            if (rep) printf("grid %d x256  ST32B    %.1f us  %.1f Gop/s\n", grid, ms * 1e3, n / ms / 1e6);
        }
    }
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
