// Dependent-chain latencies on one B200 SM (cycles per op): DADD, DMUL, DFMA,
// LDS.64, and an LDS issued right after a strong global store.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a tools/lat_fp64.cu -o /tmp/lat && /tmp/lat
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k(double* out, long long* cyc, double a, double b, double* g) {
    __shared__ double sh[256];
    sh[threadIdx.x] = threadIdx.x;
    __syncthreads();
    double x = a;
    long long t0, t1;
    constexpr int N = 256;
    // DADD chain
    t0 = clock64();
#pragma unroll
    for (int i = 0; i < N; ++i) x = __dadd_rn(x, b);
    t1 = clock64();
    cyc[0] = t1 - t0;
    t0 = clock64();
#pragma unroll
    for (int i = 0; i < N; ++i) x = __dmul_rn(x, b);
    t1 = clock64();
    cyc[1] = t1 - t0;
    t0 = clock64();
#pragma unroll
    for (int i = 0; i < N; ++i) x = __fma_rn(x, b, a);
    t1 = clock64();
    cyc[2] = t1 - t0;
    // LDS chain: address from the loaded value
    int idx = threadIdx.x & 7;
    t0 = clock64();
#pragma unroll
    for (int i = 0; i < N; ++i) idx = static_cast<int>(sh[idx]) & 7;
    t1 = clock64();
    cyc[3] = t1 - t0;
    // STG (strong) then dependent LDS chain
    t0 = clock64();
#pragma unroll 1
    for (int i = 0; i < N; ++i) {
        asm volatile("st.relaxed.gpu.global.f64 [%0], %1;" ::"l"(g + threadIdx.x), "d"(x) : "memory");
        idx = static_cast<int>(sh[idx]) & 7;
    }
    t1 = clock64();
    cyc[4] = t1 - t0;
    t0 = clock64();
#pragma unroll 1
    for (int i = 0; i < N; ++i) {
        asm volatile("st.global.f64 [%0], %1;" ::"l"(g + threadIdx.x), "d"(x) : "memory");
        idx = static_cast<int>(sh[idx]) & 7;
    }
    t1 = clock64();
    cyc[5] = t1 - t0;
    t0 = clock64();
#pragma unroll 1
    for (int i = 0; i < N; ++i) {
        idx = static_cast<int>(sh[idx]) & 7;
    }
    t1 = clock64();
    cyc[6] = t1 - t0;
    // named barrier round trip with 4 warps
    t0 = clock64();
#pragma unroll 1
    for (int i = 0; i < N; ++i) asm volatile("bar.sync 1, 128;" ::: "memory");
    t1 = clock64();
    cyc[7] = t1 - t0;
    out[threadIdx.x] = x + idx;
}
int main() {
    double *o, *g;
    long long* c;
    cudaMalloc(&o, 4096);
    cudaMalloc(&g, 4096);
    cudaMallocManaged(&c, 64 * 8);
    for (int rep = 0; rep < 2; ++rep) {
        k<<<1, 128>>>(o, c, 1.0000001, 0.9999999, g);
        cudaDeviceSynchronize();
    }
    const char* names[] = {"DADD", "DMUL", "DFMA", "LDS dep", "STG.strong+LDS (loop)", "STG+LDS (loop)", "LDS (loop)", "bar.sync 128"};
    for (int i = 0; i < 8; ++i) printf("%-24s %.1f cycles/op\n", names[i], c[i] / 256.0);
    return 0;
}
