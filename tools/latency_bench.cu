// Diagnostics: primitive latencies on this B200 (cycles), single thread.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a tools/latency_bench.cu -o /tmp/lb && /tmp/lb
#include <cstdio>
constexpr int R = 4096;
__global__ void lat(double* out, long long* cyc, double seed, volatile unsigned long long* gflag) {
    __shared__ volatile unsigned long long s[64];
    double a = seed, b = seed * 0.5 + 1.0;
    long long t0 = clock64();
    for (int i = 0; i < R; ++i) a = __dadd_rn(a, b);
    long long t1 = clock64();
    for (int i = 0; i < R; ++i) a = __dmul_rn(a, 0.999999);
    long long t2 = clock64();
    for (int i = 0; i < R; ++i) a = __fma_rn(a, 0.999999, 1e-9);
    long long t3 = clock64();
    for (int i = 0; i < R / 8; ++i) a = __ddiv_rn(b, a);
    long long t4 = clock64();
    float f = (float)seed;
    for (int i = 0; i < R; ++i) f = __fadd_rn(f, 1.0f);
    long long t5 = clock64();
    // smem ping-pong between lane 0 and lane 1 (two warps: warp 0 lane 0, warp 1 lane 0)
    out[0] = a + f;
    cyc[0] = t1 - t0; cyc[1] = t2 - t1; cyc[2] = t3 - t2; cyc[3] = (t4 - t3) * 8; cyc[4] = t5 - t4;
}
__global__ void pingpong(long long* cyc, unsigned long long* g) {
    __shared__ volatile unsigned long long s[2];
    const int w = threadIdx.x >> 5;
    if ((threadIdx.x & 31) != 0) return;
    if (w == 0) { s[0] = 0; s[1] = 0; }
    __syncthreads();
    long long t0 = clock64();
    for (unsigned long long i = 1; i <= 1000; ++i) {
        if (w == 0) { while (s[1] != i - 1) {} s[0] = i; }
        else { while (s[0] != i) {} s[1] = i; }
    }
    long long t1 = clock64();
    if (w == 0) cyc[5] = (t1 - t0) / 1000;  // one round trip = 2 hops
}
__global__ void pingpong_global(long long* cyc, unsigned long long* g, int other) {
    // CTA 0 and CTA 1 bounce a counter through global memory (L2)
    if (threadIdx.x != 0) return;
    volatile unsigned long long* p = g;
    const int me = blockIdx.x;
    long long t0 = clock64();
    for (unsigned long long i = 1; i <= 1000; ++i) {
        if (me == 0) { while (p[1] != i - 1) {} p[0] = i; }
        else { while (p[0] != i) {} p[1] = i; }
    }
    long long t1 = clock64();
    if (me == 0) cyc[6] = (t1 - t0) / 1000;
}
int main() {
    double* out; long long* cyc; unsigned long long* g;
    cudaMalloc(&out, 64); cudaMalloc(&cyc, 8 * 16); cudaMalloc(&g, 64);
    for (int rep = 0; rep < 2; ++rep) {
        lat<<<1, 1>>>(out, cyc, 1.234, g);
        pingpong<<<1, 64>>>(cyc, g);
        cudaMemset(g, 0, 64);
        pingpong_global<<<2, 32>>>(cyc, g, 0);
        cudaDeviceSynchronize();
    }
    long long h[16]; cudaMemcpy(h, cyc, 8 * 16, cudaMemcpyDeviceToHost);
    printf("DADD dependent   %.1f cycles\n", h[0] / double(R));
    printf("DMUL dependent   %.1f cycles\n", h[1] / double(R));
    printf("DFMA dependent   %.1f cycles\n", h[2] / double(R));
    printf("DDIV dependent   %.1f cycles\n", h[3] / double(R));
    printf("FADD dependent   %.1f cycles\n", h[4] / double(R));
    printf("smem ping-pong round trip (2 hops, 2 warps)  %lld cycles\n", h[5]);
    printf("global ping-pong round trip (2 hops, 2 CTAs) %lld cycles\n", h[6]);
    printf("status %s\n", cudaGetErrorString(cudaGetLastError()));
}
