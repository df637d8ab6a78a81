// Diagnostics: host<->device bandwidth on this box for the e2e path (8 MB,
// as config 2's b and x): copy engine H2D / D2H alone and together, and a
// kernel reading mapped (zero-copy) host memory, alone and beside a D2H copy.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a tools/pcie_bench.cu -o /tmp/pcie && /tmp/pcie
#include <cstdio>

__global__ void zread(const double* __restrict__ h, double* __restrict__ d, long n) {
    const long i0 = blockIdx.x * (long)blockDim.x + threadIdx.x, st = (long)gridDim.x * blockDim.x;
    for (long i = i0; i < n; i += 4 * st) {  // four loads in flight per thread
        double v[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) v[q] = i + q * st < n ? h[i + q * st] : 0.0;
#pragma unroll
        for (int q = 0; q < 4; ++q)
            if (i + q * st < n) d[i + q * st] = v[q];
    }
}

int main() {
    const long n = 1000000;  // 8 MB of doubles
    const size_t bytes = n * sizeof(double);
    double *h_in, *h_out, *d_a, *d_b;
    cudaHostAlloc(&h_in, bytes, cudaHostAllocMapped);
    cudaHostAlloc(&h_out, bytes, cudaHostAllocMapped);
    cudaMalloc(&d_a, bytes);
    cudaMalloc(&d_b, bytes);
    for (long i = 0; i < n; ++i) h_in[i] = i;
    double* h_in_dev;
    cudaHostGetDevicePointer(&h_in_dev, h_in, 0);
    cudaStream_t s1, s2;
    cudaStreamCreate(&s1);
    cudaStreamCreate(&s2);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    auto timeit = [&](const char* name, auto fn) {
        for (int w = 0; w < 3; ++w) fn();
        cudaDeviceSynchronize();
        cudaEventRecord(e0, s1);
        const int reps = 20;
        for (int r = 0; r < reps; ++r) fn();
        cudaEventRecord(e1, s1);
        cudaDeviceSynchronize();
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        ms /= reps;
        printf("%-40s %8.1f us  %6.1f GB/s (per 8 MB)\n", name, ms * 1e3, bytes / (ms * 1e-3) / 1e9);
    };
    timeit("H2D copy engine", [&] { cudaMemcpyAsync(d_a, h_in, bytes, cudaMemcpyHostToDevice, s1); });
    timeit("D2H copy engine", [&] { cudaMemcpyAsync(h_out, d_b, bytes, cudaMemcpyDeviceToHost, s1); });
    timeit("H2D + D2H (two streams)", [&] {
        cudaEventRecord(e1, s1);
        cudaStreamWaitEvent(s2, e1, 0);
        cudaMemcpyAsync(d_a, h_in, bytes, cudaMemcpyHostToDevice, s1);
        cudaMemcpyAsync(h_out, d_b, bytes, cudaMemcpyDeviceToHost, s2);
        cudaEventRecord(e1, s2);
        cudaStreamWaitEvent(s1, e1, 0);
    });
    timeit("zero-copy kernel read (148 CTAs)", [&] { zread<<<148, 512, 0, s1>>>(h_in_dev, d_a, n); });
    timeit("zero-copy kernel read (48 CTAs)", [&] { zread<<<48, 512, 0, s1>>>(h_in_dev, d_a, n); });
    timeit("zero-copy read + D2H copy", [&] {
        cudaEventRecord(e1, s1);
        cudaStreamWaitEvent(s2, e1, 0);
        zread<<<148, 512, 0, s1>>>(h_in_dev, d_a, n);
        cudaMemcpyAsync(h_out, d_b, bytes, cudaMemcpyDeviceToHost, s2);
        cudaEventRecord(e1, s2);
        cudaStreamWaitEvent(s1, e1, 0);
    });
    printf("status %s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
