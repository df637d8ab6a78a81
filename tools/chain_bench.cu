// Diagnostics: cycles per dependency step of a single-warp chain
// x[i] = (b[i] - v*x[i-1]) / d[i] passed through shared memory, under the
// scheduling variants the solve kernel could use. Build + run on a GPU box:
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a tools/chain_bench.cu -o /tmp/cb && /tmp/cb
#include <cstdio>
#include <cstdint>

constexpr unsigned long long kSent = 0xFFFFFFFFFFFFFFFFull;
constexpr int N = 4096;

template <int kVariant>
__global__ void chain(const double* b, const double* d, double* out, long long* cycles) {
    __shared__ unsigned long long sx[N];
    const int lane = threadIdx.x;
    for (int i = lane; i < N; i += 32) sx[i] = kSent;
    __syncwarp();
    long long t0 = clock64();
    int i = lane;
    double acc_div = 0;
    if (kVariant == 3) {  // divergent spin: each lane waits alone for its predecessor
        for (; i < N; i += 32) {
            const double bi = b[i], di = d[i];
            double prev = 0.0;
            if (i > 0) {
                unsigned long long v;
                while ((v = reinterpret_cast<volatile unsigned long long*>(sx)[i - 1]) == kSent) {
                }
                prev = __longlong_as_double(v);
            }
            double xr = __ddiv_rn(__dsub_rn(bi, __dmul_rn(0.5, prev)), di);
            reinterpret_cast<volatile unsigned long long*>(sx)[i] = __double_as_longlong(xr);
        }
    } else {  // converged rounds
        double bi = b[i], di = d[i];
        while (__any_sync(0xFFFFFFFFu, i < N)) {
            while (i < N) {
                double prev = 0.0;
                if (i > 0) {
                    unsigned long long v = reinterpret_cast<volatile unsigned long long*>(sx)[i - 1];
                    if (v == kSent) break;
                    prev = __longlong_as_double(v);
                }
                if (kVariant == 2) {
                    unsigned c = clock();
                    if (c == 0xFFFFFFFFu) acc_div += 1;  // keep the clock read
                }
                double num = __dsub_rn(bi, __dmul_rn(0.5, prev));
                double xr = kVariant == 1 ? __dmul_rn(num, di) : __ddiv_rn(num, di);
                reinterpret_cast<volatile unsigned long long*>(sx)[i] = __double_as_longlong(xr);
                i += 32;
                if (i < N) { bi = b[i]; di = d[i]; }
            }
        }
    }
    long long t1 = clock64();
    if (lane == 0) cycles[kVariant] = t1 - t0;
    out[lane] = acc_div + __longlong_as_double(sx[N - 1 - lane]);
}

// Same chain, but successive rows sit on successive WARPS of a 512-thread CTA
// (row i -> warp i % 16); converged rounds per warp.
__global__ void chain_warps(const double* b, const double* d, double* out, long long* cycles) {
    __shared__ unsigned long long sx[N];
    for (int i = threadIdx.x; i < N; i += blockDim.x) sx[i] = kSent;
    __syncthreads();
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31, W = blockDim.x >> 5;
    int i = w + lane * W;  // rows of this lane: w + (lane + 32 j) * W
    long long t0 = clock64();
    double bi = i < N ? b[i] : 0, di = i < N ? d[i] : 1;
    while (__any_sync(0xFFFFFFFFu, i < N)) {
        while (i < N) {
            double prev = 0.0;
            if (i > 0) {
                unsigned long long v = reinterpret_cast<volatile unsigned long long*>(sx)[i - 1];
                if (v == kSent) break;
                prev = __longlong_as_double(v);
            }
            double xr = __ddiv_rn(__dsub_rn(bi, __dmul_rn(0.5, prev)), di);
            reinterpret_cast<volatile unsigned long long*>(sx)[i] = __double_as_longlong(xr);
            i += 32 * W;
            if (i < N) { bi = b[i]; di = d[i]; }
        }
    }
    long long t1 = clock64();
    __syncthreads();
    if (threadIdx.x == 0) cycles[4] = t1 - t0;
    if (threadIdx.x < 32) out[threadIdx.x] = __longlong_as_double(sx[N - 1 - threadIdx.x]);
}

int main() {
    double *b, *d, *out;
    long long* cyc;
    cudaMalloc(&b, N * 8);
    cudaMalloc(&d, N * 8);
    cudaMalloc(&out, 64 * 8);
    cudaMalloc(&cyc, 8 * 8);
    double hb[N], hd[N];
    for (int i = 0; i < N; ++i) {
        hb[i] = 1.0 + i * 1e-3;
        hd[i] = 2.0 + (i % 7) * 0.1;
    }
    cudaMemcpy(b, hb, N * 8, cudaMemcpyHostToDevice);
    cudaMemcpy(d, hd, N * 8, cudaMemcpyHostToDevice);
    for (int rep = 0; rep < 2; ++rep) {
        chain<0><<<1, 32>>>(b, d, out, cyc);
        chain<1><<<1, 32>>>(b, d, out, cyc);
        chain<2><<<1, 32>>>(b, d, out, cyc);
        chain<3><<<1, 32>>>(b, d, out, cyc);
        chain_warps<<<1, 512>>>(b, d, out, cyc);
        cudaDeviceSynchronize();
    }
    long long h[8];
    cudaMemcpy(h, cyc, 8 * 8, cudaMemcpyDeviceToHost);
    const char* names[5] = {"rounds + ddiv", "rounds + dmul (no div)", "rounds + ddiv + clock()",
                            "divergent spin + ddiv", "rounds, rows across 16 warps"};
    for (int v = 0; v < 5; ++v) printf("%-32s %8.1f cycles/step\n", names[v], double(h[v]) / N);
    printf("status %s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
