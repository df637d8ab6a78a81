// Random 8-byte gather throughput on one B200: how many x gathers per second
// the L1/L2 (x range resident) and DRAM (x range >> L2) deliver, alone and
// beside a matrix-like stream (12 B per gather: a column index and a value),
// with and without L2 eviction-priority hints and an L2 persisting window.
// Sizes the config-5 SpMV ceiling.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/gather_probe tools/gather_probe.cu
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

__global__ void init_idx(uint32_t* idx, int64_t n, uint32_t range, uint64_t seed) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        uint64_t z = (i + 1) * 0x9E3779B97F4A7C15ull + seed;
        z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
        z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
        z ^= z >> 31;
        idx[i] = static_cast<uint32_t>(z % range);
    }
}

__device__ __forceinline__ uint64_t pol_first() {
    uint64_t p;
    asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ uint64_t pol_last() {
    uint64_t p;
    asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
    return p;
}

// mode 0: gather only (idx stream 4 B); 1: + value stream (SpMV-like); 2: 1 with L2 hints;
// 3: gather via ld.global.cg (L2 only)
template <int kMode>
__global__ void __launch_bounds__(256) gather(const uint32_t* __restrict__ idx, const double* __restrict__ val,
                                              const double* __restrict__ x, double* out, int64_t n) {
    constexpr int kPer = 8;
    double acc = 0;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    uint64_t pf = 0, pl = 0;
    if (kMode == 2) {
        pf = pol_first();
        pl = pol_last();
    }
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += stride * kPer) {
        uint32_t c[kPer];
        double v[kPer];
#pragma unroll
        for (int k = 0; k < kPer; ++k) {
            const int64_t e = i + k * stride;
            c[k] = 0;
            v[k] = 1.0;
            if (e < n) {
                if (kMode == 2) {
                    asm("ld.global.nc.L1::no_allocate.L2::cache_hint.u32 %0, [%1], %2;" : "=r"(c[k]) : "l"(idx + e), "l"(pf));
                    asm("ld.global.nc.L1::no_allocate.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v[k]) : "l"(val + e), "l"(pf));
                } else {
                    c[k] = __ldcs(idx + e);
                    if (kMode == 1) v[k] = __ldcs(val + e);
                }
            }
        }
#pragma unroll
        for (int k = 0; k < kPer; ++k) {
            double xv;
            if (kMode == 2) asm("ld.global.nc.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(xv) : "l"(x + c[k]), "l"(pl));
            else if (kMode == 3) xv = __ldcg(x + c[k]);
            else xv = __ldg(x + c[k]);
            acc += v[k] * xv;
        }
    }
    if (acc == 12345.0) out[0] = acc;
}

__global__ void stream(const double* __restrict__ a, double* out, int64_t n) {
    double acc = 0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        acc += __ldcs(a + i);
    if (acc == 12345.0) out[0] = acc;
}

int main() {
    const int64_t n = 400000000;  // gathers (config 5: 401M)
    uint32_t* idx;
    double *x, *val, *out, *flush;
    cudaMalloc(&idx, n * 4);
    cudaMalloc(&val, n * 8);
    cudaMemset(val, 0, n * 8);
    const int64_t xmax = 1ll << 28;  // 2 GiB of x
    cudaMalloc(&x, xmax * 8);
    cudaMemset(x, 0, xmax * 8);
    cudaMalloc(&out, 8);
    cudaMalloc(&flush, 512 << 20);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    int sms = 0, persist_max = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaDeviceGetAttribute(&persist_max, cudaDevAttrMaxPersistingL2CacheSize, 0);
    printf("SMs %d, max persisting L2 %d MB\n", sms, persist_max >> 20);
    cudaStream_t st;
    cudaStreamCreate(&st);
    auto run = [&](const char* what, int mode, double range_mb, bool persist) {
        const uint32_t range = static_cast<uint32_t>(range_mb * 1000000 / 8);
        init_idx<<<sms * 8, 256, 0, st>>>(idx, n, range, 7);
        if (persist) {
            cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, persist_max);
            cudaStreamAttrValue a = {};
            a.accessPolicyWindow.base_ptr = x;
            a.accessPolicyWindow.num_bytes = static_cast<size_t>(range) * 8;
            a.accessPolicyWindow.hitRatio = 1.0f;
            a.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
            a.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
            cudaStreamSetAttribute(st, cudaStreamAttributeAccessPolicyWindow, &a);
        }
        float best = 1e9;
        for (int rep = 0; rep < 3; ++rep) {
            cudaMemsetAsync(flush, rep, 512 << 20, st);
            cudaEventRecord(e0, st);
            if (mode == 0) gather<0><<<sms * 8, 256, 0, st>>>(idx, val, x, out, n);
            if (mode == 1) gather<1><<<sms * 8, 256, 0, st>>>(idx, val, x, out, n);
            if (mode == 2) gather<2><<<sms * 8, 256, 0, st>>>(idx, val, x, out, n);
            if (mode == 3) gather<3><<<sms * 8, 256, 0, st>>>(idx, val, x, out, n);
            cudaEventRecord(e1, st);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            if (ms < best) best = ms;
        }
        if (persist) {
            cudaStreamAttrValue a = {};
            a.accessPolicyWindow.num_bytes = 0;
            cudaStreamSetAttribute(st, cudaStreamAttributeAccessPolicyWindow, &a);
            cudaCtxResetPersistingL2Cache();
        }
        const double bytes = n * (mode == 0 || mode == 3 ? 4.0 : 12.0);
        printf("%-28s x range %7.2f MB: %.3f ms = %6.1f G gathers/s, stream %.2f TB/s\n", what, range_mb, best,
               n / best / 1e6, bytes / best / 1e9);
    };
    for (double r : {0.1, 1.0, 8.0, 64.0, 80.0, 160.0}) run("gather (ldg)", 0, r, false);
    for (double r : {0.1, 8.0, 64.0}) run("gather (ld.cg)", 3, r, false);
    for (double r : {20.0, 40.0, 53.0, 64.0, 80.0, 160.0}) run("gather+value stream", 1, r, false);
    for (double r : {20.0, 40.0, 53.0, 64.0, 80.0}) run("  + evict hints", 2, r, false);
    for (double r : {20.0, 40.0, 53.0, 64.0, 80.0}) run("  + persisting window", 1, r, true);
    for (int rep = 0; rep < 3; ++rep) {
        cudaEventRecord(e0);
        stream<<<sms * 8, 256>>>(x, out, xmax);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (rep == 2) printf("stream 2 GiB: %.3f ms = %.2f TB/s\n", ms, xmax * 8.0 / ms / 1e9);
    }
    return 0;
}
