// A lean sync-free round for chain units, on one CTA with a synthetic
// config-2 tile (10 x 10 x-lines of 100 rows, lower 7-point stencil, no halo):
// lane = line, each converged round every lane tries its next row; the
// chain operand (the lane's previous x) stays in a register, the y/z
// neighbours come from the shared window (sentinel = not yet), records are
// prefetched into registers two rows ahead from global memory. Reports the
// tile's solve time and cycles per round; variants (mode bits):
//   1  chain operand read back from shared memory instead of the register
//   2  records loaded when needed (no register prefetch)
//   4  division range test with an outlined __ddiv_rn fallback
//   8  records prefetched four rows ahead (a rotating register queue)
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a tools/lean_round_bench.cu -o /tmp/lrb && /tmp/lrb
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <vector>

constexpr unsigned long long kSent = ~0ull;

__device__ __forceinline__ unsigned long long lds_v(uint32_t a) {
    unsigned long long v;
    asm volatile("ld.volatile.shared.u64 %0, [%1];" : "=l"(v) : "r"(a) : "memory");
    return v;
}
__device__ __forceinline__ void sts(uint32_t a, unsigned long long v) {
    asm volatile("st.volatile.shared.u64 [%0], %1;" ::"r"(a), "l"(v) : "memory");
}
__device__ __noinline__ double ddiv_out(double a, double b) { return __ddiv_rn(a, b); }
__device__ __forceinline__ bool in_range(double v) {
    return (static_cast<unsigned>(__double2hiint(v)) & 0x7FFFFFFFu) - (523u << 20) < (1001u << 20);
}

// record of a row: vz, vy, vx, d, y (reciprocal), b, codes (z slot, y slot; -1 none) packed
struct Rec {
    double vz, vy, vx, d, y, b;
    int cz, cy;
};

template <int kMode>
__global__ void __launch_bounds__(128) lean(const Rec* rec, double* xout, long long* out, int* rounds_out) {
    extern __shared__ unsigned long long win[];  // 10000 slots + the zero word
    const uint32_t win_a = static_cast<uint32_t>(__cvta_generic_to_shared(win));
    const int tid = threadIdx.x;
    for (int i = tid; i < 10000; i += blockDim.x) win[i] = kSent;
    win[10000] = 0;  // zero word
    __syncthreads();
    const long long t0 = clock64();
    const bool active = tid < 100;
    int row = 0;  // next row of this lane's line (slot = 100 * line + row)
    const int line = tid;
    double xprev = 0.0;
    Rec n1{}, n2{}, n3{}, n4{};
    if (active) {
        n1 = rec[line * 100 + 0];
        n2 = rec[line * 100 + 1];
        if (kMode & 8) {
            n3 = rec[line * 100 + 2];
            n4 = rec[line * 100 + 3];
        }
    }
    int rounds = 0;
    while (__any_sync(0xffffffffu, active && row < 100)) {
        ++rounds;
        if (active && row < 100) {
            if (kMode & 2) n1 = rec[line * 100 + row];
            const Rec& q = n1;
            const uint32_t az = win_a + 8u * (q.cz >= 0 ? q.cz : 10000), ay = win_a + 8u * (q.cy >= 0 ? q.cy : 10000);
            const unsigned long long uz = lds_v(az), uy = lds_v(ay);
            unsigned long long ux = __double_as_longlong(xprev);
            if (kMode & 1) ux = row > 0 ? lds_v(win_a + 8u * (line * 100 + row - 1)) : 0ull;
            if (uz != kSent && uy != kSent) {
                double sp = __dmul_rn(q.vz, __longlong_as_double(uz));
                sp = __dadd_rn(sp, __dmul_rn(q.vy, __longlong_as_double(uy)));
                sp = __dadd_rn(sp, __dmul_rn(q.vx, __longlong_as_double(ux)));
                const double acc = __dadd_rn(0.0, sp);
                const double tq = __dsub_rn(q.b, acc);
                const double q0 = __dmul_rn(tq, q.y);
                double xr = __fma_rn(q.y, __fma_rn(-q.d, q0, tq), q0);
                if (kMode & 4)
                    if (!in_range(tq)) xr = ddiv_out(tq, q.d);
                sts(win_a + 8u * (line * 100 + row), __double_as_longlong(xr));
                xprev = xr;
                ++row;
                if (kMode & 8) {
                    n1 = n2;
                    n2 = n3;
                    n3 = n4;
                    if (row + 3 < 100) n4 = rec[line * 100 + row + 3];
                } else if (!(kMode & 2)) {
                    n1 = n2;
                    if (row + 1 < 100) n2 = rec[line * 100 + row + 1];
                }
            }
        }
    }
    const long long t1 = clock64();
    if (active)
        for (int r = 0; r < 100; ++r) xout[line * 100 + r] = __longlong_as_double(win[line * 100 + r]);
    if (tid == 0) {
        out[kMode] = t1 - t0;
        rounds_out[kMode] = rounds;
    }
}

int main() {
    // slot of (x, j, k) in the tile = 100 * (j + 10 k) + x; rows by line
    std::vector<Rec> rec(10000);
    for (int k = 0; k < 10; ++k)
        for (int j = 0; j < 10; ++j)
            for (int x = 0; x < 100; ++x) {
                Rec r;
                const int line = j + 10 * k;
                r.vz = k > 0 ? -1.0 : 0.0;
                r.vy = j > 0 ? -1.0 : 0.0;
                r.vx = x > 0 ? -1.0 : 0.0;
                r.d = 6.05;
                r.y = 1.0 / 6.05;
                r.b = 0.5;
                r.cz = k > 0 ? 100 * (line - 10) + x : -1;
                r.cy = j > 0 ? 100 * (line - 1) + x : -1;
                rec[line * 100 + x] = r;
            }
    Rec* drec;
    double* dx;
    long long* dout;
    int* drounds;
    cudaMalloc(&drec, rec.size() * sizeof(Rec));
    cudaMemcpy(drec, rec.data(), rec.size() * sizeof(Rec), cudaMemcpyHostToDevice);
    cudaMalloc(&dx, 10000 * sizeof(double));
    cudaMallocManaged(&dout, 64 * sizeof(long long));
    cudaMallocManaged(&drounds, 64 * sizeof(int));
#define RUN(M)                                                                                                \
    cudaFuncSetAttribute(lean<M>, cudaFuncAttributeMaxDynamicSharedMemorySize, 10001 * 8);                  \
    for (int rep = 0; rep < 3; ++rep) lean<M><<<1, 128, 10001 * 8>>>(drec, dx, dout, drounds);                \
    cudaDeviceSynchronize();                                                                                  \
    printf("mode %d: %lld cycles (%.2f us at 1.965 GHz), %d rounds, %.0f cycles/round %s\n", M, dout[M],      \
           dout[M] / 1965.0, drounds[M], double(dout[M]) / drounds[M], cudaGetErrorString(cudaGetLastError())); \
    fflush(stdout);
    RUN(0) RUN(8) RUN(9) RUN(12)
    return 0;
}
