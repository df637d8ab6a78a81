// Floor of a lockstep wavefront solve: one CTA, a
// synthetic config-2 tile (10 x 10 x-lines of 100 rows, lower 7-point stencil, no halo), lane =
// line, every warp walking a static schedule (line (y, z) runs row t - y - z at step t) with the
// leanest step this design allows:
//   * records (80 bytes: three values, d, reciprocal, b, two window codes, two source lanes,
//     the row's window slot) stored step-major in 16-byte planes and prefetched straight into
//     registers kDepth steps ahead (possible because the lanes step together);
//   * operands produced by the warp's previous step by shuffle, the chain operand in a register,
//     the others from the shared window (sentinel = not yet; one vote per attempt);
//   * the reference's sequential partial, 0 + partial, b - acc, the division on the reciprocal
//     with the range test and an outlined __ddiv_rn, the canonical-NaN test;
//   * one window store, one global store, __syncwarp.
// Prints the tile's solve time, cycles per step of warp 0 (which never waits) and of the tile,
// and checks x bitwise against a host solve.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a tools/lockstep_bench.cu -o /tmp/lsb && /tmp/lsb
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <vector>

constexpr unsigned long long kSent = ~0ull;
constexpr int kN = 10, kRows = 100, kLines = kN * kN, kDepth = 4;

__device__ __forceinline__ unsigned long long lds_v(uint32_t a) {
    unsigned long long v;
    asm volatile("ld.volatile.shared.u64 %0, [%1];" : "=l"(v) : "r"(a) : "memory");
    return v;
}
__device__ __noinline__ double ddiv_out(double a, double b) { return __ddiv_rn(a, b); }
__device__ __forceinline__ bool in_range(double v) {
    return (static_cast<unsigned>(__double2hiint(v)) & 0x7FFFFFFFu) - (523u << 20) < (1001u << 20);
}

struct Rec {  // 80 bytes = 5 planes of 16
    double vz, vy;
    double vx, d;
    double y, b;
    int cz, cy, lz, ly;
    int loc, row, pad0, pad1;
};
static_assert(sizeof(Rec) == 80, "record");

struct Stage {
    uint4 p[5];
};

__device__ __forceinline__ void load_stage(Stage& s, const uint4* base, int step, int lane) {
    const uint4* q = base + static_cast<size_t>(step) * 5 * 32 + lane;
#pragma unroll
    for (int c = 0; c < 5; ++c) s.p[c] = __ldg(q + 32 * c);
}

__global__ void __launch_bounds__(128, 1) lockstep(const uint4* rec, const int* warp_step0, const int* warp_steps,
                                                   double* xout, long long* out) {
    extern __shared__ unsigned long long win[];  // [0] scratch, [1] zero word, then 10000 slots
    const uint32_t win_a = static_cast<uint32_t>(__cvta_generic_to_shared(win)) + 16;
    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    for (int i = tid; i < kLines * kRows; i += blockDim.x) win[2 + i] = kSent;
    if (tid == 0) {
        win[0] = 0;
        win[1] = 0;
    }
    __syncthreads();
    const long long t0 = clock64();
    const uint4* base = rec + static_cast<size_t>(warp_step0[w]) * 5 * 32;
    const int ns = warp_steps[w];
    // (schedules are padded to a multiple of kDepth null steps, so the unrolled stages need no guards
    // and the compiler renames the prefetch registers instead of copying them)
    Stage st[kDepth];
#pragma unroll
    for (int k = 0; k < kDepth; ++k) load_stage(st[k], base, k, lane);
    double xprev = 0.0;
    for (int s0 = 0; s0 < ns; s0 += kDepth) {
#pragma unroll
        for (int k = 0; k < kDepth; ++k) {
            const int s = s0 + k;
            const Stage cur = st[k];
            load_stage(st[k], base, min(s + kDepth, ns - 1), lane);
            const double vz = __hiloint2double(cur.p[0].y, cur.p[0].x), vy = __hiloint2double(cur.p[0].w, cur.p[0].z);
            const double vx = __hiloint2double(cur.p[1].y, cur.p[1].x), d = __hiloint2double(cur.p[1].w, cur.p[1].z);
            const double y = __hiloint2double(cur.p[2].y, cur.p[2].x), b = __hiloint2double(cur.p[2].w, cur.p[2].z);
            const int cz = cur.p[3].x, cy = cur.p[3].y, lz = cur.p[3].z, ly = cur.p[3].w;
            const int loc = cur.p[4].x, row = cur.p[4].y;
            const double hz = __shfl_sync(0xFFFFFFFFu, xprev, lz), hy = __shfl_sync(0xFFFFFFFFu, xprev, ly);
            unsigned long long uz, uy;
            for (;;) {
                uz = lds_v(win_a + 8u * static_cast<uint32_t>(cz));
                uy = lds_v(win_a + 8u * static_cast<uint32_t>(cy));
                if (__all_sync(0xFFFFFFFFu, (__double2hiint(__longlong_as_double(uz)) != -1) &
                                                (__double2hiint(__longlong_as_double(uy)) != -1)))
                    break;
            }
            const double xz = lz >= 0 ? hz : __longlong_as_double(uz);
            const double xy = ly >= 0 ? hy : __longlong_as_double(uy);
            double sp = __dmul_rn(vz, xz);
            sp = __dadd_rn(sp, __dmul_rn(vy, xy));
            sp = __dadd_rn(sp, __dmul_rn(vx, xprev));
            const double acc = __dadd_rn(0.0, sp);
            const double t = __dsub_rn(b, acc);
            const double q0 = __dmul_rn(t, y);
            double x = __fma_rn(y, __fma_rn(-d, q0, t), q0);
            if (!in_range(t)) x = ddiv_out(t, d);
            if (__double2hiint(x) == -1) x = __longlong_as_double(0x7FF8000000000000ll);
            asm volatile("st.volatile.shared.u64 [%0], %1;" ::"r"(win_a + 8u * static_cast<uint32_t>(loc)),
                         "l"(__double_as_longlong(x))
                         : "memory");
            if (row >= 0) asm volatile("st.relaxed.gpu.global.b64 [%0], %1;" ::"l"(xout + row), "l"(__double_as_longlong(x)) : "memory");
            xprev = x;
            __syncwarp();
        }
    }
    const long long t1 = clock64();
    if (lane == 0) out[w] = t1 - t0;
}

int main() {
    // matrix: row r = x + 100 * line, line = y + 10 z; off-diagonals -1, diagonal 6 + small; b pseudo-random
    const int n = kLines * kRows;
    std::vector<double> diag(n), bv(n), xref(n);
    unsigned long long h = 12345;
    auto rnd = [&]() {
        h = h * 6364136223846793005ull + 1442695040888963407ull;
        return static_cast<double>(h >> 11) / 9007199254740992.0;
    };
    for (int r = 0; r < n; ++r) {
        diag[r] = 6.0 + 0.1 * rnd();
        bv[r] = 2.0 * rnd() - 1.0;
    }
    auto slot = [&](int line, int i) { return line * kRows + i; };  // window slot == row index here
    for (int z = 0; z < kN; ++z)
        for (int yy = 0; yy < kN; ++yy)
            for (int i = 0; i < kRows; ++i) {
                const int line = yy + kN * z, r = slot(line, i);
                double sp = (z > 0 ? -1.0 : 0.0) * (z > 0 ? xref[slot(line - kN, i)] : 0.0);
                sp = sp + (yy > 0 ? -1.0 : 0.0) * (yy > 0 ? xref[slot(line - 1, i)] : 0.0);
                sp = sp + (i > 0 ? -1.0 : 0.0) * (i > 0 ? xref[r - 1] : 0.0);
                const double acc = 0.0 + sp;
                xref[r] = (bv[r] - acc) / diag[r];
            }
    // schedules: warp w holds lines 32 w .. 32 w + 31; line (y, z) runs row t - (y + z) at global step t
    std::vector<Rec> recs;
    std::vector<int> step0(4), steps(4);
    for (int w = 0; w < 4; ++w) {
        int lo = 1 << 30, hi = -1;
        for (int l = 32 * w; l < std::min(32 * w + 32, kLines); ++l) {
            const int lv = l % kN + l / kN;
            lo = std::min(lo, lv);
            hi = std::max(hi, lv + kRows - 1);
        }
        step0[w] = static_cast<int>(recs.size() / 32);
        steps[w] = (hi - lo + 1 + kDepth - 1) / kDepth * kDepth;  // padded with null steps
        for (int t = lo; t < lo + steps[w]; ++t)
            for (int lane = 0; lane < 32; ++lane) {
                Rec q{};
                q.d = 1.0;
                q.y = 1.0;
                q.b = 1.0;
                q.cz = q.cy = -1;  // the zero word
                q.lz = q.ly = -1;
                q.loc = -2;  // scratch
                q.row = -1;
                const int l = 32 * w + lane;
                if (l < kLines) {
                    const int yy = l % kN, z = l / kN, i = t - (yy + z);
                    if (i >= 0 && i < kRows) {
                        const int r = slot(l, i);
                        q.d = diag[r];
                        q.y = 1.0 / diag[r];  // (the kernel under test refines it; the bench uses exact-enough values)
                        q.b = bv[r];
                        q.vz = z > 0 ? -1.0 : 0.0;
                        q.vy = yy > 0 ? -1.0 : 0.0;
                        q.vx = i > 0 ? -1.0 : 0.0;
                        if (z > 0) {
                            if (lane >= kN) q.lz = lane - kN;  // produced by this warp's previous step
                            else q.cz = slot(l - kN, i);
                        }
                        if (yy > 0) {
                            if (lane >= 1) q.ly = lane - 1;
                            else q.cy = slot(l - 1, i);
                        }
                        q.loc = r;
                        q.row = r;
                    }
                }
                recs.push_back(q);
            }
    }
    // plane layout: per step 5 planes of 32 x 16 bytes
    const size_t n_steps = recs.size() / 32;
    std::vector<unsigned char> planes(n_steps * 5 * 32 * 16);
    for (size_t s = 0; s < n_steps; ++s)
        for (int lane = 0; lane < 32; ++lane)
            for (int c = 0; c < 5; ++c)
                std::memcpy(&planes[((s * 5 + c) * 32 + lane) * 16], reinterpret_cast<const unsigned char*>(&recs[s * 32 + lane]) + 16 * c, 16);
    uint4* d_rec;
    int *d_s0, *d_ns;
    double* d_x;
    long long* d_out;
    cudaMalloc(&d_rec, planes.size());
    cudaMalloc(&d_s0, 16);
    cudaMalloc(&d_ns, 16);
    cudaMalloc(&d_x, n * sizeof(double));
    cudaMalloc(&d_out, 4 * sizeof(long long));
    cudaMemcpy(d_rec, planes.data(), planes.size(), cudaMemcpyHostToDevice);
    cudaMemcpy(d_s0, step0.data(), 16, cudaMemcpyHostToDevice);
    cudaMemcpy(d_ns, steps.data(), 16, cudaMemcpyHostToDevice);
    const size_t smem = (2 + static_cast<size_t>(n)) * 8;
    cudaFuncSetAttribute(lockstep, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float best = 1e9f;
    long long cyc[4] = {0, 0, 0, 0};
    for (int it = 0; it < 5; ++it) {
        cudaMemset(d_x, 0, n * sizeof(double));
        cudaEventRecord(e0);
        lockstep<<<1, 128, smem>>>(d_rec, d_s0, d_ns, d_x, d_out);
        cudaEventRecord(e1);
        if (cudaDeviceSynchronize() != cudaSuccess) {
            std::printf("kernel failed: %s\n", cudaGetErrorString(cudaGetLastError()));
            return 1;
        }
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        best = std::min(best, ms);
        cudaMemcpy(cyc, d_out, sizeof(cyc), cudaMemcpyDeviceToHost);
    }
    std::vector<double> x(n);
    cudaMemcpy(x.data(), d_x, n * sizeof(double), cudaMemcpyDeviceToHost);
    size_t bad = 0;
    for (int r = 0; r < n; ++r) bad += std::memcmp(&x[r], &xref[r], 8) != 0;
    const int levels = kRows + 2 * (kN - 1);
    std::printf("tile: %.2f us, %d levels, %.0f cycles per level (slowest warp %lld cycles); warp 0: %d steps, %.0f cycles per step; mismatches %zu\n",
                best * 1e3, levels, static_cast<double>(std::max(std::max(cyc[0], cyc[1]), std::max(cyc[2], cyc[3]))) / levels,
                std::max(std::max(cyc[0], cyc[1]), std::max(cyc[2], cyc[3])), steps[0], static_cast<double>(cyc[0]) / steps[0], bad);
    return 0;
}
