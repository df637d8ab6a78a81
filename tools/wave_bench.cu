// Cycles per step of the level-synchronous solve loop (sptrsv_wave.cu) on one
// CTA with synthetic config-2 tile records (10 x 10 lines of 100 rows, in-tile
// operands only), adding the real kernel's pieces one at a time (mode bits):
//   1   operand loads + FP chain + STS (always on below)
//   2   records from global memory (register ring, 4 steps ahead) instead of a shared ring
//   4   STG of x per row
//   8   sentinel re-poll loop on the operands
//   16  division range check with an outlined __ddiv_rn fallback
//   32  256-thread CTA: 3 idle warps + 1 exiting warp beside the 4 solving warps
//   64  globaltimer + trace store per row
//   256 (with 128) sentinel misses and out-of-range divisions OR-reduced by the
//       step's barrier (bar.red.or.pred), fixed by a uniform redo after it
//   512 (with 128, shared ring) a loader warp refills the ring with TMA bulk copies
//       (mbarrier complete_tx), confirms slab s+2 and joins every barrier
//   1024 (with 16|128) the fast quotient is stored first; a warp vote after the
//       store decides whether any lane overwrites it with __ddiv_rn
//   2048 (with 4) the STG of a step's x is issued after the step's barrier
//   128 no divergence: idle threads compute a null row; the halo test is one
//       CTA-uniform counter check per step, the division fallback a warp vote
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a tools/wave_bench.cu -o /tmp/wb && /tmp/wb
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <vector>

constexpr int kT = 128, kSteps = 118, kRing = 8, kDepth = 4;
constexpr unsigned long long kSent = ~0ull;

__device__ __forceinline__ unsigned long long lds_v(uint32_t a) {
    unsigned long long v;
    asm volatile("ld.volatile.shared.u64 %0, [%1];" : "=l"(v) : "r"(a) : "memory");
    return v;
}
__device__ __forceinline__ int4 ldg_stream(const int4* p) {
    int4 v;
    asm volatile("ld.global.nc.L1::no_allocate.v4.s32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
    return v;
}
__device__ __noinline__ double ddiv_out(double a, double b) { return __ddiv_rn(a, b); }
__device__ __forceinline__ bool in_range(double v) {
    return (static_cast<unsigned>(__double2hiint(v)) & 0x7FFFFFFFu) - (523u << 20) < (1001u << 20);
}

struct Rec {
    int4 c0, c1, c2, c3;
    bool has;
};

template <int kMode>
__global__ void __launch_bounds__(256) wave_loop(const int4* recs, const int* offs, double* x, unsigned long long* tr,
                                                 long long* out) {
    extern __shared__ __align__(128) unsigned char smem[];
    double* win = reinterpret_cast<double*>(smem + kRing * kT * 64 + 16);
    const uint32_t win_a = static_cast<uint32_t>(__cvta_generic_to_shared(win));
    __shared__ int soff[kSteps + 2];
    __shared__ unsigned halo_done;
    __shared__ __align__(8) unsigned long long mbar[kRing];
    __shared__ double dummy[kT];
    const int tid = threadIdx.x;
    for (int i = tid; i < 10000; i += blockDim.x) win[i] = 1.0 + i * 1e-6;
    for (int i = tid; i <= kSteps; i += blockDim.x) soff[i] = offs[i];
    if (tid < kT) dummy[tid] = 1.0;
    if (tid == 0) halo_done = 1u << 30;
    __syncthreads();
    for (int s = 0; s < kRing; ++s) {  // the shared ring holds steps 0..7 (reused cyclically)
        int4* dst = reinterpret_cast<int4*>(smem + s * kT * 64);
        for (int i = tid; i < 4 * (soff[s + 1] - soff[s]); i += blockDim.x) dst[i] = recs[4 * soff[s] + i];
    }
    __syncthreads();
    const uint32_t mbar_a = static_cast<uint32_t>(__cvta_generic_to_shared(&mbar[0]));
    const uint32_t ring_a = static_cast<uint32_t>(__cvta_generic_to_shared(smem));
    auto issue = [&](int s, int slot) {  // slab of step s % kSteps into ring slot `slot`
        const int ss = s % kSteps;
        const int e0 = soff[ss], bytes = (soff[ss + 1] - e0) * 64;
        const uint32_t mb = mbar_a + 8u * slot;
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(mb), "r"(bytes) : "memory");
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                         ring_a + slot * kT * 64u),
                     "l"(recs + 4 * e0), "r"(bytes), "r"(mb)
                     : "memory");
    };
    if (kMode & 512) {
        if (tid == 0) {
            for (int k = 0; k < kRing; ++k) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(mbar_a + 8u * k));
            asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        }
        __syncthreads();
        if (tid == 0)
            for (int k = 0; k < kRing; ++k) issue(k, k);
        __syncthreads();
    }
    if ((kMode & 512) && tid >= kT && tid < kT + 32) {  // loader warp
        const bool lead = tid == kT;
        auto wait = [&](int s) {
            const uint32_t mb = mbar_a + 8u * (s % kRing), par = (s / kRing) & 1;
            asm volatile("{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W_%=;\n}\n" ::"r"(mb), "r"(par) : "memory");
        };
        if (lead) wait(0), wait(1);
        __syncwarp();
        asm volatile("bar.sync 1, 160;" ::: "memory");  // start
        for (int s = 0; s < kSteps; ++s) {
            if (lead && s + 2 < kSteps) wait(s + 2);
            __syncwarp();
            asm volatile("bar.sync 1, 160;" ::: "memory");
            if (lead && s + kRing < kSteps) issue(s + kRing, s % kRing);  // step s's slot was read during step s-1
        }
        return;
    }
    if (tid >= kT) {
        if ((kMode & 32) && tid < kT + 32) return;  // the exiting (halo) warp
        if (kMode & 32) {
            __syncthreads();
            return;
        }
        return;
    }
    const long long t0 = clock64();
    auto fetch = [&](Rec& w, int s) {
        s = (kMode & 2) ? s % kSteps : (kMode & 512) ? s % kSteps : s % kRing;  // a static ring holds steps 0..7 only
        const int e0 = soff[s], cnt = soff[s + 1] - e0;
        w.has = tid < cnt;
        if (!w.has) return;
        if (kMode & 2) {
            const int4* b = recs + 4 * e0 + tid;
            w.c0 = ldg_stream(b);
            w.c1 = ldg_stream(b + cnt);
            w.c2 = ldg_stream(b + 2 * cnt);
            w.c3 = ldg_stream(b + 3 * cnt);
        } else {
            const int4* b = reinterpret_cast<const int4*>(smem + (s % kRing) * kT * 64) + tid;  // (step s's slot)
            w.c0 = b[0];
            w.c1 = b[cnt];
            w.c2 = b[2 * cnt];
            w.c3 = b[3 * cnt];
        }
    };
    Rec q[kDepth];
    if (kMode & 2) {
#pragma unroll
        for (int i = 0; i < kDepth; ++i) fetch(q[i], i);
    }
    struct Dec {
        bool has;
        uint32_t a0, a1, a2, a3, own;
    };
    const uint32_t zero_a = static_cast<uint32_t>(__cvta_generic_to_shared(smem + kRing * kT * 64 + 8));
    const uint32_t dummy_a = static_cast<uint32_t>(__cvta_generic_to_shared(&dummy[tid]));
    auto decode = [&](Rec& w) {
        Dec e;
        e.has = w.has;
        if ((kMode & 128) && !w.has) {  // null row: zero operands, b = 1, d = y = 1, into the thread's dummy slot
            e.a0 = e.a1 = e.a2 = e.a3 = zero_a;
            e.own = dummy_a;
            const double one = 1.0;
            w.c0 = w.c1 = make_int4(0, 0, 0, 0);
            w.c2 = make_int4(__double2loint(one), __double2hiint(one), __double2loint(one), __double2hiint(one));
            w.c3.z = -1;
            return e;
        }
        e.a0 = win_a + 8u * static_cast<uint32_t>(static_cast<int>(static_cast<short>(w.c3.x & 0xFFFF)));
        e.a1 = win_a + 8u * static_cast<uint32_t>(w.c3.x >> 16);
        e.a2 = win_a + 8u * static_cast<uint32_t>(static_cast<int>(static_cast<short>(w.c3.y & 0xFFFF)));
        e.a3 = win_a + 8u * static_cast<uint32_t>(w.c3.y >> 16);
        e.own = win_a + 8u * (static_cast<uint32_t>(w.c3.w) & 0xFFFFu);
        return e;
    };
    if (kMode & 512) asm volatile("bar.sync 1, 160;" ::: "memory");  // start (slabs 0, 1 confirmed)
    if (!(kMode & 2)) fetch(q[0], 0);
    Dec dc = decode(q[0]);
    double pend_x = 0.0;
    int pend_r = -1;
    auto step = [&](Rec& w, Rec& wn, int s) {
        int redo = 0;
        if ((kMode & 2048) && pend_r >= 0)
            asm volatile("st.relaxed.gpu.global.b64 [%0], %1;" ::"l"(x + pend_r), "l"(__double_as_longlong(pend_x)) : "memory");
        if (!(kMode & 2)) fetch(wn, s + 1);  // shared ring: next step's records at the start
        if ((kMode & 128) || dc.has) {
            unsigned long long u0 = lds_v(dc.a0), u1 = lds_v(dc.a1), u2 = lds_v(dc.a2), u3 = lds_v(dc.a3);
            const unsigned long long ub = lds_v(dc.own);
            if (kMode & 256) {
                redo = (u0 == kSent) | (u1 == kSent) | (u2 == kSent) | (u3 == kSent);
            }
            if ((kMode & 8) && !(kMode & 128)) {
                while (u0 == kSent || u1 == kSent || u2 == kSent || u3 == kSent) {
                    u0 = lds_v(dc.a0);
                    u1 = lds_v(dc.a1);
                    u2 = lds_v(dc.a2);
                    u3 = lds_v(dc.a3);
                }
            }
            const double v0 = __hiloint2double(w.c0.y, w.c0.x), v1 = __hiloint2double(w.c0.w, w.c0.z);
            const double v2 = __hiloint2double(w.c1.y, w.c1.x), v3 = __hiloint2double(w.c1.w, w.c1.z);
            const double d = __hiloint2double(w.c2.y, w.c2.x), y = __hiloint2double(w.c2.w, w.c2.z);
            double sp = __dmul_rn(v0, __longlong_as_double(u0));
            sp = __dadd_rn(sp, __dmul_rn(v1, __longlong_as_double(u1)));
            sp = __dadd_rn(sp, __dmul_rn(v2, __longlong_as_double(u2)));
            sp = __dadd_rn(sp, __dmul_rn(v3, __longlong_as_double(u3)));
            const double acc = __dadd_rn(0.0, sp);
            const double tq = __dsub_rn(__longlong_as_double(ub), acc);
            const double q0 = __dmul_rn(tq, y);
            double xr = __fma_rn(y, __fma_rn(-d, q0, tq), q0);
            if (kMode & 256) {
                redo |= !in_range(tq) | (__double_as_longlong(y) == -1ll);
            } else if ((kMode & 16) && (kMode & 128) && (kMode & 1024)) {
                asm volatile("st.shared.u64 [%0], %1;" ::"r"(dc.own), "l"(__double_as_longlong(xr)) : "memory");
                const bool bad = !in_range(tq) | (__double_as_longlong(y) == -1ll);
                if (__any_sync(0xffffffffu, bad)) {
                    if (bad) {
                        xr = ddiv_out(tq, d);
                        asm volatile("st.shared.u64 [%0], %1;" ::"r"(dc.own), "l"(__double_as_longlong(xr)) : "memory");
                    }
                }
            } else if ((kMode & 16) && (kMode & 128)) {
                const bool bad = !in_range(tq) | (__double_as_longlong(y) == -1ll);
                if (__any_sync(0xffffffffu, bad)) {
                    if (bad) xr = ddiv_out(tq, d);
                }
                if (static_cast<unsigned long long>(__double_as_longlong(xr)) == kSent) xr = 0.0;
            } else if (kMode & 16) {
                if (!in_range(tq) | (__double_as_longlong(y) == -1ll)) xr = ddiv_out(tq, d);
                if (static_cast<unsigned long long>(__double_as_longlong(xr)) == kSent) xr = 0.0;
            }
            if (!(kMode & 1024)) asm volatile("st.shared.u64 [%0], %1;" ::"r"(dc.own), "l"(__double_as_longlong(xr)) : "memory");
            if (kMode & 2048) {
                pend_x = xr;
                pend_r = w.c3.z;
            } else if ((kMode & 4) && w.c3.z >= 0)
                asm volatile("st.relaxed.gpu.global.b64 [%0], %1;" ::"l"(x + w.c3.z), "l"(__double_as_longlong(xr)) : "memory");
            if (kMode & 64) {
                unsigned long long tt;
                asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tt));
                tr[w.c3.z] = tt;
            }
        }
        if (kMode & 2) fetch(w, s + kDepth);
        dc = decode(wn);
        if (kMode & 256) {
            int any;
            asm volatile("{\n.reg .pred p, q;\nsetp.ne.s32 p, %1, 0;\nbar.red.or.pred q, 1, 128, p;\nselp.s32 %0, 1, 0, q;\n}\n" : "=r"(any) : "r"(redo) : "memory");
            if (any) {  // never in this bench
                if (redo) dummy[tid] = ddiv_out(2.0, 3.0);
                asm volatile("bar.sync 1, 128;" ::: "memory");
            }
            return;
        }
        if ((kMode & 8) && (kMode & 128)) {  // halo entries for the next step: a CTA-uniform counter test
            unsigned hd;
            do {
                asm volatile("ld.acquire.cta.shared.u32 %0, [%1];" : "=r"(hd) : "r"(static_cast<uint32_t>(__cvta_generic_to_shared(&halo_done))) : "memory");
            } while (hd < static_cast<unsigned>(s));
        }
        if (kMode & 512) asm volatile("bar.sync 1, 160;" ::: "memory");
        else asm volatile("bar.sync 1, 128;" ::: "memory");
    };
    if (kMode & 2) {
        for (int s0 = 0; s0 < kSteps; s0 += kDepth) {
#pragma unroll
            for (int i = 0; i < kDepth; ++i)
                if (s0 + i < kSteps) step(q[i], q[(i + 1) % kDepth], s0 + i);
        }
    } else {
        for (int s = 0; s < kSteps; ++s) {
            step(q[s & 1], q[(s + 1) & 1], s);
        }
    }
    const long long t1 = clock64();
    if (tid == 0) out[kMode] = t1 - t0;
    if (kMode & 32) __syncthreads();
}

int main() {
    // records of a 10 x 10 x 100 tile (x fastest within a line); window slot of (x, j, k) = 100 * (j + 10 k) + x
    std::vector<std::vector<int>> rows(kSteps);
    for (int k = 0; k < 10; ++k)
        for (int j = 0; j < 10; ++j)
            for (int xx = 0; xx < 100; ++xx) rows[xx + j + k].push_back(100 * (j + 10 * k) + xx);
    std::vector<int4> all;
    std::vector<int> offs{0};
    for (int s = 0; s < kSteps; ++s) {
        const int c = static_cast<int>(rows[s].size());
        std::vector<int4> ch(4 * c);
        for (int i = 0; i < c; ++i) {
            const int slot = rows[s][i], xx = slot % 100, j = (slot / 100) % 10, k = slot / 1000;
            const short cz = k > 0 ? static_cast<short>(slot - 1000) : -1, cy = j > 0 ? static_cast<short>(slot - 100) : -1,
                        cx = xx > 0 ? static_cast<short>(slot - 1) : -1;
            double v[6] = {-1, -1, -1, 0, 6.05, 1 / 6.05};
            ch[i] = *reinterpret_cast<int4*>(&v[0]);
            ch[c + i] = *reinterpret_cast<int4*>(&v[2]);
            ch[2 * c + i] = *reinterpret_cast<int4*>(&v[4]);
            int4 m;
            m.x = (static_cast<uint16_t>(cz)) | (static_cast<int>(cy) << 16);
            m.y = (static_cast<uint16_t>(cx)) | (-1 << 16);
            m.z = slot;
            m.w = slot;
            ch[3 * c + i] = m;
        }
        all.insert(all.end(), ch.begin(), ch.end());
        offs.push_back(offs.back() + c);
    }
    int4* drec;
    int* doff;
    double* dx;
    unsigned long long* dtr;
    long long* dout;
    cudaMalloc(&drec, all.size() * sizeof(int4));
    cudaMemcpy(drec, all.data(), all.size() * sizeof(int4), cudaMemcpyHostToDevice);
    cudaMalloc(&doff, offs.size() * sizeof(int));
    cudaMemcpy(doff, offs.data(), offs.size() * sizeof(int), cudaMemcpyHostToDevice);
    cudaMalloc(&dx, 20000 * sizeof(double));
    cudaMalloc(&dtr, 20000 * sizeof(unsigned long long));
    cudaMallocManaged(&dout, 256 * sizeof(long long));
    const size_t smem = kRing * kT * 64 + 16 + 10000 * 8;
#define RUN(M)                                                                                                  \
    cudaFuncSetAttribute(wave_loop<M>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));   \
    for (int rep = 0; rep < 3; ++rep) wave_loop<M><<<1, (M & 32) ? 256 : (M & 512) ? 160 : 128, smem>>>(drec, doff, dx, dtr, dout); \
    cudaDeviceSynchronize();                                                                                    \
    printf("mode %3d: %6.1f cycles/step %s\n", M, dout[M] / double(kSteps), cudaGetErrorString(cudaGetLastError())); fflush(stdout);
    RUN(641) RUN(657) RUN(661) RUN(1681) RUN(1685) RUN(2709) RUN(3733) RUN(3797)
    return 0;
}
