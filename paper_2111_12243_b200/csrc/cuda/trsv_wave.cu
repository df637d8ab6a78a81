// Wavefront record solve (sm_100a): the record kernel's blocks, windows and
// halo warp (kernels.cu "Record-driven solve rounds"), but every solving warp
// walks a schedule fixed at bind instead of polling lane by lane.
//
// lower.cpp wave_schedule() simulates the block in lockstep -- step g holds
// the rows whose in-block operands all finished at steps < g, every lane
// taking its units front to back -- and lists, per warp, the steps in which
// one of its lanes has a row. Rows of one warp step never depend on one
// another, and an operand from the same warp was produced at an earlier step
// of that warp: inside a warp no row ever waits. Operands from other warps or
// blocks (the halo) are polled by the whole warp with one vote per attempt;
// every wait is for a row of a strictly smaller simulated step (or an earlier
// block), so the schedule cannot deadlock.
//
// The schedule is stored step-major: step s of a warp is 32 slots -- a row's
// 64-byte record (trsv_build_rec), kept in four 16-byte chunk planes so a
// warp's loads are contiguous, and its row index (-1: the lane idles; its
// record is a null row that stores to a scratch word). A warp streams its
// steps through a shared-memory ring with cp.async, kWaveDepth steps ahead
// (row indices twice that, so the right-hand side b[row] can be fetched with
// the record), one commit group per step. All lanes step together, so the
// ring bookkeeping is warp-uniform and the next step's record is read from
// the ring before the current step's FP chain.
//
// Per step and lane: four window loads (operand address = window + 8 * code),
// the sentinel test and vote, the reference's sequential partial,
// acc = 0 + partial, x = (b - acc) / d on the precomputed reciprocal
// (executor.cpp:119-145; bitwise equal to __ddiv_rn, trsv_common.cuh), one
// store into the window and one into x.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>

#include "kernels.hpp"
#include "trsv_common.cuh"

namespace pscb {
namespace {

constexpr int kWaveDepth = 8;      // steps staged ahead per warp (ring slots)
constexpr int kWaveStepBytes = 32 * 64;

__host__ __device__ constexpr int wave_pad_warps(int threads) { return threads >= 128 ? 3 : 0; }

template <int kT>
struct WaveSmem {
    // per warp: ring of kWaveDepth steps, [slot][16-byte chunk][lane]
    unsigned long long rec[kT / 32][kWaveDepth][4][32][2];
    double bq[kT / 32][kWaveDepth][32];
    int rowq[kT / 32][2 * kWaveDepth][32];
    unsigned long long bar[kT / 32][kWaveDepth];  // one mbarrier per ring slot
    unsigned long long scratch, zero;  // window slots -2 (null rows store here) and -1 (padding operands)
};

struct WaveRow {
    int r, loc, slow;
    int l0, l1, l2, l3;  // operand j: the lane whose last x it is (the warp's previous step), or -1: the window
    uint32_t a0, a1, a2, a3;
    double v0, v1, v2, v3, d, y, br;
};

template <int kT, bool kDiag>
__global__ void __launch_bounds__(kT + 32 * (1 + wave_pad_warps(kT))) sptrsv_wave_kernel(WaveArgs A) {
    constexpr int kD = kWaveDepth;
    constexpr int kW = kT / 32;
    constexpr int kAll = kT + 32 * (1 + wave_pad_warps(kT));
    extern __shared__ __align__(16) unsigned char smem_raw[];
    WaveSmem<kT>& ws = *reinterpret_cast<WaveSmem<kT>*>(smem_raw);
    double* sx_raw = reinterpret_cast<double*>(smem_raw + sizeof(WaveSmem<kT>));  // window: rows, then halo
    volatile unsigned long long* sxb = reinterpret_cast<volatile unsigned long long*>(sx_raw);
    int32_t* hcol = reinterpret_cast<int32_t*>(sx_raw + A.max_rows + A.max_halo);
    __shared__ int s_blk;
    const int tid = threadIdx.x;
    const uint32_t sx_addr = static_cast<uint32_t>(__cvta_generic_to_shared(sx_raw));
    if (tid == 0) {
        ws.zero = 0ull;
        ws.scratch = 0ull;
        s_blk = atomicAdd(A.ticket, 1);
    }
    __syncthreads();
    const int blk = s_blk;
    const int U0 = A.block_unit[blk], nU = A.block_unit[blk + 1] - U0;
    const int nrows = A.block_row[blk + 1] - A.block_row[blk];
    const int H0 = A.halo_ptr[blk], nH = A.halo_ptr[blk + 1] - H0;
    for (int i = tid; i < nH; i += kAll) {
        hcol[i] = __ldg(A.halo_col + H0 + i);
        sxb[nrows + i] = kSentinel;
    }
    for (int u = tid >> 5; u < nU; u += kAll / 32) {  // sentinels in the window and in x, unit by unit
        const int r0 = __ldg(A.unit_start + U0 + u), n = __ldg(A.unit_len + U0 + u), l0 = __ldg(A.unit_loc + U0 + u);
        for (int j = tid & 31; j < n; j += 32) {
            sxb[l0 + j] = kSentinel;
            reinterpret_cast<unsigned long long*>(A.x)[r0 + j] = kSentinel;
        }
    }
    __syncthreads();
    if (tid == 0) {
        __threadfence();
        st_release_gpu(A.armed + blk, A.epoch);
        if (A.trace) {
            unsigned long long t;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
            A.trace[A.block_row[gridDim.x] + blk] = t;
        }
    }
    for (int j = tid; j < blk; j += kAll) {  // earlier blocks must be armed before their x is trusted
        while (ld_acquire_gpu(A.armed + j) != A.epoch) {
        }
    }
    __syncthreads();
    __threadfence();

    if (tid >= kT && tid < kT + 32 * wave_pad_warps(kT)) {
        // idle warps: they keep the halo warp off the first solving warps' sub-partitions
    } else if (tid >= kT) {
        // ---- halo warp: copy the halo's x entries from L2 as they are published (production order)
        const int lane = tid - kT - 32 * wave_pad_warps(kT);
        volatile unsigned long long* hx = sxb + nrows;
        for (int e = lane; e < nH;) {
            const int e1 = e + 32, e2 = e + 64, e3 = e + 96;
            const unsigned long long v0 = ld_relaxed_gpu(A.x + hcol[e]);
            const unsigned long long v1 = e1 < nH ? ld_relaxed_gpu(A.x + hcol[e1]) : 0ull;
            const unsigned long long v2 = e2 < nH ? ld_relaxed_gpu(A.x + hcol[e2]) : 0ull;
            const unsigned long long v3 = e3 < nH ? ld_relaxed_gpu(A.x + hcol[e3]) : 0ull;
            int adv = 0;
            if (v0 != kSentinel) {
                hx[e] = v0;
                adv = 1;
                if (v1 != kSentinel) {
                    if (e1 < nH) hx[e1] = v1;
                    adv = 2;
                    if (v2 != kSentinel) {
                        if (e2 < nH) hx[e2] = v2;
                        adv = 3;
                        if (v3 != kSentinel) {
                            if (e3 < nH) hx[e3] = v3;
                            adv = 4;
                        }
                    }
                }
            }
            e += 32 * adv;
        }
    } else {
        // ---- solving warps: one schedule each
        const int w = tid >> 5, lane = tid & 31;
        const int s0 = __ldg(A.wstep_ptr + blk * kW + w);
        const int ns = __ldg(A.wstep_ptr + blk * kW + w + 1) - s0;
        const char* recw = static_cast<const char*>(A.rec) + static_cast<size_t>(s0) * kWaveStepBytes;
        const int32_t* roww = A.srow + static_cast<size_t>(s0) * 32;
        const uint32_t ring0 = static_cast<uint32_t>(__cvta_generic_to_shared(&ws.rec[w][0][0][0][0]));
        const uint32_t ring = ring0 + 16u * lane;
        const uint32_t bqa = static_cast<uint32_t>(__cvta_generic_to_shared(&ws.bq[w][0][lane]));
        const uint32_t rq0 = static_cast<uint32_t>(__cvta_generic_to_shared(&ws.rowq[w][0][0]));
        const uint32_t rqa = rq0 + 4u * lane;
        const uint32_t bar0 = static_cast<uint32_t>(__cvta_generic_to_shared(&ws.bar[w][0]));
        auto ch = [&](int k, int c) -> uint32_t { return ring + 512u * static_cast<uint32_t>(k * 4 + c); };
        if (lane == 0) {
            if (ns > 0) prefetch_l2(recw, static_cast<size_t>(ns) * kWaveStepBytes, 0, 1);  // one contiguous range
#pragma unroll
            for (int k = 0; k < kD; ++k)
                asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar0 + 8u * k) : "memory");
            asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        }
        // row indices of the first 2 kD steps (plain loads), then the lane's b of the first kD
#pragma unroll
        for (int s = 0; s < 2 * kD; ++s)
            if (s < ns) sts_s32(rqa + 128u * s, __ldg(roww + static_cast<size_t>(s) * 32 + lane));
        __syncwarp();
        // one bulk copy per step: its 32 records (2048 bytes) into ring slot s % kD, and the row
        // indices of step s + kD (the lanes fetch b of step s + kD when that copy has landed)
        auto issue_step = [&](int s) {  // lane 0
            const int k = s & (kD - 1);
            const uint32_t bar = bar0 + 8u * k;
            const bool rows = s >= kD && s + kD < ns;  // rows of steps < 2 kD came with the prologue
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(rows ? 2048u + 128u : 2048u) : "memory");
            asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                             ring0 + 2048u * k),
                         "l"(recw + static_cast<size_t>(s) * kWaveStepBytes), "r"(2048u), "r"(bar)
                         : "memory");
            if (rows)
                asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                                 rq0 + 128u * ((s + kD) & (2 * kD - 1))),
                             "l"(roww + static_cast<size_t>(s + kD) * 32), "r"(128u), "r"(bar)
                             : "memory");
        };
        auto issue_b = [&](int s) {  // all lanes: b of step s (its row index is in the row ring)
            int r;
            asm volatile("ld.shared.s32 %0, [%1];" : "=r"(r) : "r"(rqa + 128u * static_cast<uint32_t>(s & (2 * kD - 1))) : "memory");
            const uint32_t bd = bqa + 256u * static_cast<uint32_t>(s & (kD - 1));
            if (r >= 0) cpa8(bd, A.b + r);
            else asm volatile("st.shared.u64 [%0], %1;" ::"r"(bd), "l"(0x3FF0000000000000ull) : "memory");  // b = 1: x = 1 / 1
        };
        auto wait_step = [&](int s) {  // the bulk copies of step s have landed
            const uint32_t bar = bar0 + 8u * (s & (kD - 1));
            const uint32_t parity = static_cast<uint32_t>(s / kD) & 1u;
            uint32_t done;
            do {
                asm volatile(
                    "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                    : "=r"(done)
                    : "r"(bar), "r"(parity)
                    : "memory");
            } while (!done);
        };
        struct Raw {
            int r, m01, m23, src, ls;
            double v0, v1, v2, v3, d, y, br;
        };
        auto load_raw = [&](Raw& q, int s) {
            const int k = s & (kD - 1);
            asm volatile("ld.shared.s32 %0, [%1];" : "=r"(q.r) : "r"(rqa + 128u * static_cast<uint32_t>(s & (2 * kD - 1))) : "memory");
            lds_f64x2(ch(k, 0), q.v0, q.v1);
            lds_f64x2(ch(k, 1), q.v2, q.v3);
            lds_f64x2(ch(k, 2), q.d, q.y);
            lds_s32x4(ch(k, 3), q.m01, q.m23, q.src, q.ls);
            asm volatile("ld.shared.f64 %0, [%1];" : "=d"(q.br) : "r"(bqa + 256u * static_cast<uint32_t>(k)) : "memory");
        };
        WaveRow cur;
        bool need0 = false, need1 = false, need2 = false, need3 = false;  // some lane takes operand j from a lane's last x
        auto adopt = [&](const Raw& q) {
            cur.r = q.r;
            cur.loc = static_cast<int>(static_cast<short>(q.ls & 0xFFFF));
            cur.slow = q.ls >> 16;
            cur.v0 = q.v0;
            cur.v1 = q.v1;
            cur.v2 = q.v2;
            cur.v3 = q.v3;
            cur.d = q.d;
            cur.y = q.y;
            cur.br = q.br;
            cur.a0 = sx_addr + 8u * static_cast<uint32_t>(static_cast<int>(static_cast<short>(q.m01 & 0xFFFF)));
            cur.a1 = sx_addr + 8u * static_cast<uint32_t>(q.m01 >> 16);
            cur.a2 = sx_addr + 8u * static_cast<uint32_t>(static_cast<int>(static_cast<short>(q.m23 & 0xFFFF)));
            cur.a3 = sx_addr + 8u * static_cast<uint32_t>(q.m23 >> 16);
            cur.l0 = static_cast<int>(static_cast<signed char>(q.src & 0xFF));
            cur.l1 = static_cast<int>(static_cast<signed char>((q.src >> 8) & 0xFF));
            cur.l2 = static_cast<int>(static_cast<signed char>((q.src >> 16) & 0xFF));
            cur.l3 = q.src >> 24;
            need0 = __any_sync(0xFFFFFFFFu, cur.l0 >= 0);
            need1 = __any_sync(0xFFFFFFFFu, cur.l1 >= 0);
            need2 = __any_sync(0xFFFFFFFFu, cur.l2 >= 0);
            need3 = __any_sync(0xFFFFFFFFu, cur.l3 >= 0);
        };
        if (ns > 0) {
            if (lane == 0) {
#pragma unroll
                for (int s = 0; s < kD; ++s)
                    if (s < ns) issue_step(s);
            }
#pragma unroll
            for (int s = 0; s < kD; ++s) {
                if (s < ns) issue_b(s);
                asm volatile("cp.async.commit_group;" ::: "memory");
            }
            asm volatile("cp.async.wait_group %0;" ::"n"(kD - 1) : "memory");
            wait_step(0);
            {
                Raw q;
                load_raw(q, 0);
                adopt(q);
            }
        }
        unsigned polls = 0;
        long long cyc_wait = 0, cyc_poll = 0, cyc_fp = 0, cyc_st = 0;
        const long long t_start = clock64();
        double xprev = 0.0;  // the lane's last x: operands produced by this warp's previous step come by shuffle
        for (int s = 0; s < ns; ++s) {
            long long c0 = 0, c1 = 0, c2 = 0, c3 = 0, c4 = 0;
            if (kDiag) c0 = clock64();
            // step s + 1: its b (cp.async group) and its records (bulk copy) have landed
            asm volatile("cp.async.wait_group %0;" ::"n"(kD - 2) : "memory");
            if (s + 1 < ns) wait_step(s + 1);
            if (kDiag) c1 = clock64();
            Raw nx;
            load_raw(nx, s + 1);
            // operands from the warp's previous step
            double h0 = 0.0, h1 = 0.0, h2 = 0.0, h3 = 0.0;
            if (need0) h0 = __shfl_sync(0xFFFFFFFFu, xprev, cur.l0);
            if (need1) h1 = __shfl_sync(0xFFFFFFFFu, xprev, cur.l1);
            if (need2) h2 = __shfl_sync(0xFFFFFFFFu, xprev, cur.l2);
            if (need3) h3 = __shfl_sync(0xFFFFFFFFu, xprev, cur.l3);
            unsigned long long u0, u1, u2, u3;
            // operands from the window (older steps, other warps, the halo): lanes re-read only
            // what is still missing
            u0 = lds_u64(cur.a0);
            u1 = lds_u64(cur.a1);
            u2 = lds_u64(cur.a2);
            u3 = lds_u64(cur.a3);
            while (!__all_sync(0xFFFFFFFFu,
                               (u0 != kSentinel) & (u1 != kSentinel) & (u2 != kSentinel) & (u3 != kSentinel))) {
                if (A.poll_ns > 0) __nanosleep(A.poll_ns);
                if (u0 == kSentinel) u0 = lds_u64(cur.a0);
                if (u1 == kSentinel) u1 = lds_u64(cur.a1);
                if (u2 == kSentinel) u2 = lds_u64(cur.a2);
                if (u3 == kSentinel) u3 = lds_u64(cur.a3);
                if (kDiag) ++polls;
            }
            if (kDiag) {
                c2 = clock64();
                cyc_wait += c1 - c0;
                cyc_poll += c2 - c1;
            }
            const double x0 = cur.l0 >= 0 ? h0 : __longlong_as_double(static_cast<long long>(u0));
            const double x1 = cur.l1 >= 0 ? h1 : __longlong_as_double(static_cast<long long>(u1));
            const double x2 = cur.l2 >= 0 ? h2 : __longlong_as_double(static_cast<long long>(u2));
            const double x3 = cur.l3 >= 0 ? h3 : __longlong_as_double(static_cast<long long>(u3));
            // exec_group + finalize_row (executor.cpp:119-145)
            double sp = __dmul_rn(cur.v0, x0);
            sp = __dadd_rn(sp, __dmul_rn(cur.v1, x1));
            sp = __dadd_rn(sp, __dmul_rn(cur.v2, x2));
            sp = __dadd_rn(sp, __dmul_rn(cur.v3, x3));
            const double acc = __dadd_rn(0.0, sp);
            const double tq = __dsub_rn(cur.br, acc);
            double xr = div_rcp_fast(tq, cur.d, cur.y);
            if (!div_rcp_range(tq) | (cur.slow != 0)) xr = ddiv_outlined(tq, cur.d);
            if (static_cast<unsigned long long>(__double_as_longlong(xr)) == kSentinel)
                xr = __longlong_as_double(static_cast<long long>(kCanonNaN));
            xprev = xr;
            if (kDiag) {
                asm volatile("" ::"d"(xr));
                c3 = clock64();
            }
            asm volatile("st.volatile.shared.u64 [%0], %1;" ::"r"(sx_addr + 8u * static_cast<uint32_t>(cur.loc)),
                         "l"(__double_as_longlong(xr))
                         : "memory");
            if (cur.r >= 0) {
                st_relaxed_gpu(A.x + cur.r, xr);
                if (kDiag && A.acc_out) A.acc_out[cur.r] = acc;
                if (kDiag && A.trace && A.trace_rows) {
                    unsigned long long tt;
                    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tt));
                    A.trace[cur.r] = tt;
                }
            }
            __syncwarp();  // the window store is visible to the warp's later steps; the ring slot of step s is free
            if (kDiag) {
                c4 = clock64();
                cyc_fp += c3 - c2;
                cyc_st += c4 - c3;
            }
            adopt(nx);
            if (s + kD < ns) {
                if (lane == 0) issue_step(s + kD);
                issue_b(s + kD);
            }
            asm volatile("cp.async.commit_group;" ::: "memory");
        }
        asm volatile("cp.async.wait_all;" ::: "memory");
        if (kDiag && A.trace && lane == 0) {  // diagnostics: steps + polls, cycles in the loop, warps, steps
            unsigned long long* stats = A.trace + A.block_row[gridDim.x] + gridDim.x;
            atomicAdd(stats + 0, static_cast<unsigned long long>(ns) + polls);
            atomicAdd(stats + 1, static_cast<unsigned long long>(clock64() - t_start));
            atomicAdd(stats + 2, 1ull);
            atomicAdd(stats + 3, static_cast<unsigned long long>(ns));
            atomicAdd(stats + 4, static_cast<unsigned long long>(cyc_wait));
            atomicAdd(stats + 5, static_cast<unsigned long long>(cyc_poll));
            if (blk == 0 && w == 0) {
                atomicAdd(stats + 6, static_cast<unsigned long long>(clock64() - t_start));
                atomicAdd(stats + 7, static_cast<unsigned long long>(ns));
                atomicAdd(stats + 8, static_cast<unsigned long long>(cyc_wait));
                atomicAdd(stats + 9, static_cast<unsigned long long>(cyc_poll));
                atomicAdd(stats + 10, static_cast<unsigned long long>(polls));
                atomicAdd(stats + 11, static_cast<unsigned long long>(cyc_fp));
                atomicAdd(stats + 12, static_cast<unsigned long long>(cyc_st));
            }
        }
    }
    __syncthreads();
    if (tid == 0) {  // the last block to finish re-arms the ticket for the next launch
        __threadfence();
        if (atomicAdd(A.ticket + 1, 1) == static_cast<int>(gridDim.x) - 1) {
            A.ticket[0] = 0;
            A.ticket[1] = 0;
        }
    }
}

// Records of the scheduled rows, written to their slots (chunk planes of the step).
__global__ void trsv_wave_pack_kernel(const int32_t* ro, const int32_t* col, const double* val, const int32_t* row_block,
                                      const int32_t* row_loc, const int32_t* block_row, const int32_t* halo_ptr,
                                      const int32_t* halo_key, const int32_t* halo_pos, const int32_t* wslot,
                                      const int32_t* wsrc, int n_rows, unsigned char* rec) {
    const int r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= n_rows) return;
    TrsvRec q = trsv_build_rec(ro, col, val, row_block, row_loc, block_row, halo_ptr, halo_key, halo_pos, r);
    // operands the warp's previous step produced come from that lane's register (wsrc: four
    // lanes, -1: the window); their window code is the zero word
    const int lanes = wsrc[r];
#pragma unroll
    for (int j = 0; j < 4; ++j)
        if (static_cast<signed char>((lanes >> (8 * j)) & 0xFF) >= 0) q.idx[j] = -1;
    q.pad[1] = (row_loc[r] & 0xFFFF) | (q.pad[0] << 16);
    q.pad[0] = lanes;
    const int slot = wslot[r];
    unsigned char* dst = rec + static_cast<size_t>(slot >> 5) * kWaveStepBytes + 16 * (slot & 31);
    const uint4* src = reinterpret_cast<const uint4*>(&q);
#pragma unroll
    for (int c = 0; c < 4; ++c) *reinterpret_cast<uint4*>(dst + 512 * c) = src[c];
}

// Idle slots: a null row (no operands, d = 1; its b is set to 1 in the ring) that stores to the scratch word below the window.
__global__ void trsv_wave_null_kernel(const int32_t* srow, int64_t n_slots, unsigned char* rec) {
    const int64_t slot = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (slot >= n_slots || srow[slot] >= 0) return;
    TrsvRec q;
    for (int j = 0; j < 4; ++j) {
        q.v[j] = 0.0;
        q.idx[j] = -1;
    }
    q.d = 1.0;
    q.y = 1.0;
    q.pad[0] = -1;              // no operand from a lane
    q.pad[1] = (-2) & 0xFFFF;   // stores to the scratch word
    unsigned char* dst = rec + static_cast<size_t>(slot >> 5) * kWaveStepBytes + 16 * (slot & 31);
    const uint4* src = reinterpret_cast<const uint4*>(&q);
#pragma unroll
    for (int c = 0; c < 4; ++c) *reinterpret_cast<uint4*>(dst + 512 * c) = src[c];
}

template <int T>
void launch_wave_t(const WaveArgs& A, cudaStream_t stream) {
    const size_t smem = sptrsv_wave_smem_bytes(T, A.max_rows, A.max_halo);
    auto go = [&](auto kern) {
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
        kern<<<A.n_blocks, T + 32 * (1 + wave_pad_warps(T)), smem, stream>>>(A);
    };
    if (A.acc_out || A.trace) go(sptrsv_wave_kernel<T, true>);
    else go(sptrsv_wave_kernel<T, false>);
}

}  // namespace

size_t sptrsv_wave_smem_bytes(int threads, int max_rows, int max_halo) {
    size_t ring = 0;
    switch (threads) {
        case 64: ring = sizeof(WaveSmem<64>); break;
        case 128: ring = sizeof(WaveSmem<128>); break;
        case 256: ring = sizeof(WaveSmem<256>); break;
        default: ring = sizeof(WaveSmem<512>); break;
    }
    return ring + static_cast<size_t>(max_rows + max_halo) * sizeof(double) + static_cast<size_t>(max_halo) * sizeof(int32_t);
}

void launch_trsv_wave_pack(const int32_t* ro, const int32_t* col, const double* val, const int32_t* row_block,
                           const int32_t* row_loc, const int32_t* block_row, const int32_t* halo_ptr,
                           const int32_t* halo_key, const int32_t* halo_pos, const int32_t* wslot, const int32_t* wsrc,
                           int n_rows, void* rec, cudaStream_t stream) {
    if (n_rows <= 0) return;
    trsv_wave_pack_kernel<<<(n_rows + 255) / 256, 256, 0, stream>>>(ro, col, val, row_block, row_loc, block_row, halo_ptr,
                                                                    halo_key, halo_pos, wslot, wsrc, n_rows,
                                                                    static_cast<unsigned char*>(rec));
}

void launch_trsv_wave_nulls(const int32_t* srow, int64_t n_slots, void* rec, cudaStream_t stream) {
    if (n_slots <= 0) return;
    trsv_wave_null_kernel<<<static_cast<unsigned>((n_slots + 255) / 256), 256, 0, stream>>>(
        srow, n_slots, static_cast<unsigned char*>(rec));
}

void launch_sptrsv_wave(const WaveArgs& A, int threads, cudaStream_t stream) {
    if (A.n_blocks <= 0) return;
    switch (threads) {
        case 64: launch_wave_t<64>(A, stream); break;
        case 128: launch_wave_t<128>(A, stream); break;
        case 512: launch_wave_t<512>(A, stream); break;
        default: launch_wave_t<256>(A, stream); break;
    }
}

}  // namespace pscb
