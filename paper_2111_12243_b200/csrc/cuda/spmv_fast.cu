// Fast-mode SpMV (PSC_MODE_FAST): the same y = A x over the plan's rows with
// the row sums reassociated (north_star: SpMV within 1e-12 normwise of the
// reference; the summation order may differ). Parity mode keeps the
// reference's dot_unit order (kernels.cu); this path balances work by entries
// and adds products in a fixed order of its own, so it is deterministic run
// to run but not bitwise equal to the reference.
//
// Column-split passes (x larger than L2, config 5): the matrix is stored as
// one entry stream per column range of x, and pass q gathers only from range
// q, which stays in L2 while its entries stream by; pass 0 stores y, later
// passes add onto it. Each row is owned by one lane (or one carry fixup) per
// pass: no atomics.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>

#include "kernels.hpp"

namespace pscb {
namespace {

__device__ __forceinline__ uint64_t policy_evict_first() {
    uint64_t p;
    asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ uint64_t policy_evict_last() {
    uint64_t p;
    asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ double ld_keep_f64(const double* a, uint64_t pol) {
    double v;
    // no L1 allocation: a random gather is never reused there (config 5: 1.980 -> 1.958 ms)
    asm("ld.global.nc.L1::no_allocate.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(a), "l"(pol));
    return v;
}

// ---- flagged entries, register-only warps ----------------------------------
// The L1 data pipe moves one wavefront per cycle per SM and a random x gather
// costs one (tools/gather_probe.cu: ~1 gather per SM-cycle, L2 hit or not);
// shared-memory traffic and shuffles go through the same pipe and come
// straight off the gather rate. So this kernel keeps the row bookkeeping in
// registers: each entry's column carries a row-end flag in bit 31, and every
// row holds at least one entry in every pass (an empty row gets one
// placeholder entry, column 0x7fffffff, which contributes +0), so the m-th
// row end of a pass is row m. A warp takes chunks of 32 x kSegPer entries
// (4 by default; chunk starts are aligned, so lane l loads its consecutive
// entries with 16-byte vector loads, issued one chunk ahead so they are in
// flight during the previous chunk's gathers); ballots count the row ends
// before each lane, the
// rows' old y (accumulating passes) is loaded beside the x gathers, each lane
// sums its rows sequentially, and one shuffle scan over the lanes (12
// shuffles per chunk) adds the partials that cross lanes to each lane's first
// row. The chunk's trailing open row goes to the per-chunk carry
// (spmv_carry_fixup_kernel), so rows may span chunks and warps.
constexpr int kSegWarps = 8;
constexpr uint32_t kNoColumn = 0x7fffffffu;

template <int kSegPer>
__device__ __forceinline__ void load_chunk(const FlagPassDev& P, int c, int lane, uint64_t pf, int4 (&c4)[kSegPer / 4],
                                           double2 (&v2)[kSegPer / 2], int& m0) {
    const int64_t k0 = static_cast<int64_t>(c) * (32 * kSegPer) + kSegPer * lane;
    const int4* cp = reinterpret_cast<const int4*>(P.colf + k0);
    const double2* vp = reinterpret_cast<const double2*>(P.val + k0);
    m0 = __ldg(P.chunk_m0 + c);
#pragma unroll
    for (int i = 0; i < kSegPer / 4; ++i)
        asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.s32 {%0,%1,%2,%3}, [%4], %5;"
                     : "=r"(c4[i].x), "=r"(c4[i].y), "=r"(c4[i].z), "=r"(c4[i].w)
                     : "l"(cp + i), "l"(pf));
#pragma unroll
    for (int i = 0; i < kSegPer / 2; ++i)
        asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v2.f64 {%0,%1}, [%2], %3;"
                     : "=d"(v2[i].x), "=d"(v2[i].y)
                     : "l"(vp + i), "l"(pf));
}

template <bool kAccum, int kSegPer, int kMinBlocks, bool kPf>
__global__ void __launch_bounds__(32 * kSegWarps, kMinBlocks) spmv_flag_kernel(FlagPassDev P, const double* __restrict__ x,
                                                                              double* __restrict__ y) {
    const int lane = threadIdx.x & 31;
    const uint32_t lt = (1u << lane) - 1u;  // lanes below this one
    const uint64_t pf = policy_evict_first(), pl = policy_evict_last();
    const int n_warps = gridDim.x * kSegWarps;
    int4 n4[kSegPer / 4];
    double2 n2[kSegPer / 2];
    int nm0 = 0;
    const int c_first = blockIdx.x * kSegWarps + (threadIdx.x >> 5);
    if (kPf && c_first < P.n_chunks) load_chunk<kSegPer>(P, c_first, lane, pf, n4, n2, nm0);
    for (int c = c_first; c < P.n_chunks; c += n_warps) {
        const int64_t k0 = static_cast<int64_t>(c) * (32 * kSegPer) + kSegPer * lane;  // this lane's entries
        int m0;
        uint32_t cf[kSegPer];
        double v[kSegPer];
        {
            int4 c4[kSegPer / 4];
            double2 v2[kSegPer / 2];
            if (kPf) {  // this chunk was loaded an iteration ago; start the next one's loads
#pragma unroll
                for (int i = 0; i < kSegPer / 4; ++i) c4[i] = n4[i];
#pragma unroll
                for (int i = 0; i < kSegPer / 2; ++i) v2[i] = n2[i];
                m0 = nm0;
                if (c + n_warps < P.n_chunks) load_chunk<kSegPer>(P, c + n_warps, lane, pf, n4, n2, nm0);
            } else {
                load_chunk<kSegPer>(P, c, lane, pf, c4, v2, m0);
            }
#pragma unroll
            for (int i = 0; i < kSegPer / 4; ++i) {
                cf[4 * i] = c4[i].x;
                cf[4 * i + 1] = c4[i].y;
                cf[4 * i + 2] = c4[i].z;
                cf[4 * i + 3] = c4[i].w;
            }
#pragma unroll
            for (int i = 0; i < kSegPer / 2; ++i) {
                v[2 * i] = v2[i].x;
                v[2 * i + 1] = v2[i].y;
            }
        }
        // row ends before this lane's run (one ballot per entry slot); this lane's rows are m, m+1, ...
        int m = m0, my_ends = 0;
#pragma unroll
        for (int i = 0; i < kSegPer; ++i) {
            const uint32_t b = __ballot_sync(0xffffffffu, cf[i] >> 31);
            m += __popc(b & lt);
            my_ends += static_cast<int>(cf[i] >> 31);
        }
        double yo[kSegPer];  // the rows' y from earlier passes, loaded beside the gathers
        if constexpr (kAccum) {
#pragma unroll
            for (int i = 0; i < kSegPer; ++i) yo[i] = i < my_ends ? y[m + i] : 0.0;
        }
        // entries past the pass's end are padding (column 0, value 0, no flag)
#pragma unroll
        for (int i = 0; i < kSegPer; ++i) {
            const uint32_t cc = cf[i] & 0x7fffffffu;
            const double xv = ld_keep_f64(x + (cc == kNoColumn ? 0u : cc), pl);
            v[i] = cc == kNoColumn ? 0.0 : v[i] * xv;
        }
        // the lane's rows: the first one is completed by the scan below
        double acc = 0.0, first = 0.0;
        int e = 0;
#pragma unroll
        for (int i = 0; i < kSegPer; ++i) {
            acc += v[i];
            if (cf[i] >> 31) {
                if (e == 0) {
                    first = acc;
                } else {
                    double out = acc;
                    if constexpr (kAccum) {
#pragma unroll
                        for (int q = 1; q < kSegPer; ++q)
                            if (q == e) out += yo[q];
                    }
                    y[m + e] = out;
                }
                ++e;
                acc = 0.0;
            }
        }
        // segmented scan over lanes of the trailing open partials: a lane with a row
        // end starts a new segment
        const uint32_t heads = __ballot_sync(0xffffffffu, my_ends > 0) | 1u;
        const int seg0 = 31 - __clz(heads & (lt | (1u << lane)));
        double s = acc;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const double u = __shfl_up_sync(0xffffffffu, s, o);
            if (lane - o >= seg0) s += u;
        }
        const double ex = __shfl_up_sync(0xffffffffu, s, 1);  // the open row's sum through the lane before
        if (my_ends > 0) {
            const double tot = lane > 0 ? ex + first : first;
            if constexpr (kAccum) y[m] = yo[0] + tot;
            else y[m] = tot;
        }
        if (lane == 31) {
            // a chunk whose last entry ends no row leaves row m + my_ends open (the
            // pass's last entry always ends a row, so the final chunk never does)
            const bool open = !(cf[kSegPer - 1] >> 31) && k0 + kSegPer < P.n_ent;
            P.carry_row[c] = open ? m + my_ends : -1;
            P.carry_val[c] = open ? s : 0.0;
        }
    }
}

// Adds each chunk's carried partial to its row: one thread per run of chunks
// that carry the same row, summing the run in chunk order.
__global__ void spmv_carry_fixup_kernel(double* __restrict__ y, const double* __restrict__ carry_val,
                                        const int32_t* __restrict__ carry_row, int n_tiles) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= n_tiles) return;
    const int32_t r = carry_row[t];
    if (r < 0 || (t > 0 && carry_row[t - 1] == r)) return;
    double s = carry_val[t];
    for (int u = t + 1; u < n_tiles && carry_row[u] == r; ++u) s += carry_val[u];
    y[r] += s;
}

}  // namespace

int flag_chunk_entries(int per) { return 32 * per; }

void launch_spmv_flag(const FlagPassDev& P, const double* x, double* y, bool accumulate, int n_sms, cudaStream_t stream) {
    if (P.n_chunks <= 0) return;
#define PSC_FLAG(PER, MB, PF)                                                                                 \
    do {                                                                                                      \
        const int grid = std::max(1, std::min((P.n_chunks + kSegWarps - 1) / kSegWarps, MB * n_sms));        \
        if (accumulate) spmv_flag_kernel<true, PER, MB, PF><<<grid, 32 * kSegWarps, 0, stream>>>(P, x, y);   \
        else spmv_flag_kernel<false, PER, MB, PF><<<grid, 32 * kSegWarps, 0, stream>>>(P, x, y);             \
    } while (0)
    // 4 entries per lane: the next chunk's loads in flight during this chunk's
    // gathers, 3 CTAs/SM (1.98 against 2.05 ms unpipelined at 6)
    if (P.per == 4) PSC_FLAG(4, 3, true);
    else PSC_FLAG(8, 4, false);
#undef PSC_FLAG
    spmv_carry_fixup_kernel<<<(P.n_chunks + 255) / 256, 256, 0, stream>>>(y, P.carry_val, P.carry_row, P.n_chunks);
}

}  // namespace pscb
