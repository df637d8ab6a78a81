// C ABI, device half: Executor, bound (HBM-resident) plans, the host-span
// run_spmv / run_sptrsv contracts, execute_plan and exec_*_codelet.
//
// Reference: /root/reference/proj/core/src/executor.cpp:252-308 (Executor,
// execute_plan, run_spmv, run_sptrsv) and :53-116 (exec_*_codelet).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <functional>
#include <mutex>
#include <string>
#include <tuple>
#include <vector>

#include "capi_types.hpp"
#include "csr.hpp"
#include "common.hpp"
#include "kernels.hpp"
#include "lower.hpp"

using namespace pscb;

namespace pscb {

inline void ck(cudaError_t e, const char* what) {
    if (e != cudaSuccess) throw CudaError(std::string(what) + ": " + cudaGetErrorString(e));
}

// Owned device allocation.
struct DevBuf {
    void* p = nullptr;
    size_t bytes = 0;
    DevBuf() = default;
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
    ~DevBuf() { release(); }
    void release() {
        if (p) cudaFree(p);
        p = nullptr;
        bytes = 0;
    }
    void ensure(size_t n) {
        if (n <= bytes && p) return;
        release();
        // +64 bytes: 16-byte-rounded bulk copies of a tail stay in bounds (spmv_fast.cu)
        ck(cudaMalloc(&p, std::max<size_t>(n, 16) + 64), "cudaMalloc");
        bytes = std::max<size_t>(n, 16);
    }
    template <class T>
    void upload(const std::vector<T>& v, cudaStream_t s) {
        ensure(v.size() * sizeof(T));
        if (!v.empty()) ck(cudaMemcpyAsync(p, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice, s), "H2D");
    }
    void upload_raw(const void* h, size_t n, cudaStream_t s) {
        ensure(n);
        if (n) ck(cudaMemcpyAsync(p, h, n, cudaMemcpyHostToDevice, s), "H2D");
    }
    template <class T>
    T* as() const {
        return static_cast<T*>(p);
    }
};

}  // namespace pscb

struct psc_bound {
    int device = 0;
    int kernel = PSC_KERNEL_SPMV;
    int mode = PSC_MODE_PARITY;
    int32_t row_begin = 0, row_end = 0, n_rows_total = 0, n_cols = 0;
    int64_t k_begin = 0, k_end = 0;
    bool canonical = true, simple = true;
    int n_chunks = 0, n_blocks = 0, max_block_rows = 0, n_sms = 148;
    int64_t n_segments = 0, long_rows = 0;
    int spmv_short = 0;  // > 0: every row holds <= spmv_short entries (thread-per-row SpMV)
    DevBuf run_items;    // spmv_short: warp items over shifted runs (spmv_run_kernel); empty: spmv_row_kernel
    int n_run_items = 0;
    // fused x exchange (sharded simple SpMV): remote column runs and per-work flags
    bool peer_ok = false;
    std::vector<int32_t> remote_runs;  // [c0, c1) pairs of columns outside the shard's rows
    DevBuf remote_block, remote_item, remote_long, peer_pieces, peer_src, peer_ctr;
    std::vector<int64_t> peer_sig;     // peer table the pieces were built for
    int n_peer_pieces = 0;
    unsigned long long peer_done = 0;  // pieces landed so far (device counter mirror)
    std::string why_general;
    DevBuf ro, col, val;
    DevBuf rsp, sst, slen, svec, chunk_row, item_seg, long_list, ticket, armed;
    DevBuf groups;      // SpMV row groups {r0, g} (segmented plans)
    int n_groups = 0;
    // column-split SpMV (kernels.hpp SplitPassDev): two CSRs by column half,
    // their chunks and long rows, and the rows' dot_unit state between passes
    int split = 0;  // column-split passes (0: none)
    DevBuf sp_j0[kMaxSplitPasses], sp_ro[kMaxSplitPasses], sp_col[kMaxSplitPasses], sp_val[kMaxSplitPasses],
        sp_items[kMaxSplitPasses], sp_long[kMaxSplitPasses], sp_state;
    int sp_n_items[kMaxSplitPasses] = {}, sp_n_long[kMaxSplitPasses] = {};
    // fast mode (simple SpMV, spmv_fast.cu): flagged entry streams, one per
    // column range of x (one range unless x outgrows the L2)
    int fast_passes = 0;  // 0: fast mode not in use
    int32_t fp_c0[kMaxSplitPasses + 1] = {};  // column ranges of the passes
    DevBuf fl_colf[kMaxSplitPasses], fl_val[kMaxSplitPasses], fl_m0[kMaxSplitPasses], fp_carry_val, fp_carry_row;
    int64_t fl_n_ent[kMaxSplitPasses] = {};
    int fl_n_chunks[kMaxSplitPasses] = {};
    int fl_per = 4;  // entries per lane (PSC_FAST_PER: 4 or 8)
    // the last pass's stream cut into row slices at chunks that start a row
    // (no carry crosses a cut), so the host path sends each slice's y down
    // while the next slice runs
    static constexpr int kFastSlices = 8;
    int32_t fsl_chunk[kFastSlices + 1] = {}, fsl_row[kFastSlices + 1] = {};
    bool chain_mode = false;
    int max_block_units = 0;
    DevBuf block_row, block_unit, unit_start;
    int32_t epoch = 0;      // per-launch arming epoch of the solve kernel
    DevBuf trace;           // PSC_TRSV_TRACE=1: per-row publish times (diagnostics)
    int trsv_threads = 256; // CTA size of the solve kernel (PSC_TRSV_THREADS)
    int trsv_lean = 0;      // solve kernel: 2 records (sptrsv_rec_kernel), 4 global queue (streaming / unit queue)
    DevBuf rec;             // trsv_lean == 2: per-row records (trsv_pack_kernel)
    DevBuf q_units, q_ends, q_next;  // trsv_lean == 4: global unit queue (chain starts / ends)
    int n_q_units = 0;
    int q_backoff = 200;  // ns a queue warp sleeps between polls of a missing operand (PSC_TRSV_BACKOFF)
    DevBuf s_pieces, s_w0;  // trsv_lean == 4, chain mode: <= 32-row pieces of the chain units (streaming kernel),
                            // and each piece's window start (its chain's previous piece)
    int n_s_pieces = 0;   // 0: the warp-per-row queue kernel
    int stream_k = 8;     // entries a lane consumes per round
    DevBuf unit_len, unit_loc, row_block, row_loc;  // trsv_lean == 2: unit tables, row -> (block, window slot)
    DevBuf halo_ptr, halo_col, halo_key, halo_pos;  // trsv_lean == 2: per block, the x entries it reads from earlier blocks
    int max_block_halo = -1;
    bool tiled = false;     // blocks grown over the unit graph (not row ranges)
    bool rec_dirty = true;  // values changed since the records were packed
    uint64_t values_version = 0;  // run_* cache: caller's tag of the values on the device (0: none)
    DevBuf hx, hy, hacc;    // scratch for the host-buffer entry points
    DevBuf naive_ticket;    // psc_csr_sptrsv_device
    // overlapped upload of b (host path, record kernel): copy stream, chunk flags
    cudaStream_t copy_stream = nullptr;
    cudaEvent_t ev_before = nullptr, ev_copied = nullptr;
    std::mutex host_mu;                  // the host-buffer entry points (host_call)
    cudaEvent_t ev_host_done = nullptr;  // end of the last host-buffer call's work
    cudaEvent_t ev_part[kMaxSplitPasses] = {};  // host path, column split: x range q landed
    static constexpr int kYSlices = 4;             // ... and the last pass in row slices, y of each sent down at once
    int32_t ysl_row[kYSlices + 1] = {}, ysl_item[kYSlices + 1] = {}, ysl_long[kYSlices + 1] = {};
    cudaEvent_t ev_slice[kYSlices > kFastSlices ? kYSlices : kFastSlices] = {};
    DevBuf b_ready, g_order;  // host path: per-unit arrival flags (+ gather ticket), gather order
    int n_units_total = 0;
    int* flag_patterns = nullptr;  // pinned, immutable: [i] = 0x01010101 * i (flags are written by the copy engine)
    ~psc_bound() {
        if (flag_patterns) cudaFreeHost(flag_patterns);
        if (copy_stream) cudaStreamDestroy(copy_stream);
        if (ev_before) cudaEventDestroy(ev_before);
        if (ev_copied) cudaEventDestroy(ev_copied);
        if (ev_host_done) cudaEventDestroy(ev_host_done);
        for (cudaEvent_t e : ev_part)
            if (e) cudaEventDestroy(e);
        for (cudaEvent_t e : ev_slice)
            if (e) cudaEventDestroy(e);
    }
    // general path
    std::vector<int64_t> part_group_ptr;
    DevBuf g_cp, g_fp, g_kind, g_m, g_n, g_form, g_base, g_so, g_si, g_tab, g_tables, g_frow, g_fdiag, g_frhs;
    // hash of the whole CSR structure (row offsets, columns, sizes): the run_* cache key check
    uint64_t structure = 0;
    uint64_t last_use = 0;  // run_* cache LRU clock

    int32_t rows() const { return row_end - row_begin; }
    SegmentsDev segs() const {
        if (simple) return {};
        return {rsp.as<int32_t>(), sst.as<int32_t>(), slen.as<int32_t>(), svec.as<int32_t>(), groups.as<int4>(), n_groups};
    }
    GeneralDev gen() const {
        return {g_cp.as<int64_t>(),  g_fp.as<int64_t>(),  g_kind.as<int32_t>(), g_m.as<int32_t>(),
                g_n.as<int32_t>(),   g_form.as<int32_t>(), g_base.as<int32_t>(), g_so.as<int32_t>(),
                g_si.as<int32_t>(),  g_tab.as<int64_t>(),  g_tables.as<int32_t>(), g_frow.as<int32_t>(),
                g_fdiag.as<int32_t>(), g_frhs.as<int32_t>()};
    }
    int64_t algorithmic_bytes() const {
        int64_t nnz = k_end - k_begin, r = rows();
        if (kernel == PSC_KERNEL_SPMV) return 12 * nnz + 4 * (r + 1) + 8LL * n_cols + 8 * r;
        return 12 * nnz + 4 * (r + 1) + 16 * r;
    }
    int64_t device_bytes() const {
        size_t t = 0;
        for (const DevBuf* b : {&ro, &col, &val, &rsp, &sst, &slen, &svec, &chunk_row, &item_seg, &long_list, &groups, &sp_ro[0], &sp_ro[1], &sp_ro[2], &sp_ro[3], &sp_col[0], &sp_col[1], &sp_col[2], &sp_col[3], &sp_val[0], &sp_val[1], &sp_val[2], &sp_val[3], &sp_j0[1], &sp_j0[2], &sp_j0[3], &sp_state, &ticket, &armed, &block_row, &block_unit, &unit_start, &rec, &q_units, &q_ends, &s_pieces, &s_w0, &g_order, &unit_len, &unit_loc, &row_block, &row_loc, &remote_block, &remote_item, &remote_long, &halo_ptr, &halo_col, &halo_key, &halo_pos, &g_cp, &g_fp,
                                &g_kind, &g_m, &g_n, &g_form, &g_base, &g_so, &g_si, &g_tab, &g_tables, &g_frow,
                                &g_fdiag, &g_frhs})
            t += b->bytes;
        t += fp_carry_val.bytes + fp_carry_row.bytes + run_items.bytes;
        for (int q = 0; q < kMaxSplitPasses; ++q)
            t += fl_colf[q].bytes + fl_val[q].bytes + fl_m0[q].bytes;
        return static_cast<int64_t>(t);
    }
};

struct psc_executor {
    int workers = 1;
    int device = 0;
    cudaStream_t stream = nullptr;
    std::mutex mu;
    // run_* cache: (plan serial, structure pointers, sizes, general flag) -> bound; a
    // hit also needs the same whole-structure hash; at most kCacheCap entries (LRU)
    std::map<std::tuple<uint64_t, const void*, const void*, int64_t, int32_t, int32_t, int>, std::unique_ptr<psc_bound>>
        cache;
    static constexpr size_t kCacheCap = 8;
    uint64_t clock = 0;
    DevBuf vx, vy, vb, vacc;
    // psc_executor_set_values_version: the caller's tag for the matrix values
    // the next run_* / execute_plan calls pass (0: unknown -- always upload)
    uint64_t values_version = 0;
};

namespace pscb {
namespace {

void use_device(int device) { ck(cudaSetDevice(device), "cudaSetDevice"); }

// Build a bound plan. force_general lowers through the exact interpreter
// (execute_plan semantics need accumulate-onto-existing for the solve).
// Column-split SpMV: two CSRs -- entries with column < n_cols / 2, then the
// rest (columns are sorted within a row, so each row splits at one point) --
// each chunked like the plan's rows (<= 256 entries and rows per chunk,
// longer rows alone). Values are bound once (psc_bind: the run_* API, which
// re-uploads values per call, does not split).
void build_split(psc_bound* b, const psc_csr_view& a, int parts, cudaStream_t s) {
    const int32_t n = a.n_rows;
    const int32_t* ro = a.row_offsets;
    // kb[q][r]: row r's first entry with column >= q * n_cols / parts (columns are sorted in a row)
    std::vector<std::vector<int32_t>> kb(static_cast<size_t>(parts) + 1, std::vector<int32_t>(n));
    for (int q = 0; q <= parts; ++q) {
        const int32_t c = static_cast<int32_t>(static_cast<int64_t>(a.n_cols) * q / parts);
        parallel_for((n + 65535) / 65536, hw_threads(0), [&](int64_t blk) {
            for (int32_t r = static_cast<int32_t>(blk * 65536); r < std::min<int64_t>(n, (blk + 1) * 65536); ++r)
                kb[q][r] = q == 0 ? ro[r] : q == parts ? ro[r + 1] :
                           static_cast<int32_t>(std::lower_bound(a.col_indices + ro[r], a.col_indices + ro[r + 1], c) -
                                                a.col_indices);
        });
    }
    for (int q = 0; q < parts; ++q) {
        std::vector<int32_t> pro(static_cast<size_t>(n) + 1, 0), j0(n);
        for (int32_t r = 0; r < n; ++r) {
            pro[r + 1] = pro[r] + (kb[q + 1][r] - kb[q][r]);
            j0[r] = kb[q][r] - ro[r];
        }
        const int64_t m = pro[n];
        std::vector<int32_t> pc(static_cast<size_t>(m));
        std::vector<double> pv(static_cast<size_t>(m));
        parallel_for((n + 65535) / 65536, hw_threads(0), [&](int64_t blk) {
            for (int32_t r = static_cast<int32_t>(blk * 65536); r < std::min<int64_t>(n, (blk + 1) * 65536); ++r) {
                std::copy(a.col_indices + kb[q][r], a.col_indices + kb[q + 1][r], pc.begin() + pro[r]);
                std::copy(a.values + kb[q][r], a.values + kb[q + 1][r], pv.begin() + pro[r]);
            }
        });
        std::vector<int32_t> items, longs;
        int32_t c0 = 0;
        auto close = [&](int32_t r1) {
            if (r1 > c0) items.insert(items.end(), {c0, r1, pro[c0], pro[r1]});
        };
        for (int32_t r = 0; r < n; ++r) {
            if (pro[r + 1] - pro[r] > kSpmvWarpCap) {
                close(r);
                longs.push_back(r);
                c0 = r + 1;
                continue;
            }
            if (pro[r + 1] - pro[c0] > kSpmvWarpCap || r + 1 - c0 > kSpmvWarpCap) {
                close(r);
                c0 = r;
            }
        }
        close(n);
        if (q == parts - 1) {  // row slices of the last pass, cut at item starts (host path: y goes down per slice)
            const int n_it = static_cast<int>(items.size() / 4);
            for (int i = 0; i <= psc_bound::kYSlices; ++i) {
                const int64_t t = static_cast<int64_t>(n) * i / psc_bound::kYSlices;
                int ia = 0;
                while (ia < n_it && items[4 * static_cast<size_t>(ia)] < t) ++ia;
                // slice 0 starts at row 0 (rows before the first chunk are long rows), the
                // last ends at n; the others start at a chunk's first row
                const int32_t cut = i == 0 ? 0 : i == psc_bound::kYSlices ? n : ia < n_it ? items[4 * static_cast<size_t>(ia)] : n;
                b->ysl_row[i] = cut;
                b->ysl_item[i] = i == 0 ? 0 : i == psc_bound::kYSlices ? n_it : ia;
                b->ysl_long[i] = static_cast<int>(std::lower_bound(longs.begin(), longs.end(), cut) - longs.begin());
            }
        }
        if (q > 0) b->sp_j0[q].upload(j0, s);
        b->sp_ro[q].upload(pro, s);
        b->sp_col[q].upload(pc, s);
        b->sp_val[q].upload(pv, s);
        b->sp_items[q].upload(items, s);
        b->sp_long[q].upload(longs, s);
        b->sp_n_items[q] = static_cast<int>(items.size() / 4);
        b->sp_n_long[q] = static_cast<int>(longs.size());
        ck(cudaStreamSynchronize(s), "split upload");  // the host staging vectors go out of scope
    }
    b->sp_state.ensure(static_cast<size_t>(n) * 4 * sizeof(double));
    b->split = parts;
}

// Fast mode over the bound rows (local CSR: ro[0..n] rebased, col/val from
// a.col_indices/values + k_begin): one pass over the whole CSR, or `parts`
// column ranges each stored as its own CSR (columns are sorted within a row,
// so a row splits at one point per range boundary).
void build_fast(psc_bound* b, const psc_csr_view& a, const std::vector<int32_t>& ro, int parts, cudaStream_t s) {
    const int32_t n = b->rows();
    const int32_t* col = a.col_indices + b->k_begin;
    const double* val = a.values + b->k_begin;
    if (const char* h = std::getenv("PSC_FAST_PER")) b->fl_per = std::atoi(h) == 8 ? 8 : 4;
    parts = std::max(1, parts);
    int64_t max_chunks = 0;
    std::vector<int32_t> lo(n), hi(n);
    for (int q = 0; q < parts; ++q) {
        const int32_t c0 = static_cast<int32_t>(static_cast<int64_t>(a.n_cols) * q / parts);
        const int32_t c1 = static_cast<int32_t>(static_cast<int64_t>(a.n_cols) * (q + 1) / parts);
        b->fp_c0[q] = c0;
        b->fp_c0[q + 1] = c1;
        // row r's entries in column range q: [lo[r], hi[r]) (columns are sorted in a row)
        parallel_for((n + 65535) / 65536, hw_threads(0), [&](int64_t blk) {
            const int32_t r1 = static_cast<int32_t>(std::min<int64_t>(n, (blk + 1) * 65536));
            for (int32_t r = static_cast<int32_t>(blk * 65536); r < r1; ++r) {
                const int32_t* rb = col + ro[r];
                const int32_t* re = col + ro[r + 1];
                lo[r] = q == 0 ? ro[r] : static_cast<int32_t>(std::lower_bound(rb, re, c0) - col);
                hi[r] = q == parts - 1 ? ro[r + 1] : static_cast<int32_t>(std::lower_bound(rb, re, c1) - col);
            }
        });
        {
            // entries in CSR order, bit 31 of the column on each row's last entry; a
            // row with no entries in this pass gets one placeholder (column
            // 0x7fffffff, value 0) so that row end m is row m; per chunk, the row
            // ends before it; padded to whole chunks (lanes load 16-byte vectors)
            const int64_t ch = flag_chunk_entries(b->fl_per);
            std::vector<int64_t> fo(static_cast<size_t>(n) + 1, 0);
            for (int32_t r = 0; r < n; ++r) fo[r + 1] = fo[r] + std::max(1, hi[r] - lo[r]);
            const int64_t mf = fo[n];
            const size_t m_pad = static_cast<size_t>((mf + ch - 1) / ch * ch);
            std::vector<int32_t> colf(m_pad, 0);
            std::vector<double> pv(m_pad, 0.0);
            parallel_for((n + 65535) / 65536, hw_threads(0), [&](int64_t blk) {
                const int32_t r1 = static_cast<int32_t>(std::min<int64_t>(n, (blk + 1) * 65536));
                for (int32_t r = static_cast<int32_t>(blk * 65536); r < r1; ++r) {
                    if (hi[r] > lo[r]) {
                        std::copy(col + lo[r], col + hi[r], colf.begin() + fo[r]);
                        std::copy(val + lo[r], val + hi[r], pv.begin() + fo[r]);
                    } else {
                        colf[fo[r]] = 0x7fffffff;
                    }
                    colf[fo[r + 1] - 1] |= static_cast<int32_t>(0x80000000u);
                }
            });
            const int64_t n_chunks = (mf + ch - 1) / ch;
            require(n_chunks < INT32_MAX && mf < INT32_MAX, "bind: too many fast-mode entries");
            std::vector<int32_t> m0(static_cast<size_t>(std::max<int64_t>(1, n_chunks)));
            {   // row ends before chunk c = the number of rows ending before entry c * ch
                int32_t r = 0;
                for (int64_t c = 0; c < n_chunks; ++c) {
                    while (r < n && fo[r + 1] <= c * ch) ++r;
                    m0[c] = r;
                }
            }
            if (q == parts - 1) {  // y slices: cut at chunks whose first entry starts a row
                int64_t cut = 0;
                b->fsl_chunk[0] = 0;
                b->fsl_row[0] = 0;
                for (int i = 1; i < psc_bound::kFastSlices; ++i) {
                    cut = std::max<int64_t>(cut, n_chunks * i / psc_bound::kFastSlices);
                    while (cut < n_chunks && fo[m0[cut]] != cut * ch) ++cut;
                    b->fsl_chunk[i] = static_cast<int32_t>(cut);
                    b->fsl_row[i] = cut < n_chunks ? m0[cut] : n;
                }
                b->fsl_chunk[psc_bound::kFastSlices] = static_cast<int32_t>(n_chunks);
                b->fsl_row[psc_bound::kFastSlices] = n;
            }
            b->fl_colf[q].upload(colf, s);
            b->fl_val[q].upload(pv, s);
            b->fl_m0[q].upload(m0, s);
            b->fl_n_ent[q] = mf;
            b->fl_n_chunks[q] = static_cast<int>(n_chunks);
            max_chunks = std::max<int64_t>(max_chunks, n_chunks);
        }
        ck(cudaStreamSynchronize(s), "fast upload");  // the staging vectors go out of scope
    }
    b->fp_carry_val.ensure(static_cast<size_t>(std::max<int64_t>(1, max_chunks)) * sizeof(double));
    b->fp_carry_row.ensure(static_cast<size_t>(std::max<int64_t>(1, max_chunks)) * sizeof(int32_t));
    b->fast_passes = parts;
}

FlagPassDev flag_pass(const psc_bound* b, int q) {
    FlagPassDev P;
    P.colf = b->fl_colf[q].as<int32_t>();
    P.val = b->fl_val[q].as<double>();
    P.chunk_m0 = b->fl_m0[q].as<int32_t>();
    P.n_ent = b->fl_n_ent[q];
    P.n_chunks = b->fl_n_chunks[q];
    P.per = b->fl_per;
    P.carry_val = b->fp_carry_val.as<double>();
    P.carry_row = b->fp_carry_row.as<int32_t>();
    return P;
}

// pass q of a fast multiply
void fast_pass_launch(const psc_bound* b, int q, const double* x, double* y, cudaStream_t s) {
    launch_spmv_flag(flag_pass(b, q), x, y, q > 0, b->n_sms, s);
}

std::unique_ptr<psc_bound> make_bound(int device, const Plan& p, const psc_csr_view& a, int mode, int64_t p0,
                                      int64_t p1, bool force_general, cudaStream_t s, bool allow_split = false) {
    if (p.kernel == PSC_KERNEL_SPTRSV) adopt_triangular(a);
    else validate_csr(a);
    // A mined plan's tables are its matrix's columns: bind it only to that
    // matrix (the structure hash its inspection recorded), or -- provenance
    // unknown (a version-1 plan file) -- after validate_plan (miner.cpp:325-395).
    if (p.mined && p.structure != 0) {
        if (structure_hash(a) != p.structure)
            throw std::logic_error("bind: the plan was inspected from a matrix with a different structure");
    } else if (p.mined) {
        validate_plan(p, a);
    }
    Lowered L = lower_plan(p, a, p0, p1, 0, force_general);
    auto b = std::make_unique<psc_bound>();
    b->device = device;
    b->kernel = p.kernel;
    b->mode = mode;
    b->row_begin = L.row_begin;
    b->row_end = L.row_end;
    b->n_rows_total = a.n_rows;
    b->n_cols = a.n_cols;
    b->k_begin = L.k_begin;
    b->k_end = L.k_end;
    b->canonical = L.canonical;
    b->simple = L.simple;
    b->why_general = L.why_general;
    use_device(device);
    if (L.canonical) {
        const int32_t nr = b->rows();
        std::vector<int32_t> ro(static_cast<size_t>(nr) + 1);
        for (int32_t r = 0; r <= nr; ++r) ro[r] = static_cast<int32_t>(a.row_offsets[r + L.row_begin] - L.k_begin);
        b->ro.upload(ro, s);
        b->col.upload_raw(a.col_indices + L.k_begin, (L.k_end - L.k_begin) * sizeof(int32_t), s);
        b->val.upload_raw(a.values + L.k_begin, (L.k_end - L.k_begin) * sizeof(double), s);
        if (!L.simple) {
            b->rsp.upload(L.row_seg_ptr, s);
            b->sst.upload(L.seg_start, s);
            b->slen.upload(L.seg_len, s);
            b->svec.upload(L.seg_vec, s);
            b->n_segments = static_cast<int64_t>(L.seg_start.size());
        }
        if (p.kernel == PSC_KERNEL_SPMV) {
            b->chunk_row.upload(L.items, s);  // warp chunks {r0, r1, k0, k1}
            b->item_seg.upload(L.item_seg, s);
            b->long_list.upload(L.long_row_list, s);
            b->n_chunks = static_cast<int>(L.items.size() / 4);
            b->groups.upload(L.groups, s);
            b->n_groups = static_cast<int>(L.groups.size() / 8);
            // x of at least PSC_SPMV_SPLIT_BYTES (default: about an L2) -> column-split passes
            // (a negative threshold disables them)
            if (mode == PSC_MODE_FAST && L.simple) {
                // fast mode: merge-path tiles; column ranges of <= PSC_FAST_SPLIT_BYTES
                // of x each once x outgrows the L2 (a negative value: never split)
                const char* v = std::getenv("PSC_FAST_SPLIT_BYTES");
                // (config 5, x = 160 MB: 2 / 3 / 4 ranges 2.27 / 2.05 / 2.31 ms; one range 4.9 ms)
                const int64_t part_bytes = v ? std::atoll(v) : 55000000LL;
                const int64_t xb = static_cast<int64_t>(a.n_cols) * 8;
                // (by default only once x outgrows ~100 MB of the L2; a set PSC_FAST_SPLIT_BYTES always applies)
                int parts = part_bytes > 0 && (v || xb > 100000000LL) ? static_cast<int>((xb + part_bytes - 1) / part_bytes) : 1;
                parts = std::max(1, std::min(kMaxSplitPasses, parts));
                // one pass over rows of <= 16 entries: the thread-per-row kernel below is
                // faster (one launch, no carries; config 1: 20.7 vs 23.6 us) and exact anyway
                int32_t mx = 0;
                for (int32_t r = L.row_begin; r < L.row_end && mx <= 16; ++r)
                    mx = std::max(mx, static_cast<int32_t>(a.row_offsets[r + 1] - a.row_offsets[r]));
                if (parts > 1 || mx > 16 || v) build_fast(b.get(), a, ro, parts, s);
            } else if (allow_split && L.simple && L.row_begin == 0 && L.row_end == a.n_rows) {
                const char* v = std::getenv("PSC_SPMV_SPLIT_BYTES");
                const int64_t min_bytes = v ? std::atoll(v) : 128000000LL;
                if (min_bytes >= 0 && static_cast<int64_t>(a.n_cols) * 8 >= min_bytes) {
                    // parts of x of at most ~60 MB each (config 5, x = 160 MB: 2 / 3 / 4 parts:
                    // 3.54 / 3.45 / 3.63 ms, unsplit 4.67 ms), 2..4 passes
                    const char* pv = std::getenv("PSC_SPMV_SPLIT_PARTS");
                    int parts = pv ? std::atoi(pv)
                                   : static_cast<int>((static_cast<int64_t>(a.n_cols) * 8 + 59999999) / 60000000);
                    parts = std::max(2, std::min(kMaxSplitPasses, parts));
                    build_split(b.get(), a, parts, s);
                }
            }
            b->long_rows = L.long_rows;
            // every row of a simple plan <= 16 entries: thread-per-row kernel (PSC_SPMV_ROWK=0 disables)
            if (L.simple && L.long_rows == 0) {
                int32_t mx = 0;
                for (int32_t r = L.row_begin; r < L.row_end; ++r)
                    mx = std::max(mx, static_cast<int32_t>(a.row_offsets[r + 1] - a.row_offsets[r]));
                b->spmv_short = mx <= 16 ? std::max<int32_t>(mx, 1) : 0;
                if (const char* rk = std::getenv("PSC_SPMV_ROWK"); rk && rk[0] == '0') b->spmv_short = 0;
                // shifted runs (stencil interiors): rows without row offsets or column loads, when
                // they cover most of the matrix (PSC_SPMV_RUNS=0 disables)
                const char* rv = std::getenv("PSC_SPMV_RUNS");
                if (b->spmv_short > 0 && !(rv && rv[0] == '0')) {
                    std::vector<int32_t> items;
                    const int64_t in_runs = build_run_items(L, a, items);
                    if (2 * in_runs >= static_cast<int64_t>(L.row_end - L.row_begin) && !items.empty()) {
                        b->run_items.upload(items, s);
                        b->n_run_items = static_cast<int>(items.size() / 20);
                    }
                }
            }
            // a shard of a simple plan: the columns it reads outside its own rows
            // (whose x other ranks own), for the fused exchange
            if (L.simple && (L.row_begin > 0 || L.row_end < a.n_rows) && a.n_cols == a.n_rows) {
                std::vector<uint8_t> used(static_cast<size_t>(a.n_cols), 0);
                auto remote = [&](int32_t c) { return c < L.row_begin || c >= L.row_end; };
                auto row_remote = [&](int32_t r) {  // local row r
                    bool any = false;
                    for (int64_t k = a.row_offsets[r + L.row_begin]; k < a.row_offsets[r + L.row_begin + 1]; ++k) {
                        const int32_t c = a.col_indices[k];
                        if (remote(c)) {
                            used[c] = 1;
                            any = true;
                        }
                    }
                    return any;
                };
                const int32_t nr = b->rows();
                std::vector<uint8_t> rrow(nr);
                for (int32_t r = 0; r < nr; ++r) rrow[r] = row_remote(r);
                std::vector<uint8_t> fb((nr + 255) / 256, 0), fi(L.items.size() / 4, 0), fl(L.long_row_list.size(), 0);
                for (int32_t r = 0; r < nr; ++r) fb[r / 256] |= rrow[r];
                for (size_t i = 0; i < fi.size(); ++i)
                    for (int32_t r = L.items[4 * i]; r < L.items[4 * i + 1]; ++r) fi[i] |= rrow[r];
                for (size_t i = 0; i < fl.size(); ++i) fl[i] = rrow[L.long_row_list[i]];
                b->remote_block.upload(fb, s);
                b->remote_item.upload(fi, s);
                b->remote_long.upload(fl, s);
                for (int32_t c = 0; c < a.n_cols;) {  // runs of used columns, gaps < 32 merged
                    if (!used[c]) {
                        ++c;
                        continue;
                    }
                    int32_t e = c + 1, last = c;
                    while (e < a.n_cols && e - last <= 32) {
                        if (used[e]) last = e;
                        ++e;
                    }
                    b->remote_runs.push_back(c);
                    b->remote_runs.push_back(last + 1);
                    c = last + 1;
                }
                b->peer_ok = true;
            }
            cudaDeviceGetAttribute(&b->n_sms, cudaDevAttrMultiProcessorCount, device);
        } else {
            // Solve kernel: the record kernel (sptrsv_rec_kernel) for simple rows
            // with <= 4 off-diagonal entries whose block window (rows + halo) fits
            // in shared memory -- in chain mode over tiled blocks
            // (tile_chain_blocks); every other canonical plan goes to a global
            // queue: the streaming kernel (chain mode, lane per row) or the unit
            // queue (row mode). PSC_TRSV_LEAN=4 forces the queue.
            int32_t max_ext = 0;
            for (int32_t r = L.row_begin; r < L.row_end; ++r)
                max_ext = std::max(max_ext, a.row_offsets[r + 1] - a.row_offsets[r] - 1);
            bool want_rec = L.simple && max_ext <= 4;
            if (const char* ln = std::getenv("PSC_TRSV_LEAN")) want_rec = want_rec && std::atoi(ln) != 4;
            auto pick_threads = [&](const Lowered& M, int max_halo) {
                int th = 256;
                if (M.chain_mode) {  // enough lanes for the units of a block
                    th = 64;
                    while (th < 512 && th < M.max_block_units) th *= 2;
                }
                if (const char* env = std::getenv("PSC_TRSV_THREADS")) th = std::atoi(env);
                int p2 = 64;  // the solve kernels are instantiated for 64, 128, 256 and 512 threads
                while (p2 < 512 && p2 < th) p2 *= 2;
                th = p2;
                while (th > 64 && sptrsv_smem_bytes(th, M.max_block_rows, M.max_block_units, max_halo) > 232448) th /= 2;
                return sptrsv_smem_bytes(th, M.max_block_rows, M.max_block_units, max_halo) <= 232448 ? th : -1;
            };
            auto recs_fit = [&](Lowered& M) {  // window indices fit int16 and the window fits
                block_halos(M, a);
                return M.max_block_rows + M.max_block_halo <= 32767 && pick_threads(M, M.max_block_halo) > 0;
            };
            b->trsv_lean = 4;
            if (want_rec) {
                bool tiles = L.chain_mode;
                if (const char* tv = std::getenv("PSC_TRSV_TILES")) tiles = tiles && tv[0] != '0';
                if (tiles) {
                    Lowered T = L;
                    if (tile_chain_blocks(T, a, L.max_block_rows) && recs_fit(T)) {
                        L = std::move(T);
                        b->trsv_lean = 2;
                    }
                }
                if (b->trsv_lean != 2) {
                    Lowered C = L;
                    unit_maps(C);
                    if (recs_fit(C)) {
                        L = std::move(C);
                        b->trsv_lean = 2;
                    }
                }
            }
            if (b->trsv_lean == 4) {
                // units over the whole matrix: chains in row order (chain mode) or
                // single rows by dependency level (row mode); both topological
                const int32_t nr = L.row_end - L.row_begin;
                std::vector<int32_t> lvl(nr, 0);  // dependency level of every row
                for (int32_t r = 0; r < nr; ++r) {
                    int32_t m = -1;
                    for (int32_t k = a.row_offsets[r + L.row_begin]; k < a.row_offsets[r + L.row_begin + 1] - 1; ++k)
                        m = std::max(m, lvl[a.col_indices[k] - L.row_begin]);
                    lvl[r] = m + 1;
                }
                std::vector<int32_t> units;
                if (L.chain_mode) {
                    // chain starts in row order: contiguous chains cannot interleave, so a
                    // chain depends only on chains that start before it -- the claim order
                    // is topological (ordering by the first row's level would not be, and
                    // could exhaust the resident warps on units waiting for unclaimed ones)
                    for (int32_t r = 0; r < nr; ++r) {
                        const int32_t gr = r + L.row_begin;
                        const int32_t k0 = a.row_offsets[gr], kd = a.row_offsets[gr + 1] - 1;
                        const bool cont = r > 0 && kd > k0 && a.col_indices[kd - 1] == gr - 1;
                        if (!cont) units.push_back(r);
                    }
                    std::vector<int32_t> en(units.size());
                    for (size_t i = 0; i < units.size(); ++i) en[i] = i + 1 < units.size() ? units[i + 1] : nr;
                    b->q_ends.upload(en, s);
                    // streaming kernel (lane per row): the chains cut into pieces of <= 32 rows
                    const char* sv = std::getenv("PSC_TRSV_STREAM");
                    if (!(sv && sv[0] == '0')) {
                        std::vector<int32_t> pieces, w0;
                        for (size_t i = 0; i < units.size(); ++i)
                            for (int32_t r = units[i]; r < en[i]; r += 32) {
                                pieces.push_back(r);
                                w0.push_back(r == units[i] ? r : r - 32);  // the previous piece of the chain
                            }
                        pieces.push_back(nr);
                        b->s_pieces.upload(pieces, s);
                        b->s_w0.upload(w0, s);
                        b->n_s_pieces = static_cast<int>(pieces.size()) - 1;
                    }
                } else {
                    units.resize(nr);
                    for (int32_t r = 0; r < nr; ++r) units[r] = r;
                    std::stable_sort(units.begin(), units.end(), [&](int32_t p, int32_t q) { return lvl[p] < lvl[q]; });
                }
                units.push_back(nr);
                b->q_units.upload(units, s);
                b->n_q_units = static_cast<int>(units.size()) - 1;
                b->q_next.ensure(sizeof(int));
                if (const char* bo = std::getenv("PSC_TRSV_BACKOFF")) b->q_backoff = std::max(0, std::atoi(bo));
                cudaDeviceGetAttribute(&b->n_sms, cudaDevAttrMultiProcessorCount, device);
            }
            b->n_blocks = static_cast<int>(L.block_row.size()) - 1;
            b->chain_mode = L.chain_mode;
            b->tiled = L.tiled;
            b->block_row.upload(L.block_row, s);
            b->block_unit.upload(L.block_unit, s);
            b->unit_start.upload(L.unit_start, s);
            b->max_block_units = L.max_block_units;
            b->max_block_halo = -1;
            if (b->trsv_lean == 2) {
                {   // host path: the order the solve needs b, unit by unit (first rows' dependency levels)
                    const int32_t nr = b->rows();
                    std::vector<int32_t> lvl(nr, 0);
                    for (int32_t r = 0; r < nr; ++r) {
                        int32_t m = -1;
                        for (int32_t k = a.row_offsets[r + L.row_begin]; k < a.row_offsets[r + L.row_begin + 1] - 1; ++k)
                            m = std::max(m, lvl[a.col_indices[k] - L.row_begin]);
                        lvl[r] = m + 1;
                    }
                    std::vector<int32_t> order(L.unit_start.size());
                    for (size_t i = 0; i < order.size(); ++i) order[i] = static_cast<int32_t>(i);
                    std::stable_sort(order.begin(), order.end(), [&](int32_t p1, int32_t p2) {
                        return lvl[L.unit_start[p1]] < lvl[L.unit_start[p2]];
                    });
                    b->g_order.upload(order, s);
                    b->n_units_total = static_cast<int>(order.size());
                }
                b->unit_len.upload(L.unit_len, s);
                b->unit_loc.upload(L.unit_loc, s);
                b->row_block.upload(L.row_block, s);
                b->row_loc.upload(L.row_loc, s);
                b->halo_ptr.upload(L.halo_ptr, s);
                b->halo_col.upload(L.halo_col, s);
                b->halo_key.upload(L.halo_key, s);
                b->halo_pos.upload(L.halo_pos, s);
                b->max_block_halo = L.max_block_halo;
                b->rec.ensure(static_cast<size_t>(b->rows()) * trsv_rec_bytes());
            }
            if (b->trsv_lean == 2) {
                const int th = pick_threads(L, b->max_block_halo);
                require(th > 0, "bind: solve block does not fit in shared memory");
                b->trsv_threads = th;
            }
            b->max_block_rows = L.max_block_rows;
            b->ticket.ensure(2 * sizeof(int32_t));
            ck(cudaMemsetAsync(b->ticket.p, 0, 2 * sizeof(int32_t), s), "memset");
            if (const char* tr = std::getenv("PSC_TRSV_TRACE"); tr && tr[0] == '1') {
                const size_t nt = static_cast<size_t>(b->rows()) + b->n_blocks + 16;
                b->trace.ensure(nt * sizeof(unsigned long long));
                ck(cudaMemsetAsync(b->trace.p, 0, nt * sizeof(unsigned long long), s), "memset");
            }
            b->armed.ensure(std::max(1, b->n_blocks) * sizeof(int32_t));
            ck(cudaMemsetAsync(b->armed.p, 0, std::max(1, b->n_blocks) * sizeof(int32_t), s), "memset");
        }
    } else {
        // general interpreter: full CSR values, descriptors and tables
        b->val.upload_raw(a.values, a.nnz * sizeof(double), s);
        auto& G = L.gen;
        b->part_group_ptr = G.part_group_ptr;
        b->g_cp.upload(G.group_codelet_ptr, s);
        b->g_fp.upload(G.group_fin_ptr, s);
        b->g_kind.upload(G.c_kind, s);
        b->g_m.upload(G.c_m, s);
        b->g_n.upload(G.c_n, s);
        b->g_form.upload(G.d_form, s);
        b->g_base.upload(G.d_base, s);
        b->g_so.upload(G.d_so, s);
        b->g_si.upload(G.d_si, s);
        b->g_tab.upload(G.d_tab, s);
        b->g_tables.upload(G.tables, s);
        b->g_frow.upload(G.f_row, s);
        b->g_fdiag.upload(G.f_diag, s);
        b->g_frhs.upload(G.f_rhs, s);
    }
    ck(cudaStreamSynchronize(s), "bind sync");
    return b;
}

void run_general(psc_bound* b, const double* gather, double* accum, const double* rhs, double* solution,
                 cudaStream_t s) {
    GeneralDev g = b->gen();
    for (size_t p = 0; p + 1 < b->part_group_ptr.size(); ++p) {
        launch_general_partition(g, b->part_group_ptr[p], b->part_group_ptr[p + 1], b->val.as<double>(), gather, accum,
                                 rhs, solution, s);
    }
    ck(cudaGetLastError(), "general kernel launch");
}

void split_passes(const psc_bound* b, SplitPassDev (&P)[kMaxSplitPasses]) {
    for (int q = 0; q < b->split; ++q) {
        P[q].j0 = q > 0 ? b->sp_j0[q].as<int32_t>() : nullptr;
        P[q].ro_pass = b->sp_ro[q].as<int32_t>();
        P[q].col = b->sp_col[q].as<int32_t>();
        P[q].val = b->sp_val[q].as<double>();
        P[q].items = b->sp_items[q].as<int4>();
        P[q].n_items = b->sp_n_items[q];
        P[q].long_rows = b->sp_long[q].as<int32_t>();
        P[q].n_long = b->sp_n_long[q];
    }
}

void bound_spmv(psc_bound* b, const double* x, double* y, cudaStream_t s) {
    use_device(b->device);
    if (b->canonical && b->fast_passes) {
        for (int q = 0; q < b->fast_passes; ++q) fast_pass_launch(b, q, x, y, s);
    } else if (b->canonical && b->split) {
        SplitPassDev P[kMaxSplitPasses];
        split_passes(b, P);
        launch_spmv_split(b->ro.as<int32_t>(), P, b->split, b->sp_state.as<double>(), x, y, false, b->n_sms, s);
    } else if (b->canonical) {
        launch_spmv_parity(b->ro.as<int32_t>(), b->col.as<int32_t>(), b->val.as<double>(), x, y,
                           b->chunk_row.as<int4>(), b->n_chunks, b->item_seg.as<int2>(), b->long_list.as<int32_t>(),
                           static_cast<int>(b->long_rows), b->segs(), false, b->n_sms, b->spmv_short, b->rows(), s,
                           nullptr, b->run_items.as<int4>(), b->n_run_items);
    } else {
        ck(cudaMemsetAsync(y, 0, static_cast<size_t>(b->rows()) * sizeof(double), s), "memset y");
        run_general(b, x, y, nullptr, nullptr, s);
    }
    ck(cudaGetLastError(), "spmv launch");
}

void bound_sptrsv(psc_bound* b, const double* rhs, double* x, double* acc, cudaStream_t s, double* x_host = nullptr,
                  const int* b_ready = nullptr, int b_shift = 0, int b_flag = 0) {
    use_device(b->device);
    if (b->canonical && b->trsv_lean == 4 && b->n_s_pieces > 0) {
        launch_sptrsv_stream(b->ro.as<int32_t>(), b->col.as<int32_t>(), b->val.as<double>(), rhs, x, acc,
                             b->s_pieces.as<int32_t>(), b->s_w0.as<int32_t>(), b->n_s_pieces, b->segs(), b->q_next.as<int>(),
                             b->trace.as<unsigned long long>(), b->rows(), b->n_sms, b->stream_k, s);
    } else if (b->canonical && b->trsv_lean == 4) {
        launch_sptrsv_queue(b->ro.as<int32_t>(), b->col.as<int32_t>(), b->val.as<double>(), rhs, x, acc,
                            b->q_units.as<int32_t>(), b->chain_mode ? b->q_ends.as<int32_t>() : nullptr, b->n_q_units,
                            !b->chain_mode, b->segs(), b->q_next.as<int>(),
                            b->trace.as<unsigned long long>(), b->rows(), b->n_sms, b->q_backoff, s);
    } else if (b->canonical) {
        if (b->trsv_lean == 2 && b->rec_dirty) {
            launch_trsv_pack(b->ro.as<int32_t>(), b->col.as<int32_t>(), b->val.as<double>(), b->row_block.as<int32_t>(),
                             b->row_loc.as<int32_t>(), b->block_row.as<int32_t>(), b->halo_ptr.as<int32_t>(),
                             b->halo_key.as<int32_t>(), b->halo_pos.as<int32_t>(), b->rows(), b->rec.p, s);
            b->rec_dirty = false;
        }
        b->epoch = b->epoch == INT32_MAX ? 1 : b->epoch + 1;
        launch_sptrsv(b->ro.as<int32_t>(), b->col.as<int32_t>(), b->val.as<double>(), rhs, x, acc,
                      b->block_row.as<int32_t>(), b->block_unit.as<int32_t>(), b->unit_start.as<int32_t>(), b->n_blocks,
                      b->max_block_rows, b->max_block_units, !b->chain_mode, b->segs(), b->ticket.as<int32_t>(),
                      b->armed.as<int32_t>(), b->epoch, b->trace.as<unsigned long long>(), b->trsv_threads,
                      b->rec.p, b->unit_len.as<int32_t>(),
                      b->unit_loc.as<int32_t>(), b->halo_ptr.as<int32_t>(), b->halo_col.as<int32_t>(), b->max_block_halo,
                      x_host, b_ready, b_shift, b_flag, s);
    } else {
        require(acc != nullptr, "sptrsv: the general path needs an acc buffer");
        ck(cudaMemsetAsync(acc, 0, static_cast<size_t>(b->rows()) * sizeof(double), s), "memset acc");
        run_general(b, x, acc, rhs, x, s);
    }
    ck(cudaGetLastError(), "sptrsv launch");
}

psc_bound* cached_bound(psc_executor* e, const psc_plan* plan, const psc_csr_view& a, bool general) {
    auto key = std::make_tuple(plan->serial, static_cast<const void*>(a.row_offsets),
                               static_cast<const void*>(a.col_indices), a.nnz, a.n_rows, a.n_cols, general ? 1 : 0);
    const uint64_t h = structure_hash(a);
    auto it = e->cache.find(key);
    if (it != e->cache.end() && it->second->structure == h) {
        it->second->last_use = ++e->clock;
        return it->second.get();
    }
    if (it != e->cache.end()) e->cache.erase(it);  // the structure changed in place: rebind
    while (e->cache.size() >= psc_executor::kCacheCap) {  // evict the least recently used binding
        auto lru = e->cache.begin();
        for (auto jt = e->cache.begin(); jt != e->cache.end(); ++jt)
            if (jt->second->last_use < lru->second->last_use) lru = jt;
        e->cache.erase(lru);
    }
    auto b = make_bound(e->device, plan->p, a, PSC_MODE_PARITY, -1, -1, general, e->stream);
    b->structure = h;
    b->last_use = ++e->clock;
    psc_bound* raw = b.get();
    e->cache[key] = std::move(b);
    return raw;
}

}  // namespace
}  // namespace pscb

extern "C" {

PSC_API psc_status psc_selftest_division(uint64_t seed, int64_t n, int32_t exp_span, int64_t* mismatches) {
    return guarded([&] {
        require(mismatches != nullptr && n >= 0 && exp_span >= 1 && exp_span <= 1000, "selftest_division: bad argument");
        const int64_t m = division_selftest(seed, n, exp_span);
        require(m >= 0, "selftest_division: CUDA error");
        *mismatches = m;
    });
}

PSC_API int32_t psc_device_count(void) {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    return n;
}

PSC_API psc_status psc_executor_create(int32_t workers, int32_t device, psc_executor** out) {
    return guarded([&] {
        require(out != nullptr, "Executor: null output");
        if (workers < 1) throw std::invalid_argument("Executor: worker count must be >= 1");
        int n = psc_device_count();
        if (n <= 0) throw CudaError("Executor: no CUDA device is available");
        require(device >= 0 && device < n, "Executor: device index out of range");
        auto e = std::make_unique<psc_executor>();
        e->workers = workers;
        e->device = device;
        use_device(device);
        ck(cudaStreamCreateWithFlags(&e->stream, cudaStreamNonBlocking), "cudaStreamCreate");
        *out = e.release();
    });
}
PSC_API int32_t psc_executor_workers(const psc_executor* e) { return e ? e->workers : 0; }
PSC_API void psc_executor_destroy(psc_executor* e) {
    if (!e) return;
    cudaSetDevice(e->device);
    e->cache.clear();
    if (e->stream) cudaStreamDestroy(e->stream);
    delete e;
}

PSC_API psc_status psc_bind(psc_executor* e, const psc_plan* plan, const psc_csr_view* a, int32_t mode,
                            psc_bound** out) {
    return guarded([&] {
        require(e && plan && a && out, "bind: null argument");
        require(mode == PSC_MODE_PARITY || mode == PSC_MODE_FAST, "bind: unknown mode");
        std::lock_guard<std::mutex> lk(e->mu);
        *out = make_bound(e->device, plan->p, *a, mode, -1, -1, false, e->stream, true).release();
    });
}
PSC_API psc_status psc_bind_partitions(psc_executor* e, const psc_plan* plan, const psc_csr_view* a, int32_t mode,
                                       int64_t part_begin, int64_t part_end, psc_bound** out) {
    return guarded([&] {
        require(e && plan && a && out, "bind_partitions: null argument");
        require(part_end >= 0, "bind_partitions: part_end must be >= 0");
        std::lock_guard<std::mutex> lk(e->mu);
        *out = make_bound(e->device, plan->p, *a, mode, part_begin, part_end, false, e->stream).release();
    });
}
PSC_API psc_status psc_bound_rows(const psc_bound* b, int32_t* row_begin, int32_t* row_end) {
    return guarded([&] {
        require(b != nullptr, "bound: null");
        if (row_begin) *row_begin = b->row_begin;
        if (row_end) *row_end = b->row_end;
    });
}
PSC_API void psc_bound_destroy(psc_bound* b) {
    if (!b) return;
    cudaSetDevice(b->device);
    delete b;
}
PSC_API psc_status psc_bound_x_runs(const psc_bound* b, int32_t* runs, int64_t cap, int64_t* n_runs) {
    return guarded([&] {
        require(b && n_runs, "x_runs: null argument");
        require(b->kernel == PSC_KERNEL_SPMV, "x_runs: not an SpMV binding");
        require(b->peer_ok, "x_runs: not a shard of a simple plan (no fused exchange)");
        *n_runs = static_cast<int64_t>(b->remote_runs.size() / 2);
        if (runs) {
            require(cap >= *n_runs, "x_runs: buffer too small");
            std::copy(b->remote_runs.begin(), b->remote_runs.end(), runs);
        }
    });
}

// The fused exchange: see PeerDev (kernels.hpp) and DESIGN.md "Multi-GPU".
PSC_API psc_status psc_bound_spmv_peers(psc_bound* b, const psc_peer_window* peers, int32_t n_peers, double* x_window,
                                        double* y, void* stream) {
    return guarded([&] {
        require(b && peers && x_window && y && n_peers >= 1, "spmv_peers: null argument");
        require(b->kernel == PSC_KERNEL_SPMV, "spmv_peers: plan was built for another kernel");
        require(b->canonical && b->peer_ok, "spmv_peers: needs a shard of a simple (one segment per row) plan");
        int32_t expect = 0;
        for (int32_t q = 0; q < n_peers; ++q) {
            require(peers[q].row_begin == expect && peers[q].row_end >= peers[q].row_begin && peers[q].base,
                    "spmv_peers: peer windows must tile the rows contiguously");
            expect = peers[q].row_end;
        }
        require(expect == b->n_cols, "spmv_peers: peer windows must cover all columns");
        cudaStream_t s = static_cast<cudaStream_t>(stream);
        use_device(b->device);
        if (b->canonical && b->fast_passes) {
            // fast mode: the copy engines pull the remote runs pass by pass (each
            // pass's column range, split by owner) on the copy stream, and every
            // pass waits only for its own range -- the pulls of later ranges
            // overlap the earlier passes' multiplies and take no SMs
            if (!b->copy_stream) {
                ck(cudaStreamCreateWithFlags(&b->copy_stream, cudaStreamNonBlocking), "stream");
                ck(cudaEventCreateWithFlags(&b->ev_before, cudaEventDisableTiming), "event");
                ck(cudaEventCreateWithFlags(&b->ev_copied, cudaEventDisableTiming), "event");
            }
            ck(cudaEventRecord(b->ev_before, s), "event");  // the caller's writes of x_window are done
            ck(cudaStreamWaitEvent(b->copy_stream, b->ev_before, 0), "wait");
            for (int q = 0; q < b->fast_passes; ++q) {
                const int32_t p0 = b->fp_c0[q], p1 = b->fp_c0[q + 1];
                for (size_t i = 0; i + 1 < b->remote_runs.size(); i += 2) {
                    int32_t c = std::max(b->remote_runs[i], p0);
                    const int32_t c1 = std::min(b->remote_runs[i + 1], p1);
                    int32_t o = 0;
                    while (c < c1) {
                        while (peers[o].row_end <= c) ++o;
                        const int32_t e = std::min(c1, peers[o].row_end);
                        if (peers[o].base != x_window)
                            ck(cudaMemcpyAsync(x_window + c, peers[o].base + c, static_cast<size_t>(e - c) * sizeof(double),
                                               cudaMemcpyDefault, b->copy_stream),
                               "peer pull");
                        c = e;
                    }
                }
                if (!b->ev_part[q]) ck(cudaEventCreateWithFlags(&b->ev_part[q], cudaEventDisableTiming), "event");
                ck(cudaEventRecord(b->ev_part[q], b->copy_stream), "event");
            }
            for (int q = 0; q < b->fast_passes; ++q) {
                ck(cudaStreamWaitEvent(s, b->ev_part[q], 0), "wait");
                fast_pass_launch(b, q, x_window, y, s);
            }
            ck(cudaGetLastError(), "spmv_peers launch");
            return;
        }
        std::vector<int64_t> sig;
        for (int32_t q = 0; q < n_peers; ++q)
            sig.insert(sig.end(), {reinterpret_cast<int64_t>(peers[q].base), peers[q].row_begin, peers[q].row_end});
        sig.push_back(reinterpret_cast<int64_t>(x_window));
        if (sig != b->peer_sig) {  // pieces {peer, c0, c1}: remote runs split by owner, <= 16384 columns
            std::vector<int32_t> pc;
            std::vector<const double*> src(n_peers);
            for (int32_t q = 0; q < n_peers; ++q) src[q] = peers[q].base;
            for (size_t i = 0; i + 1 < b->remote_runs.size(); i += 2) {
                int32_t c = b->remote_runs[i];
                const int32_t c1 = b->remote_runs[i + 1];
                int32_t q = 0;
                while (c < c1) {
                    while (peers[q].row_end <= c) ++q;
                    const int32_t e = std::min({c1, peers[q].row_end, c + 16384});
                    if (peers[q].base != x_window) pc.insert(pc.end(), {q, c, e, 0});
                    c = e;
                }
            }
            b->n_peer_pieces = static_cast<int>(pc.size() / 4);
            b->peer_pieces.upload(pc, s);
            b->peer_src.upload_raw(src.data(), src.size() * sizeof(const double*), s);
            if (!b->peer_ctr.p) {
                b->peer_ctr.ensure(2 * sizeof(unsigned long long));
                ck(cudaMemsetAsync(b->peer_ctr.p, 0, 2 * sizeof(unsigned long long), s), "memset");
                b->peer_done = 0;
            }
            b->peer_sig = sig;
        }
        PeerDev P;
        P.pieces = b->peer_pieces.as<int4>();
        P.n_pieces = b->n_peer_pieces;
        P.src = b->peer_src.as<const double*>();
        P.dst = x_window;
        P.ticket = b->peer_ctr.as<unsigned long long>();
        P.done = b->peer_ctr.as<unsigned long long>() + 1;
        P.ticket_base = 0;
        b->peer_done += static_cast<unsigned long long>(b->n_peer_pieces);
        P.done_target = b->peer_done;
        P.k_pull = std::min(b->n_peer_pieces, 64);
        P.remote_block = b->remote_block.as<uint8_t>();
        P.remote_item = b->remote_item.as<uint8_t>();
        P.remote_long = b->remote_long.as<uint8_t>();
        ck(cudaMemsetAsync(b->peer_ctr.p, 0, sizeof(unsigned long long), s), "ticket reset");
        launch_spmv_parity(b->ro.as<int32_t>(), b->col.as<int32_t>(), b->val.as<double>(), x_window, y,
                           b->chunk_row.as<int4>(), b->n_chunks, b->item_seg.as<int2>(), b->long_list.as<int32_t>(),
                           static_cast<int>(b->long_rows), b->segs(), false, b->n_sms, b->spmv_short, b->rows(), s, &P);
        ck(cudaGetLastError(), "spmv_peers launch");
    });
}

// Device memory shareable with other processes (CUDA IPC), for peer x windows.
PSC_API psc_status psc_ipc_alloc(int64_t bytes, void** ptr, uint8_t handle[64]) {
    return guarded([&] {
        require(ptr && handle && bytes > 0, "ipc_alloc: bad argument");
        ck(cudaMalloc(ptr, static_cast<size_t>(bytes)), "ipc_alloc");
        cudaIpcMemHandle_t h;
        ck(cudaIpcGetMemHandle(&h, *ptr), "ipc handle");
        std::memcpy(handle, &h, 64);
    });
}
PSC_API psc_status psc_ipc_open(const uint8_t handle[64], void** ptr) {
    return guarded([&] {
        require(ptr && handle, "ipc_open: bad argument");
        cudaIpcMemHandle_t h;
        std::memcpy(&h, handle, 64);
        ck(cudaIpcOpenMemHandle(ptr, h, cudaIpcMemLazyEnablePeerAccess), "ipc open");
    });
}
PSC_API psc_status psc_ipc_close(void* ptr) {
    return guarded([&] { ck(cudaIpcCloseMemHandle(ptr), "ipc close"); });
}
PSC_API psc_status psc_ipc_free(void* ptr) {
    return guarded([&] { ck(cudaFree(ptr), "ipc free"); });
}
PSC_API psc_status psc_copy_async(void* dst, const void* src, int64_t bytes, void* stream) {
    return guarded([&] {
        require(bytes >= 0 && (bytes == 0 || (dst && src)), "copy_async: bad argument");
        if (bytes)
            ck(cudaMemcpyAsync(dst, src, static_cast<size_t>(bytes), cudaMemcpyDefault, static_cast<cudaStream_t>(stream)),
               "copy_async");
    });
}

PSC_API psc_status psc_bound_spmv(psc_bound* b, const double* x, double* y, void* stream) {
    return guarded([&] {
        require(b && x && y, "spmv: null argument");
        require(b->kernel == PSC_KERNEL_SPMV, "run_spmv: plan was built for another kernel");
        bound_spmv(b, x, y, static_cast<cudaStream_t>(stream));
    });
}
PSC_API psc_status psc_bound_sptrsv(psc_bound* b, const double* rhs, double* x, double* acc, void* stream) {
    return guarded([&] {
        require(b && rhs && x, "sptrsv: null argument");
        require(b->kernel == PSC_KERNEL_SPTRSV, "run_sptrsv: plan was built for another kernel");
        bound_sptrsv(b, rhs, x, acc, static_cast<cudaStream_t>(stream));
    });
}
// Host-buffer variants (the e2e path): H2D of the input, the kernel and the
// D2H of the result, all enqueued on `stream`. Host memory should be pinned
// for the copies to be asynchronous.
static psc_status spmv_host_unlocked(psc_bound* b, const double* x, double* y, void* stream) {
    return guarded([&] {
        require(b && x && y, "spmv_host: null argument");
        require(b->kernel == PSC_KERNEL_SPMV, "run_spmv: plan was built for another kernel");
        cudaStream_t s = static_cast<cudaStream_t>(stream);
        use_device(b->device);
        b->hy.ensure(std::max(1, b->rows()) * sizeof(double));
        if (b->canonical && b->fast_passes >= 1) {
            // fast column-split passes: x range q goes up on the copy stream and
            // pass q waits only for it, so the later ranges' upload hides the
            // earlier passes
            if (!b->copy_stream) {
                ck(cudaStreamCreateWithFlags(&b->copy_stream, cudaStreamNonBlocking), "stream");
                ck(cudaEventCreateWithFlags(&b->ev_before, cudaEventDisableTiming), "event");
                ck(cudaEventCreateWithFlags(&b->ev_copied, cudaEventDisableTiming), "event");
            }
            for (int q = 0; q < b->fast_passes; ++q)
                if (!b->ev_part[q]) ck(cudaEventCreateWithFlags(&b->ev_part[q], cudaEventDisableTiming), "event");
            b->hx.ensure(std::max<size_t>(8, static_cast<size_t>(b->n_cols) * sizeof(double)));
            ck(cudaEventRecord(b->ev_before, s), "event");  // earlier work on s is done with hx
            ck(cudaStreamWaitEvent(b->copy_stream, b->ev_before, 0), "wait");
            for (int q = 0; q < b->fast_passes; ++q) {
                const int64_t c0 = b->fp_c0[q], c1 = b->fp_c0[q + 1];
                if (c1 > c0)
                    ck(cudaMemcpyAsync(b->hx.as<double>() + c0, x + c0, static_cast<size_t>(c1 - c0) * sizeof(double),
                                       cudaMemcpyHostToDevice, b->copy_stream), "H2D");
                ck(cudaEventRecord(b->ev_part[q], b->copy_stream), "event");
            }
            const int last = b->fast_passes - 1;
            for (int q = 0; q < last; ++q) {
                ck(cudaStreamWaitEvent(s, b->ev_part[q], 0), "wait");
                fast_pass_launch(b, q, b->hx.as<double>(), b->hy.as<double>(), s);
            }
            // the last pass slice by slice; each slice's y rows are final once it ran
            ck(cudaStreamWaitEvent(s, b->ev_part[last], 0), "wait");
            const FlagPassDev whole = flag_pass(b, last);
            const int64_t ch = flag_chunk_entries(b->fl_per);
            for (int i = 0; i < psc_bound::kFastSlices; ++i) {
                const int32_t c0 = b->fsl_chunk[i], c1 = b->fsl_chunk[i + 1];
                const int32_t r0 = b->fsl_row[i], r1 = b->fsl_row[i + 1];
                if (c1 > c0) {
                    FlagPassDev P = whole;
                    P.colf += c0 * ch;
                    P.val += c0 * ch;
                    P.chunk_m0 += c0;
                    P.carry_val += c0;
                    P.carry_row += c0;
                    P.n_chunks = c1 - c0;
                    P.n_ent = c1 == whole.n_chunks ? whole.n_ent - c0 * ch : static_cast<int64_t>(c1 - c0) * ch;
                    launch_spmv_flag(P, b->hx.as<double>(), b->hy.as<double>(), last > 0, b->n_sms, s);
                }
                if (r1 > r0) {
                    if (!b->ev_slice[i]) ck(cudaEventCreateWithFlags(&b->ev_slice[i], cudaEventDisableTiming), "event");
                    ck(cudaEventRecord(b->ev_slice[i], s), "event");
                    ck(cudaStreamWaitEvent(b->copy_stream, b->ev_slice[i], 0), "wait");
                    ck(cudaMemcpyAsync(y + r0, b->hy.as<double>() + r0, static_cast<size_t>(r1 - r0) * sizeof(double),
                                       cudaMemcpyDeviceToHost, b->copy_stream), "D2H");
                }
            }
            ck(cudaEventRecord(b->ev_copied, b->copy_stream), "event");
            ck(cudaStreamWaitEvent(s, b->ev_copied, 0), "wait");  // the caller's stream covers the copies
            ck(cudaGetLastError(), "spmv launch");
            return;
        } else if (b->canonical && b->split) {
            // Column-split passes: pass q reads only x's column range q, so the
            // ranges go up on a copy stream one by one and pass q waits for its
            // own; the upload of the later ranges hides the earlier passes.
            if (!b->copy_stream) {
                ck(cudaStreamCreateWithFlags(&b->copy_stream, cudaStreamNonBlocking), "stream");
                ck(cudaEventCreateWithFlags(&b->ev_before, cudaEventDisableTiming), "event");
                ck(cudaEventCreateWithFlags(&b->ev_copied, cudaEventDisableTiming), "event");
            }
            for (int q = 0; q < b->split; ++q)
                if (!b->ev_part[q]) ck(cudaEventCreateWithFlags(&b->ev_part[q], cudaEventDisableTiming), "event");
            b->hx.ensure(std::max<size_t>(8, static_cast<size_t>(b->n_cols) * sizeof(double)));
            ck(cudaEventRecord(b->ev_before, s), "event");  // earlier work on s is done with hx
            ck(cudaStreamWaitEvent(b->copy_stream, b->ev_before, 0), "wait");
            for (int q = 0; q < b->split; ++q) {  // the column ranges of build_split
                const int64_t c0 = static_cast<int64_t>(b->n_cols) * q / b->split;
                const int64_t c1 = static_cast<int64_t>(b->n_cols) * (q + 1) / b->split;
                if (c1 > c0)
                    ck(cudaMemcpyAsync(b->hx.as<double>() + c0, x + c0, static_cast<size_t>(c1 - c0) * sizeof(double),
                                       cudaMemcpyHostToDevice, b->copy_stream), "H2D");
                ck(cudaEventRecord(b->ev_part[q], b->copy_stream), "event");
            }
            SplitPassDev P[kMaxSplitPasses];
            split_passes(b, P);
            const int last = b->split - 1;
            for (int q = 0; q < last; ++q) {
                ck(cudaStreamWaitEvent(s, b->ev_part[q], 0), "wait");
                launch_spmv_split(b->ro.as<int32_t>(), P, q + 1, b->sp_state.as<double>(), b->hx.as<double>(),
                                  b->hy.as<double>(), false, b->n_sms, s, q);
            }
            // the last pass slice by slice; each slice's y rows are final once it ran
            ck(cudaStreamWaitEvent(s, b->ev_part[last], 0), "wait");
            const SplitPassDev whole = P[last];
            for (int i = 0; i < psc_bound::kYSlices; ++i) {
                if (!b->ev_slice[i]) ck(cudaEventCreateWithFlags(&b->ev_slice[i], cudaEventDisableTiming), "event");
                P[last].items = whole.items + b->ysl_item[i];
                P[last].n_items = b->ysl_item[i + 1] - b->ysl_item[i];
                P[last].long_rows = whole.long_rows + b->ysl_long[i];
                P[last].n_long = b->ysl_long[i + 1] - b->ysl_long[i];
                launch_spmv_split(b->ro.as<int32_t>(), P, last + 1, b->sp_state.as<double>(), b->hx.as<double>(),
                                  b->hy.as<double>(), false, b->n_sms, s, last);
                const int32_t r0 = b->ysl_row[i], r1 = b->ysl_row[i + 1];
                if (r1 > r0) {
                    ck(cudaEventRecord(b->ev_slice[i], s), "event");
                    ck(cudaStreamWaitEvent(b->copy_stream, b->ev_slice[i], 0), "wait");
                    ck(cudaMemcpyAsync(y + r0, b->hy.as<double>() + r0, static_cast<size_t>(r1 - r0) * sizeof(double),
                                       cudaMemcpyDeviceToHost, b->copy_stream), "D2H");
                }
            }
            ck(cudaEventRecord(b->ev_copied, b->copy_stream), "event");
            ck(cudaStreamWaitEvent(s, b->ev_copied, 0), "wait");  // the caller's stream covers the copies
            ck(cudaGetLastError(), "spmv launch");
            return;
        } else {
            b->hx.upload_raw(x, static_cast<size_t>(b->n_cols) * sizeof(double), s);
            bound_spmv(b, b->hx.as<double>(), b->hy.as<double>(), s);
        }
        ck(cudaMemcpyAsync(y, b->hy.p, static_cast<size_t>(b->rows()) * sizeof(double), cudaMemcpyDeviceToHost, s), "D2H");
    });
}
// CTAs of the unit gather: the SMs the solve leaves free, at least 8 (PSC_GATHER_CTAS overrides)
static int gather_ctas(int n_sms, int n_blocks) {
    static const int forced = [] {
        const char* e = std::getenv("PSC_GATHER_CTAS");
        return e ? std::atoi(e) : 0;
    }();
    return forced > 0 ? forced : std::max(8, n_sms - n_blocks);
}

static psc_status sptrsv_host_unlocked(psc_bound* b, const double* rhs, double* x, double* acc, void* stream) {
    return guarded([&] {
        require(b && rhs && x, "sptrsv_host: null argument");
        require(b->kernel == PSC_KERNEL_SPTRSV, "run_sptrsv: plan was built for another kernel");
        cudaStream_t s = static_cast<cudaStream_t>(stream);
        use_device(b->device);
        const size_t bytes = static_cast<size_t>(b->rows()) * sizeof(double);
        b->hy.ensure(std::max<size_t>(bytes, 8));
        b->hx.ensure(std::max<size_t>(bytes, 8));
        if (acc || !b->canonical) b->hacc.ensure(std::max<size_t>(bytes, 8));
        // A pinned, mapped x (UVA) is written by the record kernel directly:
        // every finished chain unit is shipped by one bulk copy, overlapping
        // the solve instead of a copy after it. A pinned b is then uploaded
        // in row-ordered chunks on a side stream while the solve runs; the
        // kernel waits per chunk on arrival flags.
        auto mapped = [](const void* p) -> const void* {
            cudaPointerAttributes at{};
            if (cudaPointerGetAttributes(&at, p) == cudaSuccess && at.type == cudaMemoryTypeHost && at.devicePointer)
                return at.devicePointer;
            (void)cudaGetLastError();
            return nullptr;
        };
        double* x_map = nullptr;
        if (b->canonical && b->trsv_lean == 2 && b->chain_mode)
            x_map = static_cast<double*>(const_cast<void*>(mapped(x)));
        // (not under a profiler: ncu serialises and replays kernels, so a solve
        // waiting on a concurrent copy would never finish)
        static const bool overlap = [] {
            const char* ov = std::getenv("PSC_HOST_OVERLAP");
            if (ov) return ov[0] != '0';
            for (const char* v : {"CUDA_INJECTION64_PATH", "NV_TPS_LAUNCH_TOKEN", "NV_NSIGHT_INJECTION_TRANSPORT_TYPE"})
                if (std::getenv(v)) return false;  // a profiler (ncu / nsys / sanitizer) is attached
            return true;
        }();
        // The solve's lanes spin on per-unit flags that the gather kernel (another
        // stream, launched after it) sets: take the overlap only when every solve
        // CTA (one per SM at most: the record kernel's shared memory) leaves at
        // least 8 SMs free for the gather, so both are resident together.
        int sms = 0;
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, b->device);
        if (overlap && x_map && b->n_blocks + 8 <= sms && mapped(rhs)) {
            // b streams in unit by unit (a gather kernel on a side stream, in the
            // order the solve needs the units); every solve lane waits for its
            // unit's rows before staging them
            const double* rhs_dev = static_cast<const double*>(mapped(rhs));
            if (!b->copy_stream) {
                ck(cudaStreamCreateWithFlags(&b->copy_stream, cudaStreamNonBlocking), "stream");
                ck(cudaEventCreateWithFlags(&b->ev_before, cudaEventDisableTiming), "event");
                ck(cudaEventCreateWithFlags(&b->ev_copied, cudaEventDisableTiming), "event");
                b->b_ready.ensure(static_cast<size_t>(b->n_units_total + 2) * sizeof(int));
                ck(cudaMemsetAsync(b->b_ready.p, 0, static_cast<size_t>(b->n_units_total + 2) * sizeof(int), s), "memset");
                prepare_gather_b_units();
                cudaDeviceGetAttribute(&b->n_sms, cudaDevAttrMultiProcessorCount, b->device);
            }
            const int next_epoch = b->epoch == INT32_MAX ? 1 : b->epoch + 1;  // the epoch bound_sptrsv will use
            const int flag = next_epoch % 1000003 + 1;
            ck(cudaEventRecord(b->ev_before, s), "event");  // earlier solves on s are done with hy
            // the solve goes first (its lanes wait per unit), then the gather
            bound_sptrsv(b, b->hy.as<double>(), b->hx.as<double>(), acc ? b->hacc.as<double>() : nullptr, s, x_map,
                         b->b_ready.as<int>(), -1, flag);
            ck(cudaStreamWaitEvent(b->copy_stream, b->ev_before, 0), "wait");
            launch_gather_b_units(rhs_dev, b->hy.as<double>(), b->g_order.as<int32_t>(), b->unit_start.as<int32_t>(),
                                  b->unit_len.as<int32_t>(), b->n_units_total,
                                  b->b_ready.as<int>() + b->n_units_total, b->b_ready.as<int>(), flag,
                                  gather_ctas(b->n_sms, b->n_blocks), b->copy_stream);
            ck(cudaGetLastError(), "gather b");
            ck(cudaEventRecord(b->ev_copied, b->copy_stream), "event");
            ck(cudaStreamWaitEvent(s, b->ev_copied, 0), "wait");
        } else {
            b->hy.upload_raw(rhs, bytes, s);
            if (!b->canonical) b->hx.upload_raw(x, bytes, s);
            bound_sptrsv(b, b->hy.as<double>(), b->hx.as<double>(), (acc || !b->canonical) ? b->hacc.as<double>() : nullptr,
                         s, x_map);
        }
        if (!x_map) ck(cudaMemcpyAsync(x, b->hx.p, bytes, cudaMemcpyDeviceToHost, s), "D2H");
        if (acc) ck(cudaMemcpyAsync(acc, b->hacc.p, bytes, cudaMemcpyDeviceToHost, s), "D2H");
    });
}
// The host-buffer entry points share the bound's scratch buffers, copy
// stream and events: calls on one bound -- from any thread, on any stream --
// are serialised (each enqueues after the previous call's work).
static psc_status host_call(psc_bound* b, void* stream, const std::function<psc_status()>& call) {
    if (!b) return call();  // reports the null argument
    std::lock_guard<std::mutex> lk(b->host_mu);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const psc_status pre = guarded([&] {
        use_device(b->device);
        if (b->ev_host_done) ck(cudaStreamWaitEvent(s, b->ev_host_done, 0), "wait");
    });
    if (pre != PSC_OK) return pre;
    const psc_status st = call();
    if (st != PSC_OK) return st;
    return guarded([&] {
        if (!b->ev_host_done) ck(cudaEventCreateWithFlags(&b->ev_host_done, cudaEventDisableTiming), "event");
        ck(cudaEventRecord(b->ev_host_done, s), "event");
    });
}

PSC_API psc_status psc_bound_spmv_host(psc_bound* b, const double* x, double* y, void* stream) {
    return host_call(b, stream, [&] { return spmv_host_unlocked(b, x, y, stream); });
}

PSC_API psc_status psc_bound_sptrsv_host(psc_bound* b, const double* rhs, double* x, double* acc, void* stream) {
    return host_call(b, stream, [&] { return sptrsv_host_unlocked(b, rhs, x, acc, stream); });
}

// Diagnostics: copies the per-row publish times of the last solve (ns,
// %globaltimer) followed by one arm time per block; needs PSC_TRSV_TRACE=1
// at bind time. Returns the number of entries copied.
PSC_API int64_t psc_bound_trace(const psc_bound* b, uint64_t* out, int64_t cap) {
    if (!b || !b->trace.p || !out) return 0;
    int64_t n = std::min<int64_t>(cap, static_cast<int64_t>(b->trace.bytes / sizeof(uint64_t)));
    if (cudaSetDevice(b->device) != cudaSuccess) return 0;
    if (cudaDeviceSynchronize() != cudaSuccess) return 0;
    if (cudaMemcpy(out, b->trace.p, n * sizeof(uint64_t), cudaMemcpyDeviceToHost) != cudaSuccess) return 0;
    return n;
}
PSC_API int32_t psc_bound_launches(const psc_bound* b) {
    if (!b) return 0;
    if (b->canonical) {
        if (b->kernel != PSC_KERNEL_SPMV) return 1;
        if (b->fast_passes) return 2 * b->fast_passes;
        if (b->split) {
            int n = 0;
            for (int q = 0; q < b->split; ++q) n += (b->sp_n_long[q] > 0) + (b->sp_n_items[q] > 0);
            return n;
        }
        const int n = (b->long_rows > 0) + (b->n_chunks > 0) + (b->n_groups > 0);
        return n > 0 ? n : 1;
    }
    return static_cast<int32_t>(b->part_group_ptr.size()) - 1;
}
PSC_API psc_status psc_bound_info(const psc_bound* b, int64_t out[8]) {
    return guarded([&] {
        require(b && out, "bound_info: null argument");
        out[0] = b->rows();
        out[1] = b->canonical ? b->n_segments : -1;
        out[2] = b->kernel == PSC_KERNEL_SPMV ? (b->n_run_items > 0 ? b->n_run_items : b->n_chunks) : b->n_blocks;
        out[3] = !b->canonical ? 1 : b->fast_passes ? 2 : 0;
        out[4] = b->algorithmic_bytes();
        out[5] = b->device_bytes();
        out[6] = b->long_rows;
        out[7] = b->kernel == PSC_KERNEL_SPMV ? std::max(b->fast_passes, b->split) : b->max_block_rows;
    });
}

PSC_API psc_status psc_csr_spmv_device(const psc_bound* b, const double* x, double* y, void* stream) {
    return guarded([&] {
        require(b && x && y, "csr_spmv: null argument");
        require(b->canonical, "csr_spmv: needs a canonical bound plan");
        use_device(b->device);
        launch_csr_spmv_naive(b->ro.as<int32_t>(), b->col.as<int32_t>(), b->val.as<double>(), x, y, b->rows(),
                              static_cast<cudaStream_t>(stream));
        ck(cudaGetLastError(), "csr_spmv launch");
    });
}

PSC_API psc_status psc_csr_sptrsv_device(psc_bound* b, const double* rhs, double* x, void* stream) {
    return guarded([&] {
        require(b && rhs && x, "csr_sptrsv: null argument");
        require(b->canonical, "csr_sptrsv: needs a canonical bound plan");
        require(b->kernel == PSC_KERNEL_SPTRSV, "csr_sptrsv: plan was built for another kernel");
        use_device(b->device);
        b->naive_ticket.ensure(sizeof(int));
        launch_csr_sptrsv_naive(b->ro.as<int32_t>(), b->col.as<int32_t>(), b->val.as<double>(), rhs, x, b->rows(),
                                b->naive_ticket.as<int>(), static_cast<cudaStream_t>(stream));
        ck(cudaGetLastError(), "csr_sptrsv launch");
    });
}

// The run_* / execute_plan calls read the matrix values live, as the
// reference does (upload on every call), unless the caller tagged them with a
// version (psc_executor_set_values_version) equal to the one on the device.
void upload_values(psc_executor* e, psc_bound* b, const double* values, cudaStream_t s) {
    if (e->values_version != 0 && b->values_version == e->values_version) return;
    b->val.upload_raw(values + b->k_begin, (b->k_end - b->k_begin) * sizeof(double), s);
    b->rec_dirty = true;
    b->values_version = e->values_version;
}

PSC_API psc_status psc_executor_set_values_version(psc_executor* e, uint64_t version) {
    return guarded([&] {
        require(e != nullptr, "set_values_version: null executor");
        std::lock_guard<std::mutex> lk(e->mu);
        e->values_version = version;
    });
}

// run_spmv, executor.cpp:274-288.
PSC_API psc_status psc_run_spmv(psc_executor* e, const psc_plan* plan, const psc_csr_view* a, const double* x,
                                int64_t nx, double* y, int64_t ny) {
    return guarded([&] {
        require(e && plan && a, "run_spmv: null argument");
        if (plan->p.kernel != PSC_KERNEL_SPMV) throw std::invalid_argument("run_spmv: plan was built for another kernel");
        if (nx != a->n_cols || ny != a->n_rows) throw std::invalid_argument("run_spmv: vector size mismatch");
        std::lock_guard<std::mutex> lk(e->mu);
        psc_bound* b = cached_bound(e, plan, *a, false);
        cudaStream_t s = e->stream;
        use_device(e->device);
        upload_values(e, b, a->values, s);  // the reference reads values live
        e->vx.upload_raw(x, nx * sizeof(double), s);
        e->vy.ensure(std::max<int64_t>(ny, 1) * sizeof(double));
        bound_spmv(b, e->vx.as<double>(), e->vy.as<double>(), s);
        if (ny) ck(cudaMemcpyAsync(y, e->vy.p, ny * sizeof(double), cudaMemcpyDeviceToHost, s), "D2H");
        ck(cudaStreamSynchronize(s), "run_spmv sync");
    });
}

// run_sptrsv, executor.cpp:290-308.
PSC_API psc_status psc_run_sptrsv(psc_executor* e, const psc_plan* plan, const psc_csr_view* l, const double* rhs,
                                  int64_t nb, double* x, int64_t nx, double* acc, int64_t nacc) {
    return guarded([&] {
        require(e && plan && l, "run_sptrsv: null argument");
        if (plan->p.kernel != PSC_KERNEL_SPTRSV)
            throw std::invalid_argument("run_sptrsv: plan was built for another kernel");
        int64_t n = l->n_rows;
        if (nb != n || nx != n || nacc != n) throw std::invalid_argument("run_sptrsv: vector size mismatch");
        std::lock_guard<std::mutex> lk(e->mu);
        psc_bound* b = cached_bound(e, plan, *l, false);
        cudaStream_t s = e->stream;
        use_device(e->device);
        upload_values(e, b, l->values, s);
        size_t bytes = std::max<int64_t>(n, 1) * sizeof(double);
        e->vb.upload_raw(rhs, n * sizeof(double), s);
        e->vx.ensure(bytes);
        e->vacc.ensure(bytes);
        if (!b->canonical && n) e->vx.upload_raw(x, n * sizeof(double), s);  // stale reads see caller's x
        bound_sptrsv(b, e->vb.as<double>(), e->vx.as<double>(), e->vacc.as<double>(), s);
        if (n) {
            ck(cudaMemcpyAsync(x, e->vx.p, n * sizeof(double), cudaMemcpyDeviceToHost, s), "D2H x");
            if (acc) ck(cudaMemcpyAsync(acc, e->vacc.p, n * sizeof(double), cudaMemcpyDeviceToHost, s), "D2H acc");
        }
        ck(cudaStreamSynchronize(s), "run_sptrsv sync");
    });
}

// execute_plan, executor.cpp:269-272: no zero-fill, accumulate onto ctx.
PSC_API psc_status psc_execute_plan(psc_executor* e, const psc_plan* plan, const psc_csr_view* a,
                                    const psc_exec_context* ctx) {
    return guarded([&] {
        require(e && plan && a && ctx, "execute_plan: null argument");
        require(ctx->matrix_values && ctx->gather && ctx->accum, "execute_plan: null context array");
        const bool solve = ctx->rhs != nullptr;
        if (solve) require(ctx->solution != nullptr, "execute_plan: solve context needs a solution array");
        std::lock_guard<std::mutex> lk(e->mu);
        psc_bound* b = cached_bound(e, plan, *a, true);
        cudaStream_t s = e->stream;
        use_device(e->device);
        const int64_t n = a->n_rows, nc = a->n_cols;
        if (!(e->values_version != 0 && b->values_version == e->values_version)) {
            b->val.upload_raw(ctx->matrix_values, a->nnz * sizeof(double), s);
            b->rec_dirty = true;
            b->values_version = e->values_version;
        }
        e->vy.upload_raw(ctx->accum, n * sizeof(double), s);
        if (solve) {
            // gather aliases solution (executor.hpp:12-23)
            e->vx.upload_raw(ctx->solution, n * sizeof(double), s);
            e->vb.upload_raw(ctx->rhs, n * sizeof(double), s);
            run_general(b, e->vx.as<double>(), e->vy.as<double>(), e->vb.as<double>(), e->vx.as<double>(), s);
            if (n) ck(cudaMemcpyAsync(ctx->solution, e->vx.p, n * sizeof(double), cudaMemcpyDeviceToHost, s), "D2H");
        } else {
            e->vx.upload_raw(ctx->gather, nc * sizeof(double), s);
            run_general(b, e->vx.as<double>(), e->vy.as<double>(), nullptr, nullptr, s);
        }
        if (n) ck(cudaMemcpyAsync(ctx->accum, e->vy.p, n * sizeof(double), cudaMemcpyDeviceToHost, s), "D2H");
        ck(cudaStreamSynchronize(s), "execute_plan sync");
    });
}

}  // extern "C"

namespace {

// Runs a general-path lowering over a raw host context with exact
// Executor::run semantics (executor.cpp:261-267): partitions in order, each
// group's codelets then its finalize records; accumulates onto ctx->accum,
// writes ctx->solution at the finalized rows. Only the index ranges the
// descriptors and finalize records touch are moved; a gather aliasing the
// solution (the solve, executor.hpp:12-16) is one device buffer.
void run_lowered_on_host_context(const Lowered& L, const psc_exec_context* ctx, const char* who) {
    const auto& G = L.gen;
    int n = psc_device_count();
    if (n <= 0) throw CudaError(std::string(who) + ": no CUDA device is available");
    int dev = 0;
    ck(cudaGetDevice(&dev), "cudaGetDevice");
    psc_bound b;
    b.device = dev;
    b.canonical = false;
    cudaStream_t s = nullptr;
    b.part_group_ptr = G.part_group_ptr;
    b.g_cp.upload(G.group_codelet_ptr, s);
    b.g_fp.upload(G.group_fin_ptr, s);
    b.g_kind.upload(G.c_kind, s);
    b.g_m.upload(G.c_m, s);
    b.g_n.upload(G.c_n, s);
    b.g_form.upload(G.d_form, s);
    b.g_base.upload(G.d_base, s);
    b.g_so.upload(G.d_so, s);
    b.g_si.upload(G.d_si, s);
    b.g_tab.upload(G.d_tab, s);
    b.g_tables.upload(G.tables, s);
    b.g_frow.upload(G.f_row, s);
    b.g_fdiag.upload(G.f_diag, s);
    b.g_frhs.upload(G.f_rhs, s);
    int64_t max_frow = -1, max_fdiag = -1, max_frhs = -1;
    for (size_t f = 0; f < G.f_row.size(); ++f) {
        max_frow = std::max<int64_t>(max_frow, G.f_row[f]);
        max_fdiag = std::max<int64_t>(max_fdiag, G.f_diag[f]);
        max_frhs = std::max<int64_t>(max_frhs, G.f_rhs[f]);
    }
    const bool finalize = max_frow >= 0;
    const int64_t nm = std::max(G.max_mat, max_fdiag) + 1, nv = G.max_vec + 1,
                  no = std::max(G.max_out, max_frow) + 1, ns = max_frow + 1, nr = max_frhs + 1;
    const std::string w(who);
    if (nm > 0) require(ctx->matrix_values != nullptr, w + ": null matrix_values");
    if (nv > 0) require(ctx->gather != nullptr, w + ": null gather");
    if (no > 0) require(ctx->accum != nullptr, w + ": null accum");
    if (finalize) require(ctx->rhs != nullptr && ctx->solution != nullptr, w + ": finalize records need rhs and solution");
    const bool alias = finalize && static_cast<const void*>(ctx->gather) == static_cast<const void*>(ctx->solution);
    b.val.upload_raw(ctx->matrix_values, std::max<int64_t>(nm, 0) * sizeof(double), s);
    DevBuf g, acc, rhs, sol;
    const int64_t ng = alias ? std::max(nv, ns) : nv;
    g.upload_raw(ctx->gather, std::max<int64_t>(ng, 0) * sizeof(double), s);
    acc.upload_raw(ctx->accum, std::max<int64_t>(no, 0) * sizeof(double), s);
    // a non-null rhs selects the solve's sequential partials (executor.cpp:53-116)
    // even without finalize records
    if (ctx->rhs) {
        if (finalize) rhs.upload_raw(ctx->rhs, nr * sizeof(double), s);
        else rhs.ensure(sizeof(double));
    }
    if (finalize && !alias) sol.upload_raw(ctx->solution, ns * sizeof(double), s);
    double* sol_dev = !finalize ? nullptr : alias ? g.as<double>() : sol.as<double>();
    run_general(&b, g.as<double>(), acc.as<double>(), ctx->rhs ? rhs.as<double>() : nullptr, sol_dev, s);
    if (no > 0) ck(cudaMemcpyAsync(ctx->accum, acc.p, no * sizeof(double), cudaMemcpyDeviceToHost, s), "D2H");
    if (finalize) ck(cudaMemcpyAsync(ctx->solution, sol_dev, ns * sizeof(double), cudaMemcpyDeviceToHost, s), "D2H");
    ck(cudaStreamSynchronize(s), "sync");
}

psc_status exec_one(int which, const psc_codelet_view* c, const psc_exec_context* ctx) {
    return guarded([&] {
        require(c && ctx, "exec_codelet: null argument");
        run_lowered_on_host_context(lower_single_codelet(*c, which), ctx, "exec_codelet");
    });
}

}  // namespace

extern "C" {
// Executor::run (executor.hpp:45, executor.cpp:261-267) on a plan that carries
// its tables (the reference's own CodeletPlan, imported with
// psc_plan_from_arrays); no matrix argument, accumulates onto ctx.
PSC_API psc_status psc_executor_run(psc_executor* e, const psc_plan* plan, const psc_exec_context* ctx) {
    return guarded([&] {
        require(e && plan && ctx, "Executor::run: null argument");
        std::lock_guard<std::mutex> lk(e->mu);
        use_device(e->device);
        run_lowered_on_host_context(lower_plan_tables(plan->p), ctx, "Executor::run");
    });
}
}  // extern "C"

extern "C" {
PSC_API psc_status psc_exec_blas_codelet(const psc_codelet_view* c, const psc_exec_context* ctx) {
    return exec_one(PSC_CODELET_BLAS, c, ctx);
}
PSC_API psc_status psc_exec_psci_codelet(const psc_codelet_view* c, const psc_exec_context* ctx) {
    return exec_one(PSC_CODELET_PSC_I, c, ctx);
}
PSC_API psc_status psc_exec_pscii_codelet(const psc_codelet_view* c, const psc_exec_context* ctx) {
    return exec_one(PSC_CODELET_PSC_II, c, ctx);
}
}
