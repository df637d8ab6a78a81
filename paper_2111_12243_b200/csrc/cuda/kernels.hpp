// Launch wrappers for the sm_100a kernels (definitions in kernels.cu).
// Rows and CSR positions are local to the bound row range: ro[] is rebased
// so ro[0] == 0, col/val hold only the bound rows' entries, y holds only the
// bound rows; x (the gathered vector) is always the full vector.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

namespace pscb {

struct SegmentsDev {
    const int32_t* row_seg_ptr = nullptr;  // null => every row is one implicit full-row segment
    const int32_t* seg_start = nullptr;
    const int32_t* seg_len = nullptr;
    const int32_t* seg_vec = nullptr;
    const int4* groups = nullptr;  // SpMV row groups, 2 int4 each (lower.hpp Lowered::groups)
    int n_groups = 0;
};

// Fused x exchange for multi-GPU SpMV: the first
// k_pull CTAs of the launch (by ticket, i.e. the first to be scheduled) copy
// every piece {peer, c0, c1} of x this shard reads from other ranks -- from
// the peers' x windows over NVLink (src[peer] + c) into the local window dst
// (the x the kernel gathers from) -- and count them into `done`; work that
// reads remote columns waits until `done` reaches done_target, everything
// else proceeds at once. Counters only grow (bases advance per launch).
struct PeerDev {
    const int4* pieces = nullptr;           // {peer, c0, c1, 0}
    int n_pieces = 0;
    const double* const* src = nullptr;     // device array: peer window base pointers
    double* dst = nullptr;                  // the local window (== x)
    unsigned long long* ticket = nullptr;   // CTA tickets (monotonic)
    unsigned long long* done = nullptr;     // landed pieces (monotonic)
    unsigned long long ticket_base = 0, done_target = 0;
    int k_pull = 0;                         // pulling CTAs of this launch (0: nothing to pull)
    const uint8_t* remote_block = nullptr;  // row kernel: per 256-row block, reads remote columns
    const uint8_t* remote_item = nullptr;   // chunk kernel: per chunk
    const uint8_t* remote_long = nullptr;   // long-row kernel: per long row
};

// y[r] = (accumulate ? y[r] : 0) + sum of row r's segment partials in plan
// order, each a 4-lane dot (executor.cpp:23-49). items: chunks of short rows
// {row begin, row end, CSR begin, CSR end} (<= 256 entries and rows each) with
// their segment ranges item_seg (segmented plans); long_rows: rows with more
// than 256 entries (kernels.cu "SpMV parity kernels"). Up to two launches.
// Column-split SpMV (simple plans whose x outgrows L2): the matrix stored as
// one CSR per column range, multiplied in passes that each gather from one
// range of x. A row's dot_unit state (its four lane sums, or its running tail
// sum) crosses from pass to pass through `state` (4 doubles per row). ro:
// the full matrix's row offsets.
constexpr int kMaxSplitPasses = 4;
struct SplitPassDev {
    const int32_t* j0 = nullptr;       // per row: index of its first entry in this pass (null: 0)
    const int32_t* ro_pass = nullptr;  // this pass's CSR
    const int32_t* col = nullptr;
    const double* val = nullptr;
    const int4* items = nullptr;       // chunks {r0, r1, k0, k1} in this pass's CSR
    int n_items = 0;
    const int32_t* long_rows = nullptr;  // rows with more than 256 entries in this pass
    int n_long = 0;
};
// passes [pass_begin, n_passes) of a column-split multiply (the ones before
// must already have run on `stream`)
void launch_spmv_split(const int32_t* ro, const SplitPassDev* passes, int n_passes, double* state, const double* x,
                       double* y, bool accumulate, int n_sms, cudaStream_t stream, int pass_begin = 0);

// Fast mode (spmv_fast.cu spmv_flag_kernel), one pass: the pass's
// entries in CSR order with bit 31 of the column set on each row's last
// entry (a row without entries in the pass holds one placeholder, column
// 0x7fffffff), and per chunk of flag_chunk_entries() entries the number of
// row ends before it.
struct FlagPassDev {
    const int32_t* colf = nullptr;
    const double* val = nullptr;
    const int32_t* chunk_m0 = nullptr;
    int64_t n_ent = 0;
    int n_chunks = 0;
    int per = 8;  // entries per lane (a chunk is 32 * per entries)
    double* carry_val = nullptr;
    int32_t* carry_row = nullptr;
};
int flag_chunk_entries(int per);
// y = (accumulate ? y : 0) + A_pass x; two launches (chunks, then the carries).
void launch_spmv_flag(const FlagPassDev& pass, const double* x, double* y, bool accumulate, int n_sms,
                      cudaStream_t stream);

void launch_spmv_parity(const int32_t* ro, const int32_t* col, const double* val, const double* x,
                        double* y, const int4* items, int n_items, const int2* item_seg,
                        const int32_t* long_rows, int n_long, SegmentsDev segs, bool accumulate, int n_sms,
                        int short_rows, int n_rows, cudaStream_t stream,
                        const PeerDev* peer = nullptr, const int4* run_items = nullptr, int n_run_items = 0);

// Sync-free blocked record solve (kernels.cu sptrsv_rec_kernel): blocks of
// rows (block_row: prefix sums of block sizes), solved by units listed in
// unit_start[block_unit[i] .. block_unit[i+1]) -- runs of consecutive rows
// (chain mode) or single rows in level order (single_row_units) -- from the
// per-row records (trsv_pack_kernel). ticket: 2 zeroed ints, left zeroed;
// armed: one int per block, epoch a per-launch counter. trace (nullable) gets
// per-row publish times followed by one arm time per block.
void launch_sptrsv(const int32_t* ro, const int32_t* col, const double* val, const double* b, double* x,
                   double* acc_out, const int32_t* block_row, const int32_t* block_unit, const int32_t* unit_start,
                   int n_blocks, int max_rows, int max_units, bool single_row_units, SegmentsDev segs,
                   int32_t* ticket, int32_t* armed, int epoch, unsigned long long* trace, int threads, const void* rec,
                   const int32_t* unit_len, const int32_t* unit_loc, const int32_t* halo_ptr, const int32_t* halo_col,
                   int max_halo, double* x_host, const int* b_ready, int b_shift, int b_flag, cudaStream_t stream);
// Global unit queue solve (long rows): units = first rows of the chains
// (units[n_units] = n_rows) or single rows, in topological order.
// Lane-per-row streaming solve over pieces of <= 32 consecutive rows
// (boundaries in `pieces`, n_pieces + 1 entries, in row order).
// piece_w0 (nullable): per piece, the first row of the previous piece of the
// same chain (== the piece's first row when it starts a chain)
void launch_sptrsv_stream(const int32_t* ro, const int32_t* col, const double* val, const double* b, double* x,
                          double* acc_out, const int32_t* pieces, const int32_t* piece_w0, int n_pieces, SegmentsDev s,
                          int* next_unit,
                          unsigned long long* trace, int n_rows, int n_sms, int k_entries, cudaStream_t stream);
void launch_sptrsv_queue(const int32_t* ro, const int32_t* col, const double* val, const double* b, double* x,
                         double* acc_out, const int32_t* units, const int32_t* unit_end, int n_units,
                         bool single_row_units, SegmentsDev s, int* next_unit, unsigned long long* trace, int n_rows,
                         int n_sms, int backoff_ns, cudaStream_t stream);
// Host path of the record kernel: b copied from mapped host memory unit by
// unit in `order`, b_ready[u] = flag when unit u's rows landed (ticket: 2
// ints, zero before the first launch, self re-arming). Call prepare first.
void prepare_gather_b_units();
void launch_gather_b_units(const double* b_host, double* b_dev, const int32_t* order, const int32_t* unit_start,
                           const int32_t* unit_len, int n_units, int* ticket, int* b_ready, int flag, int n_ctas,
                           cudaStream_t stream);
size_t trsv_rec_bytes();
void launch_trsv_pack(const int32_t* ro, const int32_t* col, const double* val, const int32_t* row_block,
                      const int32_t* row_loc, const int32_t* block_row, const int32_t* halo_ptr, const int32_t* halo_key,
                      const int32_t* halo_pos, int n_rows, void* rec, cudaStream_t stream);
// mismatches between the record kernel's division and __ddiv_rn on n random operand pairs (-1: CUDA error)
int64_t division_selftest(uint64_t seed, int64_t n, int exp_span);
size_t sptrsv_smem_bytes(int threads, int max_rows, int max_units, int max_halo);  // record kernel

// General interpreter (exact Listing-3 semantics) over groups [g0, g1) of one
// partition; one thread per region group.
struct GeneralDev {
    const int64_t* group_codelet_ptr;
    const int64_t* group_fin_ptr;
    const int32_t* c_kind;
    const int32_t* c_m;
    const int32_t* c_n;
    const int32_t* d_form;
    const int32_t* d_base;
    const int32_t* d_so;
    const int32_t* d_si;
    const int64_t* d_tab;
    const int32_t* tables;
    const int32_t* f_row;
    const int32_t* f_diag;
    const int32_t* f_rhs;
};
void launch_general_partition(GeneralDev g, int64_t g0, int64_t g1, const double* matrix_values,
                              const double* gather, double* accum, const double* rhs, double* solution,
                              cudaStream_t stream);

// Naive row-sequential CSR SpMV (spmv_csr_baseline, executor.cpp:310-323).
// sptrsv_csr_baseline on the GPU: thread per row, sync-free (ticket: 1 int).
void launch_csr_sptrsv_naive(const int32_t* ro, const int32_t* col, const double* val, const double* b, double* x,
                             int32_t n_rows, int* ticket, cudaStream_t stream);
void launch_csr_spmv_naive(const int32_t* ro, const int32_t* col, const double* val, const double* x,
                           double* y, int32_t n_rows, cudaStream_t stream);

}  // namespace pscb
