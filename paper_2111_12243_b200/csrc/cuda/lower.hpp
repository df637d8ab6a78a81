// Lowering of a codelet plan to the device layout (host side).
//
// Canonical plans (every plan the reference miner emits, and any imported
// plan with the same invariants) become per-row *segments*: codelet row i of
// codelet c contributes the contiguous CSR range [mat.base + i*mat.so, +n) to
// output row out(i), and its gather equals col_indices over that range
// (validate_plan enforces the gather identity, miner.cpp:346-366). A row's
// result is the sum of its segment partials in plan order, each partial
// formed exactly as exec_*_codelet forms it (4-lane dot for SpMV, sequential
// for the solve; executor.cpp:23-116). When every row is a single segment
// covering its whole operation range, no segment arrays are stored.
//
// Anything else (hand-built codelets with arbitrary tables, non-unit inner
// strides, rows split across groups, solve plans that read x before it is
// finalised) lowers to the general interpreter: one launch per partition, one
// thread per region group, exact Listing-3 semantics.
#pragma once

#include <cstdint>
#include <string>
#include <vector>

#include "plan.hpp"
#include "psc_b200.h"

namespace pscb {

struct Lowered {
    int kernel = PSC_KERNEL_SPMV;
    int32_t row_begin = 0, row_end = 0;  // bound rows [row_begin, row_end)
    int64_t k_begin = 0, k_end = 0;      // CSR positions of those rows
    bool canonical = true;
    bool simple = true;  // every row = one implicit full-row segment
    // segments (local rows), only when canonical && !simple
    std::vector<int32_t> row_seg_ptr;
    std::vector<int32_t> seg_start;  // local CSR position
    std::vector<int32_t> seg_len;
    std::vector<int32_t> seg_vec;  // x index of element 0 when the gather is a unit-stride run, else -1
    // SpMV work in local rows / CSR positions: chunks {r0, r1, k0, k1} of
    // consecutive short rows (<= kSpmvWarpCap entries and rows), their
    // segment ranges {s0, s1}, and the rows longer than kSpmvWarpCap
    std::vector<int32_t> items;     // 4 per chunk
    std::vector<int32_t> item_seg;  // 2 per chunk (segmented plans)
    std::vector<int32_t> long_row_list;
    int64_t long_rows = 0;
    // SpMV row groups (segmented plans): runs of 2..kGroupRows consecutive
    // rows with the same segment template -- all unit-stride gathers, tiling
    // the row in CSR order, the same lengths and x offsets -- so the rows read
    // the same x runs (the dof rows of a block stencil node). {r0, g} each;
    // their rows are in no chunk. 8 ints per group: {r0, g, k0, C, q0, S, -, -}
    // (first row, rows, first CSR position, entries per row, first segment,
    // segments per row).
    std::vector<int32_t> groups;
    // SpTRSV row blocks in local rows, and every block's rows in
    // dependency-level order (the plan's partition index, then row)
    std::vector<int32_t> block_row;
    // units solved front to back by one lane: chain mode -- runs of
    // consecutive rows each reading the row above, listed in row order; row
    // mode -- single rows listed by (level, row). block_unit = unit ranges.
    bool chain_mode = false;
    std::vector<int32_t> unit_start, block_unit;
    int32_t max_block_units = 0;
    int32_t max_block_rows = 0;
    // record kernel layout (unit_maps / tile_chain_blocks): every unit's row
    // count and first shared-memory slot in its block, every row's block and
    // slot. block_row then holds the prefix sum of block sizes; with tiled
    // blocks it no longer delimits row ranges.
    std::vector<int32_t> unit_len, unit_loc, row_block, row_loc;
    bool tiled = false;
    // per block: the distinct columns it reads from other blocks (sorted),
    // mirrored into shared memory after the block's own rows (block_halos)
    std::vector<int32_t> halo_ptr, halo_col;  // halo_col: in production (level) order
    std::vector<int32_t> halo_key, halo_pos;  // the same columns sorted, and their halo_col positions
    int32_t max_block_halo = 0;
    std::string why_general;  // reason the plan is not canonical

    // general interpreter tables (only when !canonical)
    struct General {
        std::vector<int64_t> part_group_ptr;
        std::vector<int64_t> group_codelet_ptr, group_fin_ptr;
        std::vector<int32_t> c_kind, c_m, c_n;
        std::vector<int32_t> d_form, d_base, d_so, d_si;  // 3 per codelet
        std::vector<int64_t> d_tab;                       // 3 per codelet: offset into tables
        std::vector<int32_t> tables;
        std::vector<int32_t> f_row, f_diag, f_rhs;
        int64_t max_mat = -1, max_vec = -1, max_out = -1;  // touched index ranges
    } gen;
};

constexpr int kSpmvWarpCap = 256;  // == kWarpCap in kernels.cu
constexpr int kGroupRows = 3;      // rows per SpMV row group (== kernels.cu)
constexpr int kGroupCols = 96;     // entries per row of a row group (three warp passes)

// Lower partitions [part_begin, part_end) (all partitions when part_end < 0).
// force_general lowers through the exact interpreter even when canonical
// (execute_plan accumulates onto caller-provided accum/solution arrays).
Lowered lower_plan(const Plan& p, const psc_csr_view& a, int64_t part_begin, int64_t part_end,
                   int sptrsv_block_rows, bool force_general = false);

// Fill unit_len / unit_loc / row_block / row_loc for the contiguous blocks
// lower_plan produced (SpTRSV).
void unit_maps(Lowered& L);

// Chain mode: regroup units into blocks of <= max_rows rows grown greedily
// over the unit dependency graph (a unit joins the open block once all its
// dependencies are placed, preferring the unit with most dependencies inside
// the open block, then discovery order), so blocks are compact regions and a
// dependency chain crosses few block boundaries. Blocks stay topologically
// ordered. Fills the record-kernel maps; returns false (L unchanged) when not
// applicable.
bool tile_chain_blocks(Lowered& L, const psc_csr_view& a, int max_rows);

// Fill halo_ptr / halo_col / max_block_halo from row_block (after unit_maps
// or tile_chain_blocks).
void block_halos(Lowered& L, const psc_csr_view& a);

// Warp items of the thread-per-row SpMV (simple plans whose rows hold <= 16 entries; kernels.cu
// spmv_run_kernel), 20 ints each: {first local row, rows (<= 32), first local CSR position, n,
// tmpl[16]}. n >= 0: a piece of a shifted run -- >= kRunMinRows consecutive rows of n entries each
// whose columns are the first row's plus the row distance (tmpl = the item's first row's columns);
// n = -1: consecutive rows outside such runs. Returns the rows covered by run items.
constexpr int kRunMinRows = 16;
int64_t build_run_items(const Lowered& L, const psc_csr_view& a, std::vector<int32_t>& items);

// General-path lowering of a plan with explicit tables (imported with
// psc_plan_from_arrays: the reference's own CodeletPlan) without a matrix:
// Executor::run(plan, ctx) semantics (executor.hpp:45). Index ranges come
// from the descriptors (Lowered::General::max_*).
Lowered lower_plan_tables(const Plan& p);

// Build a general-path lowering of one hand-built codelet (exec_*_codelet).
Lowered lower_single_codelet(const psc_codelet_view& c, int which);

// Shape checks of exec_*_codelet (executor.cpp:54-56, 76-78, 97-99).
void check_codelet_shape(int which, int out_form, int mat_form, int vec_form);

}  // namespace pscb
