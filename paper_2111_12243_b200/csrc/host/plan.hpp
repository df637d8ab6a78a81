// Host-side codelet plan (the reference's CodeletPlan, miner.hpp:56-89) in
// structure-of-arrays form.
//
// Mined plans (from pscb::inspect) store one compact record per codelet:
// {kind, m, n, first row, mat base, mat row stride, vec base, vec row stride}.
// Every codelet the reference miner emits is a row rectangle whose tables are
// verbatim slices of col_indices (miner.cpp:106-112, 156-164, 206-226), so the
// full AccessDesc of each codelet is a pure function of that record and the
// CSR arrays; psc_plan_to_arrays materialises it on demand.
//
// Imported plans (psc_plan_from_arrays: a reference-produced or hand-built
// plan) keep explicit descriptors and a table pool instead.
#pragma once

#include <cstdint>
#include <vector>

#include "psc_b200.h"

namespace pscb {

struct DescView {  // one AccessDesc, read-only
    int32_t form = PSC_FORM_STRIDED;
    int32_t base = 0, so = 0, si = 0;
    // table: explicit pointer, or implicit (CSR-derived) when tab == nullptr
    const int32_t* tab = nullptr;
    int64_t len = 0;
};

struct Plan {
    int32_t kernel = PSC_KERNEL_SPMV;
    int32_t n_rows = 0, n_cols = 0;
    int64_t nnz = 0;
    int32_t window = 0, target_groups = 0;
    bool mined = true;
    // structure_hash of the matrix a mined plan was inspected from (its tables
    // are that matrix's columns); 0 = unknown (a version-1 plan file)
    uint64_t structure = 0;

    std::vector<int64_t> part_group_ptr{0};
    std::vector<int32_t> g_row_begin, g_row_end;
    std::vector<uint8_t> g_strategy;
    std::vector<int64_t> g_cost;
    std::vector<int64_t> g_codelet_ptr{0};

    // compact codelets (both modes keep kind/m/n here)
    std::vector<uint8_t> c_kind;
    std::vector<int32_t> c_m, c_n;
    std::vector<int32_t> c_row, c_mat_base, c_mat_so, c_vec_base, c_vec_so;  // mined only

    // explicit descriptors (imported only): 3 per codelet
    std::vector<int32_t> d_form, d_base, d_so, d_si;
    std::vector<int64_t> d_tab_ptr{0};
    std::vector<int32_t> tables;
    // finalize records: implicit for mined sptrsv plans ({r, diag(r), r} for
    // every row of the window, miner.cpp:312-316), explicit when imported.
    std::vector<int64_t> g_fin_ptr{0};
    std::vector<int32_t> f_row, f_diag, f_rhs;

    int64_t n_partitions() const { return static_cast<int64_t>(part_group_ptr.size()) - 1; }
    int64_t n_groups() const { return static_cast<int64_t>(g_row_begin.size()); }
    int64_t n_codelets() const { return static_cast<int64_t>(c_kind.size()); }
    int64_t n_finalize() const;
    int64_t n_table() const;

    // Descriptor d (0 out, 1 mat, 2 vec) of codelet ci.
    DescView desc(int64_t ci, int d) const;
    // Table entry e of an implicit descriptor (mined plans only).
    int32_t implicit_entry(int64_t ci, int d, int64_t e, const int32_t* row_offsets,
                           const int32_t* col_indices) const;
};

// inspect (miner.cpp:281-323), bit-exact.
Plan inspect(int kernel, const psc_csr_view& a, int t, int target_groups, int threads);

// The schedule and windows of inspect (compute_access_functions validation,
// scheduler.cpp:9-105, get_consecutive_iterations miner.cpp:18-37): window w
// covers rows [begin[w], end[w]); partition p owns windows
// [part_win_ptr[p], part_win_ptr[p + 1]).
struct WindowSchedule {
    std::vector<int32_t> begin, end;
    std::vector<int64_t> part_win_ptr{0};
};
WindowSchedule schedule_windows(int kernel, const psc_csr_view& a, int t, int target_groups);

// inspect with the window mining on a GPU (cuda/inspect.cu): the same plan.
Plan inspect_device(int kernel, const psc_csr_view& a, int t, int target_groups, int device);

void plan_counts(const Plan& p, psc_plan_counts* c);
void plan_to_arrays(const Plan& p, const psc_csr_view* a, psc_plan_arrays* out);
Plan plan_from_arrays(const psc_plan_counts& c, const psc_plan_arrays& a);
uint64_t plan_hash(const Plan& p, const psc_csr_view* a);
void validate_plan(const Plan& p, const psc_csr_view& a);
int64_t codelet_cost(int kind, int m, int n, int64_t table_entries_out, int64_t table_entries_mat,
                     int64_t table_entries_vec, bool out_tab, bool mat_tab, bool vec_tab);

}  // namespace pscb
