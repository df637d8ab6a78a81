// C ABI, host half: errors, matrices, generators, inspector and plans.
// Executor / device entry points live in csrc/cuda/executor.cu.
#include <algorithm>
#include <cstring>
#include <memory>
#include <string>

#include "capi_types.hpp"
#include "common.hpp"
#include "configs.hpp"
#include "csr.hpp"
#include "plan.hpp"

namespace pscb {
namespace {
thread_local std::string g_last_error;
}
void set_last_error(const std::string& msg) { g_last_error = msg; }
}  // namespace pscb

using namespace pscb;

extern "C" {

PSC_API const char* psc_last_error(void) { return g_last_error.c_str(); }

// ---- matrices ----------------------------------------------------------------
PSC_API psc_status psc_csr_view_of(const psc_csr* m, psc_csr_view* out) {
    return guarded([&] {
        require(m && out, "psc_csr_view_of: null argument");
        *out = m->m.view();
    });
}
PSC_API void psc_csr_destroy(psc_csr* m) { delete m; }

PSC_API psc_status psc_csr_from_triplets(int32_t n_rows, int32_t n_cols, int64_t n, const int32_t* rows,
                                         const int32_t* cols, const double* vals, psc_csr** out) {
    return guarded([&] {
        std::vector<Triplet> t(n);
        for (int64_t i = 0; i < n; ++i) t[i] = {rows[i], cols[i], vals[i]};
        *out = new psc_csr{csr_from_triplets(n_rows, n_cols, std::move(t))};
    });
}
PSC_API psc_status psc_validate_csr(const psc_csr_view* a) {
    return guarded([&] {
        require(a != nullptr, "psc_validate_csr: null matrix");
        validate_csr(*a);
    });
}
PSC_API psc_status psc_lower_triangular(const psc_csr_view* a, psc_csr** out) {
    return guarded([&] { *out = new psc_csr{lower_triangular(*a)}; });
}
PSC_API psc_status psc_adopt_triangular(const psc_csr_view* a) {
    return guarded([&] { adopt_triangular(*a); });
}
// The reference's sequential baselines (executor.cpp:310-340, SURVEY.md §8a
// row A13): the NER / verification baselines of the bench report. Plain
// host loops, built without -march (no FMA contraction).
PSC_API psc_status psc_csr_spmv_baseline(const psc_csr_view* a, const double* x, int64_t nx, double* y, int64_t ny) {
    return guarded([&] {
        require(a && x && y, "spmv_csr_baseline: null argument");
        require(nx == a->n_cols && ny == a->n_rows, "spmv_csr_baseline: vector size mismatch");
        for (int32_t i = 0; i < a->n_rows; ++i) {
            double sum = 0.0;
            for (int32_t k = a->row_offsets[i]; k < a->row_offsets[i + 1]; ++k) sum += a->values[k] * x[a->col_indices[k]];
            y[i] = sum;
        }
    });
}
PSC_API psc_status psc_csr_sptrsv_baseline(const psc_csr_view* l, const double* b, int64_t nb, double* x, int64_t nx) {
    return guarded([&] {
        require(l && b && x, "sptrsv_csr_baseline: null argument");
        require(nb == l->n_rows && nx == l->n_rows, "sptrsv_csr_baseline: vector size mismatch");
        for (int32_t i = 0; i < l->n_rows; ++i) {
            double sum = 0.0;
            const int32_t diag = l->row_offsets[i + 1] - 1;  // diagonal stored last (csr_matrix.hpp:49)
            for (int32_t k = l->row_offsets[i]; k < diag; ++k) sum += l->values[k] * x[l->col_indices[k]];
            x[i] = (b[i] - sum) / l->values[diag];
        }
    });
}

PSC_API psc_status psc_generate_config(int32_t config, double scale, uint64_t seed, psc_csr** out) {
    return guarded([&] { *out = new psc_csr{generate_config(config, scale, seed)}; });
}

PSC_API void psc_seeded_vector(int64_t n, uint64_t seed, double* out) { seeded_vector(n, seed, out); }
PSC_API void psc_uniform_vector(int64_t n, uint64_t seed, double lo, double hi, double* out) {
    uniform_vector(n, seed, lo, hi, out);
}
PSC_API void psc_int_vector(int64_t n, uint64_t seed, double* out) { int_vector(n, seed, out); }

// ---- inspector / plans ----------------------------------------------------------
PSC_API psc_status psc_inspect(int32_t kernel, const psc_csr_view* a, int32_t t, int32_t target_groups,
                               int32_t threads, psc_plan** out) {
    return guarded([&] {
        require(a != nullptr && out != nullptr, "inspect: null argument");
        Plan p = inspect(kernel, *a, t, target_groups, threads);
        p.structure = structure_hash(*a);
        *out = new psc_plan(std::move(p));
    });
}
PSC_API psc_status psc_plan_get_counts(const psc_plan* plan, psc_plan_counts* out) {
    return guarded([&] {
        require(plan && out, "psc_plan_get_counts: null argument");
        plan_counts(plan->p, out);
    });
}
PSC_API psc_status psc_plan_to_arrays(const psc_plan* plan, const psc_csr_view* a, psc_plan_arrays* out) {
    return guarded([&] {
        require(plan && out, "psc_plan_to_arrays: null argument");
        plan_to_arrays(plan->p, a, out);
    });
}
PSC_API psc_status psc_plan_from_arrays(const psc_plan_counts* counts, const psc_plan_arrays* arrays,
                                        psc_plan** out) {
    return guarded([&] {
        require(counts && arrays && out, "psc_plan_from_arrays: null argument");
        *out = new psc_plan(plan_from_arrays(*counts, *arrays));
    });
}
PSC_API psc_status psc_plan_hash(const psc_plan* plan, const psc_csr_view* a, uint64_t* out) {
    return guarded([&] {
        require(plan && out, "psc_plan_hash: null argument");
        *out = plan_hash(plan->p, a);
    });
}
PSC_API psc_status psc_plan_totals(const psc_plan* plan, int64_t* total_cost, int64_t* total_ops,
                                   int64_t ops_by_kind[3]) {
    return guarded([&] {
        require(plan != nullptr, "psc_plan_totals: null plan");
        const Plan& p = plan->p;
        int64_t cost = 0, ops = 0, by[3] = {0, 0, 0};
        for (int64_t c : p.g_cost) cost += c;  // CodeletPlan::total_cost, miner.cpp:263-269
        for (int64_t c = 0; c < p.n_codelets(); ++c) {
            int64_t o = static_cast<int64_t>(p.c_m[c]) * p.c_n[c];
            ops += o;
            if (p.c_kind[c] < 3) by[p.c_kind[c]] += o;
        }
        if (total_cost) *total_cost = cost;
        if (total_ops) *total_ops = ops;
        if (ops_by_kind) std::memcpy(ops_by_kind, by, sizeof by);
    });
}
PSC_API psc_status psc_plan_partition_rows(const psc_plan* plan, int64_t part_begin, int64_t part_end,
                                           int32_t* row_begin, int32_t* row_end) {
    return guarded([&] {
        require(plan && row_begin && row_end, "psc_plan_partition_rows: null argument");
        const Plan& p = plan->p;
        require(0 <= part_begin && part_begin <= part_end && part_end <= p.n_partitions(),
                "psc_plan_partition_rows: partition range out of bounds");
        int64_t g0 = p.part_group_ptr[part_begin], g1 = p.part_group_ptr[part_end];
        int32_t rb = p.n_rows, re = 0;
        int64_t rows = 0;
        for (int64_t g = g0; g < g1; ++g) {
            rb = std::min(rb, p.g_row_begin[g]);
            re = std::max(re, p.g_row_end[g]);
            rows += p.g_row_end[g] - p.g_row_begin[g];
        }
        if (g0 == g1) rb = re = 0;
        require(rows == static_cast<int64_t>(re) - rb,
                "psc_plan_partition_rows: partitions do not cover a contiguous row range");
        *row_begin = rb;
        *row_end = re;
    });
}
PSC_API psc_status psc_validate_plan(const psc_plan* plan, const psc_csr_view* a) {
    return guarded([&] {
        require(plan && a, "psc_validate_plan: null argument");
        validate_plan(plan->p, *a);
    });
}
PSC_API void psc_plan_destroy(psc_plan* plan) { delete plan; }

}  // extern "C"
