// oracle/ref_shim.cpp — TEST INFRASTRUCTURE, not product code.
//
// A thin extern "C" shim over the UNMODIFIED reference library, compiled
// from the sources where they lie under /root/reference/proj/core/src by
// oracle/Makefile into oracle/_ref/libpsc_ref.so. It exposes the reference's
// public API (psc::inspect, psc::Executor, psc::run_spmv, psc::run_sptrsv, the
// naive baselines, exec_*_codelet, pattern generators and the test helpers)
// to the Python test-suite and to bench.py's reference arm. Nothing here
// re-implements reference behaviour; it only converts between plain arrays
// and the reference's C++ types.
#include <chrono>
#include <cstdint>
#include <cstring>
#include <exception>
#include <span>
#include <stdexcept>
#include <string>
#include <vector>

#include "psc/codelet.hpp"
#include "psc/csr_matrix.hpp"
#include "psc/executor.hpp"
#include "psc/kernel_model.hpp"
#include "psc/miner.hpp"
#include "psc/pattern_gen.hpp"
#include "psc/scheduler.hpp"
#include "support/test_helpers.hpp"  // reference tests/support (random_unit_lower, int_vector, ...)

#include "psc_b200.h"
#include "psc/matrix_market.hpp"
#include "psc_plan_hash.h"

#define REF_API extern "C" __attribute__((visibility("default")))

namespace {

thread_local std::string g_err;

template <class F>
int guard(F&& f) {
    try {
        f();
        return PSC_OK;
    } catch (const std::invalid_argument& e) {
        g_err = e.what();
        return PSC_ERR_INVALID_ARGUMENT;
    } catch (const std::logic_error& e) {
        g_err = e.what();
        return PSC_ERR_LOGIC;
    } catch (const std::exception& e) {
        g_err = e.what();
        return PSC_ERR_INTERNAL;
    }
}

psc::CsrMatrix from_view(const psc_csr_view* v) {
    psc::CsrMatrix a;
    a.n_rows = v->n_rows;
    a.n_cols = v->n_cols;
    a.row_offsets.assign(v->row_offsets, v->row_offsets + v->n_rows + 1);
    a.col_indices.assign(v->col_indices, v->col_indices + v->nnz);
    a.values.assign(v->values, v->values + v->nnz);
    return a;
}

psc::AccessDesc desc_from_view(const psc_access_desc_view& d) {
    switch (d.form) {
        case PSC_FORM_STRIDED:
            return psc::AccessDesc::strided(d.base, d.stride_outer, d.stride_inner);
        case PSC_FORM_INNER_TABLE:
            return psc::AccessDesc::inner_table(std::vector<int>(d.table, d.table + d.table_len));
        case PSC_FORM_OUTER_TABLE:
            return psc::AccessDesc::outer_table(std::vector<int>(d.table, d.table + d.table_len));
        default:
            return psc::AccessDesc::point_table(std::vector<int>(d.table, d.table + d.table_len));
    }
}

psc::Codelet codelet_from_view(const psc_codelet_view* v) {
    psc::Codelet c;
    c.kind = static_cast<psc::CodeletKind>(v->kind);
    c.outer_extent = v->outer_extent;
    c.inner_extent = v->inner_extent;
    c.out = desc_from_view(v->out);
    c.mat = desc_from_view(v->mat);
    c.vec = desc_from_view(v->vec);
    return c;
}

struct RefCsr {
    psc::CsrMatrix m;
};

}  // namespace

REF_API const char* ref_last_error() { return g_err.c_str(); }

// ---- matrices ---------------------------------------------------------------
REF_API int ref_csr_from_view(const psc_csr_view* v, void** out) {
    return guard([&] { *out = new RefCsr{from_view(v)}; });
}
REF_API int ref_csr_view(void* h, psc_csr_view* out) {
    auto* r = static_cast<RefCsr*>(h);
    out->n_rows = r->m.n_rows;
    out->n_cols = r->m.n_cols;
    out->nnz = r->m.nnz();
    out->row_offsets = r->m.row_offsets.data();
    out->col_indices = r->m.col_indices.data();
    out->values = r->m.values.data();
    return PSC_OK;
}
REF_API void ref_csr_free(void* h) { delete static_cast<RefCsr*>(h); }

// read_matrix_market_file; on a ParseError, *line = its 1-based line
REF_API int ref_read_matrix_market(const char* path, void** out, int* line) {
    *line = 0;
    return guard([&] {
        try {
            *out = new RefCsr{psc::read_matrix_market_file(path)};
        } catch (const psc::ParseError& e) {
            *line = e.line();
            throw std::invalid_argument(e.what());
        }
    });
}

REF_API int ref_generate_pattern(const char* spec, uint64_t seed, void** out) {
    return guard([&] { *out = new RefCsr{psc::generate_pattern(spec, seed)}; });
}
REF_API int ref_csr_from_triplets(int n_rows, int n_cols, int64_t n, const int* rows,
                                  const int* cols, const double* vals, void** out) {
    return guard([&] {
        std::vector<psc::Triplet> t(n);
        for (int64_t i = 0; i < n; ++i) t[i] = {rows[i], cols[i], vals[i]};
        *out = new RefCsr{psc::csr_from_triplets(n_rows, n_cols, std::move(t))};
    });
}
REF_API int ref_lower_triangular(void* h, void** out) {
    return guard([&] {
        psc::TriangularMatrix l = psc::lower_triangular(static_cast<RefCsr*>(h)->m);
        *out = new RefCsr{l.csr()};
    });
}
REF_API int ref_random_unit_lower(int n, int max_extra, uint64_t seed, void** out) {
    return guard([&] { *out = new RefCsr{psc::test::random_unit_lower(n, max_extra, seed)}; });
}
REF_API int ref_unit_lower(void* h, void** out) {
    return guard([&] { *out = new RefCsr{psc::test::unit_lower(static_cast<RefCsr*>(h)->m)}; });
}
REF_API void ref_int_values(void* h, uint64_t seed) {
    psc::test::int_values(static_cast<RefCsr*>(h)->m, seed);
}
REF_API void ref_int_vector(int n, uint64_t seed, double* out) {
    std::vector<double> v = psc::test::int_vector(n, seed);
    std::memcpy(out, v.data(), sizeof(double) * v.size());
}

// ---- inspector --------------------------------------------------------------
struct RefPlan {
    psc::CodeletPlan plan;
};

REF_API int ref_inspect(int kernel, void* h, int t, int groups, void** out) {
    return guard([&] {
        auto* p = new RefPlan;
        p->plan = psc::inspect(static_cast<psc::KernelKind>(kernel), static_cast<RefCsr*>(h)->m,
                               t, groups);
        *out = p;
    });
}
REF_API void ref_plan_free(void* p) { delete static_cast<RefPlan*>(p); }

REF_API int ref_plan_counts(void* hp, psc_plan_counts* c) {
    const psc::CodeletPlan& p = static_cast<RefPlan*>(hp)->plan;
    std::memset(c, 0, sizeof *c);
    c->kernel = static_cast<int>(p.kernel);
    c->n_rows = p.n_rows;
    c->n_cols = p.n_cols;
    c->nnz = p.nnz;
    c->window = p.window;
    c->target_groups = p.target_groups;
    c->n_partitions = static_cast<int64_t>(p.partitions.size());
    for (const auto& part : p.partitions) {
        c->n_groups += static_cast<int64_t>(part.groups.size());
        for (const auto& g : part.groups) {
            c->n_codelets += static_cast<int64_t>(g.codelets.size());
            c->n_finalize += static_cast<int64_t>(g.finalize.size());
            for (const auto& cd : g.codelets) {
                c->n_table += static_cast<int64_t>(cd.out.table.size() + cd.mat.table.size() +
                                                   cd.vec.table.size());
            }
        }
    }
    return PSC_OK;
}

REF_API int ref_plan_export(void* hp, psc_plan_arrays* a) {
    const psc::CodeletPlan& p = static_cast<RefPlan*>(hp)->plan;
    int64_t gi = 0, ci = 0, fi = 0, ti = 0;
    a->part_group_ptr[0] = 0;
    a->group_codelet_ptr[0] = 0;
    a->group_finalize_ptr[0] = 0;
    a->desc_table_ptr[0] = 0;
    for (std::size_t pi = 0; pi < p.partitions.size(); ++pi) {
        for (const auto& g : p.partitions[pi].groups) {
            a->group_row_begin[gi] = g.window.row_begin;
            a->group_row_end[gi] = g.window.row_end;
            a->group_strategy[gi] = static_cast<int>(g.strategy);
            a->group_cost[gi] = g.cost;
            for (const auto& c : g.codelets) {
                a->codelet_kind[ci] = static_cast<int>(c.kind);
                a->codelet_m[ci] = c.outer_extent;
                a->codelet_n[ci] = c.inner_extent;
                const psc::AccessDesc* ds[3] = {&c.out, &c.mat, &c.vec};
                for (int d = 0; d < 3; ++d) {
                    int64_t k = 3 * ci + d;
                    a->desc_form[k] = static_cast<int>(ds[d]->form);
                    a->desc_base[k] = ds[d]->lin.base;
                    a->desc_stride_outer[k] = ds[d]->lin.stride_outer;
                    a->desc_stride_inner[k] = ds[d]->lin.stride_inner;
                    for (int v : ds[d]->table) a->table[ti++] = v;
                    a->desc_table_ptr[k + 1] = ti;
                }
                ++ci;
            }
            for (const auto& f : g.finalize) {
                a->fin_row[fi] = f.row;
                a->fin_diag_pos[fi] = f.diag_pos;
                a->fin_rhs_index[fi] = f.rhs_index;
                ++fi;
            }
            ++gi;
            a->group_codelet_ptr[gi] = ci;
            a->group_finalize_ptr[gi] = fi;
        }
        a->part_group_ptr[pi + 1] = gi;
    }
    return PSC_OK;
}

REF_API uint64_t ref_plan_hash(void* hp) {
    const psc::CodeletPlan& p = static_cast<RefPlan*>(hp)->plan;
    uint64_t h = PSC_HASH_SEED;
    auto mix = [&](int64_t v) { h = psc_hash_mix(h, static_cast<uint64_t>(v)); };
    mix(static_cast<int>(p.kernel));
    mix(p.n_rows);
    mix(p.n_cols);
    mix(p.nnz);
    mix(p.window);
    mix(p.target_groups);
    mix(static_cast<int64_t>(p.partitions.size()));
    for (const auto& part : p.partitions) {
        mix(static_cast<int64_t>(part.groups.size()));
        for (const auto& g : part.groups) {
            mix(g.window.row_begin);
            mix(g.window.row_end);
            mix(static_cast<int>(g.strategy));
            mix(g.cost);
            mix(static_cast<int64_t>(g.codelets.size()));
            for (const auto& c : g.codelets) {
                mix(static_cast<int>(c.kind));
                mix(c.outer_extent);
                mix(c.inner_extent);
                for (const psc::AccessDesc* d : {&c.out, &c.mat, &c.vec}) {
                    mix(static_cast<int>(d->form));
                    mix(d->lin.base);
                    mix(d->lin.stride_outer);
                    mix(d->lin.stride_inner);
                    mix(static_cast<int64_t>(d->table.size()));
                    for (int v : d->table) mix(v);
                }
            }
            mix(static_cast<int64_t>(g.finalize.size()));
            for (const auto& f : g.finalize) {
                mix(f.row);
                mix(f.diag_pos);
                mix(f.rhs_index);
            }
        }
    }
    return h;
}

REF_API void ref_plan_totals(void* hp, int64_t* cost, int64_t* ops) {
    const psc::CodeletPlan& p = static_cast<RefPlan*>(hp)->plan;
    *cost = p.total_cost();
    *ops = p.total_ops();
}

// Strategy costs of one window, for strategy-minimum checks (acceptance #5).
REF_API int ref_strategy_costs(int kernel, void* h, int row_begin, int row_end, int64_t out[3]) {
    return guard([&] {
        psc::KernelModel m =
            psc::compute_access_functions(static_cast<psc::KernelKind>(kernel),
                                          static_cast<RefCsr*>(h)->m);
        psc::RowWindow w{row_begin, row_end};
        out[0] = psc::blas_first(m, w).cost;
        out[1] = psc::psci_first(m, w).cost;
        out[2] = psc::pscii_first(m, w).cost;
    });
}

// ---- executor -----------------------------------------------------------------
REF_API int ref_run_spmv(void* hp, void* ha, const double* x, double* y, int workers) {
    return guard([&] {
        const psc::CsrMatrix& a = static_cast<RefCsr*>(ha)->m;
        psc::Executor exec(workers);
        psc::run_spmv(static_cast<RefPlan*>(hp)->plan, a, std::span<const double>(x, a.n_cols),
                      std::span<double>(y, a.n_rows), exec);
    });
}
REF_API int ref_run_sptrsv(void* hp, void* hl, const double* b, double* x, double* acc,
                           int workers) {
    return guard([&] {
        psc::TriangularMatrix l = psc::TriangularMatrix::adopt(static_cast<RefCsr*>(hl)->m);
        int n = l.n();
        psc::Executor exec(workers);
        psc::run_sptrsv(static_cast<RefPlan*>(hp)->plan, l, std::span<const double>(b, n),
                        std::span<double>(x, n), std::span<double>(acc, n), exec);
    });
}
REF_API int ref_spmv_baseline(void* ha, const double* x, double* y) {
    return guard([&] {
        const psc::CsrMatrix& a = static_cast<RefCsr*>(ha)->m;
        std::vector<double> r = psc::spmv_csr_baseline(a, std::span<const double>(x, a.n_cols));
        std::memcpy(y, r.data(), sizeof(double) * r.size());
    });
}
REF_API int ref_sptrsv_baseline(void* hl, const double* b, double* x) {
    return guard([&] {
        psc::TriangularMatrix l = psc::TriangularMatrix::adopt(static_cast<RefCsr*>(hl)->m);
        std::vector<double> r = psc::sptrsv_csr_baseline(l, std::span<const double>(b, l.n()));
        std::memcpy(x, r.data(), sizeof(double) * r.size());
    });
}

// exec_*_codelet on host arrays (test_executor.cpp:37-138 known answers).
REF_API int ref_exec_codelet(int which, const psc_codelet_view* v, const psc_exec_context* c) {
    return guard([&] {
        psc::Codelet cd = codelet_from_view(v);
        psc::ExecutionContext ctx;
        ctx.matrix_values = c->matrix_values;
        ctx.gather = c->gather;
        ctx.accum = c->accum;
        ctx.rhs = c->rhs;
        ctx.solution = c->solution;
        if (which == 0) psc::exec_blas_codelet(cd, ctx);
        else if (which == 1) psc::exec_psci_codelet(cd, ctx);
        else psc::exec_pscii_codelet(cd, ctx);
    });
}

// ---- timing (bench.py --impl reference) ----------------------------------------
// One Executor for the whole run (the reference's run_bench does the same,
// bench.cpp:149); warm-up calls are untimed; each timed call is one complete
// run_spmv / run_sptrsv over the full matrix, timed with steady_clock as in
// bench.cpp:61-69.
REF_API int ref_time_spmv(void* hp, void* ha, const double* x, double* y, int workers,
                          int warmup, int reps, double* seconds) {
    return guard([&] {
        const psc::CsrMatrix& a = static_cast<RefCsr*>(ha)->m;
        psc::Executor exec(workers);
        std::span<const double> xs(x, a.n_cols);
        std::span<double> ys(y, a.n_rows);
        const psc::CodeletPlan& plan = static_cast<RefPlan*>(hp)->plan;
        for (int i = 0; i < warmup; ++i) psc::run_spmv(plan, a, xs, ys, exec);
        for (int i = 0; i < reps; ++i) {
            auto t0 = std::chrono::steady_clock::now();
            psc::run_spmv(plan, a, xs, ys, exec);
            auto t1 = std::chrono::steady_clock::now();
            seconds[i] = std::chrono::duration<double>(t1 - t0).count();
        }
    });
}
REF_API int ref_time_sptrsv(void* hp, void* hl, const double* b, double* x, double* acc,
                            int workers, int warmup, int reps, double* seconds) {
    return guard([&] {
        psc::TriangularMatrix l = psc::TriangularMatrix::adopt(static_cast<RefCsr*>(hl)->m);
        int n = l.n();
        psc::Executor exec(workers);
        const psc::CodeletPlan& plan = static_cast<RefPlan*>(hp)->plan;
        std::span<const double> bs(b, n);
        std::span<double> xs(x, n), as(acc, n);
        for (int i = 0; i < warmup; ++i) psc::run_sptrsv(plan, l, bs, xs, as, exec);
        for (int i = 0; i < reps; ++i) {
            auto t0 = std::chrono::steady_clock::now();
            psc::run_sptrsv(plan, l, bs, xs, as, exec);
            auto t1 = std::chrono::steady_clock::now();
            seconds[i] = std::chrono::duration<double>(t1 - t0).count();
        }
    });
}
REF_API int ref_time_inspect(int kernel, void* h, int t, int groups, double* seconds, void** out) {
    return guard([&] {
        auto* p = new RefPlan;
        auto t0 = std::chrono::steady_clock::now();
        p->plan = psc::inspect(static_cast<psc::KernelKind>(kernel), static_cast<RefCsr*>(h)->m,
                               t, groups);
        auto t1 = std::chrono::steady_clock::now();
        *seconds = std::chrono::duration<double>(t1 - t0).count();
        *out = p;
    });
}
