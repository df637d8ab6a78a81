/*
 * oracle/psc_oracle.c — TEST INFRASTRUCTURE ONLY (the parity checker).
 *
 * A plain-C restatement of the reference executor's arithmetic
 * (/root/reference/proj/core/src/executor.cpp) over the SoA plan view of
 * include/psc_b200.h. Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline leg may load it; the product never links or calls it.
 *
 * Parity is pinned two ways (tests/test_oracle.py): against the golden
 * vectors of the reference's own tests (test_executor.cpp known answers) and
 * bitwise against the reference library itself built from its sources
 * (oracle/_ref/libpsc_ref.so) on the 336-plan acceptance suite and on scaled
 * benchmark configs. Build flags: -ffp-contract=off, so every product is
 * rounded before it is added, as in the reference's default x86-64 build
 * (no FMA without -march).
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include "psc_b200.h"

static const char* g_msg = "";
const char* oracle_last_error(void) { return g_msg; }

/* executor.cpp:23-35 — four-lane dot product with a fixed lane order. */
static double dot_unit(const double* a, const double* b, int n) {
    double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
    int j = 0;
    for (; j + 4 <= n; j += 4) {
        s0 += a[j] * b[j];
        s1 += a[j + 1] * b[j + 1];
        s2 += a[j + 2] * b[j + 2];
        s3 += a[j + 3] * b[j + 3];
    }
    double sum = (s0 + s1) + (s2 + s3);
    for (; j < n; ++j) sum += a[j] * b[j];
    return sum;
}

/* executor.cpp:37-49 — same order through a column table. */
static double dot_gather(const double* a, const double* x, const int32_t* cols, int n) {
    double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
    int j = 0;
    for (; j + 4 <= n; j += 4) {
        s0 += a[j] * x[cols[j]];
        s1 += a[j + 1] * x[cols[j + 1]];
        s2 += a[j + 2] * x[cols[j + 2]];
        s3 += a[j + 3] * x[cols[j + 3]];
    }
    double sum = (s0 + s1) + (s2 + s3);
    for (; j < n; ++j) sum += a[j] * x[cols[j]];
    return sum;
}

static int is_table(int form) { return form != PSC_FORM_STRIDED; }

/* executor.cpp:53-73 */
static int exec_blas(const psc_codelet_view* c, const psc_exec_context* ctx) {
    if (is_table(c->out.form) || is_table(c->mat.form) || is_table(c->vec.form)) {
        g_msg = "exec_blas_codelet: descriptors must be strided";
        return PSC_ERR_INVALID_ARGUMENT;
    }
    const int n = c->inner_extent;
    const int msi = c->mat.stride_inner, vsi = c->vec.stride_inner;
    for (int i = 0; i < c->outer_extent; ++i) {
        const double* arow = ctx->matrix_values + c->mat.base + (long)i * c->mat.stride_outer;
        const double* xrow = ctx->gather + c->vec.base + (long)i * c->vec.stride_outer;
        double sum = 0.0;
        if (msi == 1 && vsi == 1 && ctx->rhs == NULL) {
            sum = dot_unit(arow, xrow, n);
        } else {
            for (int j = 0; j < n; ++j) sum += arow[j * msi] * xrow[j * vsi];
        }
        ctx->accum[c->out.base + i * c->out.stride_outer] += sum;
    }
    return PSC_OK;
}

/* executor.cpp:75-94 */
static int exec_psci(const psc_codelet_view* c, const psc_exec_context* ctx) {
    if (is_table(c->out.form) || is_table(c->mat.form) || !is_table(c->vec.form)) {
        g_msg = "exec_psci_codelet: expects one gather table";
        return PSC_ERR_INVALID_ARGUMENT;
    }
    const int32_t* cols = c->vec.table;
    const int n = c->inner_extent, msi = c->mat.stride_inner;
    for (int i = 0; i < c->outer_extent; ++i) {
        const double* arow = ctx->matrix_values + c->mat.base + (long)i * c->mat.stride_outer;
        double sum = 0.0;
        if (msi == 1 && ctx->rhs == NULL) {
            sum = dot_gather(arow, ctx->gather, cols, n);
        } else {
            for (int j = 0; j < n; ++j) sum += arow[j * msi] * ctx->gather[cols[j]];
        }
        ctx->accum[c->out.base + i * c->out.stride_outer] += sum;
    }
    return PSC_OK;
}

/* executor.cpp:96-116 */
static int exec_pscii(const psc_codelet_view* c, const psc_exec_context* ctx) {
    if (!is_table(c->out.form) || is_table(c->mat.form) || !is_table(c->vec.form)) {
        g_msg = "exec_pscii_codelet: expects output and gather tables";
        return PSC_ERR_INVALID_ARGUMENT;
    }
    const int n = c->inner_extent, msi = c->mat.stride_inner;
    const int per_point = c->vec.form == PSC_FORM_POINT_TABLE;
    for (int i = 0; i < c->outer_extent; ++i) {
        const double* arow = ctx->matrix_values + c->mat.base + (long)i * c->mat.stride_outer;
        const int32_t* cols = per_point ? c->vec.table + (long)i * n : c->vec.table;
        double sum = 0.0;
        if (msi == 1 && ctx->rhs == NULL) {
            sum = dot_gather(arow, ctx->gather, cols, n);
        } else {
            for (int j = 0; j < n; ++j) sum += arow[j * msi] * ctx->gather[cols[j]];
        }
        ctx->accum[c->out.table[i]] += sum;
    }
    return PSC_OK;
}

int oracle_exec_codelet(int which, const psc_codelet_view* c, const psc_exec_context* ctx) {
    if (which == PSC_CODELET_BLAS) return exec_blas(c, ctx);
    if (which == PSC_CODELET_PSC_I) return exec_psci(c, ctx);
    return exec_pscii(c, ctx);
}

static void codelet_at(const psc_plan_arrays* a, int64_t ci, psc_codelet_view* v) {
    psc_access_desc_view* ds[3] = {&v->out, &v->mat, &v->vec};
    v->kind = a->codelet_kind[ci];
    v->outer_extent = a->codelet_m[ci];
    v->inner_extent = a->codelet_n[ci];
    for (int d = 0; d < 3; ++d) {
        int64_t k = 3 * ci + d;
        ds[d]->form = a->desc_form[k];
        ds[d]->base = a->desc_base[k];
        ds[d]->stride_outer = a->desc_stride_outer[k];
        ds[d]->stride_inner = a->desc_stride_inner[k];
        ds[d]->table = a->table + a->desc_table_ptr[k];
        ds[d]->table_len = a->desc_table_ptr[k + 1] - a->desc_table_ptr[k];
    }
}

/* executor.cpp:120-134 (exec_codelet switch + exec_group) and 261-267
 * (partitions in order; groups of a partition are independent, so running
 * them in index order equals any worker count). */
static int run_plan(const psc_plan_counts* pc, const psc_plan_arrays* a,
                    const psc_exec_context* ctx) {
    for (int64_t p = 0; p < pc->n_partitions; ++p) {
        for (int64_t g = a->part_group_ptr[p]; g < a->part_group_ptr[p + 1]; ++g) {
            for (int64_t ci = a->group_codelet_ptr[g]; ci < a->group_codelet_ptr[g + 1]; ++ci) {
                psc_codelet_view v;
                codelet_at(a, ci, &v);
                int which = v.kind == PSC_CODELET_BLAS   ? PSC_CODELET_BLAS
                            : v.kind == PSC_CODELET_PSC_I ? PSC_CODELET_PSC_I
                                                          : PSC_CODELET_PSC_II;
                int st = oracle_exec_codelet(which, &v, ctx);
                if (st) return st;
            }
            for (int64_t f = a->group_finalize_ptr[g]; f < a->group_finalize_ptr[g + 1]; ++f) {
                int32_t r = a->fin_row[f];
                ctx->solution[r] = (ctx->rhs[a->fin_rhs_index[f]] - ctx->accum[r]) /
                                   ctx->matrix_values[a->fin_diag_pos[f]];
            }
        }
    }
    return PSC_OK;
}

/* executor.cpp:274-288 */
int oracle_run_spmv(const psc_plan_counts* pc, const psc_plan_arrays* a, const psc_csr_view* m,
                    const double* x, double* y) {
    if (pc->kernel != PSC_KERNEL_SPMV) {
        g_msg = "run_spmv: plan was built for another kernel";
        return PSC_ERR_INVALID_ARGUMENT;
    }
    memset(y, 0, sizeof(double) * (size_t)m->n_rows);
    psc_exec_context ctx = {m->values, x, y, NULL, NULL};
    return run_plan(pc, a, &ctx);
}

/* executor.cpp:290-308 */
int oracle_run_sptrsv(const psc_plan_counts* pc, const psc_plan_arrays* a, const psc_csr_view* m,
                      const double* b, double* x, double* acc) {
    if (pc->kernel != PSC_KERNEL_SPTRSV) {
        g_msg = "run_sptrsv: plan was built for another kernel";
        return PSC_ERR_INVALID_ARGUMENT;
    }
    memset(acc, 0, sizeof(double) * (size_t)m->n_rows);
    psc_exec_context ctx = {m->values, x, acc, b, x};
    return run_plan(pc, a, &ctx);
}

/* executor.cpp:310-323 */
void oracle_spmv_baseline(const psc_csr_view* m, const double* x, double* y) {
    for (int i = 0; i < m->n_rows; ++i) {
        double sum = 0.0;
        for (int k = m->row_offsets[i]; k < m->row_offsets[i + 1]; ++k)
            sum += m->values[k] * x[m->col_indices[k]];
        y[i] = sum;
    }
}

/* executor.cpp:325-340 (diagonal stored last, csr_matrix.hpp:49) */
void oracle_sptrsv_baseline(const psc_csr_view* m, const double* b, double* x) {
    for (int i = 0; i < m->n_rows; ++i) {
        double sum = 0.0;
        int diag = m->row_offsets[i + 1] - 1;
        for (int k = m->row_offsets[i]; k < diag; ++k) sum += m->values[k] * x[m->col_indices[k]];
        x[i] = (b[i] - sum) / m->values[diag];
    }
}
