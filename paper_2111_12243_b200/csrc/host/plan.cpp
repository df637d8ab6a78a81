// Plan storage, export/import, canonical hash and validate_plan.
#include "plan.hpp"

#include <algorithm>
#include <string>

#include "common.hpp"
#include "csr.hpp"
#include "psc_plan_hash.h"

namespace pscb {

int64_t Plan::n_finalize() const {
    if (!mined) return static_cast<int64_t>(f_row.size());
    return kernel == PSC_KERNEL_SPTRSV ? n_rows : 0;
}

int64_t Plan::n_table() const {
    if (!mined) return static_cast<int64_t>(tables.size());
    int64_t total = 0;
    for (int64_t c = 0; c < n_codelets(); ++c) {
        int64_t m = c_m[c], n = c_n[c];
        if (c_kind[c] == PSC_CODELET_PSC_I) total += n;
        else if (c_kind[c] == PSC_CODELET_PSC_II) total += m + m * n;
    }
    return total;
}

DescView Plan::desc(int64_t ci, int d) const {
    DescView v;
    if (!mined) {
        int64_t k = 3 * ci + d;
        v.form = d_form[k];
        v.base = d_base[k];
        v.so = d_so[k];
        v.si = d_si[k];
        v.len = d_tab_ptr[k + 1] - d_tab_ptr[k];
        v.tab = tables.data() + d_tab_ptr[k];
        return v;
    }
    const int kind = c_kind[ci];
    const int m = c_m[ci], n = c_n[ci];
    // Descriptor factories exactly as miner.cpp:110-112, 160-164, 210-226.
    if (d == 0) {
        if (kind == PSC_CODELET_PSC_II) {
            v.form = PSC_FORM_OUTER_TABLE;
            v.len = m;
        } else {
            v.base = c_row[ci];
            v.so = m > 1 ? 1 : 0;
        }
    } else if (d == 1) {
        v.base = c_mat_base[ci];
        v.so = c_mat_so[ci];
        v.si = 1;
    } else {
        if (kind == PSC_CODELET_BLAS) {
            v.base = c_vec_base[ci];
            v.so = c_vec_so[ci];
            v.si = 1;
        } else if (kind == PSC_CODELET_PSC_I || m == 1) {
            v.form = PSC_FORM_INNER_TABLE;
            v.len = n;
        } else {
            v.form = PSC_FORM_POINT_TABLE;
            v.len = static_cast<int64_t>(m) * n;
        }
    }
    return v;
}

int32_t Plan::implicit_entry(int64_t ci, int d, int64_t e, const int32_t*,
                             const int32_t* col) const {
    if (d == 0) return c_row[ci] + static_cast<int32_t>(e);  // PSC_II out table r..r+m-1
    const int n = c_n[ci];
    if (c_kind[ci] == PSC_CODELET_PSC_I || c_m[ci] == 1) return col[c_mat_base[ci] + e];
    int64_t i = e / n, j = e % n;  // point table: col_indices[mat.at(i, j)]
    return col[c_mat_base[ci] + i * c_mat_so[ci] + j];
}

void plan_counts(const Plan& p, psc_plan_counts* c) {
    c->kernel = p.kernel;
    c->n_rows = p.n_rows;
    c->n_cols = p.n_cols;
    c->window = p.window;
    c->target_groups = p.target_groups;
    c->nnz = p.nnz;
    c->n_partitions = p.n_partitions();
    c->n_groups = p.n_groups();
    c->n_codelets = p.n_codelets();
    c->n_finalize = p.n_finalize();
    c->n_table = p.n_table();
}

namespace {

void check_matrix_for(const Plan& p, const psc_csr_view* a) {
    require(a != nullptr, "plan: a mined plan needs its matrix to materialise tables");
    require(a->n_rows == p.n_rows && a->nnz == p.nnz, "plan: matrix does not match the plan");
}

// Visit the finalize records of group g: fn(row, diag_pos, rhs_index).
template <class F>
void for_finalize(const Plan& p, const psc_csr_view* a, int64_t g, F&& fn) {
    if (!p.mined) {
        for (int64_t f = p.g_fin_ptr[g]; f < p.g_fin_ptr[g + 1]; ++f) fn(p.f_row[f], p.f_diag[f], p.f_rhs[f]);
        return;
    }
    if (p.kernel != PSC_KERNEL_SPTRSV) return;
    for (int32_t r = p.g_row_begin[g]; r < p.g_row_end[g]; ++r) fn(r, a->row_offsets[r + 1] - 1, r);
}

}  // namespace

void plan_to_arrays(const Plan& p, const psc_csr_view* a, psc_plan_arrays* o) {
    if (p.mined) check_matrix_for(p, a);
    const int64_t G = p.n_groups(), C = p.n_codelets();
    std::copy(p.part_group_ptr.begin(), p.part_group_ptr.end(), o->part_group_ptr);
    std::copy(p.g_row_begin.begin(), p.g_row_begin.end(), o->group_row_begin);
    std::copy(p.g_row_end.begin(), p.g_row_end.end(), o->group_row_end);
    for (int64_t g = 0; g < G; ++g) o->group_strategy[g] = p.g_strategy[g];
    std::copy(p.g_cost.begin(), p.g_cost.end(), o->group_cost);
    std::copy(p.g_codelet_ptr.begin(), p.g_codelet_ptr.end(), o->group_codelet_ptr);
    int64_t fi = 0;
    o->group_finalize_ptr[0] = 0;
    for (int64_t g = 0; g < G; ++g) {
        for_finalize(p, a, g, [&](int32_t r, int32_t dpos, int32_t rhs) {
            o->fin_row[fi] = r;
            o->fin_diag_pos[fi] = dpos;
            o->fin_rhs_index[fi] = rhs;
            ++fi;
        });
        o->group_finalize_ptr[g + 1] = fi;
    }
    int64_t ti = 0;
    o->desc_table_ptr[0] = 0;
    for (int64_t c = 0; c < C; ++c) {
        o->codelet_kind[c] = p.c_kind[c];
        o->codelet_m[c] = p.c_m[c];
        o->codelet_n[c] = p.c_n[c];
        for (int d = 0; d < 3; ++d) {
            DescView v = p.desc(c, d);
            int64_t k = 3 * c + d;
            o->desc_form[k] = v.form;
            o->desc_base[k] = v.base;
            o->desc_stride_outer[k] = v.so;
            o->desc_stride_inner[k] = v.si;
            for (int64_t e = 0; e < v.len; ++e)
                o->table[ti++] = v.tab ? v.tab[e] : p.implicit_entry(c, d, e, a->row_offsets, a->col_indices);
            o->desc_table_ptr[k + 1] = ti;
        }
    }
}

Plan plan_from_arrays(const psc_plan_counts& c, const psc_plan_arrays& a) {
    require(c.kernel == PSC_KERNEL_SPMV || c.kernel == PSC_KERNEL_SPTRSV, "plan: unknown kernel");
    require(c.n_rows >= 0 && c.n_cols >= 0 && c.nnz >= 0 && c.n_partitions >= 0 && c.n_groups >= 0 &&
                c.n_codelets >= 0 && c.n_finalize >= 0 && c.n_table >= 0,
            "plan: negative count");
    Plan p;
    p.mined = false;
    p.kernel = c.kernel;
    p.n_rows = c.n_rows;
    p.n_cols = c.n_cols;
    p.nnz = c.nnz;
    p.window = c.window;
    p.target_groups = c.target_groups;
    p.part_group_ptr.assign(a.part_group_ptr, a.part_group_ptr + c.n_partitions + 1);
    require(p.part_group_ptr.front() == 0 && p.part_group_ptr.back() == c.n_groups,
            "plan: partition/group offsets inconsistent");
    p.g_row_begin.assign(a.group_row_begin, a.group_row_begin + c.n_groups);
    p.g_row_end.assign(a.group_row_end, a.group_row_end + c.n_groups);
    p.g_strategy.resize(c.n_groups);
    for (int64_t g = 0; g < c.n_groups; ++g) p.g_strategy[g] = static_cast<uint8_t>(a.group_strategy[g]);
    p.g_cost.assign(a.group_cost, a.group_cost + c.n_groups);
    p.g_codelet_ptr.assign(a.group_codelet_ptr, a.group_codelet_ptr + c.n_groups + 1);
    p.g_fin_ptr.assign(a.group_finalize_ptr, a.group_finalize_ptr + c.n_groups + 1);
    require(p.g_codelet_ptr.front() == 0 && p.g_codelet_ptr.back() == c.n_codelets,
            "plan: group/codelet offsets inconsistent");
    require(p.g_fin_ptr.front() == 0 && p.g_fin_ptr.back() == c.n_finalize,
            "plan: group/finalize offsets inconsistent");
    for (int64_t i = 0; i + 1 < static_cast<int64_t>(p.part_group_ptr.size()); ++i)
        require(p.part_group_ptr[i] <= p.part_group_ptr[i + 1], "plan: partition offsets not monotone");
    for (int64_t g = 0; g < c.n_groups; ++g)
        require(p.g_codelet_ptr[g] <= p.g_codelet_ptr[g + 1] && p.g_fin_ptr[g] <= p.g_fin_ptr[g + 1],
                "plan: group offsets not monotone");
    p.c_kind.resize(c.n_codelets);
    for (int64_t i = 0; i < c.n_codelets; ++i) p.c_kind[i] = static_cast<uint8_t>(a.codelet_kind[i]);
    p.c_m.assign(a.codelet_m, a.codelet_m + c.n_codelets);
    p.c_n.assign(a.codelet_n, a.codelet_n + c.n_codelets);
    p.d_form.assign(a.desc_form, a.desc_form + 3 * c.n_codelets);
    p.d_base.assign(a.desc_base, a.desc_base + 3 * c.n_codelets);
    p.d_so.assign(a.desc_stride_outer, a.desc_stride_outer + 3 * c.n_codelets);
    p.d_si.assign(a.desc_stride_inner, a.desc_stride_inner + 3 * c.n_codelets);
    p.d_tab_ptr.assign(a.desc_table_ptr, a.desc_table_ptr + 3 * c.n_codelets + 1);
    require(p.d_tab_ptr.front() == 0 && p.d_tab_ptr.back() == c.n_table, "plan: table offsets inconsistent");
    for (int64_t k = 0; k < 3 * c.n_codelets; ++k) {
        require(p.d_tab_ptr[k] <= p.d_tab_ptr[k + 1], "plan: table offsets not monotone");
        require(p.d_form[k] >= PSC_FORM_STRIDED && p.d_form[k] <= PSC_FORM_POINT_TABLE, "plan: bad descriptor form");
    }
    p.tables.assign(a.table, a.table + c.n_table);
    p.f_row.assign(a.fin_row, a.fin_row + c.n_finalize);
    p.f_diag.assign(a.fin_diag_pos, a.fin_diag_pos + c.n_finalize);
    p.f_rhs.assign(a.fin_rhs_index, a.fin_rhs_index + c.n_finalize);
    return p;
}

uint64_t plan_hash(const Plan& p, const psc_csr_view* a) {
    if (p.mined) check_matrix_for(p, a);
    uint64_t h = PSC_HASH_SEED;
    auto mix = [&](int64_t v) { h = psc_hash_mix(h, static_cast<uint64_t>(v)); };
    mix(p.kernel);
    mix(p.n_rows);
    mix(p.n_cols);
    mix(p.nnz);
    mix(p.window);
    mix(p.target_groups);
    mix(p.n_partitions());
    for (int64_t part = 0; part < p.n_partitions(); ++part) {
        mix(p.part_group_ptr[part + 1] - p.part_group_ptr[part]);
        for (int64_t g = p.part_group_ptr[part]; g < p.part_group_ptr[part + 1]; ++g) {
            mix(p.g_row_begin[g]);
            mix(p.g_row_end[g]);
            mix(p.g_strategy[g]);
            mix(p.g_cost[g]);
            mix(p.g_codelet_ptr[g + 1] - p.g_codelet_ptr[g]);
            for (int64_t c = p.g_codelet_ptr[g]; c < p.g_codelet_ptr[g + 1]; ++c) {
                mix(p.c_kind[c]);
                mix(p.c_m[c]);
                mix(p.c_n[c]);
                for (int d = 0; d < 3; ++d) {
                    DescView v = p.desc(c, d);
                    mix(v.form);
                    mix(v.base);
                    mix(v.so);
                    mix(v.si);
                    mix(v.len);
                    for (int64_t e = 0; e < v.len; ++e)
                        mix(v.tab ? v.tab[e] : p.implicit_entry(c, d, e, a->row_offsets, a->col_indices));
                }
            }
            int64_t nf = 0;
            for_finalize(p, a, g, [&](int32_t, int32_t, int32_t) { ++nf; });
            mix(nf);
            for_finalize(p, a, g, [&](int32_t r, int32_t dpos, int32_t rhs) {
                mix(r);
                mix(dpos);
                mix(rhs);
            });
        }
    }
    return h;
}

int64_t codelet_cost(int, int m, int n, int64_t te_out, int64_t te_mat, int64_t te_vec, bool out_tab,
                     bool mat_tab, bool vec_tab) {
    int64_t dims = (m > 1 ? 1 : 0) + (n > 1 ? 1 : 0);
    if (dims == 0) dims = 1;
    return int64_t(m) * n + 3 + (out_tab ? te_out : dims) + (mat_tab ? te_mat : dims) +
           (vec_tab ? te_vec : dims);
}

// validate_plan, miner.cpp:325-395, over the generic descriptor view.
void validate_plan(const Plan& p, const psc_csr_view& a) {
    if (p.kernel == PSC_KERNEL_SPTRSV) adopt_triangular(a);
    else validate_csr(a);
    if (p.n_rows != a.n_rows) throw std::logic_error("plan: row count does not match the kernel model");
    const int sp = p.kernel == PSC_KERNEL_SPTRSV ? 1 : 0;
    const int32_t* ro = a.row_offsets;
    // flat_of_mat: operation index of each stored position, -1 for non-ops.
    require(p.nnz >= a.nnz, "plan: nnz smaller than the matrix");
    std::vector<int64_t> flat_of_mat(static_cast<std::size_t>(p.nnz), -1);
    std::vector<int32_t> out_of(static_cast<std::size_t>(a.nnz));
    int64_t points = 0;
    for (int r = 0; r < a.n_rows; ++r) {
        for (int32_t k = ro[r]; k < ro[r + 1] - sp; ++k) {
            flat_of_mat[k] = points++;
            out_of[k] = r;
        }
    }
    std::vector<uint8_t> seen(points, 0);
    int64_t covered = 0;
    std::vector<int32_t> finalized;
    for (int64_t g = 0; g < p.n_groups(); ++g) {
        for (int64_t c = p.g_codelet_ptr[g]; c < p.g_codelet_ptr[g + 1]; ++c) {
            const int m = p.c_m[c], n = p.c_n[c];
            if (m < 1 || n < 1) throw std::logic_error("plan: empty codelet");
            DescView ds[3] = {p.desc(c, 0), p.desc(c, 1), p.desc(c, 2)};
            int tables = (ds[0].form != 0) + (ds[1].form != 0) + (ds[2].form != 0);
            if (tables == 3) throw std::invalid_argument("codelet: all three descriptors are tables");
            if (tables != p.c_kind[c]) throw std::logic_error("plan: codelet kind does not match descriptors");
            auto at = [&](int d, int i, int j) -> int64_t {
                const DescView& v = ds[d];
                int64_t e;
                switch (v.form) {
                    case PSC_FORM_STRIDED:
                        return static_cast<int64_t>(v.base) + static_cast<int64_t>(i) * v.so +
                               static_cast<int64_t>(j) * v.si;
                    case PSC_FORM_INNER_TABLE: e = j; break;
                    case PSC_FORM_OUTER_TABLE: e = i; break;
                    default: e = static_cast<int64_t>(i) * n + j; break;
                }
                if (e >= v.len) throw std::logic_error("plan: table shorter than the codelet extent");
                return v.tab ? v.tab[e] : p.implicit_entry(c, d, e, a.row_offsets, a.col_indices);
            };
            for (int i = 0; i < m; ++i) {
                for (int j = 0; j < n; ++j) {
                    int64_t k = at(1, i, j);
                    if (k < 0 || k >= p.nnz || flat_of_mat[k] < 0)
                        throw std::logic_error("plan: matrix index outside operation set");
                    int64_t f = flat_of_mat[k];
                    if (seen[f]) throw std::logic_error("plan: operation covered twice");
                    seen[f] = 1;
                    ++covered;
                    if (at(0, i, j) != out_of[k]) throw std::logic_error("plan: wrong output index");
                    if (at(2, i, j) != a.col_indices[k]) throw std::logic_error("plan: wrong gather index");
                    int row = out_of[k];
                    if (row < p.g_row_begin[g] || row >= p.g_row_end[g])
                        throw std::logic_error("plan: operation outside its window");
                }
            }
        }
        bool bad = false;
        for_finalize(p, &a, g, [&](int32_t r, int32_t dpos, int32_t rhs) {
            if (p.kernel != PSC_KERNEL_SPTRSV) throw std::logic_error("plan: finalize record in a non-sptrsv plan");
            if (r < 0 || r >= p.n_rows || dpos != ro[r + 1] - 1 || rhs != r) bad = true;
            finalized.push_back(r);
        });
        if (bad) throw std::logic_error("plan: bad finalize record");
    }
    if (covered != points) throw std::logic_error("plan: uncovered operations");
    if (p.kernel == PSC_KERNEL_SPTRSV) {
        std::sort(finalized.begin(), finalized.end());
        for (int r = 0; r < p.n_rows; ++r) {
            if (r >= static_cast<int>(finalized.size()) || finalized[r] != r)
                throw std::logic_error("plan: finalize records do not cover every row once");
        }
        if (static_cast<int>(finalized.size()) != p.n_rows) throw std::logic_error("plan: surplus finalize records");
    }
}

}  // namespace pscb
