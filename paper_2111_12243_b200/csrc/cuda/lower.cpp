// Plan -> device layout lowering (see lower.hpp).
#include "lower.hpp"

#include <algorithm>
#include <cstdlib>

#include "common.hpp"

namespace pscb {

void check_codelet_shape(int which, int out_form, int mat_form, int vec_form) {
    bool ot = out_form != PSC_FORM_STRIDED, mt = mat_form != PSC_FORM_STRIDED, vt = vec_form != PSC_FORM_STRIDED;
    if (which == PSC_CODELET_BLAS) {
        if (ot || mt || vt) throw std::invalid_argument("exec_blas_codelet: descriptors must be strided");
    } else if (which == PSC_CODELET_PSC_I) {
        if (ot || mt || !vt) throw std::invalid_argument("exec_psci_codelet: expects one gather table");
    } else {
        if (!ot || mt || !vt) throw std::invalid_argument("exec_pscii_codelet: expects output and gather tables");
    }
}

namespace {

int dispatch_kind(int kind) {  // exec_codelet switch, executor.cpp:120-126
    return kind == PSC_CODELET_BLAS ? PSC_CODELET_BLAS : kind == PSC_CODELET_PSC_I ? PSC_CODELET_PSC_I : PSC_CODELET_PSC_II;
}

struct SegRec {
    int32_t row;  // local
    int32_t start, len, vec;
};

// Table entry e of descriptor d of codelet c, bounds-checked.
int64_t tab_at(const Plan& p, const DescView& v, int64_t c, int d, int64_t e, const psc_csr_view& a) {
    if (e >= v.len) throw std::invalid_argument("codelet: table shorter than the codelet extent");
    return v.tab ? v.tab[e] : p.implicit_entry(c, d, e, a.row_offsets, a.col_indices);
}

void build_general(const Plan& p, const psc_csr_view& a, Lowered& L) {
    auto& G = L.gen;
    const int64_t C = p.n_codelets();
    G.part_group_ptr = p.part_group_ptr;
    G.group_codelet_ptr = p.g_codelet_ptr;
    G.c_kind.resize(C);
    G.c_m.resize(C);
    G.c_n.resize(C);
    G.d_form.resize(3 * C);
    G.d_base.resize(3 * C);
    G.d_so.resize(3 * C);
    G.d_si.resize(3 * C);
    G.d_tab.resize(3 * C);
    for (int64_t c = 0; c < C; ++c) {
        const int which = dispatch_kind(p.c_kind[c]);
        const int m = p.c_m[c], n = p.c_n[c];
        G.c_kind[c] = which;
        G.c_m[c] = m;
        G.c_n[c] = n;
        DescView ds[3] = {p.desc(c, 0), p.desc(c, 1), p.desc(c, 2)};
        check_codelet_shape(which, ds[0].form, ds[1].form, ds[2].form);
        for (int d = 0; d < 3; ++d) {
            G.d_form[3 * c + d] = ds[d].form;
            G.d_base[3 * c + d] = ds[d].base;
            G.d_so[3 * c + d] = ds[d].so;
            G.d_si[3 * c + d] = ds[d].si;
            G.d_tab[3 * c + d] = static_cast<int64_t>(G.tables.size());
            if (ds[d].form != PSC_FORM_STRIDED) {
                for (int64_t e = 0; e < ds[d].len; ++e) G.tables.push_back(static_cast<int32_t>(tab_at(p, ds[d], c, d, e, a)));
            }
        }
        if (m <= 0 || n <= 0) continue;  // the reference loops do nothing
        // Index ranges the executor will touch (exec_* semantics).
        auto lin = [&](int d, int64_t i, int64_t j) {
            return static_cast<int64_t>(ds[d].base) + i * ds[d].so + j * ds[d].si;
        };
        auto track = [](int64_t& mx, int64_t v) {
            if (v < 0) throw std::invalid_argument("codelet: negative index");
            mx = std::max(mx, v);
        };
        for (int64_t i : {int64_t(0), int64_t(m - 1)})
            for (int64_t j : {int64_t(0), int64_t(n - 1)}) track(G.max_mat, lin(1, i, j));
        if (which == PSC_CODELET_BLAS) {
            for (int64_t i : {int64_t(0), int64_t(m - 1)}) {
                track(G.max_out, lin(0, i, 0));
                for (int64_t j : {int64_t(0), int64_t(n - 1)}) track(G.max_vec, lin(2, i, j));
            }
        } else {
            if (which == PSC_CODELET_PSC_I) {
                for (int64_t i : {int64_t(0), int64_t(m - 1)}) track(G.max_out, lin(0, i, 0));
            } else {
                for (int64_t i = 0; i < m; ++i) track(G.max_out, tab_at(p, ds[0], c, 0, i, a));
            }
            bool per_point = which == PSC_CODELET_PSC_II && ds[2].form == PSC_FORM_POINT_TABLE;
            int64_t cnt = per_point ? static_cast<int64_t>(m) * n : n;
            for (int64_t e = 0; e < cnt; ++e) track(G.max_vec, tab_at(p, ds[2], c, 2, e, a));
        }
    }
    // finalize records
    G.group_fin_ptr.assign(p.n_groups() + 1, 0);
    for (int64_t g = 0; g < p.n_groups(); ++g) {
        if (!p.mined) {
            for (int64_t f = p.g_fin_ptr[g]; f < p.g_fin_ptr[g + 1]; ++f) {
                G.f_row.push_back(p.f_row[f]);
                G.f_diag.push_back(p.f_diag[f]);
                G.f_rhs.push_back(p.f_rhs[f]);
            }
        } else if (p.kernel == PSC_KERNEL_SPTRSV) {
            for (int32_t r = p.g_row_begin[g]; r < p.g_row_end[g]; ++r) {
                G.f_row.push_back(r);
                G.f_diag.push_back(a.row_offsets[r + 1] - 1);
                G.f_rhs.push_back(r);
            }
        }
        G.group_fin_ptr[g + 1] = static_cast<int64_t>(G.f_row.size());
    }
    for (std::size_t f = 0; f < G.f_row.size(); ++f) {
        if (G.f_row[f] < 0 || G.f_row[f] >= a.n_rows || G.f_rhs[f] < 0 || G.f_rhs[f] >= a.n_rows ||
            G.f_diag[f] < 0 || G.f_diag[f] >= a.nnz)
            throw std::invalid_argument("finalize record index out of range");
    }
    if (G.max_mat >= a.nnz) throw std::invalid_argument("codelet: matrix index out of range");
    if (G.max_vec >= a.n_cols) throw std::invalid_argument("codelet: gather index out of range");
    if (G.max_out >= a.n_rows) throw std::invalid_argument("codelet: output index out of range");
}

}  // namespace

Lowered lower_plan(const Plan& p, const psc_csr_view& a, int64_t part_begin, int64_t part_end,
                   int sptrsv_block_rows, bool force_general) {
    require(p.n_rows == a.n_rows && p.n_cols == a.n_cols && p.nnz == a.nnz,
            "bind: matrix does not match the plan");
    const int32_t* ro = a.row_offsets;
    const int sp = p.kernel == PSC_KERNEL_SPTRSV ? 1 : 0;
    Lowered L;
    L.kernel = p.kernel;
    const bool partial = part_end >= 0;
    if (!partial) {
        part_begin = 0;
        part_end = p.n_partitions();
        L.row_begin = 0;
        L.row_end = p.n_rows;
    } else {
        require(p.kernel == PSC_KERNEL_SPMV, "bind_partitions: only SpMV plans shard by partition");
        require(0 <= part_begin && part_begin <= part_end && part_end <= p.n_partitions(),
                "bind_partitions: partition range out of bounds");
        int64_t g0 = p.part_group_ptr[part_begin], g1 = p.part_group_ptr[part_end];
        int32_t rb = p.n_rows, re = 0;
        int64_t rows = 0;
        for (int64_t g = g0; g < g1; ++g) {
            rb = std::min(rb, p.g_row_begin[g]);
            re = std::max(re, p.g_row_end[g]);
            rows += p.g_row_end[g] - p.g_row_begin[g];
        }
        if (g0 == g1) rb = re = 0;
        require(rows == static_cast<int64_t>(re) - rb, "bind_partitions: partitions do not cover a contiguous row range");
        L.row_begin = rb;
        L.row_end = re;
    }
    L.k_begin = ro[L.row_begin];
    L.k_end = ro[L.row_end];
    const int32_t nr = L.row_end - L.row_begin;
    const int64_t g0 = p.part_group_ptr[part_begin], g1 = p.part_group_ptr[part_end];
    if (force_general) {
        require(!partial, "bind_partitions: the general interpreter binds whole plans only");
        L.canonical = false;
        L.why_general = "execute_plan accumulates onto the caller's arrays";
        build_general(p, a, L);
        return L;
    }

    // ---- collect segments in plan order; decide canonicality ----
    std::vector<int32_t> count(static_cast<std::size_t>(nr) + 1, 0);
    std::vector<SegRec> segs;
    auto non_canonical = [&](const std::string& why) {
        if (L.canonical) L.why_general = why;
        L.canonical = false;
    };
    std::vector<int64_t> fin_part;      // sptrsv: partition of each row's finalize
    std::vector<int64_t> fin_group;
    if (p.kernel == PSC_KERNEL_SPTRSV) {
        fin_part.assign(p.n_rows, -1);
        fin_group.assign(p.n_rows, -1);
        for (int64_t part = part_begin; part < part_end && L.canonical; ++part) {
            for (int64_t g = p.part_group_ptr[part]; g < p.part_group_ptr[part + 1]; ++g) {
                auto visit = [&](int32_t r, int32_t dpos, int32_t rhs) {
                    if (r < 0 || r >= p.n_rows || dpos != ro[r + 1] - 1 || rhs != r || fin_part[r] >= 0) {
                        non_canonical("finalize records are not one {r, diag(r), r} per row");
                        return;
                    }
                    fin_part[r] = part;
                    fin_group[r] = g;
                };
                if (p.mined) {
                    for (int32_t r = p.g_row_begin[g]; r < p.g_row_end[g]; ++r) visit(r, ro[r + 1] - 1, r);
                } else {
                    for (int64_t f = p.g_fin_ptr[g]; f < p.g_fin_ptr[g + 1]; ++f) visit(p.f_row[f], p.f_diag[f], p.f_rhs[f]);
                }
            }
        }
        for (int32_t r = 0; r < p.n_rows && L.canonical; ++r)
            if (fin_part[r] < 0) non_canonical("a row has no finalize record");
    }
    segs.reserve(static_cast<std::size_t>(p.g_codelet_ptr[g1] - p.g_codelet_ptr[g0]));
    for (int64_t part = part_begin; part < part_end && L.canonical; ++part) {
        for (int64_t g = p.part_group_ptr[part]; g < p.part_group_ptr[part + 1] && L.canonical; ++g) {
            for (int64_t c = p.g_codelet_ptr[g]; c < p.g_codelet_ptr[g + 1] && L.canonical; ++c) {
                const int m = p.c_m[c], n = p.c_n[c];
                if (p.mined) {
                    const bool blas = p.c_kind[c] == PSC_CODELET_BLAS;
                    for (int i = 0; i < m; ++i) {
                        int32_t r = p.c_row[c] + i;
                        int64_t s = static_cast<int64_t>(p.c_mat_base[c]) + static_cast<int64_t>(i) * p.c_mat_so[c];
                        segs.push_back({r - L.row_begin, static_cast<int32_t>(s - L.k_begin), n,
                                        blas ? p.c_vec_base[c] + i * p.c_vec_so[c] : -1});
                        ++count[r - L.row_begin];
                    }
                    continue;
                }
                // imported codelet: check every canonical invariant
                const int which = dispatch_kind(p.c_kind[c]);
                DescView ds[3] = {p.desc(c, 0), p.desc(c, 1), p.desc(c, 2)};
                check_codelet_shape(which, ds[0].form, ds[1].form, ds[2].form);
                if (m <= 0 || n <= 0) continue;
                if (n > 1 && ds[1].si != 1) {
                    non_canonical("non-unit matrix inner stride");
                    break;
                }
                if (p.kernel == PSC_KERNEL_SPMV && which == PSC_CODELET_BLAS && n >= 4 && ds[2].si != 1) {
                    non_canonical("BLAS gather with non-unit inner stride takes the sequential branch");
                    break;
                }
                for (int i = 0; i < m && L.canonical; ++i) {
                    int64_t o = which == PSC_CODELET_PSC_II ? tab_at(p, ds[0], c, 0, i, a)
                                                            : static_cast<int64_t>(ds[0].base) + static_cast<int64_t>(i) * ds[0].so;
                    if (o < L.row_begin || o >= L.row_end) {
                        non_canonical("output index outside the bound rows");
                        break;
                    }
                    int64_t s = static_cast<int64_t>(ds[1].base) + static_cast<int64_t>(i) * ds[1].so;
                    if (s < ro[o] || s + n > static_cast<int64_t>(ro[o + 1]) - sp) {
                        non_canonical("codelet row does not lie in its output row");
                        break;
                    }
                    bool unit_run = which == PSC_CODELET_BLAS && (ds[2].si == 1 || n == 1);
                    int64_t v0 = 0;
                    for (int j = 0; j < n; ++j) {
                        int64_t xv;
                        if (which == PSC_CODELET_BLAS) {
                            xv = static_cast<int64_t>(ds[2].base) + static_cast<int64_t>(i) * ds[2].so +
                                 static_cast<int64_t>(j) * ds[2].si;
                        } else {
                            bool per_point = which == PSC_CODELET_PSC_II && ds[2].form == PSC_FORM_POINT_TABLE;
                            xv = tab_at(p, ds[2], c, 2, per_point ? static_cast<int64_t>(i) * n + j : j, a);
                        }
                        if (j == 0) v0 = xv;
                        if (xv != a.col_indices[s + j]) {
                            non_canonical("gather differs from col_indices");
                            break;
                        }
                    }
                    if (!L.canonical) break;
                    if (p.kernel == PSC_KERNEL_SPTRSV) {
                        // must run before its row's finalize, in the same group
                        // when in the same partition, after every x it reads
                        if (fin_part[o] < part || (fin_part[o] == part && fin_group[o] != g)) {
                            non_canonical("codelet of a row runs outside its finalize group");
                            break;
                        }
                        for (int j = 0; j < n; ++j) {
                            if (fin_part[a.col_indices[s + j]] >= part) {
                                non_canonical("codelet reads x before it is finalised");
                                break;
                            }
                        }
                        if (!L.canonical) break;
                    }
                    segs.push_back({static_cast<int32_t>(o - L.row_begin), static_cast<int32_t>(s - L.k_begin), n,
                                    unit_run ? static_cast<int32_t>(v0) : -1});
                    ++count[o - L.row_begin];
                }
            }
        }
    }
    if (p.kernel == PSC_KERNEL_SPTRSV && p.mined && L.canonical) {
        // level sets guarantee finalize-before-read; nothing to check
    }

    if (!L.canonical) {
        require(!partial, "bind_partitions: plan is not canonical (" + L.why_general + ")");
        segs.clear();
        segs.shrink_to_fit();
        build_general(p, a, L);
        return L;
    }

    // ---- per-row segment lists (stable by plan order) ----
    L.row_seg_ptr.assign(static_cast<std::size_t>(nr) + 1, 0);
    for (int32_t r = 0; r < nr; ++r) L.row_seg_ptr[r + 1] = L.row_seg_ptr[r] + count[r];
    const int64_t S = static_cast<int64_t>(segs.size());
    require(S <= INT32_MAX, "bind: too many segments");
    L.seg_start.resize(S);
    L.seg_len.resize(S);
    L.seg_vec.resize(S);
    {
        std::vector<int32_t> cur(L.row_seg_ptr.begin(), L.row_seg_ptr.end() - 1);
        for (const SegRec& s : segs) {
            int32_t k = cur[s.row]++;
            L.seg_start[k] = s.start;
            L.seg_len[k] = s.len;
            L.seg_vec[k] = s.vec;
        }
    }
    segs.clear();
    segs.shrink_to_fit();
    L.simple = true;
    for (int32_t r = 0; r < nr && L.simple; ++r) {
        int32_t gr = r + L.row_begin;
        int32_t ext = ro[gr + 1] - ro[gr] - sp;
        int32_t c = L.row_seg_ptr[r + 1] - L.row_seg_ptr[r];
        if (c == 0) {
            L.simple = ext == 0;
        } else if (c == 1) {
            int32_t k = L.row_seg_ptr[r];
            L.simple = L.seg_start[k] == ro[gr] - L.k_begin && L.seg_len[k] == ext;
        } else {
            L.simple = false;
        }
    }
    if (L.simple) {
        L.row_seg_ptr.clear();
        L.seg_start.clear();
        L.seg_len.clear();
        L.seg_vec.clear();
        L.row_seg_ptr.shrink_to_fit();
        L.seg_start.shrink_to_fit();
        L.seg_len.shrink_to_fit();
        L.seg_vec.shrink_to_fit();
    }

    // ---- work units ----
    if (p.kernel == PSC_KERNEL_SPMV) {
        auto k_of = [&](int32_t r) { return static_cast<int32_t>(ro[r + L.row_begin] - L.k_begin); };
        auto s_of = [&](int32_t r) { return L.simple ? 0 : L.row_seg_ptr[r]; };
        // row groups (segmented plans): rows whose segments are unit-stride
        // gathers tiling the row in CSR order, consecutive rows with the same
        // lengths and x offsets
        std::vector<int32_t> group_len(nr, 0);  // > 0 at a group's first row
        const char* gv = std::getenv("PSC_SPMV_GROUPS");
        const char* sgv = std::getenv("PSC_SPMV_GROUP_SHIFT");
        const bool shift_groups = !(sgv && sgv[0] == '0');
        if (!L.simple && !(gv && gv[0] == '0')) {
            auto templ = [&](int32_t r) {  // row r qualifies as a template
                const int32_t q0 = L.row_seg_ptr[r], q1 = L.row_seg_ptr[r + 1];
                const int32_t len = k_of(r + 1) - k_of(r);
                if (q1 - q0 < 1 || q1 - q0 > 32 || len < 1 || len > kGroupCols) return false;
                int32_t at = k_of(r);
                for (int32_t q = q0; q < q1; ++q) {
                    if (L.seg_vec[q] < 0 || L.seg_start[q] != at) return false;
                    at += L.seg_len[q];
                }
                return at == k_of(r + 1);
            };
            auto same = [&](int32_t r, int32_t t) {  // row t has row r's template
                const int32_t q0 = L.row_seg_ptr[r], q1 = L.row_seg_ptr[r + 1], d = L.row_seg_ptr[t] - q0;
                if (L.row_seg_ptr[t + 1] - L.row_seg_ptr[t] != q1 - q0) return false;
                for (int32_t q = q0; q < q1; ++q)
                    if (L.seg_len[q + d] != L.seg_len[q] || L.seg_vec[q + d] != L.seg_vec[q]) return false;
                return true;
            };
            for (int32_t r = 0; r < nr;) {
                int32_t g = 1;
                if (templ(r))
                    while (g < kGroupRows && r + g < nr && templ(r + g) && same(r, r + g)) ++g;
                if (g >= 2) {
                    group_len[r] = g;
                    const int32_t q0 = L.row_seg_ptr[r], S = L.row_seg_ptr[r + 1] - q0;
                    const int32_t k0 = k_of(r), C = k_of(r + 1) - k0;
                    // A group whose template is the previous group's shifted by a constant column
                    // distance (the next node of a stencil line) takes its columns and segment
                    // table from that group's template: {.., q0_t, S, k0_t, shift}; the line's
                    // groups then read one template (L2-resident) instead of their own columns.
                    int32_t qt = q0, kt = k0, shift = 0;
                    if (shift_groups && !L.groups.empty()) {
                        const int32_t* pg = L.groups.data() + L.groups.size() - 8;
                        const int32_t pr = pg[0], pk = pg[2], pq = L.row_seg_ptr[pr];
                        bool ok = pr + pg[1] == r && pg[3] == C && pg[5] == S;
                        for (int32_t q = 0; q < S && ok; ++q) ok = L.seg_len[pq + q] == L.seg_len[q0 + q];
                        const int64_t kb = L.k_begin;
                        const int32_t d = ok ? a.col_indices[kb + k0] - a.col_indices[kb + pk] : 0;
                        for (int32_t c = 0; c < C && ok; ++c) ok = a.col_indices[kb + k0 + c] == a.col_indices[kb + pk + c] + d;
                        if (ok) {
                            qt = pg[4];
                            kt = pg[6];
                            shift = pg[7] + d;
                        }
                    }
                    L.groups.insert(L.groups.end(), {r, g, k0, C, qt, S, kt, shift});
                }
                r += g;
            }
        }
        int32_t c0 = 0;  // start of the open chunk
        auto close = [&](int32_t r1) {
            if (r1 > c0) {
                L.items.insert(L.items.end(), {c0, r1, k_of(c0), k_of(r1)});
                L.item_seg.insert(L.item_seg.end(), {s_of(c0), s_of(r1)});
            }
        };
        for (int32_t r = 0; r < nr; ++r) {
            if (group_len[r] > 0) {  // a row group: not in any chunk
                close(r);
                r += group_len[r] - 1;
                c0 = r + 1;
                continue;
            }
            const int64_t len = ro[r + L.row_begin + 1] - ro[r + L.row_begin];
            if (len > kSpmvWarpCap) {  // a long row is handled on its own
                close(r);
                L.long_row_list.push_back(r);
                c0 = r + 1;
                continue;
            }
            if (static_cast<int64_t>(k_of(r + 1)) - k_of(c0) > kSpmvWarpCap || r + 1 - c0 > kSpmvWarpCap) {
                close(r);
                c0 = r;
            }
        }
        close(nr);
        L.long_rows = static_cast<int64_t>(L.long_row_list.size());
    } else {
        // Units: a row continues the unit of the row above when it reads it
        // (its last off-diagonal entry is column r-1).
        std::vector<uint8_t> cont(nr, 0);
        int64_t n_units = 0;
        for (int32_t r = 0; r < nr; ++r) {
            const int32_t gr = r + L.row_begin;
            const int32_t k0 = ro[gr], kd = ro[gr + 1] - 1;
            cont[r] = r > 0 && kd > k0 && a.col_indices[kd - 1] == gr - 1;
            n_units += !cont[r];
        }
        const double avg_unit = n_units ? static_cast<double>(nr) / static_cast<double>(n_units) : 0.0;
        int mode = -1;  // PSC_TRSV_MODE: 0 rows, 1 chains; default by average unit length
        if (const char* env = std::getenv("PSC_TRSV_MODE")) mode = std::atoi(env);
        L.chain_mode = mode == 1 || (mode != 0 && avg_unit >= 4.0);
        int R = sptrsv_block_rows;
        if (R <= 0) {
            if (const char* env = std::getenv("PSC_SPTRSV_BLOCK_ROWS")) R = std::atoi(env);
        }
        L.block_row.push_back(0);
        {
            const int cap = L.chain_mode ? 12000 : 9000;  // shared-memory rows per CTA (kernels.cu smem layout)
            if (R <= 0) R = std::max(1024, (nr + 99) / 100);  // ~100 blocks
            R = std::max(1, std::min({R, cap, std::max(1, nr)}));
            for (int32_t r = 0; r < nr;) {
                int32_t e = static_cast<int32_t>(std::min<int64_t>(nr, static_cast<int64_t>(r) + R));
                L.block_row.push_back(e);
                L.max_block_rows = std::max(L.max_block_rows, e - r);
                r = e;
            }
        }
        if (L.chain_mode) {
            L.block_unit.push_back(0);
            for (size_t bi = 0; bi + 1 < L.block_row.size(); ++bi) {
                const int32_t b0 = L.block_row[bi], b1 = L.block_row[bi + 1];
                const int64_t u0 = static_cast<int64_t>(L.unit_start.size());
                for (int32_t r = b0; r < b1; ++r)
                    if (r == b0 || !cont[r]) L.unit_start.push_back(r);
                L.block_unit.push_back(static_cast<int32_t>(L.unit_start.size()));
                L.max_block_units = std::max<int32_t>(L.max_block_units, static_cast<int32_t>(L.unit_start.size() - u0));
            }
        } else {
            // level of every row = partition of its finalize record; within a
            // block, rows are listed by (level, row) so threads take them in a
            // dependency-respecting order
            std::vector<int32_t> lvl(nr, 0);
            if (!fin_part.empty()) {
                for (int32_t r = 0; r < nr; ++r) lvl[r] = static_cast<int32_t>(fin_part[r]);
            }
            L.unit_start.resize(nr);
            for (size_t bi = 0; bi + 1 < L.block_row.size(); ++bi) {
                int32_t b0 = L.block_row[bi], b1 = L.block_row[bi + 1];
                for (int32_t r = b0; r < b1; ++r) L.unit_start[r] = r;
                std::stable_sort(L.unit_start.begin() + b0, L.unit_start.begin() + b1,
                                 [&](int32_t u, int32_t v) { return lvl[u] < lvl[v]; });
            }
            L.block_unit = L.block_row;  // one unit per row
            L.max_block_units = L.max_block_rows;
        }
    }
    return L;
}

void unit_maps(Lowered& L) {
    const int32_t nr = L.row_end - L.row_begin;
    const size_t nu = L.unit_start.size();
    L.unit_len.assign(nu, 1);
    L.unit_loc.assign(nu, 0);
    L.row_block.assign(nr, 0);
    L.row_loc.assign(nr, 0);
    for (size_t bi = 0; bi + 1 < L.block_row.size(); ++bi) {
        const int32_t b0 = L.block_row[bi], b1 = L.block_row[bi + 1];
        for (int32_t r = b0; r < b1; ++r) {
            L.row_block[r] = static_cast<int32_t>(bi);
            L.row_loc[r] = r - b0;
        }
        const int32_t u0 = L.block_unit[bi], u1 = L.block_unit[bi + 1];
        for (int32_t u = u0; u < u1; ++u) {
            L.unit_loc[u] = L.unit_start[u] - b0;
            if (L.chain_mode) L.unit_len[u] = (u + 1 < u1 ? L.unit_start[u + 1] : b1) - L.unit_start[u];
        }
    }
    L.tiled = false;
}

bool tile_chain_blocks(Lowered& L, const psc_csr_view& a, int max_rows) {
    if (!L.chain_mode || L.row_begin != 0) return false;
    const int32_t nr = L.row_end;
    unit_maps(L);  // contiguous unit lengths
    const int32_t nu = static_cast<int32_t>(L.unit_start.size());
    if (nu < 2) return false;
    std::vector<int32_t> start(L.unit_start), len(L.unit_len);
    std::vector<int32_t> unit_of(nr);
    for (int32_t u = 0; u < nu; ++u)
        for (int32_t r = start[u]; r < start[u] + len[u]; ++r) unit_of[r] = u;
    // dependency lists (deduplicated) and dependents
    std::vector<int64_t> dep_ptr(nu + 1, 0);
    std::vector<int32_t> deps;
    std::vector<int32_t> seen(nu, -1);
    for (int32_t u = 0; u < nu; ++u) {
        for (int32_t r = start[u]; r < start[u] + len[u]; ++r) {
            for (int64_t k = a.row_offsets[r]; k < a.row_offsets[r + 1] - 1; ++k) {
                const int32_t v = unit_of[a.col_indices[k]];
                if (v != u && seen[v] != u) {
                    seen[v] = u;
                    deps.push_back(v);
                }
            }
        }
        dep_ptr[u + 1] = static_cast<int64_t>(deps.size());
    }
    std::vector<int64_t> out_ptr(nu + 1, 0);
    for (int32_t v : deps) ++out_ptr[v + 1];
    for (int32_t u = 0; u < nu; ++u) out_ptr[u + 1] += out_ptr[u];
    std::vector<int32_t> outs(deps.size());
    {
        std::vector<int64_t> fill(out_ptr.begin(), out_ptr.end() - 1);
        for (int32_t u = 0; u < nu; ++u)
            for (int64_t k = dep_ptr[u]; k < dep_ptr[u + 1]; ++k) outs[fill[deps[k]]++] = u;
    }
    std::vector<int32_t> remaining(nu), block_of(nu, -1), affinity(nu, 0);
    // ready units: `pool` (FIFO by discovery, affinity to earlier blocks only)
    // and `heap` (became ready while the open block grew: (affinity, -order))
    std::vector<int32_t> pool;
    size_t pool_head = 0;
    std::vector<std::pair<std::pair<int32_t, int64_t>, int32_t>> heap;
    int64_t order = 0;
    std::vector<int64_t> disc(nu, 0);
    for (int32_t u = 0; u < nu; ++u) {
        remaining[u] = static_cast<int32_t>(dep_ptr[u + 1] - dep_ptr[u]);
        if (remaining[u] == 0) {
            disc[u] = order++;
            pool.push_back(u);
        }
    }
    std::vector<int32_t> new_unit_start, new_block_unit{0}, new_block_row{0}, new_len;
    int32_t cur_block = 0, cur_rows = 0, placed = 0;
    auto close_block = [&] {
        if (cur_rows == 0) return;
        new_block_unit.push_back(static_cast<int32_t>(new_unit_start.size()));
        new_block_row.push_back(new_block_row.back() + cur_rows);
        ++cur_block;
        cur_rows = 0;
        for (auto& e : heap) pool.push_back(e.second);  // no affinity to the next block
        heap.clear();
    };
    while (placed < nu) {
        int32_t u = -1;
        if (!heap.empty()) {
            std::pop_heap(heap.begin(), heap.end());
            u = heap.back().second;
            heap.pop_back();
        } else {
            while (pool_head < pool.size() && block_of[pool[pool_head]] >= 0) ++pool_head;
            if (pool_head == pool.size()) return false;  // cycle: not a triangle
            u = pool[pool_head++];
        }
        if (block_of[u] >= 0) continue;
        if (cur_rows > 0 && cur_rows + len[u] > max_rows) {
            close_block();
            // u has no affinity to the new block; it seeds it
        }
        block_of[u] = cur_block;
        new_unit_start.push_back(start[u]);
        new_len.push_back(len[u]);
        cur_rows += len[u];
        ++placed;
        for (int64_t k = out_ptr[u]; k < out_ptr[u + 1]; ++k) {
            const int32_t w = outs[k];
            ++affinity[w];
            if (--remaining[w] == 0) {
                disc[w] = order++;
                // affinity = dependencies of w inside the open block
                int32_t in = 0;
                for (int64_t j = dep_ptr[w]; j < dep_ptr[w + 1]; ++j) in += block_of[deps[j]] == cur_block;
                heap.push_back({{in, -disc[w]}, w});
                std::push_heap(heap.begin(), heap.end());
            }
        }
    }
    close_block();
    // adopt the tiled layout
    const int32_t nb = static_cast<int32_t>(new_block_row.size()) - 1;
    L.unit_start = std::move(new_unit_start);
    L.unit_len = std::move(new_len);
    L.block_unit = std::move(new_block_unit);
    L.block_row = std::move(new_block_row);
    L.unit_loc.assign(L.unit_start.size(), 0);
    L.row_block.assign(nr, 0);
    L.row_loc.assign(nr, 0);
    L.max_block_rows = 0;
    L.max_block_units = 0;
    for (int32_t bi = 0; bi < nb; ++bi) {
        int32_t loc = 0;
        for (int32_t u = L.block_unit[bi]; u < L.block_unit[bi + 1]; ++u) {
            L.unit_loc[u] = loc;
            for (int32_t j = 0; j < L.unit_len[u]; ++j) {
                L.row_block[L.unit_start[u] + j] = bi;
                L.row_loc[L.unit_start[u] + j] = loc + j;
            }
            loc += L.unit_len[u];
        }
        L.max_block_rows = std::max(L.max_block_rows, loc);
        L.max_block_units = std::max(L.max_block_units, L.block_unit[bi + 1] - L.block_unit[bi]);
    }
    L.tiled = true;
    return true;
}

int64_t build_run_items(const Lowered& L, const psc_csr_view& a, std::vector<int32_t>& items) {
    const int32_t nr = L.row_end - L.row_begin;
    const int64_t kb = a.row_offsets[L.row_begin];
    items.clear();
    int64_t in_runs = 0;
    auto emit = [&](int32_t r0, int32_t count, int32_t n) {  // local rows [r0, r0 + count)
        const int64_t k0 = a.row_offsets[r0 + L.row_begin];
        items.push_back(r0);
        items.push_back(count);
        items.push_back(static_cast<int32_t>(k0 - kb));
        items.push_back(n);
        for (int j = 0; j < 16; ++j) items.push_back(j < n ? a.col_indices[k0 + j] : 0);
    };
    int32_t loose0 = -1;  // open range of rows outside runs
    auto flush_loose = [&](int32_t end) {
        for (int32_t r = loose0; loose0 >= 0 && r < end; r += 32) emit(r, std::min<int32_t>(32, end - r), -1);
        loose0 = -1;
    };
    int32_t r = 0;
    while (r < nr) {
        const int64_t k0 = a.row_offsets[r + L.row_begin];
        const int32_t n = static_cast<int32_t>(a.row_offsets[r + L.row_begin + 1] - k0);
        int32_t e = r + 1;
        if (n >= 1 && n <= 16) {
            while (e < nr) {
                const int64_t ke = a.row_offsets[e + L.row_begin];
                if (a.row_offsets[e + L.row_begin + 1] - ke != n) break;
                bool same = true;
                for (int32_t j = 0; j < n && same; ++j) same = a.col_indices[ke + j] == a.col_indices[k0 + j] + (e - r);
                if (!same) break;
                ++e;
            }
        }
        if (e - r >= kRunMinRows) {
            flush_loose(r);
            for (int32_t q = r; q < e; q += 32) emit(q, std::min<int32_t>(32, e - q), n);
            in_runs += e - r;
        } else if (loose0 < 0) {
            loose0 = r;
        }
        r = e;
    }
    flush_loose(nr);
    return in_runs;
}

void block_halos(Lowered& L, const psc_csr_view& a) {
    const int32_t nb = static_cast<int32_t>(L.block_row.size()) - 1;
    const int32_t nr = L.row_end - L.row_begin;
    // dependency level of every row (longest path from a row without
    // off-diagonal entries): the halo is listed in the order its entries are
    // produced, so the halo warp's lanes rarely wait behind a late entry
    std::vector<int32_t> lvl(nr, 0);
    for (int32_t r = 0; r < nr; ++r) {
        const int32_t gr = r + L.row_begin;
        int32_t m = -1;
        for (int64_t k = a.row_offsets[gr]; k < a.row_offsets[gr + 1] - 1; ++k) {
            const int32_t c = a.col_indices[k] - L.row_begin;
            if (c >= 0 && c < r) m = std::max(m, lvl[c]);
        }
        lvl[r] = m + 1;
    }
    L.halo_ptr.assign(1, 0);
    L.halo_col.clear();
    L.halo_key.clear();
    L.halo_pos.clear();
    L.max_block_halo = 0;
    std::vector<int32_t> cols, pos;
    for (int32_t bi = 0; bi < nb; ++bi) {
        cols.clear();
        for (int32_t u = L.block_unit[bi]; u < L.block_unit[bi + 1]; ++u) {
            for (int32_t r = L.unit_start[u]; r < L.unit_start[u] + L.unit_len[u]; ++r) {
                const int32_t gr = r + L.row_begin;
                for (int64_t k = a.row_offsets[gr]; k < a.row_offsets[gr + 1] - 1; ++k) {
                    const int32_t c = a.col_indices[k];
                    if (L.row_block[c - L.row_begin] != bi) cols.push_back(c);
                }
            }
        }
        std::sort(cols.begin(), cols.end());
        cols.erase(std::unique(cols.begin(), cols.end()), cols.end());
        L.halo_key.insert(L.halo_key.end(), cols.begin(), cols.end());  // by column, for lookups
        pos.resize(cols.size());
        for (size_t i = 0; i < cols.size(); ++i) pos[i] = static_cast<int32_t>(i);
        std::stable_sort(pos.begin(), pos.end(), [&](int32_t p, int32_t q) {
            return lvl[cols[p] - L.row_begin] < lvl[cols[q] - L.row_begin];
        });
        std::vector<int32_t> where(cols.size());
        for (size_t i = 0; i < pos.size(); ++i) {
            L.halo_col.push_back(cols[pos[i]]);
            where[pos[i]] = static_cast<int32_t>(i);
        }
        L.halo_pos.insert(L.halo_pos.end(), where.begin(), where.end());
        L.halo_ptr.push_back(static_cast<int32_t>(L.halo_col.size()));
        L.max_block_halo = std::max(L.max_block_halo, static_cast<int32_t>(cols.size()));
    }
}

Lowered lower_plan_tables(const Plan& p) {
    require(!p.mined,
            "Executor::run: a plan mined by psc_inspect keeps its tables in the matrix (col_indices); "
            "run it with psc_execute_plan / run_spmv / run_sptrsv, which take the matrix");
    Lowered L;
    L.kernel = p.kernel;
    L.canonical = false;
    L.why_general = "Executor::run over a raw context";
    psc_csr_view none{INT32_MAX, INT32_MAX, INT64_MAX, nullptr, nullptr, nullptr};
    build_general(p, none, L);
    return L;
}

Lowered lower_single_codelet(const psc_codelet_view& cv, int which) {
    check_codelet_shape(which, cv.out.form, cv.mat.form, cv.vec.form);
    Plan p;
    p.mined = false;
    p.kernel = PSC_KERNEL_SPMV;
    p.part_group_ptr = {0, 1};
    p.g_row_begin = {0};
    p.g_row_end = {0};
    p.g_strategy = {0};
    p.g_cost = {0};
    p.g_codelet_ptr = {0, 1};
    p.g_fin_ptr = {0, 0};
    p.c_kind = {static_cast<uint8_t>(which)};
    p.c_m = {cv.outer_extent};
    p.c_n = {cv.inner_extent};
    const psc_access_desc_view* ds[3] = {&cv.out, &cv.mat, &cv.vec};
    p.d_tab_ptr = {0};
    for (int d = 0; d < 3; ++d) {
        p.d_form.push_back(ds[d]->form);
        p.d_base.push_back(ds[d]->base);
        p.d_so.push_back(ds[d]->stride_outer);
        p.d_si.push_back(ds[d]->stride_inner);
        if (ds[d]->form != PSC_FORM_STRIDED && ds[d]->table_len > 0) {
            require(ds[d]->table != nullptr, "codelet: null table");
            p.tables.insert(p.tables.end(), ds[d]->table, ds[d]->table + ds[d]->table_len);
        }
        p.d_tab_ptr.push_back(static_cast<int64_t>(p.tables.size()));
    }
    Lowered L;
    L.canonical = false;
    L.why_general = "single codelet";
    psc_csr_view none{0, 0, INT32_MAX, nullptr, nullptr, nullptr};
    none.n_rows = INT32_MAX;
    none.n_cols = INT32_MAX;
    build_general(p, none, L);
    return L;
}

}  // namespace pscb
