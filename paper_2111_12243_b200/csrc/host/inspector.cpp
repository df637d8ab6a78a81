// Host inspector: a bit-exact restatement of the reference's Algorithm 1
// (/root/reference/proj/core/src/miner.cpp:18-323, scheduler.cpp:9-105,
// kernel_model.cpp:38-76, codelet.cpp:45-57) that produces the same
// partitions, windows, strategy choices, costs and codelets.
//
// Differences are purely in *how*: the access functions are evaluated from
// the CSR arrays on the fly instead of being tabulated (3 x nnz int32 in the
// reference's KernelModel), codelets are compact records instead of
// heap-allocated AccessDesc tables, level sets come from one pass in row order
// (rows only depend on smaller rows in a lower triangle, so row order is a
// topological order and the longest-path levels equal the Kahn levels of
// scheduler.cpp:27-65), and independent windows are mined on all host
// threads with results stitched back in window order.
#include <algorithm>
#include <atomic>
#include <numeric>

#include "common.hpp"
#include "csr.hpp"
#include "plan.hpp"

namespace pscb {

namespace {

struct Rec {
    uint8_t kind;
    int32_t m, n, row, mat_base, mat_so, vec_base, vec_so;
};

// The kernel model of kernel_model.cpp:38-76 evaluated on demand: row r has
// ext(r) operations at positions 0..ext-1; Mat(r,j) = row_offsets[r]+j,
// Vec(r,j) = col_indices[Mat(r,j)], Out(r,j) = r. For the solve the diagonal
// (stored last) is excluded.
struct Model {
    const int32_t* ro;
    const int32_t* col;
    int sp;  // 1 for sptrsv

    int ext(int r) const { return ro[r + 1] - ro[r] - sp; }
    int mat(int r, int j) const { return ro[r] + j; }
    int vec(int r, int j) const { return col[ro[r] + j]; }
    int64_t flat(int r) const { return static_cast<int64_t>(ro[r]) - static_cast<int64_t>(sp) * r; }
};

// CoverMap of miner.cpp:42-56.
struct Cover {
    const Model* md = nullptr;
    int64_t base = 0;
    std::vector<uint8_t> bits;

    void reset(const Model& m, int rb, int re) {
        md = &m;
        base = m.flat(rb);
        bits.assign(static_cast<std::size_t>(m.flat(re) - base), 0);
    }
    bool covered(int r, int p) const { return bits[md->flat(r) + p - base] != 0; }
    void cover(int r, int p) { bits[md->flat(r) + p - base] = 1; }
};

inline int64_t dims_of(int m, int n) {
    int d = (m > 1 ? 1 : 0) + (n > 1 ? 1 : 0);
    return d == 0 ? 1 : d;
}
// codelet.cpp:45-57 for the three mined shapes.
inline int64_t cost_blas(int m, int n) { return int64_t(m) * n + 3 + 3 * dims_of(m, n); }
inline int64_t cost_psci(int m, int n) { return int64_t(m) * n + 3 + 2 * dims_of(m, n) + n; }
inline int64_t cost_pscii(int m, int n) { return int64_t(m) * n + 3 + m + dims_of(m, n) + int64_t(m) * n; }

// miner.cpp:63-120
void mine_blas(const Model& md, int rb, int re, Cover& cv, std::vector<Rec>& out, int64_t& cost) {
    for (int r = rb; r < re; ++r) {
        int extent = md.ext(r);
        int p = 0;
        while (p < extent) {
            if (cv.covered(r, p)) {
                ++p;
                continue;
            }
            int q = p + 1;
            while (q < extent && !cv.covered(r, q) && md.vec(r, q) == md.vec(r, q - 1) + 1) ++q;
            int width = q - p;
            if (width < 2) {
                p = q;
                continue;
            }
            int rows = 1, mat_delta = 0, vec_delta = 0;
            while (r + rows < re) {
                int rn = r + rows;
                if (md.ext(rn) < p + width) break;
                bool ok = true;
                for (int j = p; j < q && ok; ++j) ok = !cv.covered(rn, j);
                for (int j = p + 1; j < q && ok; ++j) ok = md.vec(rn, j) == md.vec(rn, j - 1) + 1;
                if (!ok) break;
                int mdl = md.mat(rn, p) - md.mat(rn - 1, p);
                int vdl = md.vec(rn, p) - md.vec(rn - 1, p);
                if (rows == 1) {
                    mat_delta = mdl;
                    vec_delta = vdl;
                } else if (mdl != mat_delta || vdl != vec_delta) {
                    break;
                }
                ++rows;
            }
            out.push_back({PSC_CODELET_BLAS, rows, width, r, md.mat(r, p), rows > 1 ? mat_delta : 0,
                           md.vec(r, p), rows > 1 ? vec_delta : 0});
            cost += cost_blas(rows, width);
            for (int i = 0; i < rows; ++i)
                for (int j = p; j < q; ++j) cv.cover(r + i, j);
            p = q;
        }
    }
}

// miner.cpp:125-172 (shared gather) and 176-234 (tabulated); the two differ
// only in the identical-columns condition and in the emitted kind.
template <bool SharedGather>
void mine_psc(const Model& md, int rb, int re, Cover& cv, std::vector<Rec>& out, int64_t& cost) {
    for (int r = rb; r < re; ++r) {
        int extent = md.ext(r);
        int p = 0;
        while (p < extent) {
            if (cv.covered(r, p)) {
                ++p;
                continue;
            }
            int q = p + 1;
            while (q < extent && !cv.covered(r, q)) ++q;
            int width = q - p;
            int rows = 1, mat_delta = 0;
            while (r + rows < re) {
                int rn = r + rows;
                int ext_n = md.ext(rn);
                if (ext_n < q) break;
                bool ok = (p == 0 || cv.covered(rn, p - 1)) && (q == ext_n || cv.covered(rn, q));
                for (int j = p; j < q && ok; ++j) ok = !cv.covered(rn, j);
                if (SharedGather) {
                    for (int j = p; j < q && ok; ++j) ok = md.vec(rn, j) == md.vec(r, j);
                }
                if (!ok) break;
                int mdl = md.mat(rn, p) - md.mat(rn - 1, p);
                if (rows == 1) {
                    mat_delta = mdl;
                } else if (mdl != mat_delta) {
                    break;
                }
                ++rows;
            }
            out.push_back({static_cast<uint8_t>(SharedGather ? PSC_CODELET_PSC_I : PSC_CODELET_PSC_II),
                           rows, width, r, md.mat(r, p), rows > 1 ? mat_delta : 0, -1, 0});
            cost += SharedGather ? cost_psci(rows, width) : cost_pscii(rows, width);
            for (int i = 0; i < rows; ++i)
                for (int j = p; j < q; ++j) cv.cover(r + i, j);
            p = q;
        }
    }
}

struct Window {
    int32_t begin, end;
};

// get_consecutive_iterations, miner.cpp:18-37.
void consecutive_windows(const int32_t* rows, int64_t count, int t, std::vector<Window>& out) {
    int64_t i = 0;
    while (i < count) {
        int64_t j = i + 1;
        while (j < count && rows[j] == rows[j - 1] + 1) ++j;
        for (int64_t k = i; k < j; k += t) {
            int64_t last = std::min(j, k + t) - 1;
            out.push_back({rows[k], rows[last] + 1});
        }
        i = j;
    }
}

struct BlockResult {
    std::vector<uint8_t> strategy;
    std::vector<int64_t> cost;
    std::vector<int32_t> n_codelets;
    std::vector<Rec> codelets;
};

}  // namespace

WindowSchedule schedule_windows(int kernel, const psc_csr_view& a, int t, int target_groups) {
    require(t >= 1, "inspect: t must be >= 1");
    require(target_groups >= 1, "inspect: target_groups must be >= 1");
    require(kernel == PSC_KERNEL_SPMV || kernel == PSC_KERNEL_SPTRSV, "inspect: unknown kernel");
    // compute_access_functions: validate_csr, plus adopt() for the solve.
    if (kernel == PSC_KERNEL_SPTRSV) {
        adopt_triangular(a);
    } else {
        validate_csr(a);
    }
    const int n = a.n_rows;
    const int32_t* ro = a.row_offsets;
    Model md{ro, a.col_indices, kernel == PSC_KERNEL_SPTRSV ? 1 : 0};

    // ---- schedule (scheduler.cpp:9-105) ----
    // Dependencies exist iff some stored entry is off the diagonal; without
    // edges the schedule is balanced ranges even for the solve.
    bool has_edges = false;
    if (kernel == PSC_KERNEL_SPTRSV) {
        for (int r = 0; r < n && !has_edges; ++r) has_edges = md.ext(r) > 0;
    }
    std::vector<int32_t> part_rows;     // rows of all partitions, concatenated
    std::vector<int64_t> part_ptr{0};   // partition boundaries into part_rows
    if (!has_edges) {
        // balanced_ranges, scheduler.cpp:67-89
        if (n > 0) {
            int groups = std::min(target_groups, n);
            long long total = a.nnz, acc = 0;
            int row = 0;
            part_rows.resize(n);
            std::iota(part_rows.begin(), part_rows.end(), 0);
            for (int g = 0; g < groups; ++g) {
                long long threshold = total * (g + 1) / groups;
                int last_allowed = n - (groups - 1 - g);
                bool last = g == groups - 1;
                int begin = row;
                while (row < last_allowed && (last || row == begin || acc < threshold)) {
                    acc += ro[row + 1] - ro[row];
                    ++row;
                }
                part_ptr.push_back(row);
            }
        }
    } else {
        // level_sets, scheduler.cpp:27-65: longest-path level of every row.
        std::vector<int32_t> level(n, 0);
        int32_t max_level = 0;
        for (int r = 0; r < n; ++r) {
            int32_t lv = 0;
            for (int32_t k = ro[r]; k < ro[r + 1] - 1; ++k) lv = std::max(lv, level[a.col_indices[k]] + 1);
            level[r] = lv;
            max_level = std::max(max_level, lv);
        }
        std::vector<int64_t> cnt(static_cast<std::size_t>(max_level) + 2, 0);
        for (int r = 0; r < n; ++r) ++cnt[level[r] + 1];
        for (int32_t l = 0; l <= max_level; ++l) cnt[l + 1] += cnt[l];
        part_rows.resize(n);
        std::vector<int64_t> cur(cnt.begin(), cnt.end() - 1);
        for (int r = 0; r < n; ++r) part_rows[cur[level[r]]++] = r;  // ascending within a level
        part_ptr.assign(cnt.begin(), cnt.end());
    }
    const int64_t n_parts = static_cast<int64_t>(part_ptr.size()) - 1;

    // ---- windows ----
    std::vector<Window> windows;
    WindowSchedule ws;
    windows.reserve(static_cast<std::size_t>(n / t + n_parts + 1));
    for (int64_t p = 0; p < n_parts; ++p) {
        consecutive_windows(part_rows.data() + part_ptr[p], part_ptr[p + 1] - part_ptr[p], t, windows);
        ws.part_win_ptr.push_back(static_cast<int64_t>(windows.size()));
    }
    ws.begin.resize(windows.size());
    ws.end.resize(windows.size());
    for (std::size_t w = 0; w < windows.size(); ++w) {
        ws.begin[w] = windows[w].begin;
        ws.end[w] = windows[w].end;
    }
    return ws;
}

Plan inspect(int kernel, const psc_csr_view& a, int t, int target_groups, int threads) {
    WindowSchedule ws = schedule_windows(kernel, a, t, target_groups);
    threads = hw_threads(threads);
    Model md{a.row_offsets, a.col_indices, kernel == PSC_KERNEL_SPTRSV ? 1 : 0};
    std::vector<Window> windows(ws.begin.size());
    for (std::size_t w = 0; w < windows.size(); ++w) windows[w] = {ws.begin[w], ws.end[w]};
    const std::vector<int64_t>& part_win_ptr = ws.part_win_ptr;

    // ---- mine every window (miner.cpp:298-320), in parallel blocks ----
    const int64_t n_win = static_cast<int64_t>(windows.size());
    const int64_t block = 2048;
    const int64_t n_blocks = (n_win + block - 1) / block;
    std::vector<BlockResult> results(n_blocks);
    parallel_for(n_blocks, threads, [&](int64_t b) {
        BlockResult& res = results[b];
        Cover cover;
        std::vector<Rec> cand[3];
        int64_t w0 = b * block, w1 = std::min(n_win, w0 + block);
        res.strategy.reserve(w1 - w0);
        res.cost.reserve(w1 - w0);
        res.n_codelets.reserve(w1 - w0);
        for (int64_t w = w0; w < w1; ++w) {
            int rb = windows[w].begin, re = windows[w].end;
            int64_t cost[3] = {0, 0, 0};
            for (auto& c : cand) c.clear();
            cover.reset(md, rb, re);  // blas_first
            mine_blas(md, rb, re, cover, cand[0], cost[0]);
            mine_psc<true>(md, rb, re, cover, cand[0], cost[0]);
            cover.reset(md, rb, re);  // psci_first
            mine_psc<true>(md, rb, re, cover, cand[1], cost[1]);
            cover.reset(md, rb, re);  // pscii_first
            mine_psc<false>(md, rb, re, cover, cand[2], cost[2]);
            int best = 0;  // min cost, ties in strategy order (miner.cpp:301-306)
            for (int s = 1; s < 3; ++s)
                if (cost[s] < cost[best]) best = s;
            res.strategy.push_back(static_cast<uint8_t>(best));
            res.cost.push_back(cost[best]);
            res.n_codelets.push_back(static_cast<int32_t>(cand[best].size()));
            res.codelets.insert(res.codelets.end(), cand[best].begin(), cand[best].end());
        }
    });

    // ---- stitch ----
    Plan plan;
    plan.kernel = kernel;
    plan.n_rows = a.n_rows;
    plan.n_cols = a.n_cols;
    plan.nnz = a.nnz;
    plan.window = t;
    plan.target_groups = target_groups;
    plan.mined = true;
    plan.part_group_ptr.assign(part_win_ptr.begin(), part_win_ptr.end());
    plan.g_row_begin.resize(n_win);
    plan.g_row_end.resize(n_win);
    plan.g_strategy.resize(n_win);
    plan.g_cost.resize(n_win);
    plan.g_codelet_ptr.assign(n_win + 1, 0);
    std::vector<int64_t> block_codelet_base(n_blocks + 1, 0);
    for (int64_t b = 0; b < n_blocks; ++b)
        block_codelet_base[b + 1] = block_codelet_base[b] + static_cast<int64_t>(results[b].codelets.size());
    const int64_t n_cod = block_codelet_base[n_blocks];
    plan.c_kind.resize(n_cod);
    plan.c_m.resize(n_cod);
    plan.c_n.resize(n_cod);
    plan.c_row.resize(n_cod);
    plan.c_mat_base.resize(n_cod);
    plan.c_mat_so.resize(n_cod);
    plan.c_vec_base.resize(n_cod);
    plan.c_vec_so.resize(n_cod);
    parallel_for(n_blocks, threads, [&](int64_t b) {
        BlockResult& res = results[b];
        int64_t w0 = b * block;
        int64_t c = block_codelet_base[b];
        for (std::size_t i = 0; i < res.strategy.size(); ++i) {
            int64_t w = w0 + static_cast<int64_t>(i);
            plan.g_row_begin[w] = windows[w].begin;
            plan.g_row_end[w] = windows[w].end;
            plan.g_strategy[w] = res.strategy[i];
            plan.g_cost[w] = res.cost[i];
        }
        for (const Rec& r : res.codelets) {
            plan.c_kind[c] = r.kind;
            plan.c_m[c] = r.m;
            plan.c_n[c] = r.n;
            plan.c_row[c] = r.row;
            plan.c_mat_base[c] = r.mat_base;
            plan.c_mat_so[c] = r.mat_so;
            plan.c_vec_base[c] = r.vec_base;
            plan.c_vec_so[c] = r.vec_so;
            ++c;
        }
    });
    for (int64_t b = 0, w = 0; b < n_blocks; ++b) {
        int64_t c = block_codelet_base[b];
        for (int32_t k : results[b].n_codelets) {
            c += k;
            plan.g_codelet_ptr[++w] = c;
        }
    }
    return plan;
}

}  // namespace pscb
