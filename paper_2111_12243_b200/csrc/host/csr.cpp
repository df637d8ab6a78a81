// CSR construction and validation (the checks of /root/reference/proj/core/
// src/csr_matrix.cpp:9-130, same messages and exception types). The
// benchmark input generators live in configs.cpp.
#include "csr.hpp"

#include <algorithm>
#include <cmath>
#include <numeric>

#include "common.hpp"

namespace pscb {

// Triplets -> CSR with the reference's semantics (csr_matrix.cpp:9-45): rows
// and columns in order, duplicates summed in input order. Built as a stable
// counting sort by row, then an insertion sort of each row's (column, input
// position) keys, so equal columns stay in input order.
Csr csr_from_triplets(int32_t n_rows, int32_t n_cols, std::vector<Triplet> entries) {
    require(n_rows >= 0 && n_cols >= 0, "csr_from_triplets: negative dimension");
    std::vector<int64_t> start(static_cast<std::size_t>(n_rows) + 1, 0);
    for (const Triplet& t : entries) {
        if (t.row < 0 || t.row >= n_rows || t.col < 0 || t.col >= n_cols) {
            throw std::invalid_argument("csr_from_triplets: entry (" + std::to_string(t.row) +
                                        ", " + std::to_string(t.col) + ") out of range");
        }
        ++start[t.row + 1];
    }
    for (int32_t r = 0; r < n_rows; ++r) start[r + 1] += start[r];
    std::vector<int64_t> order(entries.size());  // input positions grouped by row, in input order
    {
        std::vector<int64_t> next(start.begin(), start.end() - 1);
        for (std::size_t i = 0; i < entries.size(); ++i) order[next[entries[i].row]++] = static_cast<int64_t>(i);
    }
    Csr a;
    a.n_rows = n_rows;
    a.n_cols = n_cols;
    a.row_offsets.assign(static_cast<std::size_t>(n_rows) + 1, 0);
    for (int32_t r = 0; r < n_rows; ++r) {
        const auto first = order.begin() + start[r], last = order.begin() + start[r + 1];
        std::stable_sort(first, last, [&](int64_t p, int64_t q) { return entries[p].col < entries[q].col; });
        for (auto it = first; it != last;) {
            const int32_t c = entries[*it].col;
            double sum = 0.0;
            for (; it != last && entries[*it].col == c; ++it) sum += entries[*it].value;
            a.col_indices.push_back(c);
            a.values.push_back(sum);
        }
        a.row_offsets[r + 1] = static_cast<int32_t>(a.col_indices.size());
    }
    return a;
}

namespace {
// The first row (in row order) for which bad(row) returns a nonzero code,
// searched over row blocks on every host thread: the same row -- and so the
// same error -- as a sequential scan.
template <class F>
std::pair<int32_t, int> first_bad_row(int32_t n_rows, F&& bad) {
    constexpr int32_t kBlock = 1 << 16;
    const int64_t n_blocks = (static_cast<int64_t>(n_rows) + kBlock - 1) / kBlock;
    std::vector<std::pair<int32_t, int>> found(static_cast<std::size_t>(n_blocks), {-1, 0});
    parallel_for(n_blocks, hw_threads(0), [&](int64_t b) {
        const int32_t r0 = static_cast<int32_t>(b * kBlock);
        const int32_t r1 = static_cast<int32_t>(std::min<int64_t>(n_rows, r0 + static_cast<int64_t>(kBlock)));
        for (int32_t row = r0; row < r1; ++row) {
            if (const int code = bad(row)) {
                found[b] = {row, code};
                return;
            }
        }
    });
    for (const auto& f : found)
        if (f.first >= 0) return f;
    return {-1, 0};
}
}  // namespace

void validate_csr(const psc_csr_view& a) {
    require(a.n_rows >= 0 && a.n_cols >= 0, "csr: negative dimension");
    require(a.row_offsets != nullptr, "csr: row_offsets size mismatch");
    require(a.row_offsets[0] == 0 && a.row_offsets[a.n_rows] == a.nnz,
            "csr: row_offsets endpoints mismatch");
    require(a.nnz <= INT32_MAX, "csr: more than 2^31-1 stored entries");
    const auto [row, code] = first_bad_row(a.n_rows, [&](int32_t r) {
        const int32_t b = a.row_offsets[r], e = a.row_offsets[r + 1];
        if (b > e) return 1;
        for (int32_t k = b; k < e; ++k) {
            const int32_t c = a.col_indices[k];
            if (c < 0 || c >= a.n_cols) return 2;
            if (k > b && c <= a.col_indices[k - 1]) return 3;
        }
        return 0;
    });
    if (code == 1) throw std::invalid_argument("csr: row_offsets not monotone at row " + std::to_string(row));
    if (code == 2) throw std::invalid_argument("csr: column out of range in row " + std::to_string(row));
    if (code == 3) throw std::invalid_argument("csr: columns not strictly increasing in row " + std::to_string(row));
}

void adopt_triangular(const psc_csr_view& a) {
    validate_csr(a);
    require(a.n_rows == a.n_cols, "triangular: matrix not square");
    // every entry above the diagonal is reported before any diagonal problem
    if (first_bad_row(a.n_rows, [&](int32_t r) {
            for (int32_t k = a.row_offsets[r]; k < a.row_offsets[r + 1]; ++k)
                if (a.col_indices[k] > r) return 1;
            return 0;
        }).second)
        throw std::invalid_argument("triangular: entry above the diagonal");
    const auto [row, code] = first_bad_row(a.n_rows, [&](int32_t r) {
        const int32_t last = a.row_offsets[r + 1] - 1;
        if (last < a.row_offsets[r] || a.col_indices[last] != r) return 1;
        if (a.values[last] == 0.0) return 2;
        return 0;
    });
    if (code == 1) throw std::invalid_argument("triangular: missing diagonal at row " + std::to_string(row));
    if (code == 2) throw std::invalid_argument("triangular: zero diagonal at row " + std::to_string(row));
}

Csr lower_triangular(const psc_csr_view& a) {
    validate_csr(a);
    require(a.n_rows == a.n_cols, "lower_triangular: matrix not square");
    Csr l;
    l.n_rows = a.n_rows;
    l.n_cols = a.n_cols;
    l.row_offsets.assign(static_cast<std::size_t>(a.n_rows) + 1, 0);
    for (int32_t row = 0; row < a.n_rows; ++row) {
        for (int32_t k = a.row_offsets[row]; k < a.row_offsets[row + 1]; ++k) {
            if (a.col_indices[k] <= row) {
                l.col_indices.push_back(a.col_indices[k]);
                l.values.push_back(a.values[k]);
            }
        }
        l.row_offsets[row + 1] = static_cast<int32_t>(l.col_indices.size());
    }
    adopt_triangular(l.view());
    return l;
}

// 64-bit hash of the CSR structure -- sizes, every row offset and column --
// over blocks on every host thread, combined in block order (so it does not
// depend on the thread count). Plans mined from a matrix record it, so a
// plan bound to another matrix is refused (executor.cpp binds), and the run_*
// cache re-checks it on every call: the reference re-reads the structure on
// every call (executor.cpp:274-308), so an in-place edit must rebind. O(nnz),
// cheaper than the values upload a run_* call does anyway.
uint64_t structure_hash(const psc_csr_view& a) {
    auto mix = [](uint64_t h, uint64_t v) {
        h ^= v + 0x9E3779B97F4A7C15ull + (h << 6) + (h >> 2);
        return h * 0xFF51AFD7ED558CCDull;
    };
    constexpr int64_t kBlock = 1 << 20;
    const int64_t n_ro = a.row_offsets ? static_cast<int64_t>(a.n_rows) + 1 : 0;
    const int64_t n_ci = a.col_indices ? a.nnz : 0;
    const int64_t total = n_ro + n_ci;
    const int64_t n_blocks = (total + kBlock - 1) / kBlock;
    std::vector<uint64_t> part(static_cast<size_t>(n_blocks));
    parallel_for(n_blocks, hw_threads(0), [&](int64_t blk) {
        uint64_t h = static_cast<uint64_t>(blk) + 1;
        const int64_t i1 = std::min(total, (blk + 1) * kBlock);
        for (int64_t i = blk * kBlock; i < i1; ++i) {
            const int32_t v = i < n_ro ? a.row_offsets[i] : a.col_indices[i - n_ro];
            h = (h ^ static_cast<uint32_t>(v)) * 0x100000001B3ull;
        }
        part[blk] = h;
    });
    uint64_t h = mix(mix(mix(0x5157u, static_cast<uint64_t>(a.n_rows)), static_cast<uint64_t>(a.n_cols)),
                     static_cast<uint64_t>(a.nnz));
    for (uint64_t p : part) h = mix(h, p);
    return h;
}

}  // namespace pscb
