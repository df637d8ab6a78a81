// CSR storage and validation (host side).
#pragma once

#include <cstdint>
#include <vector>

#include "psc_b200.h"

namespace pscb {

// Owned CSR, the same layout as psc::CsrMatrix (csr_matrix.hpp:9-20):
// int32 offsets and columns (sorted, unique per row), fp64 values.
struct Csr {
    int32_t n_rows = 0;
    int32_t n_cols = 0;
    std::vector<int32_t> row_offsets;
    std::vector<int32_t> col_indices;
    std::vector<double> values;

    int64_t nnz() const { return static_cast<int64_t>(col_indices.size()); }
    psc_csr_view view() const {
        return {n_rows, n_cols, nnz(), row_offsets.data(), col_indices.data(), values.data()};
    }
};

struct Triplet {
    int32_t row, col;
    double value;
};

// csr_matrix.cpp:9-45 semantics: rows and columns in order, duplicates summed in input order.
Csr csr_from_triplets(int32_t n_rows, int32_t n_cols, std::vector<Triplet> entries);
// csr_matrix.cpp:47-76
void validate_csr(const psc_csr_view& a);
// csr_matrix.cpp:87-109 (square, lower, diagonal stored last and nonzero)
void adopt_triangular(const psc_csr_view& a);
// csr_matrix.cpp:111-130
Csr lower_triangular(const psc_csr_view& a);
// 64-bit hash of sizes, row offsets and columns (not values), thread-count independent.
uint64_t structure_hash(const psc_csr_view& a);

}  // namespace pscb
