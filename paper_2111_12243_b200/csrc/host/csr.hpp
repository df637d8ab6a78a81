// CSR storage and the input generators (host side).
#pragma once

#include <cstdint>
#include <string>
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

// csr_matrix.cpp:9-45: stable sort by (row, col), duplicates summed in order.
Csr csr_from_triplets(int32_t n_rows, int32_t n_cols, std::vector<Triplet> entries);
// csr_matrix.cpp:47-76
void validate_csr(const psc_csr_view& a);
// csr_matrix.cpp:87-109 (square, lower, diagonal stored last and nonzero)
void adopt_triangular(const psc_csr_view& a);
// csr_matrix.cpp:111-130
Csr lower_triangular(const psc_csr_view& a);

// pattern_gen.cpp restated (test inputs of the reference suite).
Csr dense_block(int n);
Csr banded(int n, int bandwidth, bool lower_only);
Csr scattered_gather(int rows, std::vector<int> cols);
Csr random_uniform(int rows, int cols, double density, uint64_t seed);
Csr generate_pattern(const std::string& spec, uint64_t default_seed);

// BASELINE.json configs 1..5.
Csr generate_config(int config, double scale, uint64_t seed);

double to_unit(uint64_t bits);  // (bits >> 11) * 2^-53, pattern_gen.cpp:12-14

}  // namespace pscb
