// Benchmark inputs: BASELINE.json configs 1..5 and seeded vectors
// (configs.cpp). Self-contained (needs csr.hpp's Csr and common.hpp only), so
// oracle/Makefile can compile it into the reference arm's library as well.
#pragma once

#include <cstdint>

#include "csr.hpp"

namespace pscb {

double to_unit(uint64_t bits);  // (bits >> 11) * 2^-53
// BASELINE.json configs 1..5; scale in (0, 1] shrinks the grid / n; seed 0
// selects the config's default stream.
Csr generate_config(int config, double scale, uint64_t seed);
void seeded_vector(int64_t n, uint64_t seed, double* out);                     // 0.5 + U[0,1)
void uniform_vector(int64_t n, uint64_t seed, double lo, double hi, double* out);  // U[lo, hi)
void int_vector(int64_t n, uint64_t seed, double* out);                        // 1 + (bits mod 9)

}  // namespace pscb
