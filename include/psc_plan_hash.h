/*
 * psc_plan_hash.h — the canonical plan stream digest shared by the product
 * (paper_2111_12243_b200/csrc/host/plan.cpp) and the reference shim
 * (oracle/ref_shim.cpp), so a plan mined by either side can be compared at
 * full benchmark size without exporting gigabytes of tables.
 *
 * Stream (every field widened to 64 bits, in this order):
 *   kernel n_rows n_cols nnz window target_groups n_partitions
 *   per partition: n_groups
 *     per group: row_begin row_end strategy cost n_codelets
 *       per codelet: kind m n, then for out, mat, vec:
 *         form base stride_outer stride_inner table_len table[0..len)
 *       n_finalize, per record: row diag_pos rhs_index
 * Strided descriptors carry an empty table; table descriptors carry a zero
 * StridedAccess, exactly as the reference's AccessDesc factories build them
 * (codelet.hpp:43-54).
 */
#ifndef PSC_PLAN_HASH_H
#define PSC_PLAN_HASH_H

#include <stdint.h>

static inline uint64_t psc_hash_mix(uint64_t h, uint64_t v) {
    v *= 0x9E3779B97F4A7C15ULL;
    v ^= v >> 29;
    h ^= v;
    h = (h << 27) | (h >> 37);
    return h * 0x94D049BB133111EBULL + 0x632BE59BD9B4E019ULL;
}

#define PSC_HASH_SEED 0x2111122430000000ULL

#endif
