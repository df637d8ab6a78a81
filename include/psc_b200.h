/*
 * psc_b200.h — C ABI of the B200-native DDF codelet executor.
 *
 * This is the drop-in boundary for the reference's executor path
 * (/root/reference/proj/core/include/psc/executor.hpp:17-65) and for the
 * inspector output it consumes (miner.hpp:23-98). Every entry point takes
 * plain pointers and sizes; no C++ or torch types cross the boundary. Each
 * function returns a psc_status; on failure psc_last_error() returns a
 * thread-local message. Status codes map one-to-one onto the exception types
 * the reference throws:
 *   PSC_ERR_INVALID_ARGUMENT  <->  std::invalid_argument
 *   PSC_ERR_LOGIC             <->  std::logic_error   (validate_plan)
 * The remaining codes (CUDA, memory) have no reference counterpart.
 *
 * Ownership mirrors the reference: the caller owns matrices, plans and
 * vectors; an executor owns its device state (the reference Executor owns its
 * thread pool, executor.hpp:36-51).
 */
#ifndef PSC_B200_H
#define PSC_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#if defined(__GNUC__)
#define PSC_API __attribute__((visibility("default")))
#else
#define PSC_API
#endif

/* ---- status -------------------------------------------------------------- */
typedef int psc_status;
enum {
    PSC_OK = 0,
    PSC_ERR_INVALID_ARGUMENT = 1, /* std::invalid_argument */
    PSC_ERR_LOGIC = 2,            /* std::logic_error */
    PSC_ERR_CUDA = 3,             /* CUDA runtime failure / no device */
    PSC_ERR_NOMEM = 4,
    PSC_ERR_INTERNAL = 5
};
PSC_API const char* psc_last_error(void);

/* ---- enums (reference enum order, so integer values match static_cast) --- */
enum { PSC_KERNEL_SPMV = 0, PSC_KERNEL_SPTRSV = 1 };                   /* kernel_model.hpp:10 */
enum { PSC_CODELET_BLAS = 0, PSC_CODELET_PSC_I = 1, PSC_CODELET_PSC_II = 2 }; /* codelet.hpp:8 */
enum {                                                                  /* codelet.hpp:29 */
    PSC_FORM_STRIDED = 0,
    PSC_FORM_INNER_TABLE = 1,
    PSC_FORM_OUTER_TABLE = 2,
    PSC_FORM_POINT_TABLE = 3
};
enum { PSC_STRATEGY_BLAS_FIRST = 0, PSC_STRATEGY_PSCI_FIRST = 1, PSC_STRATEGY_PSCII_FIRST = 2 }; /* miner.hpp:46 */

/* ---- CSR view (csr_matrix.hpp:9-20) --------------------------------------- */
typedef struct psc_csr_view {
    int32_t n_rows;
    int32_t n_cols;
    int64_t nnz;
    const int32_t* row_offsets; /* n_rows + 1 */
    const int32_t* col_indices; /* nnz */
    const double* values;       /* nnz */
} psc_csr_view;

/* ---- one codelet (codelet.hpp:12-71) -------------------------------------- */
typedef struct psc_access_desc_view {
    int32_t form;         /* PSC_FORM_* */
    int32_t base;         /* StridedAccess lin (zero for tables) */
    int32_t stride_outer;
    int32_t stride_inner;
    const int32_t* table; /* NULL for strided */
    int64_t table_len;
} psc_access_desc_view;

typedef struct psc_codelet_view {
    int32_t kind;         /* PSC_CODELET_* */
    int32_t outer_extent; /* m */
    int32_t inner_extent; /* n */
    psc_access_desc_view out, mat, vec;
} psc_codelet_view;

/* ---- whole plan as SoA arrays (miner.hpp:56-89) ---------------------------
 * Partition p owns groups [part_group_ptr[p], part_group_ptr[p+1]); group g
 * owns codelets [group_codelet_ptr[g], +1) and finalize records
 * [group_finalize_ptr[g], +1). Descriptor d of codelet c (d = 0 out, 1 mat,
 * 2 vec) lives at index 3*c+d; its table is
 * table[desc_table_ptr[3c+d] .. desc_table_ptr[3c+d+1]).
 * psc_plan_to_arrays() fills caller-allocated arrays sized by
 * psc_plan_get_counts(); psc_plan_from_arrays() reads them.
 */
typedef struct psc_plan_counts {
    int32_t kernel;
    int32_t n_rows;
    int32_t n_cols;
    int32_t window;        /* t */
    int32_t target_groups;
    int64_t nnz;
    int64_t n_partitions;
    int64_t n_groups;
    int64_t n_codelets;
    int64_t n_finalize;
    int64_t n_table;       /* total table entries */
} psc_plan_counts;

typedef struct psc_plan_arrays {
    int64_t* part_group_ptr;     /* n_partitions + 1 */
    int32_t* group_row_begin;    /* n_groups */
    int32_t* group_row_end;
    int32_t* group_strategy;
    int64_t* group_cost;
    int64_t* group_codelet_ptr;  /* n_groups + 1 */
    int64_t* group_finalize_ptr; /* n_groups + 1 */
    int32_t* codelet_kind;       /* n_codelets */
    int32_t* codelet_m;
    int32_t* codelet_n;
    int32_t* desc_form;          /* 3 * n_codelets */
    int32_t* desc_base;
    int32_t* desc_stride_outer;
    int32_t* desc_stride_inner;
    int64_t* desc_table_ptr;     /* 3 * n_codelets + 1 */
    int32_t* table;              /* n_table */
    int32_t* fin_row;            /* n_finalize */
    int32_t* fin_diag_pos;
    int32_t* fin_rhs_index;
} psc_plan_arrays;

typedef struct psc_plan psc_plan;         /* CodeletPlan */
typedef struct psc_executor psc_executor; /* Executor */
typedef struct psc_bound psc_bound;       /* plan + matrix resident in HBM */
typedef struct psc_exec_context psc_exec_context; /* ExecutionContext, defined below */

/* ---- inspector (miner.hpp:95, inspect) -------------------------------------
 * Bit-exact restatement of the reference inspector: same partitions,
 * windows, strategy choice, costs, codelets, descriptors and finalize records.
 * threads <= 0 uses every hardware thread; the plan never depends on it. */
PSC_API psc_status psc_inspect(int32_t kernel, const psc_csr_view* a, int32_t t,
                               int32_t target_groups, int32_t threads, psc_plan** out);
/* The same inspection with the window mining on GPU `device` (one thread per
 * window, the three strategies of miner.cpp:298-320, cuda/inspect.cu); the
 * schedule and windows are computed on the host. Returns the same plan as
 * psc_inspect, bit for bit. */
PSC_API psc_status psc_inspect_device(int32_t kernel, const psc_csr_view* a, int32_t t,
                                      int32_t target_groups, int32_t device, psc_plan** out);
PSC_API psc_status psc_plan_get_counts(const psc_plan* plan, psc_plan_counts* out);
/* Mined plans keep their tables implicit (verbatim slices of col_indices,
 * miner.cpp:156-164, 206-226), so export needs the matrix they came from. */
PSC_API psc_status psc_plan_to_arrays(const psc_plan* plan, const psc_csr_view* a,
                                      psc_plan_arrays* out);
PSC_API psc_status psc_plan_from_arrays(const psc_plan_counts* counts,
                                        const psc_plan_arrays* arrays, psc_plan** out);
/* 64-bit digest of the canonical plan stream; equal plans
 * hash equal here and in oracle/ref_shim.cpp's ref_plan_hash. */
PSC_API psc_status psc_plan_hash(const psc_plan* plan, const psc_csr_view* a, uint64_t* out);
PSC_API psc_status psc_plan_totals(const psc_plan* plan, int64_t* total_cost, int64_t* total_ops,
                                   int64_t ops_by_kind[3]);
/* Rows covered by partitions [part_begin, part_end): the union of their
 * windows, which must be one contiguous range (SpMV balanced ranges,
 * scheduler.cpp:67-89). Used to shard a plan over GPUs. */
PSC_API psc_status psc_plan_partition_rows(const psc_plan* plan, int64_t part_begin, int64_t part_end,
                                           int32_t* row_begin, int32_t* row_end);
/* validate_plan (miner.cpp:325-395): PSC_ERR_LOGIC on violation. */
PSC_API psc_status psc_validate_plan(const psc_plan* plan, const psc_csr_view* a);
PSC_API void psc_plan_destroy(psc_plan* plan);

/* Binary plan files (the reference only writes a JSON dump,
 * plan_io.cpp:52-83): the plan as held in memory, reloadable without
 * re-inspection. Validate a loaded plan against its matrix with
 * psc_validate_plan before executing it. */
PSC_API psc_status psc_plan_save(const psc_plan* plan, const char* path);
PSC_API psc_status psc_plan_load(const char* path, psc_plan** out);

/* ---- executor (executor.hpp:36-51) -----------------------------------------
 * workers < 1 -> PSC_ERR_INVALID_ARGUMENT (executor.cpp:253-255). The worker
 * count is accepted for API compatibility; the GPU schedule never depends on
 * it, so results are bitwise identical for every value (executor.hpp:29-35). */
PSC_API psc_status psc_executor_create(int32_t workers, int32_t device, psc_executor** out);
PSC_API int32_t psc_executor_workers(const psc_executor* exec);
/* The run_* / execute_plan calls read the matrix values on every call, as the
 * reference does (they may change between calls). A caller whose values do
 * not change tags them with a nonzero version: a call whose bound plan already
 * holds values of that version skips their upload; any other version uploads
 * them again. 0 (the default) means "unknown": always upload. Not in the
 * reference (it has no device copy to keep). */
PSC_API psc_status psc_executor_set_values_version(psc_executor* exec, uint64_t version);
PSC_API void psc_executor_destroy(psc_executor* exec);

/* Bind a plan and its matrix: lowers the plan to device segments and uploads
 * CSR + plan once (inspector-executor amortisation). The matrix view points to
 * HOST memory. mode: 0 = parity (bitwise equal to the reference executor),
 * 1 = fast: SpMV plans whose rows are single codelet rows (configs 1, 5) run
 * with reassociated row sums (spmv_fast.cu; deterministic, within 1e-12
 * normwise of the reference); other plans and SpTRSV run the parity kernels
 * in either mode. */
enum { PSC_MODE_PARITY = 0, PSC_MODE_FAST = 1 };
PSC_API psc_status psc_bind(psc_executor* exec, const psc_plan* plan, const psc_csr_view* a,
                            int32_t mode, psc_bound** out);
/* Bind only partitions [part_begin, part_end) of a SpMV plan (multi-GPU
 * row shards, scheduler.cpp:67-89 ranges). y receives rows
 * [row_begin, row_end) of the shard at y[0..). */
PSC_API psc_status psc_bind_partitions(psc_executor* exec, const psc_plan* plan,
                                       const psc_csr_view* a, int32_t mode, int64_t part_begin,
                                       int64_t part_end, psc_bound** out);
PSC_API psc_status psc_bound_rows(const psc_bound* b, int32_t* row_begin, int32_t* row_end);
PSC_API void psc_bound_destroy(psc_bound* b);

/* Device-pointer execution on a CUDA stream (cudaStream_t passed as void*;
 * NULL = legacy default stream). Asynchronous: returns after enqueue. */
PSC_API psc_status psc_bound_spmv(psc_bound* b, const double* x_dev, double* y_dev, void* stream);
PSC_API psc_status psc_bound_sptrsv(psc_bound* b, const double* b_dev, double* x_dev,
                                    double* acc_dev /* nullable */, void* stream);
/* Host-buffer variants (the end-to-end path): H2D of the input vector, the
 * kernel, and D2H of the result, enqueued on `stream` (pinned host memory
 * makes the copies asynchronous). They share the bound's scratch buffers:
 * calls on one bound from several threads or streams are serialised, each
 * enqueued after the previous call's work. */
PSC_API psc_status psc_bound_spmv_host(psc_bound* b, const double* x_host, double* y_host, void* stream);
PSC_API psc_status psc_bound_sptrsv_host(psc_bound* b, const double* b_host, double* x_host,
                                         double* acc_host /* nullable */, void* stream);
/* Diagnostics (PSC_TRSV_TRACE=1 at bind): per-row publish times of the last
 * solve in ns (%globaltimer), then one arm time per row block. Returns the
 * number of entries copied (0 when tracing is off). */
PSC_API int64_t psc_bound_trace(const psc_bound* b, uint64_t* out, int64_t cap);
/* Number of kernel launches one psc_bound_* call enqueues. */
PSC_API int32_t psc_bound_launches(const psc_bound* b);
/* Lowering diagnostics, out[0..7]: rows, segments (0 = every row is one
 * implicit full-row segment), work units (SpMV chunks, or the warp items of
 * the shifted-run kernel when it is in use / SpTRSV row blocks),
 * path (0 parity kernels, 1 general interpreter, 2 fast-mode SpMV),
 * algorithmic bytes per call, device bytes held, long rows,
 * column passes (SpMV; 0 = one pass over all of x) / max block rows (SpTRSV). */
PSC_API psc_status psc_bound_info(const psc_bound* b, int64_t out[8]);
/* ---- multi-GPU SpMV: fused x exchange over peer memory --------------------
 * A rank that bound a shard (psc_bind_partitions) of a simple SpMV plan reads
 * x entries owned by other ranks. Replaces the reference's none (the
 * reference is single-node, single-process); DESIGN.md "Multi-GPU". */
typedef struct psc_peer_window {
    const double* base;  /* rank q's full-length x window (a peer pointer, or x_window itself) */
    int32_t row_begin;   /* rows (= x entries) rank q owns: [row_begin, row_end) */
    int32_t row_end;
} psc_peer_window;

/* The column runs [runs[2i], runs[2i+1]) outside the shard's own rows that
 * its multiply reads (runs may be NULL to query the count). */
PSC_API psc_status psc_bound_x_runs(const psc_bound* b, int32_t* runs, int64_t cap, int64_t* n_runs);

/* y = A_shard x in one launch sequence: the kernel's first CTAs pull the
 * runs this shard reads from the peers' windows into x_window (which already
 * holds this rank's own x entries); work that reads only own columns starts
 * at once, the rest waits for the pulled pieces. Peers must tile the columns
 * in rank order. The caller orders ranks around it (every window written
 * before any rank launches; no window rewritten until every rank's launch
 * finished). Bitwise equal to psc_bound_spmv on the gathered x. */
PSC_API psc_status psc_bound_spmv_peers(psc_bound* b, const psc_peer_window* peers, int32_t n_peers, double* x_window,
                                        double* y, void* stream);

/* CUDA IPC helpers for peer windows: allocate shareable device memory and
 * export its 64-byte handle; open / close a peer's handle; free. */
PSC_API psc_status psc_ipc_alloc(int64_t bytes, void** ptr, uint8_t handle[64]);
PSC_API psc_status psc_ipc_open(const uint8_t handle[64], void** ptr);
PSC_API psc_status psc_ipc_close(void* ptr);
PSC_API psc_status psc_ipc_free(void* ptr);
/* Stream-ordered copy between any two (device or host) addresses. */
PSC_API psc_status psc_copy_async(void* dst, const void* src, int64_t bytes, void* stream);

/* Diagnostic: count mismatches between the solve kernels' division (exact
 * reciprocal refinement + final correction, __ddiv_rn outside exponents
 * [-500, 500]) and IEEE division on n random operand pairs whose exponents
 * lie in [-exp_span, exp_span]. Replaces no reference interface. */
PSC_API psc_status psc_selftest_division(uint64_t seed, int64_t n, int32_t exp_span, int64_t* mismatches);

PSC_API int32_t psc_device_count(void);

/* Host-span entry points with the reference's contracts (executor.cpp:274-308):
 * size checks, zero-fill of y / acc, H2D of inputs, D2H of results. The bound
 * device plan is cached per (plan, matrix arrays) inside the executor. */
PSC_API psc_status psc_run_spmv(psc_executor* exec, const psc_plan* plan, const psc_csr_view* a,
                                const double* x, int64_t nx, double* y, int64_t ny);
PSC_API psc_status psc_run_sptrsv(psc_executor* exec, const psc_plan* plan,
                                  const psc_csr_view* l, const double* b, int64_t nb, double* x,
                                  int64_t nx, double* acc, int64_t nacc);

/* execute_plan (executor.cpp:269-272): runs the plan over a raw context
 * WITHOUT zero-filling accum (accumulates onto its contents). The matrix view
 * supplies the CSR structure of the plan's implicit tables; values come from
 * ctx->matrix_values. rhs != NULL selects the solve. Host pointers. */
PSC_API psc_status psc_execute_plan(psc_executor* exec, const psc_plan* plan, const psc_csr_view* a,
                                    const psc_exec_context* ctx);

/* Executor::run (executor.hpp:45, executor.cpp:261-267) on a plan that
 * carries its tables -- the reference's own CodeletPlan imported with
 * psc_plan_from_arrays -- over a raw host context, no matrix argument:
 * partitions in order, each group's codelets then its finalize records,
 * accumulating onto ctx->accum (execute_plan(plan, ctx, workers) is a
 * temporary executor's run). A plan mined by psc_inspect keeps its tables
 * in the matrix: PSC_ERR_INVALID_ARGUMENT (use psc_execute_plan). */
PSC_API psc_status psc_executor_run(psc_executor* exec, const psc_plan* plan, const psc_exec_context* ctx);

/* Single-codelet execution on the GPU with exact exec_*_codelet semantics
 * (executor.cpp:53-116), including hand-built codelets with arbitrary tables.
 * Pointers are HOST memory laid out as in ExecutionContext (executor.hpp:17-23);
 * the touched index range is derived from the descriptors. */
struct psc_exec_context {
    const double* matrix_values;
    const double* gather;
    double* accum;
    const double* rhs; /* non-NULL selects the solve (sequential-sum) branch */
    double* solution;
};
PSC_API psc_status psc_exec_blas_codelet(const psc_codelet_view* c, const psc_exec_context* ctx);
PSC_API psc_status psc_exec_psci_codelet(const psc_codelet_view* c, const psc_exec_context* ctx);
PSC_API psc_status psc_exec_pscii_codelet(const psc_codelet_view* c, const psc_exec_context* ctx);

/* Naive CSR kernels on the GPU, the device analogue of spmv_csr_baseline /
 * sptrsv_csr_baseline (executor.cpp:310-340); device pointers. */
PSC_API psc_status psc_csr_spmv_device(const psc_bound* b, const double* x_dev, double* y_dev,
                                       void* stream);
/* Forward substitution, one thread per row, sync-free (b: an SpTRSV bound
 * plan; its CSR is used, the plan is not). x_dev is overwritten. */
PSC_API psc_status psc_csr_sptrsv_device(psc_bound* b, const double* b_dev, double* x_dev, void* stream);

/* ---- matrices: construction, validation, Matrix Market, benchmark configs -- */
typedef struct psc_csr psc_csr; /* owned CSR */
PSC_API psc_status psc_csr_view_of(const psc_csr* m, psc_csr_view* out);
PSC_API void psc_csr_destroy(psc_csr* m);
PSC_API psc_status psc_csr_from_triplets(int32_t n_rows, int32_t n_cols, int64_t n,
                                         const int32_t* rows, const int32_t* cols,
                                         const double* vals, psc_csr** out);
/* The reference's sequential CSR baselines on host arrays (spmv_csr_baseline /
 * sptrsv_csr_baseline, executor.cpp:310-340): y = A x, and forward
 * substitution on a lower triangle with the diagonal stored last. */
PSC_API psc_status psc_csr_spmv_baseline(const psc_csr_view* a, const double* x, int64_t nx, double* y, int64_t ny);
PSC_API psc_status psc_csr_sptrsv_baseline(const psc_csr_view* l, const double* b, int64_t nb, double* x, int64_t nx);

/* Matrix Market coordinate files (matrix_market.hpp:24-34): read real,
 * integer or pattern / general or symmetric (mirrored), duplicates summed,
 * 0-based; errors are PSC_ERR_INVALID_ARGUMENT "line N: ..." (the reference's
 * ParseError). Write: coordinate real general, 1-based, 17 significant digits. */
PSC_API psc_status psc_csr_read_matrix_market(const char* path, psc_csr** out);
PSC_API psc_status psc_csr_write_matrix_market(const psc_csr_view* a, const char* path);

PSC_API psc_status psc_validate_csr(const psc_csr_view* a);
PSC_API psc_status psc_lower_triangular(const psc_csr_view* a, psc_csr** out);
PSC_API psc_status psc_adopt_triangular(const psc_csr_view* a); /* TriangularMatrix::adopt checks */
/* BASELINE.json configs 1..5; scale in (0,1] shrinks the
 * grid / n for tests; seed selects the value stream. */
PSC_API psc_status psc_generate_config(int32_t config, double scale, uint64_t seed, psc_csr** out);
/* std::mt19937_64 streams used by the reference's benches and tests. */
PSC_API void psc_seeded_vector(int64_t n, uint64_t seed, double* out);           /* bench.cpp:50-57 */
PSC_API void psc_uniform_vector(int64_t n, uint64_t seed, double lo, double hi, double* out);
PSC_API void psc_int_vector(int64_t n, uint64_t seed, double* out);              /* test_helpers.hpp:45-50 */

#ifdef __cplusplus
}
#endif
#endif /* PSC_B200_H */
