// GPU window mining: the inspector's hot loop (miner.cpp:298-320: three
// strategies per window, the cheapest kept) run one thread per window.
//
// The schedule and the windows come from the host (schedule_windows in
// host/inspector.cpp: level sets are one pass in row order); windows are
// independent, so each thread mines its window's rows with
// the three strategies of miner.cpp:301-306 -- blas_first (mine_blas, then
// the shared-gather PSC miner), psci_first, pscii_first -- exactly as the host
// restatement does (host/inspector.cpp, itself pinned bit-exact to the
// reference), against a cover map that is one byte per operation in a
// matrix-wide array (windows own disjoint ranges of it). Pass 0 keeps each
// window's cheapest strategy (ties in strategy order), its cost and its
// codelet count; after a prefix sum on the host, pass 1 re-mines that
// strategy and writes the codelet records {kind, m, n, row, mat base, mat
// row stride, vec base, vec row stride} at the window's offset.
#include <cuda_runtime.h>

#include <chrono>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "capi_types.hpp"
#include "common.hpp"
#include "plan.hpp"

namespace pscb {

namespace {

// The kernel model of kernel_model.cpp:38-76, evaluated on demand (as the
// host restatement's Model): row r has ext(r) operations; Mat(r, j) =
// row_offsets[r] + j, Vec(r, j) = col_indices[Mat(r, j)], Out(r, j) = r; the
// solve excludes the diagonal (stored last).
struct DevModel {
    const int32_t* ro;
    const int32_t* col;
    int sp;
    __device__ int ext(int r) const { return ro[r + 1] - ro[r] - sp; }
    __device__ int mat(int r, int j) const { return ro[r] + j; }
    __device__ int vec(int r, int j) const { return col[ro[r] + j]; }
    __device__ int64_t flat(int r) const { return static_cast<int64_t>(ro[r]) - static_cast<int64_t>(sp) * r; }
};

// CoverMap (miner.cpp:42-56) over the whole matrix's flat operation index.
struct DevCover {
    const DevModel* md;
    uint8_t* bits;
    __device__ bool covered(int r, int p) const { return bits[md->flat(r) + p] != 0; }
    __device__ void cover(int r, int p) { bits[md->flat(r) + p] = 1; }
    __device__ void reset(int rb, int re) {
        for (int64_t i = md->flat(rb), e = md->flat(re); i < e; ++i) bits[i] = 0;
    }
};

struct DevCodelets {  // pass 1 output
    uint8_t* kind;
    int32_t *m, *n, *row, *mat_base, *mat_so, *vec_base, *vec_so;
};

// Codelet emission: counts and costs (pass 0) or writes (pass 1).
struct Emit {
    int64_t cost = 0;
    int32_t count = 0;
    const DevCodelets* out = nullptr;  // null: count only
    int64_t at = 0;
    __device__ void operator()(int kind, int m, int n, int row, int mat_base, int mat_so, int vec_base, int vec_so,
                               int64_t c) {
        cost += c;
        if (out) {
            const int64_t k = at + count;
            out->kind[k] = static_cast<uint8_t>(kind);
            out->m[k] = m;
            out->n[k] = n;
            out->row[k] = row;
            out->mat_base[k] = mat_base;
            out->mat_so[k] = mat_so;
            out->vec_base[k] = vec_base;
            out->vec_so[k] = vec_so;
        }
        ++count;
    }
};

__device__ __forceinline__ int64_t dims_of(int m, int n) {
    const int d = (m > 1 ? 1 : 0) + (n > 1 ? 1 : 0);
    return d == 0 ? 1 : d;
}
// codelet.cpp:45-57 for the three mined shapes
__device__ __forceinline__ int64_t cost_blas(int m, int n) { return int64_t(m) * n + 3 + 3 * dims_of(m, n); }
__device__ __forceinline__ int64_t cost_psci(int m, int n) { return int64_t(m) * n + 3 + 2 * dims_of(m, n) + n; }
__device__ __forceinline__ int64_t cost_pscii(int m, int n) {
    return int64_t(m) * n + 3 + m + dims_of(m, n) + int64_t(m) * n;
}

// mine_blas, miner.cpp:63-120
__device__ void mine_blas(const DevModel& md, int rb, int re, DevCover& cv, Emit& em) {
    for (int r = rb; r < re; ++r) {
        const int extent = md.ext(r);
        int p = 0;
        while (p < extent) {
            if (cv.covered(r, p)) {
                ++p;
                continue;
            }
            int q = p + 1;
            while (q < extent && !cv.covered(r, q) && md.vec(r, q) == md.vec(r, q - 1) + 1) ++q;
            const int width = q - p;
            if (width < 2) {
                p = q;
                continue;
            }
            int rows = 1, mat_delta = 0, vec_delta = 0;
            while (r + rows < re) {
                const int rn = r + rows;
                if (md.ext(rn) < p + width) break;
                bool ok = true;
                for (int j = p; j < q && ok; ++j) ok = !cv.covered(rn, j);
                for (int j = p + 1; j < q && ok; ++j) ok = md.vec(rn, j) == md.vec(rn, j - 1) + 1;
                if (!ok) break;
                const int mdl = md.mat(rn, p) - md.mat(rn - 1, p);
                const int vdl = md.vec(rn, p) - md.vec(rn - 1, p);
                if (rows == 1) {
                    mat_delta = mdl;
                    vec_delta = vdl;
                } else if (mdl != mat_delta || vdl != vec_delta) {
                    break;
                }
                ++rows;
            }
            em(PSC_CODELET_BLAS, rows, width, r, md.mat(r, p), rows > 1 ? mat_delta : 0, md.vec(r, p),
               rows > 1 ? vec_delta : 0, cost_blas(rows, width));
            for (int i = 0; i < rows; ++i)
                for (int j = p; j < q; ++j) cv.cover(r + i, j);
            p = q;
        }
    }
}

// miner.cpp:125-172 (shared gather) and 176-234 (tabulated)
template <bool kShared>
__device__ void mine_psc(const DevModel& md, int rb, int re, DevCover& cv, Emit& em) {
    for (int r = rb; r < re; ++r) {
        const int extent = md.ext(r);
        int p = 0;
        while (p < extent) {
            if (cv.covered(r, p)) {
                ++p;
                continue;
            }
            int q = p + 1;
            while (q < extent && !cv.covered(r, q)) ++q;
            const int width = q - p;
            int rows = 1, mat_delta = 0;
            while (r + rows < re) {
                const int rn = r + rows;
                const int ext_n = md.ext(rn);
                if (ext_n < q) break;
                bool ok = (p == 0 || cv.covered(rn, p - 1)) && (q == ext_n || cv.covered(rn, q));
                for (int j = p; j < q && ok; ++j) ok = !cv.covered(rn, j);
                if (kShared) {
                    for (int j = p; j < q && ok; ++j) ok = md.vec(rn, j) == md.vec(r, j);
                }
                if (!ok) break;
                const int mdl = md.mat(rn, p) - md.mat(rn - 1, p);
                if (rows == 1) {
                    mat_delta = mdl;
                } else if (mdl != mat_delta) {
                    break;
                }
                ++rows;
            }
            em(kShared ? PSC_CODELET_PSC_I : PSC_CODELET_PSC_II, rows, width, r, md.mat(r, p),
               rows > 1 ? mat_delta : 0, -1, 0, kShared ? cost_psci(rows, width) : cost_pscii(rows, width));
            for (int i = 0; i < rows; ++i)
                for (int j = p; j < q; ++j) cv.cover(r + i, j);
            p = q;
        }
    }
}

__device__ void mine_strategy(const DevModel& md, int s, int rb, int re, DevCover& cv, Emit& em) {
    cv.reset(rb, re);
    if (s == 0) {  // blas_first
        mine_blas(md, rb, re, cv, em);
        mine_psc<true>(md, rb, re, cv, em);
    } else if (s == 1) {  // psci_first
        mine_psc<true>(md, rb, re, cv, em);
    } else {  // pscii_first
        mine_psc<false>(md, rb, re, cv, em);
    }
}

__global__ void __launch_bounds__(128) mine_count_kernel(DevModel md, uint8_t* cover, const int32_t* __restrict__ wb,
                                                         const int32_t* __restrict__ we, int64_t n_win,
                                                         uint8_t* strategy, int64_t* cost, int32_t* count) {
    const int64_t w = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (w >= n_win) return;
    const int rb = wb[w], re = we[w];
    DevCover cv{&md, cover};
    int best = 0;
    int64_t best_cost = 0;
    int32_t best_count = 0;
    for (int s = 0; s < 3; ++s) {  // min cost, ties in strategy order (miner.cpp:301-306)
        Emit em;
        mine_strategy(md, s, rb, re, cv, em);
        if (s == 0 || em.cost < best_cost) {
            best = s;
            best_cost = em.cost;
            best_count = em.count;
        }
    }
    strategy[w] = static_cast<uint8_t>(best);
    cost[w] = best_cost;
    count[w] = best_count;
}

__global__ void __launch_bounds__(128) mine_write_kernel(DevModel md, uint8_t* cover, const int32_t* __restrict__ wb,
                                                         const int32_t* __restrict__ we, int64_t n_win,
                                                         const uint8_t* __restrict__ strategy,
                                                         const int64_t* __restrict__ offset, DevCodelets out) {
    const int64_t w = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (w >= n_win) return;
    DevCover cv{&md, cover};
    Emit em;
    em.out = &out;
    em.at = offset[w];
    mine_strategy(md, strategy[w], wb[w], we[w], cv, em);
}

void ck(cudaError_t e, const char* what) {
    if (e != cudaSuccess) throw CudaError(std::string("inspect_device: ") + what + ": " + cudaGetErrorString(e));
}

struct Buf {  // device allocation freed on scope exit
    void* p = nullptr;
    explicit Buf(size_t bytes) { ck(cudaMalloc(&p, bytes ? bytes : 1), "cudaMalloc"); }
    ~Buf() { cudaFree(p); }
    Buf(const Buf&) = delete;
    Buf& operator=(const Buf&) = delete;
    template <class T>
    T* as() const { return static_cast<T*>(p); }
};

template <class T>
void down(std::vector<T>& dst, const Buf& src, size_t n) {
    dst.resize(n);
    if (n) ck(cudaMemcpy(dst.data(), src.p, n * sizeof(T), cudaMemcpyDeviceToHost), "download");
}

}  // namespace

Plan inspect_device(int kernel, const psc_csr_view& a, int t, int target_groups, int device) {
    static const bool trace = std::getenv("PSC_INSPECT_TRACE") != nullptr;  // stage times on stderr
    auto t_last = std::chrono::steady_clock::now();
    auto stage = [&](const char* what) {
        if (!trace) return;
        cudaDeviceSynchronize();
        const auto now = std::chrono::steady_clock::now();
        std::fprintf(stderr, "inspect_device %-10s %8.2f ms\n", what,
                     std::chrono::duration<double, std::milli>(now - t_last).count());
        t_last = now;
    };
    WindowSchedule ws = schedule_windows(kernel, a, t, target_groups);  // validates the matrix
    stage("schedule");
    ck(cudaSetDevice(device), "cudaSetDevice");
    const int n = a.n_rows;
    const int sp = kernel == PSC_KERNEL_SPTRSV ? 1 : 0;
    const int64_t n_win = static_cast<int64_t>(ws.begin.size());
    const int64_t flat_total = a.nnz - static_cast<int64_t>(sp) * n;

    Plan plan;
    plan.kernel = kernel;
    plan.n_rows = a.n_rows;
    plan.n_cols = a.n_cols;
    plan.nnz = a.nnz;
    plan.window = t;
    plan.target_groups = target_groups;
    plan.mined = true;
    plan.part_group_ptr = ws.part_win_ptr;
    plan.g_row_begin = ws.begin;
    plan.g_row_end = ws.end;
    plan.g_codelet_ptr.assign(static_cast<size_t>(n_win) + 1, 0);
    if (n_win == 0) return plan;

    Buf ro((static_cast<size_t>(n) + 1) * sizeof(int32_t)), col(static_cast<size_t>(a.nnz) * sizeof(int32_t));
    Buf cover(static_cast<size_t>(flat_total)), wb(n_win * sizeof(int32_t)), we(n_win * sizeof(int32_t));
    Buf strategy(n_win), cost(n_win * sizeof(int64_t)), count(n_win * sizeof(int32_t)), offset(n_win * sizeof(int64_t));
    ck(cudaMemcpy(ro.p, a.row_offsets, (static_cast<size_t>(n) + 1) * sizeof(int32_t), cudaMemcpyHostToDevice), "upload");
    ck(cudaMemcpy(col.p, a.col_indices, static_cast<size_t>(a.nnz) * sizeof(int32_t), cudaMemcpyHostToDevice), "upload");
    ck(cudaMemcpy(wb.p, ws.begin.data(), n_win * sizeof(int32_t), cudaMemcpyHostToDevice), "upload");
    ck(cudaMemcpy(we.p, ws.end.data(), n_win * sizeof(int32_t), cudaMemcpyHostToDevice), "upload");
    stage("upload");

    const DevModel md{ro.as<int32_t>(), col.as<int32_t>(), sp};
    const unsigned grid = static_cast<unsigned>((n_win + 127) / 128);
    mine_count_kernel<<<grid, 128>>>(md, cover.as<uint8_t>(), wb.as<int32_t>(), we.as<int32_t>(), n_win,
                                     strategy.as<uint8_t>(), cost.as<int64_t>(), count.as<int32_t>());
    ck(cudaGetLastError(), "mine_count_kernel");
    stage("count");

    std::vector<int32_t> cnt;
    down(cnt, count, n_win);
    for (int64_t w = 0; w < n_win; ++w) plan.g_codelet_ptr[w + 1] = plan.g_codelet_ptr[w] + cnt[w];
    const int64_t n_cod = plan.g_codelet_ptr[n_win];
    ck(cudaMemcpy(offset.p, plan.g_codelet_ptr.data(), n_win * sizeof(int64_t), cudaMemcpyHostToDevice), "upload");
    stage("offsets");

    Buf kind(n_cod), m(n_cod * 4), nn(n_cod * 4), row(n_cod * 4), mb(n_cod * 4), mso(n_cod * 4), vb(n_cod * 4),
        vso(n_cod * 4);
    const DevCodelets out{kind.as<uint8_t>(), m.as<int32_t>(), nn.as<int32_t>(), row.as<int32_t>(),
                          mb.as<int32_t>(), mso.as<int32_t>(), vb.as<int32_t>(), vso.as<int32_t>()};
    mine_write_kernel<<<grid, 128>>>(md, cover.as<uint8_t>(), wb.as<int32_t>(), we.as<int32_t>(), n_win,
                                     strategy.as<uint8_t>(), offset.as<int64_t>(), out);
    ck(cudaGetLastError(), "mine_write_kernel");
    stage("write");

    down(plan.g_strategy, strategy, n_win);
    down(plan.g_cost, cost, n_win);
    down(plan.c_kind, kind, n_cod);
    down(plan.c_m, m, n_cod);
    down(plan.c_n, nn, n_cod);
    down(plan.c_row, row, n_cod);
    down(plan.c_mat_base, mb, n_cod);
    down(plan.c_mat_so, mso, n_cod);
    down(plan.c_vec_base, vb, n_cod);
    down(plan.c_vec_so, vso, n_cod);
    stage("download");
    return plan;
}

}  // namespace pscb

// inspect (miner.hpp:95) with the window mining on the GPU: the same plan as
// psc_inspect, bit for bit (tests/test_gpu_parity.py checks the digests).
PSC_API psc_status psc_inspect_device(int32_t kernel, const psc_csr_view* a, int32_t t, int32_t target_groups,
                                      int32_t device, psc_plan** out) {
    return pscb::guarded([&] {
        pscb::require(a != nullptr && out != nullptr, "inspect: null argument");
        pscb::Plan p = pscb::inspect_device(kernel, *a, t, target_groups, device);
        p.structure = pscb::structure_hash(*a);
        *out = new psc_plan(std::move(p));
    });
}
