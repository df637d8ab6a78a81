// Drop-in replacement of the reference's psc/executor.hpp (TEST
// INFRASTRUCTURE): the same declarations (executor.hpp:10-65), implemented by
// the B200 executor through include/psc_b200.hpp. Put this directory ahead of
// the reference's include path and the reference's own executor tests
// (tests/test_executor.cpp) compile unchanged and run on the GPU; the
// reference's executor.cpp is not linked.
#pragma once

#include <memory>
#include <span>
#include <stdexcept>
#include <vector>

#include "psc/codelet.hpp"
#include "psc/csr_matrix.hpp"
#include "psc/miner.hpp"
#include "psc_b200.hpp"

namespace psc {

struct ExecutionContext {
    const double* matrix_values = nullptr;
    const double* gather = nullptr;
    double* accum = nullptr;
    const double* rhs = nullptr;
    double* solution = nullptr;
};

inline void exec_blas_codelet(const Codelet& c, const ExecutionContext& ctx) { psc_b200::exec_blas_codelet(c, ctx); }
inline void exec_psci_codelet(const Codelet& c, const ExecutionContext& ctx) { psc_b200::exec_psci_codelet(c, ctx); }
inline void exec_pscii_codelet(const Codelet& c, const ExecutionContext& ctx) { psc_b200::exec_pscii_codelet(c, ctx); }

class Executor {
  public:
    explicit Executor(int workers) : e_(std::make_unique<psc_b200::Executor>(workers)) {}
    Executor(const Executor&) = delete;
    Executor& operator=(const Executor&) = delete;
    int workers() const { return e_->workers(); }
    void run(const CodeletPlan& plan, const ExecutionContext& ctx) { e_->run(plan, ctx); }
    psc_b200::Executor& impl() { return *e_; }

  private:
    std::unique_ptr<psc_b200::Executor> e_;
};

inline void execute_plan(const CodeletPlan& plan, const ExecutionContext& ctx, int workers) {
    psc_b200::execute_plan(plan, ctx, workers);
}
inline void run_spmv(const CodeletPlan& plan, const CsrMatrix& a, std::span<const double> x, std::span<double> y,
                     Executor& exec) {
    psc_b200::run_spmv(plan, a, x, y, exec.impl());
}
inline void run_sptrsv(const CodeletPlan& plan, const TriangularMatrix& l, std::span<const double> b,
                       std::span<double> x, std::span<double> acc, Executor& exec) {
    psc_b200::run_sptrsv(plan, l, b, x, acc, exec.impl());
}
// the naive baselines (executor.cpp:310-340) from this library's host half
inline std::vector<double> spmv_csr_baseline(const CsrMatrix& a, std::span<const double> x) {
    std::vector<double> y(a.n_rows);
    psc_csr_view v = psc_b200::view_of(a);
    psc_b200::check(psc_csr_spmv_baseline(&v, x.data(), static_cast<int64_t>(x.size()), y.data(),
                                          static_cast<int64_t>(y.size())));
    return y;
}
inline std::vector<double> sptrsv_csr_baseline(const TriangularMatrix& l, std::span<const double> b) {
    std::vector<double> x(l.n());
    psc_csr_view v = psc_b200::view_of(l);
    psc_b200::check(psc_csr_sptrsv_baseline(&v, b.data(), static_cast<int64_t>(b.size()), x.data(),
                                            static_cast<int64_t>(x.size())));
    return x;
}

}  // namespace psc
