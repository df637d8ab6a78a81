// psc_b200.hpp -- header-only C++ layer over the C ABI (psc_b200.h) that gives
// code written against the reference library the same executor calls:
//
//   reference (/root/reference/proj/core/include/psc/executor.hpp)   here
//   psc::Executor exec(workers);                       psc_b200::Executor exec(workers);
//   psc::run_spmv(plan, a, x, y, exec);                psc_b200::run_spmv(plan, a, x, y, exec);
//   psc::run_sptrsv(plan, l, b, x, acc, exec);         psc_b200::run_sptrsv(plan, l, b, x, acc, exec);
//   exec.run(plan, ctx);                               exec.run(plan, ctx);
//   psc::execute_plan(plan, ctx, workers);             psc_b200::execute_plan(plan, ctx, workers);
//   psc::exec_{blas,psci,pscii}_codelet(c, ctx);       psc_b200::exec_*_codelet(c, ctx);
//
// `plan` may be the reference's own psc::CodeletPlan (miner.hpp:73-89) -- it is
// flattened through psc_plan_from_arrays and cached per plan object -- or a
// psc_b200::Plan mined by this library's bit-exact inspector. `a` / `l` are any
// CSR type with the fields of psc::CsrMatrix (csr_matrix.hpp:9-20) or
// psc::TriangularMatrix (csr() accessor). Status codes come back as the
// reference's exception types: std::invalid_argument, std::logic_error.
#pragma once

#include <cstdint>
#include <memory>
#include <span>
#include <stdexcept>
#include <string>
#include <type_traits>
#include <unordered_map>
#include <vector>

#include "psc_b200.h"

namespace psc_b200 {

inline void check(psc_status st) {
    if (st == PSC_OK) return;
    std::string msg = psc_last_error();
    if (st == PSC_ERR_INVALID_ARGUMENT) throw std::invalid_argument(msg);
    if (st == PSC_ERR_LOGIC) throw std::logic_error(msg);
    throw std::runtime_error(msg);
}

// ---- CSR views of reference-shaped matrices --------------------------------
template <class M>
auto& csr_of(const M& m) {
    if constexpr (requires { m.csr(); }) return m.csr();  // TriangularMatrix
    else return m;
}

template <class M>
psc_csr_view view_of(const M& m) {
    const auto& a = csr_of(m);
    return {a.n_rows, a.n_cols, static_cast<int64_t>(a.col_indices.size()), a.row_offsets.data(),
            a.col_indices.data(), a.values.data()};
}

// ---- plans -------------------------------------------------------------------
// A plan mined by this library (psc_inspect), owning its handle.
class Plan {
  public:
    Plan() = default;
    explicit Plan(psc_plan* h) : h_(h, &psc_plan_destroy) {}
    psc_plan* handle() const { return h_.get(); }

  private:
    std::shared_ptr<psc_plan> h_;
};

enum class KernelKind { Spmv = PSC_KERNEL_SPMV, Sptrsv = PSC_KERNEL_SPTRSV };

template <class M>
Plan inspect(KernelKind kernel, const M& a, int t, int target_groups, int threads = 0) {
    psc_csr_view v = view_of(a);
    psc_plan* h = nullptr;
    check(psc_inspect(static_cast<int32_t>(kernel), &v, t, target_groups, threads, &h));
    return Plan(h);
}

// Flatten a reference-shaped CodeletPlan (partitions -> groups -> codelets /
// finalize records, AccessDesc {form, lin, table}) into a library plan.
template <class P>
Plan import_plan(const P& p) {
    psc_plan_counts c{};
    c.kernel = static_cast<int32_t>(p.kernel);
    c.n_rows = p.n_rows;
    c.n_cols = p.n_cols;
    c.nnz = p.nnz;
    c.window = p.window;
    c.target_groups = p.target_groups;
    c.n_partitions = static_cast<int64_t>(p.partitions.size());
    for (const auto& part : p.partitions) {
        c.n_groups += static_cast<int64_t>(part.groups.size());
        for (const auto& g : part.groups) {
            c.n_codelets += static_cast<int64_t>(g.codelets.size());
            c.n_finalize += static_cast<int64_t>(g.finalize.size());
            for (const auto& cd : g.codelets)
                c.n_table += static_cast<int64_t>(cd.out.table.size() + cd.mat.table.size() + cd.vec.table.size());
        }
    }
    std::vector<int64_t> pg(c.n_partitions + 1), gc(c.n_groups + 1), gf(c.n_groups + 1), cost(c.n_groups),
        tp(3 * c.n_codelets + 1);
    std::vector<int32_t> rb(c.n_groups), re(c.n_groups), st(c.n_groups), kind(c.n_codelets), m(c.n_codelets),
        n(c.n_codelets), form(3 * c.n_codelets), base(3 * c.n_codelets), so(3 * c.n_codelets),
        si(3 * c.n_codelets), tab(c.n_table), fr(c.n_finalize), fd(c.n_finalize), fh(c.n_finalize);
    int64_t gi = 0, ci = 0, fi = 0, ti = 0;
    for (std::size_t pi = 0; pi < p.partitions.size(); ++pi) {
        for (const auto& g : p.partitions[pi].groups) {
            rb[gi] = g.window.row_begin;
            re[gi] = g.window.row_end;
            st[gi] = static_cast<int32_t>(g.strategy);
            cost[gi] = g.cost;
            for (const auto& cd : g.codelets) {
                kind[ci] = static_cast<int32_t>(cd.kind);
                m[ci] = cd.outer_extent;
                n[ci] = cd.inner_extent;
                const decltype(cd.out)* ds[3] = {&cd.out, &cd.mat, &cd.vec};
                for (int d = 0; d < 3; ++d) {
                    const int64_t k = 3 * ci + d;
                    form[k] = static_cast<int32_t>(ds[d]->form);
                    base[k] = ds[d]->lin.base;
                    so[k] = ds[d]->lin.stride_outer;
                    si[k] = ds[d]->lin.stride_inner;
                    for (int v : ds[d]->table) tab[ti++] = v;
                    tp[k + 1] = ti;
                }
                ++ci;
            }
            for (const auto& f : g.finalize) {
                fr[fi] = f.row;
                fd[fi] = f.diag_pos;
                fh[fi] = f.rhs_index;
                ++fi;
            }
            ++gi;
            gc[gi] = ci;
            gf[gi] = fi;
        }
        pg[pi + 1] = gi;
    }
    psc_plan_arrays a{pg.data(),   rb.data(),   re.data(),   st.data(), cost.data(), gc.data(), gf.data(),
                      kind.data(), m.data(),    n.data(),    form.data(), base.data(), so.data(), si.data(),
                      tp.data(),   tab.data(),  fr.data(),   fd.data(),  fh.data()};
    psc_plan* h = nullptr;
    check(psc_plan_from_arrays(&c, &a, &h));
    return Plan(h);
}

// ---- executor (executor.hpp:36-51) -------------------------------------------
class Executor {
  public:
    explicit Executor(int workers, int device = 0) {
        psc_executor* e = nullptr;
        check(psc_executor_create(workers, device, &e));
        e_.reset(e);
    }
    int workers() const { return psc_executor_workers(e_.get()); }
    // psc_executor_set_values_version: skip re-uploading unchanged matrix values
    void set_values_version(uint64_t version) { check(psc_executor_set_values_version(e_.get(), version)); }
    psc_executor* handle() const { return e_.get(); }

    // Executor::run (executor.hpp:45): the plan over a raw ExecutionContext,
    // accumulating onto ctx.accum. The plan must carry its tables (the
    // reference's CodeletPlan); plans mined by this library's inspector keep
    // them in the matrix -- use execute_plan(plan, a, ctx, workers).
    template <class P, class Ctx>
    void run(const P& plan, const Ctx& ctx) {
        psc_exec_context c{ctx.matrix_values, ctx.gather, ctx.accum, ctx.rhs, ctx.solution};
        check(psc_executor_run(e_.get(), plan_for(plan).handle(), &c));
    }

    // Library plan for `plan`: itself, or the cached import of a reference plan.
    template <class P>
    const Plan& plan_for(const P& plan) {
        if constexpr (std::is_same_v<P, Plan>) {
            return plan;
        } else {
            auto it = imported_.find(&plan);
            if (it == imported_.end() || it->second.first != signature(plan))
                it = imported_.insert_or_assign(&plan, std::make_pair(signature(plan), import_plan(plan))).first;
            return it->second.second;
        }
    }

  private:
    struct Del {
        void operator()(psc_executor* e) const { psc_executor_destroy(e); }
    };
    template <class P>
    static int64_t signature(const P& p) {
        int64_t s = p.nnz * 1315423911LL + p.n_rows;
        for (const auto& part : p.partitions) s = s * 31 + static_cast<int64_t>(part.groups.size());
        return s;
    }
    std::unique_ptr<psc_executor, Del> e_;
    std::unordered_map<const void*, std::pair<int64_t, Plan>> imported_;
};

// run_spmv, executor.cpp:274-288
template <class P, class M>
void run_spmv(const P& plan, const M& a, std::span<const double> x, std::span<double> y, Executor& exec) {
    psc_csr_view v = view_of(a);
    check(psc_run_spmv(exec.handle(), exec.plan_for(plan).handle(), &v, x.data(), static_cast<int64_t>(x.size()),
                       y.data(), static_cast<int64_t>(y.size())));
}

// run_sptrsv, executor.cpp:290-308
template <class P, class L>
void run_sptrsv(const P& plan, const L& l, std::span<const double> b, std::span<double> x, std::span<double> acc,
                Executor& exec) {
    psc_csr_view v = view_of(l);
    check(psc_run_sptrsv(exec.handle(), exec.plan_for(plan).handle(), &v, b.data(), static_cast<int64_t>(b.size()),
                         x.data(), static_cast<int64_t>(x.size()), acc.data(), static_cast<int64_t>(acc.size())));
}

// execute_plan, executor.cpp:269-272 (executor.hpp:54): a temporary
// executor's run over a raw context
template <class P, class Ctx>
void execute_plan(const P& plan, const Ctx& ctx, int workers) {
    Executor exec(workers);
    exec.run(plan, ctx);
}

// The same for plans mined by this library (implicit tables): the matrix
// supplies the CSR structure; values come from ctx.matrix_values
template <class P, class M, class Ctx>
void execute_plan(const P& plan, const M& a, const Ctx& ctx, int workers) {
    Executor exec(workers);
    psc_csr_view v = view_of(a);
    psc_exec_context c{ctx.matrix_values, ctx.gather, ctx.accum, ctx.rhs, ctx.solution};
    check(psc_execute_plan(exec.handle(), exec.plan_for(plan).handle(), &v, &c));
}

// exec_*_codelet, executor.cpp:53-116, for reference-shaped codelets
template <class C>
psc_codelet_view codelet_view(const C& c) {
    auto d = [](const auto& a) {
        return psc_access_desc_view{static_cast<int32_t>(a.form), a.lin.base, a.lin.stride_outer, a.lin.stride_inner,
                                    a.table.empty() ? nullptr : a.table.data(),
                                    static_cast<int64_t>(a.table.size())};
    };
    return {static_cast<int32_t>(c.kind), c.outer_extent, c.inner_extent, d(c.out), d(c.mat), d(c.vec)};
}
template <class C, class Ctx>
void exec_blas_codelet(const C& c, const Ctx& ctx) {
    psc_codelet_view v = codelet_view(c);
    psc_exec_context x{ctx.matrix_values, ctx.gather, ctx.accum, ctx.rhs, ctx.solution};
    check(psc_exec_blas_codelet(&v, &x));
}
template <class C, class Ctx>
void exec_psci_codelet(const C& c, const Ctx& ctx) {
    psc_codelet_view v = codelet_view(c);
    psc_exec_context x{ctx.matrix_values, ctx.gather, ctx.accum, ctx.rhs, ctx.solution};
    check(psc_exec_psci_codelet(&v, &x));
}
template <class C, class Ctx>
void exec_pscii_codelet(const C& c, const Ctx& ctx) {
    psc_codelet_view v = codelet_view(c);
    psc_exec_context x{ctx.matrix_values, ctx.gather, ctx.accum, ctx.rhs, ctx.solution};
    check(psc_exec_pscii_codelet(&v, &x));
}

}  // namespace psc_b200
