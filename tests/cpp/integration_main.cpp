// Drop-in integration test (TEST INFRASTRUCTURE): code written against the
// reference library -- its own inspector, matrices and plans -- switches the
// executor to include/psc_b200.hpp and must get bitwise the reference
// executor's results. Links the unmodified reference objects
// (oracle/_ref/obj) and libpsc_b200.so; built by oracle/Makefile into
// oracle/_ref/integration_test; run by tests/test_integration.py on a GPU.
#include <cmath>
#include <cstdio>
#include <cstring>
#include <random>
#include <span>
#include <vector>

#include "psc/executor.hpp"
#include "psc/miner.hpp"
#include "psc/pattern_gen.hpp"
#include "psc_b200.hpp"
#include "support/test_helpers.hpp"

static int failures = 0;
static void report(bool ok, const char* what) {
    std::printf("[%s] %s\n", ok ? "PASS" : "FAIL", what);
    if (!ok) ++failures;
}
static bool bitwise(const std::vector<double>& a, const std::vector<double>& b) {
    return a.size() == b.size() && std::memcmp(a.data(), b.data(), a.size() * sizeof(double)) == 0;
}

int main() {
    psc_b200::Executor gpu(4);
    psc::Executor cpu(1);
    int cases = 0, ok = 0;
    // the acceptance suite's generators, both kernels, t in {1,2,3,8}, groups in {1,4}
    const char* specs[] = {"dense_block(16)", "banded(32,2)", "banded(32,3,lower)", "scattered_gather(64,0:3:7:12:18:25)",
                           "random_uniform(128,128,0.05,7)", "random_uniform(256,256,0.03,1)"};
    for (const char* spec : specs) {
        psc::CsrMatrix a = psc::generate_pattern(spec);
        psc::TriangularMatrix l = psc::lower_triangular(psc::test::unit_lower(a));
        std::vector<double> x = psc::test::int_vector(a.n_cols, 7);
        std::vector<double> b = psc::test::int_vector(l.n(), 9);
        for (int t : {1, 2, 3, 8}) {
            for (int groups : {1, 4}) {
                psc::CodeletPlan plan = psc::inspect(psc::KernelKind::Spmv, a, t, groups);  // reference inspector
                std::vector<double> y_ref(a.n_rows), y_gpu(a.n_rows, NAN);
                psc::run_spmv(plan, a, x, y_ref, cpu);
                psc_b200::run_spmv(plan, a, x, y_gpu, gpu);  // same call, GPU executor
                ok += bitwise(y_ref, y_gpu);
                ++cases;
                psc::CodeletPlan splan = psc::inspect(psc::KernelKind::Sptrsv, l.csr(), t, groups);
                std::vector<double> xs_ref(l.n()), xs_gpu(l.n(), NAN), acc_ref(l.n()), acc_gpu(l.n(), NAN);
                psc::run_sptrsv(splan, l, b, xs_ref, acc_ref, cpu);
                psc_b200::run_sptrsv(splan, l, b, xs_gpu, acc_gpu, gpu);
                ok += bitwise(xs_ref, xs_gpu) && bitwise(acc_ref, acc_gpu);
                ++cases;
            }
        }
    }
    char buf[128];
    std::snprintf(buf, sizeof buf, "reference plans on the GPU executor: %d/%d bitwise (x and acc)", ok, cases);
    report(ok == cases, buf);

    // the library's own inspector yields the same plan digest and results
    {
        psc::CsrMatrix a = psc::generate_pattern("random_uniform(200,200,0.04,3)");
        psc::CodeletPlan ref = psc::inspect(psc::KernelKind::Spmv, a, 3, 4);
        psc_b200::Plan mine = psc_b200::inspect(psc_b200::KernelKind::Spmv, a, 3, 4);
        std::vector<double> x = psc::test::int_vector(a.n_cols, 1), y1(a.n_rows), y2(a.n_rows);
        psc::run_spmv(ref, a, x, y1, cpu);
        psc_b200::run_spmv(mine, a, x, y2, gpu);
        report(bitwise(y1, y2), "library inspector + GPU executor == reference inspector + executor");
    }

    // errors map onto the reference's exception types (test_executor.cpp:243-258)
    {
        psc::CsrMatrix a = psc::dense_block(3);
        psc::CodeletPlan plan = psc::inspect(psc::KernelKind::Spmv, a, 3, 1);
        std::vector<double> x(3), y(3), short_x(2);
        bool threw = false;
        try {
            psc_b200::run_spmv(plan, a, short_x, y, gpu);
        } catch (const std::invalid_argument&) {
            threw = true;
        }
        bool threw2 = false;
        try {
            psc_b200::Executor bad(0);
        } catch (const std::invalid_argument&) {
            threw2 = true;
        }
        report(threw && threw2, "size mismatch and workers < 1 throw std::invalid_argument");
    }

    // hand-built codelets (test_executor.cpp:37-87)
    {
        psc::Codelet c;
        c.kind = psc::CodeletKind::PscI;
        c.outer_extent = 3;
        c.inner_extent = 3;
        c.out = psc::AccessDesc::strided(0, 1, 0);
        c.mat = psc::AccessDesc::strided(0, 3, 1);
        c.vec = psc::AccessDesc::inner_table({0, 2, 5});
        std::vector<double> ax{1, 2, 3, 4, 5, 6, 7, 8, 9}, x{10, 0, 20, 0, 0, 30}, acc(3, 0.0);
        psc::ExecutionContext ctx;
        ctx.matrix_values = ax.data();
        ctx.gather = x.data();
        ctx.accum = acc.data();
        psc_b200::exec_psci_codelet(c, ctx);
        report(acc == std::vector<double>{140, 320, 500}, "exec_psci_codelet known answer on the GPU");
    }
    return failures == 0 ? 0 : 1;
}
