"""TEST INFRASTRUCTURE: loaders for the two parity checkers.

* ``Oracle``  -- build/liboracle.so, the plain-C restatement of the reference
  executor (psc_oracle.c); always available (gcc).
* ``Ref``     -- _ref/libpsc_ref.so, the reference library itself compiled from
  /root/reference by oracle/Makefile, behind ref_shim.cpp. Present in this
  container and on the GPU box when it was built here (the .so travels);
  ``Ref.available()`` says whether it can be used.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
arm may import this module. The product never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from ctypes import POINTER, c_char_p, c_double, c_int, c_int64, c_uint64, c_void_p

import numpy as np

from paper_2111_12243_b200._capi import CodeletView, CsrView, ExecContext, PlanArrays, PlanCounts

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "build", "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libpsc_ref.so")
REF_SRC = "/root/reference/proj/core/src/executor.cpp"


def build(ref: bool = True) -> None:
    targets = ["oracle"] + (["ref"] if ref and os.path.exists(REF_SRC) else [])
    subprocess.run(["make", "-s", "-C", HERE, "-j8", *targets], check=True)


def _dp(a):
    return a.ctypes.data_as(POINTER(c_double)) if a is not None else None


class Oracle:
    _lib = None

    @classmethod
    def lib(cls):
        if cls._lib is None:
            if not os.path.exists(ORACLE_SO):
                build(ref=False)
            lib = C.CDLL(ORACLE_SO)
            lib.oracle_last_error.restype = c_char_p
            lib.oracle_run_spmv.argtypes = [POINTER(PlanCounts), POINTER(PlanArrays), POINTER(CsrView),
                                            POINTER(c_double), POINTER(c_double)]
            lib.oracle_run_sptrsv.argtypes = [POINTER(PlanCounts), POINTER(PlanArrays), POINTER(CsrView),
                                              POINTER(c_double), POINTER(c_double), POINTER(c_double)]
            lib.oracle_exec_codelet.argtypes = [c_int, POINTER(CodeletView), POINTER(ExecContext)]
            lib.oracle_spmv_baseline.argtypes = [POINTER(CsrView), POINTER(c_double), POINTER(c_double)]
            lib.oracle_spmv_baseline.restype = None
            lib.oracle_sptrsv_baseline.argtypes = [POINTER(CsrView), POINTER(c_double), POINTER(c_double)]
            lib.oracle_sptrsv_baseline.restype = None
            cls._lib = lib
        return cls._lib

    @classmethod
    def _check(cls, st):
        if st != 0:
            raise RuntimeError(f"oracle: {cls.lib().oracle_last_error().decode()} (status {st})")

    @classmethod
    def run_spmv(cls, plan_export, csr_view, x):
        counts, arrays, _keep = plan_export
        y = np.empty(csr_view.n_rows, dtype=np.float64)
        cls._check(cls.lib().oracle_run_spmv(C.byref(counts), C.byref(arrays), C.byref(csr_view), _dp(x), _dp(y)))
        return y

    @classmethod
    def run_sptrsv(cls, plan_export, csr_view, b):
        counts, arrays, _keep = plan_export
        n = csr_view.n_rows
        x = np.zeros(n, dtype=np.float64)
        acc = np.empty(n, dtype=np.float64)
        cls._check(cls.lib().oracle_run_sptrsv(C.byref(counts), C.byref(arrays), C.byref(csr_view), _dp(b),
                                               _dp(x), _dp(acc)))
        return x, acc

    @classmethod
    def exec_codelet(cls, which, codelet_view, ctx):
        cls._check(cls.lib().oracle_exec_codelet(which, C.byref(codelet_view), C.byref(ctx)))

    @classmethod
    def spmv_baseline(cls, csr_view, x):
        y = np.empty(csr_view.n_rows, dtype=np.float64)
        cls.lib().oracle_spmv_baseline(C.byref(csr_view), _dp(x), _dp(y))
        return y

    @classmethod
    def sptrsv_baseline(cls, csr_view, b):
        x = np.empty(csr_view.n_rows, dtype=np.float64)
        cls.lib().oracle_sptrsv_baseline(C.byref(csr_view), _dp(b), _dp(x))
        return x


def alloc_plan_arrays(counts: PlanCounts):
    """Allocate numpy storage for every PlanArrays field; returns (arrays, keepalive dict)."""
    from paper_2111_12243_b200._capi import PLAN_ARRAY_FIELDS

    arrays = PlanArrays()
    keep = {}
    for name, ct, length in PLAN_ARRAY_FIELDS:
        dtype = np.int64 if ct is C.c_int64 else np.int32
        buf = np.zeros(max(1, int(length(counts))), dtype=dtype)
        keep[name] = buf
        setattr(arrays, name, buf.ctypes.data_as(POINTER(ct)))
    return arrays, keep


class RefCsr:
    """A psc::CsrMatrix owned by the reference library."""

    def __init__(self, handle):
        self.h = c_void_p(handle) if not isinstance(handle, c_void_p) else handle

    def view(self) -> CsrView:
        v = CsrView()
        Ref.lib().ref_csr_view(self.h, C.byref(v))
        return v

    def arrays(self):
        v = self.view()
        ro = np.ctypeslib.as_array(v.row_offsets, shape=(v.n_rows + 1,)).copy()
        if v.nnz:
            ci = np.ctypeslib.as_array(v.col_indices, shape=(v.nnz,)).copy()
            va = np.ctypeslib.as_array(v.values, shape=(v.nnz,)).copy()
        else:
            ci = np.zeros(0, np.int32)
            va = np.zeros(0, np.float64)
        return v.n_rows, v.n_cols, ro, ci, va

    def __del__(self):
        try:
            Ref.lib().ref_csr_free(self.h)
        except Exception:
            pass


class RefPlan:
    def __init__(self, handle):
        self.h = c_void_p(handle) if not isinstance(handle, c_void_p) else handle

    def counts(self) -> PlanCounts:
        c = PlanCounts()
        Ref.lib().ref_plan_counts(self.h, C.byref(c))
        return c

    def export(self):
        c = self.counts()
        arrays, keep = alloc_plan_arrays(c)
        Ref.lib().ref_plan_export(self.h, C.byref(arrays))
        return c, arrays, keep

    def hash(self) -> int:
        return int(Ref.lib().ref_plan_hash(self.h))

    def totals(self):
        cost, ops = c_int64(), c_int64()
        Ref.lib().ref_plan_totals(self.h, C.byref(cost), C.byref(ops))
        return cost.value, ops.value

    def __del__(self):
        try:
            Ref.lib().ref_plan_free(self.h)
        except Exception:
            pass


class Ref:
    _lib = None

    @classmethod
    def available(cls) -> bool:
        if os.path.exists(REF_SO):
            return True
        if os.path.exists(REF_SRC):
            build(ref=True)
            return os.path.exists(REF_SO)
        return False

    @classmethod
    def lib(cls):
        if cls._lib is None:
            if not cls.available():
                raise RuntimeError("reference library oracle/_ref/libpsc_ref.so is not available")
            lib = C.CDLL(REF_SO)
            vp = POINTER(c_void_p)
            lib.ref_last_error.restype = c_char_p
            lib.ref_csr_from_view.argtypes = [POINTER(CsrView), vp]
            lib.ref_csr_view.argtypes = [c_void_p, POINTER(CsrView)]
            lib.ref_csr_free.argtypes = [c_void_p]
            lib.ref_csr_free.restype = None
            lib.ref_generate_pattern.argtypes = [c_char_p, c_uint64, vp]
            lib.ref_generate_config.argtypes = [c_int, c_double, c_uint64, vp]
            lib.ref_uniform_vector.argtypes = [c_int64, c_uint64, c_double, c_double, POINTER(c_double)]
            lib.ref_uniform_vector.restype = None
            lib.ref_read_matrix_market.argtypes = [c_char_p, vp, POINTER(C.c_int)]
            lib.ref_csr_from_triplets.argtypes = [c_int, c_int, c_int64, POINTER(C.c_int32), POINTER(C.c_int32),
                                                  POINTER(c_double), vp]
            lib.ref_lower_triangular.argtypes = [c_void_p, vp]
            lib.ref_random_unit_lower.argtypes = [c_int, c_int, c_uint64, vp]
            lib.ref_unit_lower.argtypes = [c_void_p, vp]
            lib.ref_int_values.argtypes = [c_void_p, c_uint64]
            lib.ref_int_values.restype = None
            lib.ref_int_vector.argtypes = [c_int, c_uint64, POINTER(c_double)]
            lib.ref_int_vector.restype = None
            lib.ref_inspect.argtypes = [c_int, c_void_p, c_int, c_int, vp]
            lib.ref_plan_free.argtypes = [c_void_p]
            lib.ref_plan_free.restype = None
            lib.ref_plan_counts.argtypes = [c_void_p, POINTER(PlanCounts)]
            lib.ref_plan_export.argtypes = [c_void_p, POINTER(PlanArrays)]
            lib.ref_plan_hash.argtypes = [c_void_p]
            lib.ref_plan_hash.restype = c_uint64
            lib.ref_plan_totals.argtypes = [c_void_p, POINTER(c_int64), POINTER(c_int64)]
            lib.ref_plan_totals.restype = None
            lib.ref_strategy_costs.argtypes = [c_int, c_void_p, c_int, c_int, POINTER(c_int64)]
            lib.ref_run_spmv.argtypes = [c_void_p, c_void_p, POINTER(c_double), POINTER(c_double), c_int]
            lib.ref_run_sptrsv.argtypes = [c_void_p, c_void_p, POINTER(c_double), POINTER(c_double),
                                           POINTER(c_double), c_int]
            lib.ref_spmv_baseline.argtypes = [c_void_p, POINTER(c_double), POINTER(c_double)]
            lib.ref_sptrsv_baseline.argtypes = [c_void_p, POINTER(c_double), POINTER(c_double)]
            lib.ref_exec_codelet.argtypes = [c_int, POINTER(CodeletView), POINTER(ExecContext)]
            lib.ref_time_spmv.argtypes = [c_void_p, c_void_p, POINTER(c_double), POINTER(c_double), c_int, c_int,
                                          c_int, POINTER(c_double)]
            lib.ref_time_sptrsv.argtypes = [c_void_p, c_void_p, POINTER(c_double), POINTER(c_double),
                                            POINTER(c_double), c_int, c_int, c_int, POINTER(c_double)]
            lib.ref_time_inspect.argtypes = [c_int, c_void_p, c_int, c_int, POINTER(c_double), vp]
            lib.ref_paired_timing.argtypes = [c_void_p, c_void_p, c_int, POINTER(c_double), c_int, c_int,
                                              POINTER(c_double)]
            lib.ref_run_bench.argtypes = [c_int, c_void_p, c_int, c_int, c_int, c_int, c_uint64, POINTER(c_double)]
            cls._lib = lib
        return cls._lib

    @classmethod
    def _check(cls, st):
        if st == 1:
            raise ValueError(cls.lib().ref_last_error().decode())
        if st == 2:
            raise RuntimeError("logic_error: " + cls.lib().ref_last_error().decode())
        if st != 0:
            raise RuntimeError(cls.lib().ref_last_error().decode())

    # -- matrices
    @classmethod
    def csr(cls, view: CsrView) -> RefCsr:
        h = c_void_p()
        cls._check(cls.lib().ref_csr_from_view(C.byref(view), C.byref(h)))
        return RefCsr(h)

    @classmethod
    def read_matrix_market(cls, path):
        """(RefCsr, None) or (None, (parse-error line, message))."""
        h, line = c_void_p(), C.c_int(0)
        st = cls.lib().ref_read_matrix_market(str(path).encode(), C.byref(h), C.byref(line))
        if st != 0:
            return None, (line.value, cls.lib().ref_last_error().decode())
        return RefCsr(h), None

    @classmethod
    def generate_pattern(cls, spec: str, seed: int = 42) -> RefCsr:
        h = c_void_p()
        cls._check(cls.lib().ref_generate_pattern(spec.encode(), seed, C.byref(h)))
        return RefCsr(h)

    @classmethod
    def generate_config(cls, config: int, scale: float = 1.0, seed: int = 0) -> RefCsr:
        """BASELINE.json config (the product's configs.cpp compiled into the reference library)."""
        h = c_void_p()
        cls._check(cls.lib().ref_generate_config(config, float(scale), seed, C.byref(h)))
        return RefCsr(h)

    @classmethod
    def uniform_vector(cls, n: int, seed: int, lo: float = -1.0, hi: float = 1.0) -> np.ndarray:
        v = np.empty(n, dtype=np.float64)
        cls.lib().ref_uniform_vector(n, seed, lo, hi, _dp(v))
        return v

    @classmethod
    def lower_triangular(cls, a: RefCsr) -> RefCsr:
        h = c_void_p()
        cls._check(cls.lib().ref_lower_triangular(a.h, C.byref(h)))
        return RefCsr(h)

    @classmethod
    def unit_lower(cls, a: RefCsr) -> RefCsr:
        h = c_void_p()
        cls._check(cls.lib().ref_unit_lower(a.h, C.byref(h)))
        return RefCsr(h)

    @classmethod
    def random_unit_lower(cls, n: int, max_extra: int, seed: int) -> RefCsr:
        h = c_void_p()
        cls._check(cls.lib().ref_random_unit_lower(n, max_extra, seed, C.byref(h)))
        return RefCsr(h)

    @classmethod
    def int_values(cls, a: RefCsr, seed: int) -> None:
        cls.lib().ref_int_values(a.h, seed)

    @classmethod
    def int_vector(cls, n: int, seed: int) -> np.ndarray:
        v = np.empty(n, dtype=np.float64)
        cls.lib().ref_int_vector(n, seed, _dp(v))
        return v

    # -- inspector
    @classmethod
    def inspect(cls, kernel: int, a: RefCsr, t: int, groups: int) -> RefPlan:
        h = c_void_p()
        cls._check(cls.lib().ref_inspect(kernel, a.h, t, groups, C.byref(h)))
        return RefPlan(h)

    @classmethod
    def strategy_costs(cls, kernel, a: RefCsr, rb, re):
        out = (c_int64 * 3)()
        cls._check(cls.lib().ref_strategy_costs(kernel, a.h, rb, re, out))
        return list(out)

    # -- executor
    @classmethod
    def run_spmv(cls, plan: RefPlan, a: RefCsr, x, workers=1):
        v = a.view()
        y = np.empty(v.n_rows, dtype=np.float64)
        cls._check(cls.lib().ref_run_spmv(plan.h, a.h, _dp(x), _dp(y), workers))
        return y

    @classmethod
    def run_sptrsv(cls, plan: RefPlan, l: RefCsr, b, workers=1):
        v = l.view()
        x = np.zeros(v.n_rows, dtype=np.float64)
        acc = np.empty(v.n_rows, dtype=np.float64)
        cls._check(cls.lib().ref_run_sptrsv(plan.h, l.h, _dp(b), _dp(x), _dp(acc), workers))
        return x, acc

    @classmethod
    def spmv_baseline(cls, a: RefCsr, x):
        y = np.empty(a.view().n_rows, dtype=np.float64)
        cls._check(cls.lib().ref_spmv_baseline(a.h, _dp(x), _dp(y)))
        return y

    @classmethod
    def sptrsv_baseline(cls, l: RefCsr, b):
        x = np.empty(l.view().n_rows, dtype=np.float64)
        cls._check(cls.lib().ref_sptrsv_baseline(l.h, _dp(b), _dp(x)))
        return x

    @classmethod
    def exec_codelet(cls, which, codelet_view, ctx):
        cls._check(cls.lib().ref_exec_codelet(which, C.byref(codelet_view), C.byref(ctx)))

    # -- timing (bench.py reference arm)
    @classmethod
    def time_spmv(cls, plan, a, x, workers, warmup, reps):
        y = np.empty(a.view().n_rows, dtype=np.float64)
        t = np.empty(reps, dtype=np.float64)
        cls._check(cls.lib().ref_time_spmv(plan.h, a.h, _dp(x), _dp(y), workers, warmup, reps, _dp(t)))
        return t, y

    @classmethod
    def time_sptrsv(cls, plan, l, b, workers, warmup, reps):
        n = l.view().n_rows
        x = np.zeros(n, dtype=np.float64)
        acc = np.empty(n, dtype=np.float64)
        t = np.empty(reps, dtype=np.float64)
        cls._check(cls.lib().ref_time_sptrsv(plan.h, l.h, _dp(b), _dp(x), _dp(acc), workers, warmup, reps,
                                             _dp(t)))
        return t, x

    @classmethod
    def run_bench(cls, kernel, a: RefCsr, t, groups, workers, repeats, seed=42) -> dict:
        """psc::run_bench (bench.cpp:118-187): the reference's own paired-median measurement."""
        out = (c_double * 6)()
        cls._check(cls.lib().ref_run_bench(kernel, a.h, t, groups, workers, repeats, seed, out))
        keys = ["inspector_seconds", "baseline_seconds", "executor_seconds", "gflops", "max_rel_error", "ner"]
        return dict(zip(keys, [float(v) for v in out]))

    @classmethod
    def paired_timing(cls, plan: RefPlan, a: RefCsr, kernel: int, vec, workers: int, repeats: int):
        """(baseline, executor) median seconds, bench.cpp:88-104 over an existing plan."""
        out = (c_double * 2)()
        cls._check(cls.lib().ref_paired_timing(plan.h, a.h, kernel, _dp(vec), workers, repeats, out))
        return float(out[0]), float(out[1])

    @classmethod
    def time_inspect(cls, kernel, a, t, groups):
        h = c_void_p()
        s = c_double()
        cls._check(cls.lib().ref_time_inspect(kernel, a.h, t, groups, C.byref(s), C.byref(h)))
        return RefPlan(h), s.value
