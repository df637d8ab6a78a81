"""Python mirror of the reference's ``psc::`` API, backed by libpsc_b200.so.

Names, argument meaning and error behaviour follow the reference headers
(/root/reference/proj/core/include/psc/*.hpp) so parity tests read like the
reference's own tests:

* ``std::invalid_argument`` -> :class:`InvalidArgument` (a ``ValueError``)
* ``std::logic_error``      -> :class:`LogicError` (a ``RuntimeError``)

The inspector runs on the host (C++, bit-exact with the reference). Every
executor entry point runs on the GPU; there is no CPU execution path.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from enum import IntEnum
from typing import List, Optional, Sequence

import numpy as np

from . import _capi
from ._capi import CodeletView, CsrView, ExecContext, PlanArrays, PlanCounts

# ---------------------------------------------------------------------------
# errors


class InvalidArgument(ValueError):
    """std::invalid_argument"""


class LogicError(RuntimeError):
    """std::logic_error"""


class CudaError(RuntimeError):
    pass


def _check(status: int) -> None:
    if status == _capi.OK:
        return
    msg = _capi.lib().psc_last_error().decode(errors="replace")
    if status == _capi.ERR_INVALID_ARGUMENT:
        raise InvalidArgument(msg)
    if status == _capi.ERR_LOGIC:
        raise LogicError(msg)
    if status == _capi.ERR_CUDA:
        raise CudaError(msg)
    if status == _capi.ERR_NOMEM:
        raise MemoryError(msg)
    raise RuntimeError(msg)


def _dp(a: Optional[np.ndarray]):
    return None if a is None else a.ctypes.data_as(C.POINTER(C.c_double))


def _ip(a: Optional[np.ndarray]):
    return None if a is None else a.ctypes.data_as(C.POINTER(C.c_int32))


# ---------------------------------------------------------------------------
# enums (reference order)


class KernelKind(IntEnum):
    Spmv = 0
    Sptrsv = 1


class CodeletKind(IntEnum):
    Blas = 0
    PscI = 1
    PscII = 2


class MineStrategy(IntEnum):
    BlasFirst = 0
    PsciFirst = 1
    PsciiFirst = 2


class Form(IntEnum):
    Strided = 0
    InnerTable = 1
    OuterTable = 2
    PointTable = 3


def kernel_name(k) -> str:
    return "spmv" if int(k) == 0 else "sptrsv"


def codelet_kind_name(k) -> str:
    return ("BLAS", "PSC_I", "PSC_II")[min(int(k), 2)]


def strategy_name(s) -> str:
    return ("blas_first", "psci_first", "pscii_first")[min(int(s), 2)]


# ---------------------------------------------------------------------------
# matrices (csr_matrix.hpp)


class CsrMatrix:
    """CSR with int32 offsets/columns and fp64 values (csr_matrix.hpp:9-20)."""

    def __init__(self, n_rows=0, n_cols=0, row_offsets=None, col_indices=None, values=None):
        self.n_rows = int(n_rows)
        self.n_cols = int(n_cols)
        self.row_offsets = np.ascontiguousarray(
            row_offsets if row_offsets is not None else np.zeros(self.n_rows + 1), dtype=np.int32)
        self.col_indices = np.ascontiguousarray(col_indices if col_indices is not None else [], dtype=np.int32)
        self.values = np.ascontiguousarray(values if values is not None else [], dtype=np.float64)

    def nnz(self) -> int:
        return int(self.col_indices.size)

    def row_extent(self, row: int) -> int:
        return int(self.row_offsets[row + 1] - self.row_offsets[row])

    def view(self) -> CsrView:
        # keep arrays contiguous and alive as long as self
        self.row_offsets = np.ascontiguousarray(self.row_offsets, dtype=np.int32)
        self.col_indices = np.ascontiguousarray(self.col_indices, dtype=np.int32)
        self.values = np.ascontiguousarray(self.values, dtype=np.float64)
        return CsrView(self.n_rows, self.n_cols, self.nnz(), _ip(self.row_offsets), _ip(self.col_indices),
                       _dp(self.values))

    def __eq__(self, other) -> bool:
        return (isinstance(other, CsrMatrix) and self.n_rows == other.n_rows and self.n_cols == other.n_cols
                and np.array_equal(self.row_offsets, other.row_offsets)
                and np.array_equal(self.col_indices, other.col_indices)
                and np.array_equal(self.values, other.values))

    def __repr__(self):
        return f"CsrMatrix({self.n_rows}x{self.n_cols}, nnz={self.nnz()})"

    @classmethod
    def _take(cls, handle: C.c_void_p) -> "CsrMatrix":
        v = CsrView()
        try:
            _check(_capi.lib().psc_csr_view_of(handle, C.byref(v)))
            ro = np.ctypeslib.as_array(v.row_offsets, shape=(v.n_rows + 1,)).copy()
            if v.nnz:
                ci = np.ctypeslib.as_array(v.col_indices, shape=(v.nnz,)).copy()
                va = np.ctypeslib.as_array(v.values, shape=(v.nnz,)).copy()
            else:
                ci, va = np.zeros(0, np.int32), np.zeros(0, np.float64)
            return cls(v.n_rows, v.n_cols, ro, ci, va)
        finally:
            _capi.lib().psc_csr_destroy(handle)


def spmv_csr_baseline(a: CsrMatrix, x: np.ndarray) -> np.ndarray:
    """The reference's sequential SpMV baseline (executor.cpp:310-323), host."""
    x = np.ascontiguousarray(x, dtype=np.float64)
    y = np.empty(a.n_rows)
    _check(_capi.lib().psc_csr_spmv_baseline(C.byref(a.view()), _dp(x), x.size, _dp(y), y.size))
    return y


def sptrsv_csr_baseline(l, b: np.ndarray) -> np.ndarray:
    """The reference's forward substitution (executor.cpp:325-340), host."""
    m = l.csr() if isinstance(l, TriangularMatrix) else l
    b = np.ascontiguousarray(b, dtype=np.float64)
    x = np.empty(m.n_rows)
    _check(_capi.lib().psc_csr_sptrsv_baseline(C.byref(m.view()), _dp(b), b.size, _dp(x), x.size))
    return x


def read_matrix_market(path) -> CsrMatrix:
    """Matrix Market coordinate file -> CSR (read_matrix_market_file,
    matrix_market.hpp:24-29); parse errors raise InvalidArgument "line N: ..."."""
    h = C.c_void_p()
    _check(_capi.lib().psc_csr_read_matrix_market(str(path).encode(), C.byref(h)))
    return CsrMatrix._take(h)


def write_matrix_market(a: CsrMatrix, path) -> None:
    """CSR -> coordinate real general, 1-based (write_matrix_market_file)."""
    _check(_capi.lib().psc_csr_write_matrix_market(C.byref(a.view()), str(path).encode()))


@dataclass
class Triplet:
    row: int = 0
    col: int = 0
    value: float = 0.0


def csr_from_triplets(n_rows: int, n_cols: int, entries) -> CsrMatrix:
    """csr_matrix.cpp:9-45: stable sort by (row, col), duplicates summed."""
    t = [(e.row, e.col, e.value) if isinstance(e, Triplet) else tuple(e) for e in entries]
    rows = np.array([e[0] for e in t], dtype=np.int32)
    cols = np.array([e[1] for e in t], dtype=np.int32)
    vals = np.array([e[2] for e in t], dtype=np.float64)
    h = C.c_void_p()
    _check(_capi.lib().psc_csr_from_triplets(n_rows, n_cols, len(t), _ip(rows), _ip(cols), _dp(vals), C.byref(h)))
    return CsrMatrix._take(h)


def validate_csr(a: CsrMatrix) -> None:
    _check(_capi.lib().psc_validate_csr(C.byref(a.view())))


def is_lower_triangular(a: CsrMatrix) -> bool:
    for r in range(a.n_rows):
        if np.any(a.col_indices[a.row_offsets[r]:a.row_offsets[r + 1]] > r):
            return False
    return True


class TriangularMatrix:
    """Lower triangle with the diagonal stored last and nonzero (csr_matrix.hpp:41-54)."""

    def __init__(self, m: CsrMatrix):
        self._m = m

    @staticmethod
    def adopt(a: CsrMatrix) -> "TriangularMatrix":
        _check(_capi.lib().psc_adopt_triangular(C.byref(a.view())))
        return TriangularMatrix(a)

    def csr(self) -> CsrMatrix:
        return self._m

    def n(self) -> int:
        return self._m.n_rows

    def diag_pos(self, row: int) -> int:
        return int(self._m.row_offsets[row + 1] - 1)


def lower_triangular(a: CsrMatrix) -> TriangularMatrix:
    h = C.c_void_p()
    _check(_capi.lib().psc_lower_triangular(C.byref(a.view()), C.byref(h)))
    return TriangularMatrix(CsrMatrix._take(h))


# ---- benchmark inputs (configs.cpp) ----

def generate_config(config: int, scale: float = 1.0, seed: int = 0) -> CsrMatrix:
    """BASELINE.json configs 1..5; seed 0 = the config's default stream."""
    h = C.c_void_p()
    _check(_capi.lib().psc_generate_config(config, float(scale), seed, C.byref(h)))
    return CsrMatrix._take(h)


def seeded_vector(n: int, seed: int) -> np.ndarray:
    v = np.empty(n, dtype=np.float64)
    _capi.lib().psc_seeded_vector(n, seed, _dp(v))
    return v


def uniform_vector(n: int, seed: int, lo: float = -1.0, hi: float = 1.0) -> np.ndarray:
    v = np.empty(n, dtype=np.float64)
    _capi.lib().psc_uniform_vector(n, seed, lo, hi, _dp(v))
    return v


def int_vector(n: int, seed: int) -> np.ndarray:
    v = np.empty(n, dtype=np.float64)
    _capi.lib().psc_int_vector(n, seed, _dp(v))
    return v


# ---------------------------------------------------------------------------
# codelets (codelet.hpp)


@dataclass
class StridedAccess:
    base: int = 0
    stride_outer: int = 0
    stride_inner: int = 0

    def at(self, i: int, j: int) -> int:
        return self.base + i * self.stride_outer + j * self.stride_inner


@dataclass
class AccessDesc:
    form: Form = Form.Strided
    lin: StridedAccess = field(default_factory=StridedAccess)
    table: List[int] = field(default_factory=list)

    def is_table(self) -> bool:
        return self.form != Form.Strided

    def at(self, i: int, j: int, inner_extent: int) -> int:
        if self.form == Form.Strided:
            return self.lin.at(i, j)
        if self.form == Form.InnerTable:
            return self.table[j]
        if self.form == Form.OuterTable:
            return self.table[i]
        return self.table[i * inner_extent + j]

    @staticmethod
    def strided(base, stride_outer, stride_inner) -> "AccessDesc":
        return AccessDesc(Form.Strided, StridedAccess(base, stride_outer, stride_inner), [])

    @staticmethod
    def inner_table(t) -> "AccessDesc":
        return AccessDesc(Form.InnerTable, StridedAccess(), list(t))

    @staticmethod
    def outer_table(t) -> "AccessDesc":
        return AccessDesc(Form.OuterTable, StridedAccess(), list(t))

    @staticmethod
    def point_table(t) -> "AccessDesc":
        return AccessDesc(Form.PointTable, StridedAccess(), list(t))


@dataclass
class Codelet:
    kind: CodeletKind = CodeletKind.Blas
    outer_extent: int = 0
    inner_extent: int = 0
    out: AccessDesc = field(default_factory=AccessDesc)
    mat: AccessDesc = field(default_factory=AccessDesc)
    vec: AccessDesc = field(default_factory=AccessDesc)

    def ops(self) -> int:
        return self.outer_extent * self.inner_extent


def table_count(k) -> int:
    return {0: 0, 1: 1}.get(int(k), 2)


def kind_from_descriptors(out: AccessDesc, mat: AccessDesc, vec: AccessDesc) -> CodeletKind:
    tables = int(out.is_table()) + int(mat.is_table()) + int(vec.is_table())
    if tables == 3:
        raise InvalidArgument("codelet: all three descriptors are tables")
    return CodeletKind(tables)


@dataclass
class CostModelResult:
    ops: int = 0
    fns: int = 0
    descriptors: int = 0
    total: int = 0


def codelet_cost(c: Codelet) -> CostModelResult:
    """Eq. (1), codelet.cpp:45-57."""
    dims = (1 if c.outer_extent > 1 else 0) + (1 if c.inner_extent > 1 else 0)
    dims = dims or 1
    size = lambda d: len(d.table) if d.is_table() else dims  # noqa: E731
    r = CostModelResult(c.ops(), 3, size(c.out) + size(c.mat) + size(c.vec))
    r.total = r.ops + r.fns + r.descriptors
    return r


def plan_cost(cs) -> int:
    return sum(codelet_cost(c).total for c in cs)


# ---------------------------------------------------------------------------
# plans (miner.hpp)


@dataclass
class RowWindow:
    row_begin: int = 0
    row_end: int = 0

    def rows(self) -> int:
        return self.row_end - self.row_begin


@dataclass
class FinalizeRecord:
    row: int = 0
    diag_pos: int = 0
    rhs_index: int = 0


@dataclass
class RegionGroup:
    window: RowWindow = field(default_factory=RowWindow)
    strategy: MineStrategy = MineStrategy.PsciiFirst
    cost: int = 0
    codelets: List[Codelet] = field(default_factory=list)
    finalize: List[FinalizeRecord] = field(default_factory=list)


@dataclass
class PartitionPlan:
    groups: List[RegionGroup] = field(default_factory=list)


def _alloc_arrays(counts: PlanCounts):
    arrays = PlanArrays()
    keep = {}
    for name, ct, length in _capi.PLAN_ARRAY_FIELDS:
        dtype = np.int64 if ct is C.c_int64 else np.int32
        buf = np.zeros(max(1, int(length(counts))), dtype=dtype)
        keep[name] = buf
        setattr(arrays, name, buf.ctypes.data_as(C.POINTER(ct)))
    return arrays, keep


class CodeletPlan:
    """Handle to a host plan (CodeletPlan, miner.hpp:73-89).

    Mined plans keep their tables implicit in the CSR arrays; the plan holds a
    reference to the matrix it was mined from so it can materialise them.
    """

    def __init__(self, handle: C.c_void_p, matrix: Optional[CsrMatrix]):
        self._h = handle
        self._matrix = matrix
        self._partitions = None
        c = PlanCounts()
        _check(_capi.lib().psc_plan_get_counts(self._h, C.byref(c)))
        self._counts = c
        self.kernel = KernelKind(c.kernel)
        self.n_rows, self.n_cols, self.nnz = c.n_rows, c.n_cols, c.nnz
        self.window, self.target_groups = c.window, c.target_groups

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            try:
                _capi.lib().psc_plan_destroy(h)
            except Exception:
                pass
            self._h = None

    @property
    def handle(self):
        return self._h

    def counts(self) -> PlanCounts:
        return self._counts

    def _view(self):
        return C.byref(self._matrix.view()) if self._matrix is not None else None

    def export_arrays(self):
        arrays, keep = _alloc_arrays(self._counts)
        _check(_capi.lib().psc_plan_to_arrays(self._h, self._view(), C.byref(arrays)))
        return self._counts, arrays, keep

    def hash(self) -> int:
        out = C.c_uint64()
        _check(_capi.lib().psc_plan_hash(self._h, self._view(), C.byref(out)))
        return out.value

    def save(self, path: str) -> None:
        """Write the plan to a binary plan file (psc_plan_save)."""
        _check(_capi.lib().psc_plan_save(self._h, str(path).encode()))

    @staticmethod
    def load(path: str, matrix: Optional[CsrMatrix] = None) -> "CodeletPlan":
        """Read a binary plan file (psc_plan_load). Mined plans need the matrix
        they were mined from to materialise their tables; it is validated."""
        h = C.c_void_p()
        _check(_capi.lib().psc_plan_load(str(path).encode(), C.byref(h)))
        plan = CodeletPlan(h, matrix)
        if matrix is not None:
            validate_plan(plan, matrix)
        return plan

    def totals(self):
        cost, ops = C.c_int64(), C.c_int64()
        by = (C.c_int64 * 3)()
        _check(_capi.lib().psc_plan_totals(self._h, C.byref(cost), C.byref(ops), by))
        return cost.value, ops.value, list(by)

    def total_cost(self) -> int:
        return self.totals()[0]

    def total_ops(self) -> int:
        return self.totals()[1]

    @property
    def partitions(self) -> List[PartitionPlan]:
        if self._partitions is None:
            counts, arrays, keep = self.export_arrays()  # `keep` owns the buffers `arrays` points into
            self._partitions = _arrays_to_partitions(counts, arrays, self._counts)
            del keep
        return self._partitions

    @staticmethod
    def from_partitions(kernel, n_rows, n_cols, nnz, window, target_groups, partitions) -> "CodeletPlan":
        """Import a plan built from Python objects (e.g. a hand-built or
        reference-produced plan) through psc_plan_from_arrays."""
        counts, arrays, keep = _partitions_to_arrays(kernel, n_rows, n_cols, nnz, window, target_groups, partitions)
        return CodeletPlan.from_arrays(counts, arrays, keep)

    @staticmethod
    def from_arrays(counts: PlanCounts, arrays: PlanArrays, keep=None, matrix=None) -> "CodeletPlan":
        h = C.c_void_p()
        _check(_capi.lib().psc_plan_from_arrays(C.byref(counts), C.byref(arrays), C.byref(h)))
        return CodeletPlan(h, matrix)


def _arrays_to_partitions(counts: PlanCounts, arrays: PlanArrays, c: PlanCounts) -> List[PartitionPlan]:
    def arr(name, n):
        ct = dict((f[0], f[1]) for f in _capi.PLAN_ARRAY_FIELDS)[name]
        if n <= 0:
            return np.zeros(0, dtype=np.int64 if ct is C.c_int64 else np.int32)
        return np.ctypeslib.as_array(getattr(arrays, name), shape=(n,))

    pg = arr("part_group_ptr", c.n_partitions + 1)
    rb, re = arr("group_row_begin", c.n_groups), arr("group_row_end", c.n_groups)
    st, co = arr("group_strategy", c.n_groups), arr("group_cost", c.n_groups)
    gc, gf = arr("group_codelet_ptr", c.n_groups + 1), arr("group_finalize_ptr", c.n_groups + 1)
    kind, m, n = arr("codelet_kind", c.n_codelets), arr("codelet_m", c.n_codelets), arr("codelet_n", c.n_codelets)
    form, base = arr("desc_form", 3 * c.n_codelets), arr("desc_base", 3 * c.n_codelets)
    so, si = arr("desc_stride_outer", 3 * c.n_codelets), arr("desc_stride_inner", 3 * c.n_codelets)
    tp, tab = arr("desc_table_ptr", 3 * c.n_codelets + 1), arr("table", c.n_table)
    fr, fd, fh = arr("fin_row", c.n_finalize), arr("fin_diag_pos", c.n_finalize), arr("fin_rhs_index", c.n_finalize)
    parts = []
    for p in range(c.n_partitions):
        groups = []
        for g in range(int(pg[p]), int(pg[p + 1])):
            cods = []
            for ci in range(int(gc[g]), int(gc[g + 1])):
                ds = []
                for d in range(3):
                    k = 3 * ci + d
                    ds.append(AccessDesc(Form(int(form[k])), StridedAccess(int(base[k]), int(so[k]), int(si[k])),
                                         [int(v) for v in tab[int(tp[k]):int(tp[k + 1])]]))
                cods.append(Codelet(CodeletKind(int(kind[ci])), int(m[ci]), int(n[ci]), ds[0], ds[1], ds[2]))
            fins = [FinalizeRecord(int(fr[f]), int(fd[f]), int(fh[f])) for f in range(int(gf[g]), int(gf[g + 1]))]
            groups.append(RegionGroup(RowWindow(int(rb[g]), int(re[g])), MineStrategy(int(st[g])), int(co[g]), cods,
                                      fins))
        parts.append(PartitionPlan(groups))
    return parts


def _partitions_to_arrays(kernel, n_rows, n_cols, nnz, window, target_groups, partitions):
    c = PlanCounts()
    c.kernel, c.n_rows, c.n_cols, c.window, c.target_groups, c.nnz = int(kernel), n_rows, n_cols, window, \
        target_groups, nnz
    groups = [g for p in partitions for g in p.groups]
    cods = [cd for g in groups for cd in g.codelets]
    c.n_partitions, c.n_groups, c.n_codelets = len(partitions), len(groups), len(cods)
    c.n_finalize = sum(len(g.finalize) for g in groups)
    c.n_table = sum(len(d.table) for cd in cods for d in (cd.out, cd.mat, cd.vec))
    arrays, keep = _alloc_arrays(c)
    k = keep
    gi = ci = fi = ti = 0
    k["part_group_ptr"][0] = 0
    k["group_codelet_ptr"][0] = 0
    k["group_finalize_ptr"][0] = 0
    k["desc_table_ptr"][0] = 0
    for pi, p in enumerate(partitions):
        for g in p.groups:
            k["group_row_begin"][gi], k["group_row_end"][gi] = g.window.row_begin, g.window.row_end
            k["group_strategy"][gi], k["group_cost"][gi] = int(g.strategy), g.cost
            for cd in g.codelets:
                k["codelet_kind"][ci], k["codelet_m"][ci], k["codelet_n"][ci] = int(cd.kind), cd.outer_extent, \
                    cd.inner_extent
                for d, desc in enumerate((cd.out, cd.mat, cd.vec)):
                    kk = 3 * ci + d
                    k["desc_form"][kk] = int(desc.form)
                    k["desc_base"][kk] = desc.lin.base
                    k["desc_stride_outer"][kk] = desc.lin.stride_outer
                    k["desc_stride_inner"][kk] = desc.lin.stride_inner
                    for v in desc.table:
                        k["table"][ti] = v
                        ti += 1
                    k["desc_table_ptr"][kk + 1] = ti
                ci += 1
            for f in g.finalize:
                k["fin_row"][fi], k["fin_diag_pos"][fi], k["fin_rhs_index"][fi] = f.row, f.diag_pos, f.rhs_index
                fi += 1
            gi += 1
            k["group_codelet_ptr"][gi], k["group_finalize_ptr"][gi] = ci, fi
        k["part_group_ptr"][pi + 1] = gi
    return c, arrays, keep


def inspect(kernel, a: CsrMatrix, t: int, target_groups: int, threads: int = 0) -> CodeletPlan:
    """inspect (miner.hpp:95): bit-exact with the reference inspector."""
    h = C.c_void_p()
    _check(_capi.lib().psc_inspect(int(kernel), C.byref(a.view()), t, target_groups, threads, C.byref(h)))
    return CodeletPlan(h, a)


def inspect_device(kernel, a: CsrMatrix, t: int, target_groups: int, device: int = 0) -> CodeletPlan:
    """inspect with the window mining on GPU `device` (psc_inspect_device):
    the same plan as inspect(), bit for bit."""
    h = C.c_void_p()
    _check(_capi.lib().psc_inspect_device(int(kernel), C.byref(a.view()), t, target_groups, device, C.byref(h)))
    return CodeletPlan(h, a)


def validate_plan(plan: CodeletPlan, a: CsrMatrix) -> None:
    _check(_capi.lib().psc_validate_plan(plan.handle, C.byref(a.view())))


def operation_breakdown(plan: CodeletPlan):
    """bench.cpp:34-48: fraction of operations per codelet kind."""
    _, total, by = plan.totals()
    if total == 0:
        return (0.0, 0.0, 0.0)
    return tuple(b / total for b in by)


# ---------------------------------------------------------------------------
# executor (executor.hpp) — GPU only


@dataclass
class ExecutionContext:
    matrix_values: Optional[np.ndarray] = None
    gather: Optional[np.ndarray] = None
    accum: Optional[np.ndarray] = None
    rhs: Optional[np.ndarray] = None
    solution: Optional[np.ndarray] = None

    def _c(self) -> ExecContext:
        for name in ("matrix_values", "gather", "accum", "rhs", "solution"):
            v = getattr(self, name)
            if v is not None and (v.dtype != np.float64 or not v.flags.c_contiguous):
                raise InvalidArgument(f"ExecutionContext.{name} must be a contiguous float64 array")
        return ExecContext(_dp(self.matrix_values), _dp(self.gather), _dp(self.accum), _dp(self.rhs),
                           _dp(self.solution))


def _codelet_view(c: Codelet):
    keep = []

    def desc(d: AccessDesc):
        t = np.ascontiguousarray(d.table, dtype=np.int32)
        keep.append(t)
        return _capi.AccessDescView(int(d.form), d.lin.base, d.lin.stride_outer, d.lin.stride_inner,
                                    _ip(t) if t.size else None, t.size)

    v = CodeletView(int(c.kind), c.outer_extent, c.inner_extent, desc(c.out), desc(c.mat), desc(c.vec))
    return v, keep


def _exec(fn, c: Codelet, ctx: ExecutionContext):
    v, keep = _codelet_view(c)
    cc = ctx._c()
    _check(fn(C.byref(v), C.byref(cc)))
    del keep


def exec_blas_codelet(c: Codelet, ctx: ExecutionContext) -> None:
    _exec(_capi.lib().psc_exec_blas_codelet, c, ctx)


def exec_psci_codelet(c: Codelet, ctx: ExecutionContext) -> None:
    _exec(_capi.lib().psc_exec_psci_codelet, c, ctx)


def exec_pscii_codelet(c: Codelet, ctx: ExecutionContext) -> None:
    _exec(_capi.lib().psc_exec_pscii_codelet, c, ctx)


class Executor:
    """Executor(workers) (executor.hpp:36-51). Runs on one GPU; the worker
    count is validated and kept for API compatibility only."""

    def __init__(self, workers: int, device: int = 0):
        h = C.c_void_p()
        _check(_capi.lib().psc_executor_create(int(workers), int(device), C.byref(h)))
        self._h = h
        self.device = device

    def workers(self) -> int:
        return int(_capi.lib().psc_executor_workers(self._h))

    def set_values_version(self, version: int) -> None:
        """Tag the matrix values of the following run_* calls (0: unknown, always
        upload them; a nonzero tag equal to the bound plan's skips the upload)."""
        _check(_capi.lib().psc_executor_set_values_version(self._h, int(version)))

    @property
    def handle(self):
        return self._h

    def run(self, plan: CodeletPlan, ctx: ExecutionContext, matrix: Optional[CsrMatrix] = None) -> None:
        a = matrix if matrix is not None else plan._matrix
        if a is None:
            raise InvalidArgument("Executor.run: the plan's matrix structure is required")
        _check(_capi.lib().psc_execute_plan(self._h, plan.handle, C.byref(a.view()), C.byref(ctx._c())))

    def close(self):
        if getattr(self, "_h", None):
            _capi.lib().psc_executor_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def execute_plan(plan: CodeletPlan, ctx: ExecutionContext, workers: int, matrix: Optional[CsrMatrix] = None):
    """execute_plan (executor.cpp:269-272)."""
    exe = Executor(workers)
    try:
        exe.run(plan, ctx, matrix)
    finally:
        exe.close()


def _f64(v, name):
    if not isinstance(v, np.ndarray) or v.dtype != np.float64 or not v.flags.c_contiguous:
        raise InvalidArgument(f"{name} must be a contiguous float64 numpy array")
    return v


def run_spmv(plan: CodeletPlan, a: CsrMatrix, x, y, exe: Executor) -> None:
    """y = A x through a plan; y is overwritten (executor.cpp:274-288)."""
    x, y = _f64(x, "x"), _f64(y, "y")
    _check(_capi.lib().psc_run_spmv(exe.handle, plan.handle, C.byref(a.view()), _dp(x), x.size, _dp(y), y.size))


def run_sptrsv(plan: CodeletPlan, l: TriangularMatrix, b, x, acc, exe: Executor) -> None:
    """Solves L x = b through a plan (executor.cpp:290-308)."""
    b, x, acc = _f64(b, "b"), _f64(x, "x"), _f64(acc, "acc")
    m = l.csr() if isinstance(l, TriangularMatrix) else l
    _check(_capi.lib().psc_run_sptrsv(exe.handle, plan.handle, C.byref(m.view()), _dp(b), b.size, _dp(x), x.size,
                                      _dp(acc), acc.size))


# ---------------------------------------------------------------------------
# HBM-resident execution (the hot path used by bench.py)


class BoundPlan:
    """A plan and its matrix lowered and resident on the GPU. Vectors are
    torch CUDA tensors (float64); calls enqueue on the given stream (default:
    torch's current stream) and return without synchronising."""

    def __init__(self, exe: Executor, plan: CodeletPlan, a: CsrMatrix, mode: int = 0,
                 partitions: Optional[tuple] = None):
        h = C.c_void_p()
        m = a.csr() if isinstance(a, TriangularMatrix) else a
        if partitions is None:
            _check(_capi.lib().psc_bind(exe.handle, plan.handle, C.byref(m.view()), mode, C.byref(h)))
        else:
            _check(_capi.lib().psc_bind_partitions(exe.handle, plan.handle, C.byref(m.view()), mode,
                                                   int(partitions[0]), int(partitions[1]), C.byref(h)))
        self._h = h
        self.kernel = plan.kernel
        self.device = exe.device
        rb, re = C.c_int32(), C.c_int32()
        _check(_capi.lib().psc_bound_rows(self._h, C.byref(rb), C.byref(re)))
        self.row_begin, self.row_end = rb.value, re.value

    @staticmethod
    def _stream(stream):
        if stream is None:
            import torch
            return C.c_void_p(torch.cuda.current_stream().cuda_stream)
        if isinstance(stream, int):
            return C.c_void_p(stream)
        return C.c_void_p(stream.cuda_stream)

    def spmv(self, x, y, stream=None) -> None:
        _check(_capi.lib().psc_bound_spmv(self._h, C.c_void_p(x.data_ptr()), C.c_void_p(y.data_ptr()),
                                          self._stream(stream)))

    def x_runs(self) -> np.ndarray:
        """Column runs [c0, c1) outside this shard's rows that its multiply reads (shape (n, 2))."""
        n = C.c_int64()
        _check(_capi.lib().psc_bound_x_runs(self._h, None, 0, C.byref(n)))
        out = np.zeros(2 * n.value, dtype=np.int32)
        _check(_capi.lib().psc_bound_x_runs(self._h, out.ctypes.data_as(C.POINTER(C.c_int32)), n.value, C.byref(n)))
        return out.reshape(-1, 2)

    def spmv_peers(self, peers, x_window, y, stream=None) -> None:
        """Fused exchange + multiply (psc_bound_spmv_peers): `peers` lists every
        rank's (window device pointer, row_begin, row_end) in rank order;
        x_window (this rank's window, a torch CUDA tensor of all columns) holds
        this rank's own entries."""
        arr = (_capi.PeerWindow * len(peers))()
        for i, (ptr, r0, r1) in enumerate(peers):
            arr[i].base, arr[i].row_begin, arr[i].row_end = int(ptr), int(r0), int(r1)
        xw = x_window if isinstance(x_window, int) else x_window.data_ptr()
        _check(_capi.lib().psc_bound_spmv_peers(self._h, C.cast(arr, C.c_void_p), len(peers), C.c_void_p(xw),
                                                C.c_void_p(y.data_ptr()), self._stream(stream)))

    def sptrsv(self, b, x, acc=None, stream=None) -> None:
        _check(_capi.lib().psc_bound_sptrsv(self._h, C.c_void_p(b.data_ptr()), C.c_void_p(x.data_ptr()),
                                            C.c_void_p(acc.data_ptr()) if acc is not None else None,
                                            self._stream(stream)))

    def spmv_host(self, x: np.ndarray, y: np.ndarray, stream=None) -> None:
        """H2D x, kernel, D2H y on `stream` (host arrays; pin them for async copies)."""
        _check(_capi.lib().psc_bound_spmv_host(self._h, _dp(x), _dp(y), self._stream(stream)))

    def sptrsv_host(self, b: np.ndarray, x: np.ndarray, acc: Optional[np.ndarray] = None, stream=None) -> None:
        _check(_capi.lib().psc_bound_sptrsv_host(self._h, _dp(b), _dp(x), _dp(acc), self._stream(stream)))

    def csr_spmv_naive(self, x, y, stream=None) -> None:
        """spmv_csr_baseline on the GPU (executor.cpp:310-322) over this plan's matrix."""
        _check(_capi.lib().psc_csr_spmv_device(self._h, C.c_void_p(x.data_ptr()), C.c_void_p(y.data_ptr()),
                                               self._stream(stream)))

    def csr_sptrsv_naive(self, b, x, stream=None) -> None:
        """sptrsv_csr_baseline on the GPU (executor.cpp:325-340): thread per row, sync-free."""
        _check(_capi.lib().psc_csr_sptrsv_device(self._h, C.c_void_p(b.data_ptr()), C.c_void_p(x.data_ptr()),
                                                 self._stream(stream)))

    def launches(self) -> int:
        return int(_capi.lib().psc_bound_launches(self._h))

    def info(self) -> dict:
        out = (C.c_int64 * 8)()
        _check(_capi.lib().psc_bound_info(self._h, out))
        keys = ["rows", "segments", "work_units", "path", "algorithmic_bytes", "device_bytes", "long_rows",
                "passes_or_block_rows"]
        return dict(zip(keys, [int(v) for v in out]))

    def close(self):
        if getattr(self, "_h", None):
            _capi.lib().psc_bound_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def device_count() -> int:
    return int(_capi.lib().psc_device_count())


def partition_rows(plan: CodeletPlan, part_begin: int, part_end: int):
    """Contiguous row range [begin, end) covered by partitions [part_begin, part_end)."""
    rb, re = C.c_int32(), C.c_int32()
    _check(_capi.lib().psc_plan_partition_rows(plan.handle, part_begin, part_end, C.byref(rb), C.byref(re)))
    return rb.value, re.value
