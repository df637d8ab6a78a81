"""Bench reports in the reference's format (bench.hpp:13-94, bench.cpp:18-336;
SURVEY.md §8f item 3), run on the GPU executor.

``run_bench`` inspects once (timed), times the reference's sequential CSR
baseline and the executor through the host-array API (``run_spmv`` /
``run_sptrsv``: H2D, kernels, D2H -- what the reference's ``run_*`` calls do
on its host arrays), one warm-up then the median of ``repeats`` runs each, and
verifies the executor against the baseline (elementwise relative error with
a 1e-300 floor, bench.cpp:106-114). NER = inspector / (baseline - executor).
Reports render as CSV (the reference's header, then GPU columns), JSON
(fixed key order) or text. Command line:

    python -m paper_2111_12243_b200.bench_report --config 1 --format csv
"""
from __future__ import annotations

import argparse
import json
import math
import statistics
import sys
import time
from dataclasses import dataclass, field
from typing import List, Optional

import numpy as np

from . import psc as P

CSV_HEADER = ("matrix,kernel,n_rows,n_cols,nnz,t,groups,workers,repeats,inspector_s,executor_s,baseline_s,gflops,"
              "ner,frac_blas,frac_psc1,frac_psc2,verified,max_rel_error,n_gpus,executor_gbps,normwise_error")


def compute_ner(inspector_seconds: float, baseline_seconds: float, executor_seconds: float):
    """(ner, amortizable): runs of the executor that pay off the inspection
    (bench.cpp:18-25); +inf when the executor is not faster than the baseline."""
    amortizable = executor_seconds < baseline_seconds
    if not amortizable:
        return math.inf, False
    return inspector_seconds / (baseline_seconds - executor_seconds), True


def theoretical_flops(kernel, n_rows: int, nnz: int) -> int:
    return 2 * nnz if P.KernelKind(kernel) == P.KernelKind.Spmv else 2 * nnz - n_rows


@dataclass
class BenchConfig:
    matrix_name: str = ""
    kernel: int = P.KernelKind.Spmv
    t: int = 3
    groups: int = 0  # 0: use the worker count
    workers: int = 1
    repeats: int = 5
    verify_tol: float = 1e-12
    baseline_only: bool = False
    seed: int = 42


@dataclass
class BenchReport:
    matrix: str = ""
    kernel: str = ""
    n_rows: int = 0
    n_cols: int = 0
    nnz: int = 0
    t: int = 0
    groups: int = 0
    workers: int = 0
    repeats: int = 0
    baseline_only: bool = False
    inspector_seconds: float = 0.0
    executor_seconds: float = 0.0
    baseline_seconds: float = 0.0
    gflops: float = 0.0
    ner: float = 0.0
    amortizable: bool = False
    breakdown: List[float] = field(default_factory=lambda: [0.0, 0.0, 0.0])
    verified: bool = False
    max_rel_error: float = 0.0
    # GPU columns
    n_gpus: int = 1
    executor_gbps: float = 0.0
    normwise_error: float = 0.0


def _median_seconds(fn, repeats: int) -> float:
    fn()  # warm-up
    times = []
    for _ in range(max(1, repeats)):
        t0 = time.perf_counter()
        fn()
        times.append(time.perf_counter() - t0)
    return statistics.median(times)


def run_bench(cfg: BenchConfig, a: P.CsrMatrix, exe: Optional[P.Executor] = None) -> BenchReport:
    kernel = P.KernelKind(cfg.kernel)
    if kernel == P.KernelKind.Sptrsv and not P.is_lower_triangular(a):
        a = P.lower_triangular(a).csr()
    groups = cfg.groups or cfg.workers
    r = BenchReport(matrix=cfg.matrix_name, kernel=P.kernel_name(kernel), n_rows=a.n_rows, n_cols=a.n_cols,
                    nnz=a.nnz(), t=cfg.t, groups=groups, workers=cfg.workers, repeats=cfg.repeats,
                    baseline_only=cfg.baseline_only, n_gpus=1)
    vec = P.seeded_vector(a.n_cols if kernel == P.KernelKind.Spmv else a.n_rows, cfg.seed)
    if kernel == P.KernelKind.Spmv:
        base = lambda: P.spmv_csr_baseline(a, vec)  # noqa: E731
    else:
        tri = P.TriangularMatrix.adopt(a)
        base = lambda: P.sptrsv_csr_baseline(tri, vec)  # noqa: E731
    r.baseline_seconds = _median_seconds(base, cfg.repeats)
    want = base()
    if cfg.baseline_only:
        r.verified = True
        return r
    t0 = time.perf_counter()
    plan = P.inspect(kernel, a, cfg.t, groups)
    r.inspector_seconds = time.perf_counter() - t0
    exe = exe or P.Executor(cfg.workers)
    out = np.empty(a.n_rows)
    if kernel == P.KernelKind.Spmv:
        run = lambda: P.run_spmv(plan, a, vec, out, exe)  # noqa: E731
    else:
        acc = np.empty(a.n_rows)
        run = lambda: P.run_sptrsv(plan, tri, vec, out, acc, exe)  # noqa: E731
    r.executor_seconds = _median_seconds(run, cfg.repeats)
    run()
    r.gflops = theoretical_flops(kernel, a.n_rows, a.nnz()) / r.executor_seconds / 1e9
    r.ner, r.amortizable = compute_ner(r.inspector_seconds, r.baseline_seconds, r.executor_seconds)
    r.breakdown = list(P.operation_breakdown(plan))
    den = np.maximum(np.abs(want), 1e-300)
    r.max_rel_error = float(np.max(np.abs(out - want) / den)) if a.n_rows else 0.0
    r.verified = bool(r.max_rel_error <= cfg.verify_tol)
    nrm = float(np.linalg.norm(want))
    r.normwise_error = float(np.linalg.norm(out - want) / nrm) if nrm > 0 else float(np.linalg.norm(out - want))
    algo = 12 * a.nnz() + 4 * (a.n_rows + 1) + (8 * a.n_cols + 8 * a.n_rows if kernel == P.KernelKind.Spmv
                                                 else 16 * a.n_rows)
    r.executor_gbps = algo / r.executor_seconds / 1e9
    return r


def _num(v) -> str:
    return repr(float(v)) if isinstance(v, float) else str(v)  # shortest round-trip


def _csv_field(s: str) -> str:
    if not any(ch in s for ch in ',"\n'):
        return s
    return '"' + s.replace('"', '""') + '"'


def _csv_row(r: BenchReport) -> str:
    head = [_csv_field(r.matrix), r.kernel, str(r.n_rows), str(r.n_cols), str(r.nnz), str(r.t), str(r.groups),
            str(r.workers), str(r.repeats)]
    if r.baseline_only:
        return ",".join(head + ["", "", _num(r.baseline_seconds)] + [""] * 10)
    return ",".join(head + [_num(r.inspector_seconds), _num(r.executor_seconds), _num(r.baseline_seconds),
                            _num(r.gflops), _num(r.ner) if r.amortizable else "not_amortizable",
                            _num(r.breakdown[0]), _num(r.breakdown[1]), _num(r.breakdown[2]),
                            "1" if r.verified else "0", _num(r.max_rel_error), str(r.n_gpus),
                            _num(r.executor_gbps), _num(r.normwise_error)])


def _json_obj(r: BenchReport) -> dict:
    o = {"matrix": r.matrix, "kernel": r.kernel, "n_rows": r.n_rows, "n_cols": r.n_cols, "nnz": r.nnz, "t": r.t,
         "groups": r.groups, "workers": r.workers, "repeats": r.repeats, "baseline_only": r.baseline_only,
         "baseline_seconds": r.baseline_seconds}
    done = not r.baseline_only
    o["inspector_seconds"] = r.inspector_seconds if done else None
    o["executor_seconds"] = r.executor_seconds if done else None
    o["gflops"] = r.gflops if done else None
    o["ner"] = (r.ner if r.amortizable else None) if done else None
    o["amortizable"] = r.amortizable if done else None
    o["breakdown"] = ({"blas": r.breakdown[0], "psc1": r.breakdown[1], "psc2": r.breakdown[2]} if done else None)
    o["verified"] = r.verified
    o["max_rel_error"] = r.max_rel_error if done else None
    o["n_gpus"] = r.n_gpus
    o["executor_gbps"] = r.executor_gbps if done else None
    o["normwise_error"] = r.normwise_error if done else None
    return o


def emit_reports(reports: List[BenchReport], fmt: str) -> str:
    if fmt == "csv":
        return "\n".join([CSV_HEADER] + [_csv_row(r) for r in reports]) + "\n"
    if fmt == "json":
        return json.dumps([_json_obj(r) for r in reports], indent=2) + "\n"
    if fmt == "text":
        blocks = []
        for r in reports:
            lines = [f"matrix {r.matrix} ({r.kernel}, {r.n_rows}x{r.n_cols}, nnz {r.nnz})",
                     f"  t {r.t}, groups {r.groups}, workers {r.workers}, repeats {r.repeats}",
                     f"  baseline  {r.baseline_seconds * 1e3:.3f} ms"]
            if not r.baseline_only:
                lines += [f"  inspector {r.inspector_seconds * 1e3:.3f} ms",
                          f"  executor  {r.executor_seconds * 1e3:.3f} ms ({r.gflops:.2f} GFLOP/s, "
                          f"{r.executor_gbps:.1f} GB/s, {r.n_gpus} GPU)",
                          f"  NER       {r.ner:.3f}" if r.amortizable else "  NER       not amortizable",
                          f"  ops       blas {r.breakdown[0]:.3f} psc1 {r.breakdown[1]:.3f} psc2 {r.breakdown[2]:.3f}",
                          f"  verified  {'yes' if r.verified else 'NO'} (max rel err {r.max_rel_error:.3e}, "
                          f"normwise {r.normwise_error:.3e})"]
            blocks.append("\n".join(lines))
        return "\n\n".join(blocks) + "\n"
    raise P.InvalidArgument(f"unknown report format '{fmt}'")


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(description=__doc__.split("\n")[0])
    ap.add_argument("--config", type=int, action="append", help="BASELINE.json config (repeatable)")
    ap.add_argument("--mtx", action="append", help="a Matrix Market file (repeatable)")
    ap.add_argument("--kernel", choices=["spmv", "sptrsv"], help="for --mtx inputs (default spmv)")
    ap.add_argument("--scale", type=float, default=1.0)
    ap.add_argument("--t", type=int, default=3)
    ap.add_argument("--groups", type=int, default=8)
    ap.add_argument("--repeats", type=int, default=5)
    ap.add_argument("--baseline-only", action="store_true")
    ap.add_argument("--format", default="text", choices=["csv", "json", "text"])
    args = ap.parse_args(argv)
    reports = []
    config_kernel = {1: P.KernelKind.Spmv, 2: P.KernelKind.Sptrsv, 3: P.KernelKind.Spmv, 4: P.KernelKind.Sptrsv,
                     5: P.KernelKind.Spmv}
    exe = None if args.baseline_only else P.Executor(1)
    for c in args.config or []:
        cfg = BenchConfig(matrix_name=f"config{c}", kernel=config_kernel[c], t=args.t, groups=args.groups,
                          repeats=args.repeats, baseline_only=args.baseline_only)
        reports.append(run_bench(cfg, P.generate_config(c, args.scale), exe))
    for path in args.mtx or []:
        k = P.KernelKind.Sptrsv if args.kernel == "sptrsv" else P.KernelKind.Spmv
        cfg = BenchConfig(matrix_name=path, kernel=k, t=args.t, groups=args.groups, repeats=args.repeats,
                          baseline_only=args.baseline_only)
        reports.append(run_bench(cfg, P.read_matrix_market(path), exe))
    sys.stdout.write(emit_reports(reports, args.format))
    return 0 if all(r.verified for r in reports) else 1


if __name__ == "__main__":
    sys.exit(main())
