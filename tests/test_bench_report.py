"""Bench reports (bench.hpp:13-94): NER, formats, and a verified GPU run."""
import json
import math

import pytest

import paper_2111_12243_b200 as P
from paper_2111_12243_b200 import bench_report as B


def test_compute_ner():
    ner, ok = B.compute_ner(2.0, 5.0, 1.0)
    assert ok and ner == pytest.approx(0.5)
    ner, ok = B.compute_ner(2.0, 1.0, 1.0)  # not faster than the baseline
    assert not ok and math.isinf(ner)
    assert B.theoretical_flops(P.KernelKind.Spmv, 10, 30) == 60
    assert B.theoretical_flops(P.KernelKind.Sptrsv, 10, 30) == 50


def test_baseline_only_reports_in_every_format():
    a = P.generate_config(1, 0.002)
    r = B.run_bench(B.BenchConfig(matrix_name='m,"1"', kernel=P.KernelKind.Spmv, repeats=2, baseline_only=True), a)
    assert r.verified and r.baseline_seconds > 0
    csv = B.emit_reports([r], "csv").splitlines()
    assert csv[0] == B.CSV_HEADER
    row = csv[1]
    assert row.startswith('"m,""1"""')  # quoted as the reference quotes
    assert row.count(",") == csv[0].count(",") + 1  # +1: the comma inside the quoted matrix name
    j = json.loads(B.emit_reports([r], "json"))[0]
    assert j["executor_seconds"] is None and j["ner"] is None and j["baseline_only"] is True
    assert "baseline" in B.emit_reports([r], "text")
    with pytest.raises(P.InvalidArgument):
        B.emit_reports([r], "xml")


@pytest.mark.gpu
def test_gpu_report_verifies():
    reports = []
    for c, k in ((1, P.KernelKind.Spmv), (2, P.KernelKind.Sptrsv)):
        cfg = B.BenchConfig(matrix_name=f"config{c}", kernel=k, groups=8, repeats=2)
        r = B.run_bench(cfg, P.generate_config(c, 0.01))
        assert r.verified and r.executor_seconds > 0 and r.gflops > 0
        assert r.normwise_error <= (1e-12 if k == P.KernelKind.Spmv else 1e-10)
        reports.append(r)
    csv = B.emit_reports(reports, "csv").splitlines()
    assert len(csv) == 3 and all(len(line.split(",")) == len(B.CSV_HEADER.split(",")) for line in csv[1:])
    assert B.main(["--config", "2", "--scale", "0.01", "--repeats", "1", "--format", "json"]) == 0
