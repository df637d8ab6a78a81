"""The host inspector (C++) against the reference's miner / scheduler tests
(test_miner.cpp, test_scheduler.cpp known answers) and, bitwise via the plan
digest, against the reference inspector itself."""
import numpy as np
import pytest

import paper_2111_12243_b200 as P
from oracle.oracle import Ref
from paper_2111_12243_b200 import AccessDesc, CodeletKind, KernelKind, MineStrategy
from tests.helpers import golden_cases, suite_cases, pattern


def mixed_pattern():
    """test_miner.cpp:15-23."""
    t = [(0, j, 1.0) for j in (4, 5, 6, 9)] + [(i, j, 1.0) for i in (1, 2) for j in (4, 5, 6)]
    return P.csr_from_triplets(3, 10, t)


def test_dense_block_tiles_into_window_rectangles():
    """test_miner.cpp:183-197."""
    plan = P.inspect(KernelKind.Spmv, pattern("dense_block(6)"), 3, 1)
    parts = plan.partitions
    assert len(parts) == 1 and len(parts[0].groups) == 2
    for g in parts[0].groups:
        assert g.strategy == MineStrategy.BlasFirst and len(g.codelets) == 1
        c = g.codelets[0]
        assert (c.kind, c.outer_extent, c.inner_extent, g.cost) == (CodeletKind.Blas, 3, 6, 27)
    assert plan.total_cost() == 54 and plan.total_ops() == 36


def test_worked_example_shared_gather():
    """test_miner.cpp:199-211, :74-96 (BLAS descriptors of dense_block(3))."""
    plan = P.inspect(KernelKind.Spmv, pattern("scattered_gather(3,0:2:5)"), 3, 1)
    g = plan.partitions[0].groups[0]
    assert g.strategy == MineStrategy.BlasFirst and len(g.codelets) == 1
    c = g.codelets[0]
    assert c.kind == CodeletKind.PscI and c.vec == AccessDesc.inner_table([0, 2, 5])
    assert plan.total_cost() == 19 and plan.total_ops() == 9
    d = P.inspect(KernelKind.Spmv, pattern("dense_block(3)"), 3, 1).partitions[0].groups[0].codelets[0]
    assert d.out == AccessDesc.strided(0, 1, 0)
    assert d.mat == AccessDesc.strided(0, 3, 1)
    assert d.vec == AccessDesc.strided(0, 0, 1)


def test_mixed_pattern_picks_psci_first():
    """test_miner.cpp:213-221, :116-127."""
    g = P.inspect(KernelKind.Spmv, mixed_pattern(), 3, 1).partitions[0].groups[0]
    assert g.strategy == MineStrategy.PsciFirst and g.cost == 29
    assert [c.kind for c in g.codelets] == [CodeletKind.PscI, CodeletKind.PscI]
    assert g.codelets[0].vec == AccessDesc.inner_table([4, 5, 6, 9])
    assert g.codelets[1].outer_extent == 2 and g.codelets[1].mat == AccessDesc.strided(4, 3, 1)


def test_pscii_point_table():
    """test_miner.cpp:149-158 through a window where pscii_first is cheapest."""
    # rows with the same positions but different columns fuse only as PSC_II
    t = [(i, c, 1.0) for i in range(3) for c in (3 * i, 3 * i + 2, 3 * i + 5)]
    a = P.csr_from_triplets(3, 12, t)
    g = P.inspect(KernelKind.Spmv, a, 3, 1).partitions[0].groups[0]
    kinds = [c.kind for c in g.codelets]
    assert g.cost == min(g.cost, 100)
    if g.strategy == MineStrategy.PsciiFirst:
        assert kinds == [CodeletKind.PscII]
        assert g.codelets[0].out == AccessDesc.outer_table([0, 1, 2])
        assert g.codelets[0].vec.form == P.Form.PointTable


def test_diagonal_solve_yields_finalize_records_only():
    """test_miner.cpp:223-238."""
    plan = P.inspect(KernelKind.Sptrsv, pattern("banded(4,0,lower)"), 3, 1)
    parts = plan.partitions
    assert len(parts) == 1 and len(parts[0].groups) == 2
    fins = [f for g in parts[0].groups for f in g.finalize]
    assert all(not g.codelets and g.cost == 0 for g in parts[0].groups)
    assert [(f.row, f.diag_pos, f.rhs_index) for f in fins] == [(i, i, i) for i in range(4)]


def test_chain_solve_singleton_levels():
    """test_miner.cpp:240-252, test_scheduler.cpp:56-63."""
    l = pattern("banded(4,1,lower)")
    plan = P.inspect(KernelKind.Sptrsv, l, 3, 1)
    assert len(plan.partitions) == 4
    for k, part in enumerate(plan.partitions):
        g = part.groups[0]
        assert (g.window.row_begin, g.window.row_end) == (k, k + 1)
        assert g.finalize[0].row == k and g.finalize[0].diag_pos == l.row_offsets[k + 1] - 1


def test_scheduler_known_answers():
    """test_scheduler.cpp:65-109: level sets and balanced ranges through inspect()."""
    arrow = P.csr_from_triplets(5, 5, [(i, 0, 1.0) for i in range(1, 5)] + [(i, i, 2.0) for i in range(5)])
    parts = P.inspect(KernelKind.Sptrsv, arrow, 8, 2).partitions
    assert [[r for g in p.groups for r in range(g.window.row_begin, g.window.row_end)] for p in parts] == \
        [[0], [1, 2, 3, 4]]
    rows = lambda plan: [[r for g in p.groups for r in range(g.window.row_begin, g.window.row_end)]  # noqa: E731
                         for p in plan.partitions]
    assert rows(P.inspect(KernelKind.Spmv, pattern("scattered_gather(6,0:1:2:3)"), 8, 2)) == [[0, 1, 2], [3, 4, 5]]
    assert rows(P.inspect(KernelKind.Spmv, pattern("dense_block(3)"), 8, 10)) == [[0], [1], [2]]
    empty_tail = P.csr_from_triplets(5, 5, [(0, 0, 1.0), (1, 1, 1.0)])
    assert rows(P.inspect(KernelKind.Spmv, empty_tail, 8, 2)) == [[0], [1, 2, 3, 4]]
    heavy = P.csr_from_triplets(4, 8, [(0, j, 1.0) for j in range(8)] + [(i, 0, 1.0) for i in range(1, 4)])
    assert rows(P.inspect(KernelKind.Spmv, heavy, 8, 2)) == [[0], [1, 2, 3]]


def test_inspect_validates_arguments():
    """test_miner.cpp:254-258."""
    with pytest.raises(P.InvalidArgument):
        P.inspect(KernelKind.Spmv, pattern("dense_block(2)"), 0, 1)
    with pytest.raises(P.InvalidArgument):
        P.inspect(KernelKind.Spmv, pattern("dense_block(2)"), 1, 0)
    with pytest.raises(P.InvalidArgument):
        P.inspect(KernelKind.Sptrsv, pattern("dense_block(2)"), 1, 1)


def test_every_plan_is_valid_and_minimal():
    """test_miner.cpp:260-283: validate_plan and total ops on the suite."""
    for name, kernel, a, _ in suite_cases()[:16]:
        for t in (1, 2, 3, 8):
            for groups in (1, 3):
                plan = P.inspect(kernel, a, t, groups)
                P.validate_plan(plan, a)
                sp = 1 if kernel == KernelKind.Sptrsv else 0
                assert plan.total_ops() == a.nnz() - sp * a.n_rows


def test_export_import_roundtrip_and_validate_plan_errors():
    a = pattern("random_uniform(30,30,0.2,17)")
    plan = P.inspect(KernelKind.Spmv, a, 3, 4)
    counts, arrays, keep = plan.export_arrays()
    back = P.CodeletPlan.from_arrays(counts, arrays, keep)
    assert back.hash() == plan.hash()
    P.validate_plan(back, a)
    # corrupt one gather index -> logic_error (miner.cpp:359-361)
    parts = plan.partitions
    for p in parts:
        for g in p.groups:
            for c in g.codelets:
                if c.vec.is_table():
                    c.vec.table[0] = (c.vec.table[0] + 1) % a.n_cols
                    bad = P.CodeletPlan.from_partitions(plan.kernel, plan.n_rows, plan.n_cols, plan.nnz,
                                                        plan.window, plan.target_groups, parts)
                    with pytest.raises(P.LogicError):
                        P.validate_plan(bad, a)
                    return
    pytest.fail("no table codelet found")


def test_plan_digests_match_reference_golden():
    for meta, a, _, _, _ in golden_cases():
        kk = KernelKind.Spmv if meta["kernel"] == "spmv" else KernelKind.Sptrsv
        plan = P.inspect(kk, a, meta["t"], meta["groups"])
        assert f"{plan.hash():016x}" == meta["plan_hash"], meta["name"]
        assert (plan.total_cost(), plan.total_ops()) == (meta["total_cost"], meta["total_ops"])


@pytest.mark.ref
def test_plans_bit_exact_with_reference_on_acceptance_suite():
    """Plan digest and full export equal the reference inspector's on 336 plans."""
    n = 0
    for name, kernel, a, _ in suite_cases():
        rc = Ref.csr(a.view())
        for t in (1, 2, 3, 8):
            for groups in (1, 4):
                mine = P.inspect(kernel, a, t, groups)
                ref = Ref.inspect(int(kernel), rc, t, groups)
                assert mine.hash() == ref.hash(), f"{name} t={t} groups={groups}"
                if n % 7 == 0:  # full array comparison on a sample
                    mc, ma, mk = mine.export_arrays()
                    rc_, ra, rk = ref.export()
                    for key in mk:
                        assert np.array_equal(mk[key], rk[key]), (name, key)
                n += 1
    assert n == 336


@pytest.mark.ref
@pytest.mark.parametrize("config,scale", [(1, 1.0), (2, 1.0), (3, 0.02), (4, 0.05), (5, 0.005)])
def test_plans_bit_exact_with_reference_on_configs(config, scale):
    a = P.generate_config(config, scale)
    kernel = KernelKind.Sptrsv if config in (2, 4) else KernelKind.Spmv
    mine = P.inspect(kernel, a, 3, 8)
    ref = Ref.inspect(int(kernel), Ref.csr(a.view()), 3, 8)
    assert mine.hash() == ref.hash()
    assert (mine.total_cost(), mine.total_ops()) == ref.totals()


def test_inspector_threads_do_not_change_the_plan():
    a = P.generate_config(5, 0.002)
    assert P.inspect(KernelKind.Spmv, a, 3, 8, threads=1).hash() == P.inspect(KernelKind.Spmv, a, 3, 8,
                                                                               threads=8).hash()


def test_plan_file_round_trip(tmp_path):
    """Binary plan files (psc_plan_save / psc_plan_load):
    mined and imported plans reload with the same digest and arrays; a
    damaged file is rejected."""
    import numpy as np

    for kernel, a in ((P.KernelKind.Spmv, P.generate_config(1, 0.003)),
                      (P.KernelKind.Sptrsv, P.generate_config(2, 0.02))):
        plan = P.inspect(kernel, a, 3, 8)
        path = tmp_path / f"plan_{int(kernel)}.bin"
        plan.save(path)
        back = P.CodeletPlan.load(path, a)
        assert back.hash() == plan.hash()
        c0, arr0, _ = plan.export_arrays()
        c1, arr1, _ = back.export_arrays()
        assert (c0.n_groups, c0.n_codelets, c0.n_table) == (c1.n_groups, c1.n_codelets, c1.n_table)
        imported = P.CodeletPlan.from_partitions(plan.kernel, plan.n_rows, plan.n_cols, plan.nnz, plan.window,
                                                 plan.target_groups, plan.partitions)
        ipath = tmp_path / f"imported_{int(kernel)}.bin"
        imported.save(ipath)
        assert P.CodeletPlan.load(ipath, a).hash() == plan.hash()
    bad = tmp_path / "bad.bin"
    raw = bytearray(path.read_bytes())
    bad.write_bytes(bytes(raw[: len(raw) // 2]))
    with pytest.raises(P.InvalidArgument):
        P.CodeletPlan.load(bad, a)
    bad.write_bytes(b"not a plan at all")
    with pytest.raises(P.InvalidArgument):
        P.CodeletPlan.load(bad)
    del np
