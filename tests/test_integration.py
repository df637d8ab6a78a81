"""Drop-in integration (tests/cpp/integration_main.cpp): code written against
the reference library -- its inspector, matrices, plans and executor calls --
switches to include/psc_b200.hpp and gets the reference executor's results
bitwise on the GPU. The binary links the unmodified reference objects, so it
is built where /root/reference exists (oracle/Makefile `integration`)."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "oracle", "_ref", "integration_test")


@pytest.mark.gpu
def test_reference_code_switches_executor():
    if not os.path.exists(BIN):
        pytest.skip("integration binary not built (needs /root/reference at build time)")
    out = subprocess.run([BIN], capture_output=True, text=True, timeout=600)
    print(out.stdout)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "[FAIL]" not in out.stdout


@pytest.mark.gpu
def test_reference_executor_unit_tests_on_the_gpu():
    """The reference's own tests/test_executor.cpp (17 cases: exec_*_codelet
    known answers and shape errors, planned multiply / solve vs the baselines,
    bitwise across worker counts, zero-fill, size and kernel errors,
    execute_plan(plan, ctx, workers)), compiled where it lies against
    tests/cpp/shim/psc/executor.hpp -- the reference's executor header
    re-implemented over include/psc_b200.hpp -- so every executor call runs on
    this library (oracle/Makefile `reftests`)."""
    binary = os.path.join(ROOT, "oracle", "_ref", "ref_test_executor")
    if not os.path.exists(binary):
        pytest.skip("reference unit-test binary not built (needs /root/reference at build time)")
    out = subprocess.run([binary], capture_output=True, text=True, timeout=600)
    print(out.stdout)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "test cases: 17 | 17 passed | 0 failed" in out.stdout, out.stdout


def test_wrapper_header_compiles_standalone():
    """include/psc_b200.hpp compiles with only the C ABI header (no reference)."""
    src = '#include "psc_b200.hpp"\nint main() { return 0; }\n'
    r = subprocess.run(["g++", "-std=c++20", "-fsyntax-only", "-I", os.path.join(ROOT, "include"), "-x", "c++", "-"],
                       input=src, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
