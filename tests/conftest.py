import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

_LIB = os.path.join(ROOT, "paper_2111_12243_b200", "libpsc_b200.so")
_ORACLE = os.path.join(ROOT, "oracle", "build", "liboracle.so")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA GPU (B200, sm_100a)")
    config.addinivalue_line("markers", "ref: needs the reference library oracle/_ref/libpsc_ref.so")
    # Build in-tree artefacts once if they are missing (nvcc/gcc are in the image).
    if not os.path.exists(_LIB):
        subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "paper_2111_12243_b200", "csrc"), "-j8"], check=True)
    if not os.path.exists(_ORACLE):
        subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "oracle"), "oracle"], check=True)


def _has_gpu():
    try:
        import paper_2111_12243_b200 as P

        return P.device_count() > 0
    except Exception:
        return False


def pytest_collection_modifyitems(config, items):
    from oracle.oracle import Ref

    gpu = _has_gpu()
    ref = Ref.available()
    for item in items:
        if "gpu" in item.keywords and not gpu:
            item.add_marker(pytest.mark.skip(reason="no CUDA device"))
        if "ref" in item.keywords and not ref:
            item.add_marker(pytest.mark.skip(reason="reference library not built"))


@pytest.fixture(scope="session")
def exe():
    import paper_2111_12243_b200 as P

    e = P.Executor(1, 0)
    yield e
    e.close()
