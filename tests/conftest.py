import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (sm_100a) device")
    config.addinivalue_line("markers", "slow: long-running (full-size configs)")
    # the library is built in-tree (nvcc cross-compiles without a GPU) before any test module imports
    # the package; _build.py is loaded by path because the package import needs the library.
    import importlib.util
    spec = importlib.util.spec_from_file_location("_srmra_build",
                                                  os.path.join(ROOT, "paper_2204_04754_b200", "_build.py"))
    b = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(b)
    b.build()


@pytest.fixture(scope="session")
def oracle_mod():
    import oracle
    oracle.build()
    return oracle
