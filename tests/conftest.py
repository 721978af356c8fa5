import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
for _p in (ROOT, os.path.join(ROOT, "tests")):
    if _p not in sys.path:
        sys.path.insert(0, _p)

# A fresh checkout has no libscl.so (git-ignored); build it before any test
# module imports the package (nvcc cross-compiles for sm_100a without a GPU).
if not os.path.exists(os.path.join(ROOT, "paper_2212_07597_b200", "libscl.so")):
    import __graft_entry__
    __graft_entry__.build()


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (CUDA device) -- parity tests through the C-ABI")
    config.addinivalue_line("markers", "slow: long-running CPU test")


@pytest.fixture(scope="session", autouse=True)
def _built_cpu_libs():
    """Compile the oracle (plain C) and the trace generator once per session."""
    import oracle
    import tracegen
    oracle.build()
    tracegen.build()
    yield
