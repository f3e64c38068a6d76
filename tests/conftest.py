import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA GPU (B200, sm_100a); run with -m gpu")
    config.addinivalue_line("markers", "slow: long-running CPU test")
    # the suites load libfz.so / liboracle.so: (re)build them when missing or older than their sources
    # (nvcc cross-compiles sm_100a without a GPU; a no-op when both are up to date)
    import __graft_entry__

    __graft_entry__.build()


def read_golden_csv(name):
    rows = []
    with open(os.path.join(GOLDEN, name)) as f:
        header = None
        for line in f:
            line = line.strip()
            if not line or line.startswith("#"):
                continue
            parts = line.split(",")
            if header is None:
                header = parts
                continue
            rows.append(dict(zip(header, parts)))
    return rows


def parse_gens(s):
    return tuple(int(x) for x in s.split(";"))


@pytest.fixture(scope="session")
def corc():
    from oracle import oracle

    return oracle.C()
