import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs through the CUDA C-ABI)")


def pytest_sessionstart(session):
    """Build libpoetx_b200.so once if it is missing (nvcc cross-compiles for
    sm_100a without a GPU); an existing build is used as is."""
    so = os.path.join(ROOT, "paper_2603_05500_b200", "libpoetx_b200.so")
    if not os.path.exists(so):
        from paper_2603_05500_b200.build import build

        build(force=True)
