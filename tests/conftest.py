import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs through the CUDA C-ABI)")


def pytest_sessionstart(session):
    """Build libpoetx_b200.so if it is missing or older than its sources (a
    content hash of csrc/ + the header, so a stale build whose struct layout
    no longer matches is never tested; nvcc cross-compiles for sm_100a
    without a GPU).  _native.lib() also checks the ABI version on load."""
    from paper_2603_05500_b200.build import build

    build()
