"""Shared pytest configuration.

`-m gpu` tests need a B200 and call the product through its C-ABI;
everything else runs on the CPU (oracle vs golden fixtures, host logic,
library symbol checks, gloo multi-process tests).
"""

import sys
from pathlib import Path

REPO = Path(__file__).resolve().parents[1]
if str(REPO) not in sys.path:
    sys.path.insert(0, str(REPO))
TESTS = Path(__file__).resolve().parent
if str(TESTS) not in sys.path:
    sys.path.insert(0, str(TESTS))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
