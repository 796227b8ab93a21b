import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

# GPU parity runs start from a poisoned arena (0xFF = NaN in bf16/fp32): a
# read of a page this run has not yet written cannot pass by finding the same
# bytes an earlier run of the same job left there (salus.Context poison)
os.environ.setdefault("SALUS_POISON", "1")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) and the built CUDA library")
    config.addinivalue_line("markers", "slow: long-running CPU test")
