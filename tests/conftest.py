import os
import sys

import pytest

# The reference pins BLAS to one thread (pkg/tests/conftest.py:10-16) and the
# golden vectors were generated that way; multi-threaded OpenBLAS changes low
# bits of GEMM results, so the oracle is compared bitwise only single-threaded.
for _v in ("OPENBLAS_NUM_THREADS", "OMP_NUM_THREADS", "MKL_NUM_THREADS"):
    os.environ.setdefault(_v, "1")
try:
    from threadpoolctl import threadpool_limits

    _BLAS_LIMIT = threadpool_limits(1)
except Exception:  # pragma: no cover
    _BLAS_LIMIT = None

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (run with -m gpu)")
    config.addinivalue_line("markers", "slow: large-size parity runs")


@pytest.fixture(scope="session")
def golden():
    import numpy as np

    return np.load(os.path.join(GOLDEN, "golden.npz"), allow_pickle=False)


@pytest.fixture(scope="session")
def cuda():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch.device("cuda", 0)
