"""dcsvd.densecore (densecore.py) -> paper_2508_11467_b200.blas / _lib."""
from paper_2508_11467_b200._lib import ConvergenceError  # noqa: F401
from paper_2508_11467_b200.blas import *  # noqa: F401,F403
from paper_2508_11467_b200.blas import (  # noqa: F401
    GivensRotation, HouseholderReflector, as_dense, dense_matrix, givens_generate, householder_generate,
    matmul_accumulate, matvec_accumulate, triangular_solve)
