"""B200-native fp64 divide-and-conquer SVD (arxiv 2508.11467), drop-in for
the reference ``dcsvd`` package's SVD path.

Public surface mirrors pkg/src/dcsvd/__init__.py:18-129 for the hot path:
``gesdd`` (alias ``svd``), ``phase_profile``, ``SVDOptions``, ``SVDResult``,
``PhaseProfile``, ``PHASE_NAMES``; ``gebrd_blocked`` (alias
``bidiagonalize``), ``labrd_panel``, ``gebrd_unblocked``,
``BidiagonalFactorization``, ``PanelWorkspace``; ``bdsdc`` (alias ``bdc``),
``BidiagonalProblem``, ``SubproblemSVD``, ``build_z``, ``deflate``,
``DeflationOutcome``, ``merge_vectors``; ``geqrf_blocked``, ``orgqr``,
``QRFactorization``; ``ormqr_like``, ``ormlq_like``, ``ReflectorSequence``,
``column_reflectors``, ``row_reflectors``; ``matmul_accumulate``,
``matvec_accumulate``; ``ConvergenceError``; the harness (``MatrixSpec``,
``generate_matrix``, ``prescribed_singular_values``, ``accuracy``,
``AccuracyReport``, ``read_matrix``, ``write_matrix``, ``cli_main``); plus
``gesdd_batched``.

Every numeric entry point runs hand-written sm_100a CUDA kernels from
``libdcsvd_b200.so`` through ctypes.  There is no CPU fallback.
"""

from ._lib import ConvergenceError, launch_count
from .bidiagonal import (
    BidiagonalFactorization,
    PanelWorkspace,
    gebrd_blocked,
    gebrd_unblocked,
    labrd_panel,
)
from .blas import (
    GivensRotation,
    HouseholderReflector,
    as_dense,
    dense_matrix,
    givens_generate,
    householder_generate,
    matmul_accumulate,
    matvec_accumulate,
    triangular_solve,
)
from .dc import (
    BidiagonalProblem,
    DeflationOutcome,
    build_z,
    deflate,
    merge_vectors,
    SecularRoots,
    SecularSystem,
    SubproblemSVD,
    bdsdc,
    bdsqr_base,
    recompute_z,
    secular_vectors,
    solve_all_roots,
    solve_secular,
    split,
)
from .householder import (
    CompactWYBlock,
    QRFactorization,
    apply_block_reflector_left,
    apply_block_reflector_right,
    build_tinv,
    geqrf_panel,
    ReflectorSequence,
    column_reflectors,
    geqrf_blocked,
    orgqr,
    ormlq_like,
    ormqr_like,
    row_reflectors,
)
from .harness import (
    AccuracyReport,
    MatrixSpec,
    accuracy,
    cli_main,
    generate_matrix,
    prescribed_singular_values,
    read_matrix,
    write_matrix,
)
from .svd import PHASE_NAMES, PhaseProfile, SVDOptions, SVDResult, gesdd, gesdd_batched, phase_profile, svd

bidiagonalize = gebrd_blocked
bdc = bdsdc

__version__ = "0.1.0"

__all__ = [
    "AccuracyReport",
    "MatrixSpec",
    "accuracy",
    "cli_main",
    "generate_matrix",
    "prescribed_singular_values",
    "read_matrix",
    "write_matrix",
    "CompactWYBlock",
    "GivensRotation",
    "HouseholderReflector",
    "SecularRoots",
    "SecularSystem",
    "apply_block_reflector_left",
    "apply_block_reflector_right",
    "bdsqr_base",
    "build_tinv",
    "geqrf_panel",
    "givens_generate",
    "householder_generate",
    "recompute_z",
    "secular_vectors",
    "solve_all_roots",
    "solve_secular",
    "split",
    "triangular_solve",
    "BidiagonalFactorization",
    "BidiagonalProblem",
    "DeflationOutcome",
    "build_z",
    "deflate",
    "merge_vectors",
    "ConvergenceError",
    "PHASE_NAMES",
    "PanelWorkspace",
    "PhaseProfile",
    "QRFactorization",
    "ReflectorSequence",
    "SVDOptions",
    "SVDResult",
    "SubproblemSVD",
    "as_dense",
    "bdc",
    "bdsdc",
    "bidiagonalize",
    "column_reflectors",
    "dense_matrix",
    "gebrd_blocked",
    "gebrd_unblocked",
    "geqrf_blocked",
    "gesdd",
    "gesdd_batched",
    "labrd_panel",
    "launch_count",
    "matmul_accumulate",
    "matvec_accumulate",
    "orgqr",
    "ormlq_like",
    "ormqr_like",
    "phase_profile",
    "row_reflectors",
    "svd",
]
