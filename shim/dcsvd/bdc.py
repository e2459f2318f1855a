"""dcsvd.bdc (bdc.py) -> paper_2508_11467_b200.dc."""
from paper_2508_11467_b200.dc import (  # noqa: F401
    BidiagonalProblem, DeflationOutcome, SecularRoots, SecularSystem, SubproblemSVD, bdsdc, bdsqr_base, build_z,
    deflate, merge_vectors, recompute_z, secular_vectors, solve_all_roots, solve_secular, split)
