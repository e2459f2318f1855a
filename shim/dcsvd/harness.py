"""dcsvd.harness (harness.py) -> paper_2508_11467_b200.harness."""
from paper_2508_11467_b200.harness import (  # noqa: F401
    EPS, KINDS, AccuracyReport, MatrixSpec, accuracy, cli_main, generate_matrix, main, prescribed_singular_values,
    read_matrix, write_matrix, _Stream)
