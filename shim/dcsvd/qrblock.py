"""dcsvd.qrblock (qrblock.py) -> paper_2508_11467_b200.householder."""
from paper_2508_11467_b200.householder import (  # noqa: F401
    CompactWYBlock, QRFactorization, apply_block_reflector_left, apply_block_reflector_right, build_tinv,
    geqrf_blocked, geqrf_panel, orgqr)
