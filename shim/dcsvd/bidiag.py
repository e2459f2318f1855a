"""dcsvd.bidiag (bidiag.py) -> paper_2508_11467_b200.bidiagonal."""
from paper_2508_11467_b200.bidiagonal import (  # noqa: F401
    BidiagonalFactorization, PanelWorkspace, gebrd_blocked, gebrd_unblocked, labrd_panel)
