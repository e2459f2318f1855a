"""dcsvd.backtransform (backtransform.py) -> paper_2508_11467_b200.householder."""
from paper_2508_11467_b200.householder import (  # noqa: F401
    ReflectorSequence, column_reflectors, ormlq_like, ormqr_like, row_reflectors)
