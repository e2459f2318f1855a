"""dcsvd.driver (driver.py) -> paper_2508_11467_b200.svd."""
from paper_2508_11467_b200.svd import (  # noqa: F401
    PHASE_NAMES, PhaseProfile, SVDOptions, SVDResult, gesdd, phase_profile)
