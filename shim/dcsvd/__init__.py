"""`dcsvd` shim: the reference package's module layout
(pkg/src/dcsvd/__init__.py and its submodules) mapped onto the GPU engine, so
unchanged `import dcsvd` code -- including the reference's own test-suite --
runs on the B200.  Put ``shim/`` first on ``sys.path``."""

import os as _os
import sys as _sys

_sys.path.insert(0, _os.path.dirname(_os.path.dirname(_os.path.dirname(_os.path.abspath(__file__)))))

from paper_2508_11467_b200 import *  # noqa: F401,F403,E402
from paper_2508_11467_b200 import __all__ as _all  # noqa: E402
from paper_2508_11467_b200 import __version__  # noqa: F401,E402

from . import backtransform, bdc, bidiag, densecore, driver, harness, qrblock  # noqa: F401,E402

__all__ = list(_all)
