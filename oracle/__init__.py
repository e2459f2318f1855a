"""CPU oracle for the fp64 divide-and-conquer SVD path.

TEST INFRASTRUCTURE ONLY.  This package is a numpy restatement of the
reference algorithm (arxiv 2508.11467 / the ``dcsvd`` package under
/root/reference/pkg/src/dcsvd) written for this repository: every function
cites the reference file:line it follows.  Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import it, and only as the checker or the timed
CPU baseline.  The product path (``paper_2508_11467_b200``) never imports it
and fails loudly when the CUDA library is missing.

Parity is pinned by ``tests/golden/`` fixtures produced by running the real
reference in the build container (``tests/golden/make_golden.py``) and checked
by ``tests/test_oracle.py``.
"""

from .dense_ref import (  # noqa: F401
    larfg,
    lartg,
    gebd2,
    labrd,
    gebrd,
    geqr2,
    geqrf,
    orgqr,
    cwy_y,
    cwy_tinv,
    cwy_apply_left,
    cwy_apply_right,
    apply_u1,
    apply_v1t,
)
from .dc_ref import (  # noqa: F401
    Bidiag,
    NodeSVD,
    leaf_svd,
    split_rows,
    merge_inputs,
    deflate_entries,
    secular_roots,
    loewner_z,
    secular_vecs,
    bdc,
)
from .svd_ref import svd, phase_times, PHASES  # noqa: F401
from .gen_ref import philox_uniforms, philox_normals, make_matrix, accuracy_metrics  # noqa: F401
