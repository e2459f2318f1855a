"""Reference singular values for the full-size BASELINE configs C2, C3, C5.

Runs the REAL reference (/root/reference, dcsvd 0.1.0) values-only
(``SVDOptions(want_vectors=False)``; its sigma is bitwise equal to the
vector-mode sigma, ``bdc.py:14-21`` / ``test_driver.py:57-64``) on the exact
input bytes of each config -- ``generate_matrix(MatrixSpec(...))``
(``harness.py:131-147``), which the GPU regenerates bit-identically with its
Philox port -- and stores sigma as small fixtures that the ``-m gpu`` tests
and ``bench.py`` compare against (the GPU box has no /root/reference).

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_large_sigma.py c5 c3 c2

Outputs: ``c2_sigma.npz`` (8192^2, seed 2), ``c3_sigma.npz`` (65536x1024,
seed 3), ``c5_sigma.npz`` (2048^2, seeds 1000..1000+C5_COUNT-1).
"""

import os
import sys
import time
from concurrent.futures import ProcessPoolExecutor

HERE = os.path.dirname(os.path.abspath(__file__))
C5_COUNT = 64


def _ref():
    sys.path.insert(0, "/root/reference/pkg/src")
    import dcsvd
    return dcsvd


def _sigma(kind, m, n, seed):
    import numpy as np
    dcsvd = _ref()
    a = dcsvd.generate_matrix(dcsvd.MatrixSpec(kind, m, n, seed=seed))
    t0 = time.perf_counter()
    r = dcsvd.gesdd(a, dcsvd.SVDOptions(want_vectors=False))
    return np.asarray(r.sigma), time.perf_counter() - t0


def _c5_item(i):
    os.environ["OPENBLAS_NUM_THREADS"] = "1"
    return _sigma("random", 2048, 2048, 1000 + i)


def main(which):
    import numpy as np
    if "c5" in which:
        # one BLAS thread per process, one process per core (SURVEY 8d CPU plan)
        with ProcessPoolExecutor(max_workers=os.cpu_count(),
                                 initializer=os.environ.__setitem__,
                                 initargs=("OPENBLAS_NUM_THREADS", "1")) as ex:
            res = list(ex.map(_c5_item, range(C5_COUNT)))
        sig = np.stack([r[0] for r in res])
        secs = np.array([r[1] for r in res])
        np.savez_compressed(os.path.join(HERE, "c5_sigma.npz"), sigma=sig,
                            seeds=np.arange(1000, 1000 + C5_COUNT), seconds=secs)
        print(f"C5 {C5_COUNT} x 2048^2 values-only: {secs.mean():.2f} s each (1 thread)")
    for tag, (m, n, seed) in (("c3", (65536, 1024, 3)), ("c2", (8192, 8192, 2))):
        if tag not in which:
            continue
        sig, t = _sigma("random", m, n, seed)
        np.savez_compressed(os.path.join(HERE, f"{tag}_sigma.npz"), sigma=sig,
                            spec=np.array([m, n, seed]), seconds=np.array(t),
                            threads=np.array(os.cpu_count()))
        print(f"{tag.upper()} {m}x{n} seed {seed} values-only: {t:.1f} s")


if __name__ == "__main__":
    main(set(sys.argv[1:]) or {"c2", "c3", "c5"})
