"""End-to-end oracle driver (pkg/src/dcsvd/driver.py:97-170).
TEST INFRASTRUCTURE ONLY (see oracle/__init__.py)."""

import time

import numpy as np

from .dc_ref import Bidiag, bdc
from .dense_ref import apply_u1, apply_v1t, gebrd, geqrf, orgqr

PHASES = ("geqrf", "orgqr", "gebrd", "bdcdc", "ormqr+ormlq", "gemm")


class _Clock:
    def __init__(self, on):
        self.t = {p: 0.0 for p in PHASES} if on else None

    def run(self, name, fn, *args, **kw):
        if self.t is None:
            return fn(*args, **kw)
        t0 = time.perf_counter()
        try:
            return fn(*args, **kw)
        finally:
            self.t[name] += time.perf_counter() - t0


def _core(a, o, clk):
    # driver.py:97-118
    m, n = a.shape
    d, e, tq, tp = clk.run("gebrd", gebrd, a, o["bidiag_block"])
    node = clk.run("bdcdc", bdc, Bidiag(d, e, False), o["want_vectors"], o["leaf_size"], o["deflation_multiple"])
    if not o["want_vectors"]:
        return node.vals, None, None

    def back():
        u = np.zeros((m, n), order="F")
        u[:n, :] = node.W
        apply_u1(a, tq, u, o["apply_block"], trans=False)
        vt = np.asfortranarray(node.Q.T)
        apply_v1t(a, tp, vt, o["apply_block"], trans=True)
        return u, vt

    u, vt = clk.run("ormqr+ormlq", back)
    return node.vals, u, vt


def _svd(a, o, clk):
    # driver.py:121-144
    m, n = a.shape
    if m < 1 or n < 1:
        raise ValueError("empty matrix")
    if m < n:
        s, u, vt = _svd(np.asfortranarray(a.T), o, clk)
        return s, (None if vt is None else np.asfortranarray(vt.T)), (None if u is None else np.asfortranarray(u.T))
    if m > n and m >= o["ts_crossover"] * n:
        tau = clk.run("geqrf", geqrf, a, o["qr_block"])
        r = np.asfortranarray(np.triu(a[:n, :]))
        s, u0, vt = _core(r, o, clk)
        if not o["want_vectors"]:
            return s, None, None
        q = clk.run("orgqr", orgqr, a, tau, n, o["orgqr_block"])
        u = clk.run("gemm", lambda: np.asfortranarray(q @ u0))
        return s, u, vt
    return _core(a, o, clk)


DEFAULTS = dict(want_vectors=True, bidiag_block=32, qr_block=32, orgqr_block=64,
                apply_block=64, leaf_size=32, ts_crossover=5.0 / 3.0, deflation_multiple=8.0)


def svd(a, **opts):
    """Economy SVD (sigma descending, U m x k, Vt k x n); input untouched."""
    o = dict(DEFAULTS, **opts)
    a = np.array(a, dtype=np.float64, order="F", copy=True)
    return _svd(a, o, _Clock(False))


def phase_times(a, **opts):
    """(list of (phase, seconds), total) like driver.phase_profile."""
    o = dict(DEFAULTS, **opts)
    a = np.array(a, dtype=np.float64, order="F", copy=True)
    clk = _Clock(True)
    t0 = time.perf_counter()
    _svd(a, o, clk)
    return [(p, clk.t[p]) for p in PHASES], time.perf_counter() - t0
