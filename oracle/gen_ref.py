"""Input generators and accuracy metrics, restating
pkg/src/dcsvd/harness.py:69-187.  TEST INFRASTRUCTURE ONLY.

The word stream is numpy's Philox-4x64-10 keyed by the seed
(harness.py:72-74); word -> uniform ((w >> 11) + 0.5) * 2^-53
(harness.py:76-78); Box-Muller normals (harness.py:80-88).
"""

import numpy as np


class WordStream:
    def __init__(self, seed):
        self.bits = np.random.Philox(key=seed)

    def uniforms(self, count):
        w = self.bits.random_raw(count)
        return ((w >> np.uint64(11)).astype(np.float64) + 0.5) * 2.0 ** -53

    def normals(self, count):
        k = (count + 1) // 2
        u = self.uniforms(2 * k)
        rad = np.sqrt(-2.0 * np.log(u[0::2]))
        ang = 2.0 * np.pi * u[1::2]
        out = np.empty(2 * k)
        out[0::2] = rad * np.cos(ang)
        out[1::2] = rad * np.sin(ang)
        return out[:count]


def philox_uniforms(seed, count):
    return WordStream(seed).uniforms(count)


def philox_normals(seed, count):
    return WordStream(seed).normals(count)


def _spectrum(kind, n, cond, ws):
    # harness.py:91-105
    i = np.arange(n, dtype=np.float64)
    if kind == "logrand":
        return np.sort(np.exp(-np.log(cond) * ws.uniforms(n)))[::-1].copy()
    if kind == "arith":
        return np.ones(1) if n == 1 else 1.0 - (i / (n - 1)) * (1.0 - 1.0 / cond)
    if kind == "geo":
        return np.ones(1) if n == 1 else cond ** (-i / (n - 1))
    raise ValueError(kind)


def _haar(ws, rows, cols):
    # harness.py:117-128 (Q of the blocked QR with diag(R) signs absorbed)
    from .dense_ref import geqrf, orgqr

    g = np.asfortranarray(ws.normals(rows * cols).reshape((rows, cols), order="F"))
    tau = geqrf(g, 32)
    q = orgqr(g, tau, cols)
    flip = np.diag(g)[:cols] < 0.0
    q[:, flip] = -q[:, flip]
    return q


def make_matrix(kind, m, n, cond=1.0e6, seed=0):
    """generate_matrix(MatrixSpec(kind, m, n, cond, seed)) (harness.py:131-147)."""
    ws = WordStream(seed)
    if kind == "random":
        return np.asfortranarray(ws.uniforms(m * n).reshape((m, n), order="F"))
    k = min(m, n)
    s = _spectrum(kind, k, cond, ws)
    u = _haar(ws, m, k)
    v = _haar(ws, n, k)
    return np.asfortranarray((u * s) @ v.T)


def accuracy_metrics(a, sigma, u=None, vt=None, ref_sigma=None):
    """Reference metrics (harness.py:150-187) plus the north-star scaled
    checks: sigma_rel = max|s - s_ref| / s_max, resid = ||A - U S Vt||_F /
    (||A||_F n), orth_u/orth_v = ||U^T U - I||_F / n."""
    out = {}
    k = sigma.size
    n = max(a.shape[1], 1) if a is not None else max(k, 1)
    if ref_sigma is not None:
        ref = np.asarray(ref_sigma)
        out["e_sigma"] = float(np.linalg.norm(sigma - ref) / ref.size)
        smax = max(float(np.max(np.abs(ref))), np.finfo(float).tiny)
        out["sigma_rel"] = float(np.max(np.abs(sigma - ref)) / smax)
    if u is not None and vt is not None:
        r = np.linalg.norm(a - (u * sigma) @ vt)
        na = np.linalg.norm(a)
        out["e_svd"] = float(r / na) if na > 0 else float(r)
        out["orth_u"] = float(np.linalg.norm(u.T @ u - np.eye(k)))
        out["orth_v"] = float(np.linalg.norm(vt @ vt.T - np.eye(k)))
        out["resid_scaled"] = out["e_svd"] / n
        out["orth_u_scaled"] = out["orth_u"] / n
        out["orth_v_scaled"] = out["orth_v"] / n
    return out
