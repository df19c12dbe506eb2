"""BLAS-order probe: the LoD kernels reproduce numpy's
float paths bit for bit by hard-coding the FMA chains OpenBLAS takes for the
reference's BLAS-backed calls.  This probe asserts that the host numpy takes
exactly those paths, so a GPU-vs-reference bit-exactness claim made on this
host is sound:

  * `np.linalg.norm(v)` of a 3-vector (d_root, hspt.py:150; spt.py:82) is the
    ddot chain  sqrt(fma(z, z, fma(y, y, x·x)))          — lod.cu droot
  * `np.linalg.norm(a, axis=1)` (hierarchy.py:259, hspt.py:139, spt.py:54)
    is the plain  sqrt((x² + y²) + z²)                     — lod.cu dist
  * `c @ P[:, :3].T + P[:, 3]` (core.py:370): dgemm for ≥ 2 rows
    fma(c2, p2, fma(c1, p1, c0·p0)), dgemv for 1 row
    fma(c2, p2, fma(c0, p0, c1·p1)), then + d              — lod.cu sphere_in_frustum
  * `(μ − p) @ Wᵀ` (renderer.py:83) for ≥ 2 rows: the dgemm chain  — raster.cu t

The same check runs in the CPU suite and (marked gpu) inside GPUTEST on the
B200 host, whose numpy/OpenBLAS build is what the GPU parity tests compare
against.  Exact FMA is evaluated in rational arithmetic (Fraction → float
is correctly rounded)."""
from __future__ import annotations

import math
import platform
from fractions import Fraction

import numpy as np
import pytest


def fma(a, b, c):
    return float(Fraction(float(a)) * Fraction(float(b)) + Fraction(float(c)))


def _vectors(rng, n):
    mag = 10.0 ** rng.uniform(-3, 4, (n, 1))
    return rng.normal(size=(n, 3)) * mag


def probe(seed=0, n=3000):
    rng = np.random.default_rng(seed)
    bad = {}
    # 1-D norm: ddot chain
    v = _vectors(rng, n)
    for x, y, z in v:
        got = float(np.linalg.norm(np.array([x, y, z])))
        want = math.sqrt(fma(z, z, fma(y, y, x * x)))
        if got != want:
            bad["norm_1d"] = bad.get("norm_1d", 0) + 1
    # axis=1 norm: plain, several batch sizes
    for m in (1, 2, 3, 7, 64, 1000):
        a = _vectors(rng, m)
        got = np.linalg.norm(a, axis=1)
        want = np.sqrt((a[:, 0] * a[:, 0] + a[:, 1] * a[:, 1]) + a[:, 2] * a[:, 2])
        if not np.array_equal(got, want):
            bad["norm_axis1"] = bad.get("norm_axis1", 0) + int(np.sum(got != want))
    # frustum matmul, n = 1..64 rows
    for m in list(range(1, 65)) + [257]:
        P = rng.normal(size=(6, 4))
        c = _vectors(rng, m)
        got = c @ P[:, :3].T + P[:, 3]
        for i in range(m):
            for k in range(6):
                p0, p1, p2, d = P[k]
                c0, c1, c2 = c[i]
                s = fma(c2, p2, fma(c0, p0, c1 * p1)) if m == 1 else fma(c2, p2, fma(c1, p1, c0 * p0))
                if got[i, k] != s + d:
                    key = "frustum_gemv" if m == 1 else "frustum_gemm"
                    bad[key] = bad.get(key, 0) + 1
    # render depth/camera transform, ≥ 2 rows (dgemm with a 3×3 operand)
    for m in (2, 5, 64, 4096):
        W = np.linalg.qr(rng.normal(size=(3, 3)))[0]
        mu = _vectors(rng, m)
        got = mu @ W.T
        for i in range(0, m, max(1, m // 200)):
            for k in range(3):
                s = fma(mu[i, 2], W[k, 2], fma(mu[i, 1], W[k, 1], mu[i, 0] * W[k, 0]))
                if got[i, k] != s:
                    bad["camera_gemm"] = bad.get("camera_gemm", 0) + 1
    return bad


def _config():
    try:
        cfg = np.show_config(mode="dicts")
        blas = cfg.get("Build Dependencies", {}).get("blas", {})
        return f"{blas.get('name')} {blas.get('version')} on {platform.processor() or platform.machine()}"
    except Exception:        # pragma: no cover - informational only
        return "unknown"


def test_blas_order_probe():
    bad = probe()
    assert not bad, f"host numpy/BLAS float paths differ from the ones the kernels hard-code: {bad} ({_config()})"


@pytest.mark.gpu
def test_blas_order_probe_on_gpu_host():
    """The same probe inside GPUTEST (the B200 host's numpy)."""
    bad = probe(seed=1)
    assert not bad, f"B200 host BLAS paths differ: {bad} ({_config()})"
