"""Seeded synthetic test problems (numpy, deterministic).  Shapes and spectra
follow BASELINE.json's recipes at sizes the CPU oracle finishes in seconds."""
from __future__ import annotations

import numpy as np


def c2_like_sigma(r, k, p):
    """sigma_1..k = 1, sigma_{k+1..p} linear 0.99 -> 0.90, tail 0.8/(i-p)."""
    top = np.ones(k)
    mid = np.linspace(0.99, 0.90, p - k)
    tail = 0.8 / np.arange(1, r - p + 1)
    return np.concatenate([top, mid, tail])[:r]


def planted_dense(d, n, k=3, p=6, seed=0, sigma=None, noise=0.0):
    """X = U diag(sigma) V^T (+ noise * G / sqrt(n)), U, V Haar-orthonormal (QR of
    Gaussians); returns X (d x n), U (d x r) and sigma."""
    rng = np.random.default_rng(seed)
    r = min(d, n)
    sig = c2_like_sigma(r, k, p) if sigma is None else np.asarray(sigma, dtype=np.float64)
    r = len(sig)
    U, _ = np.linalg.qr(rng.standard_normal((d, r)))
    V, _ = np.linalg.qr(rng.standard_normal((n, r)))
    X = (U * sig) @ V.T
    if noise:
        X = X + noise * rng.standard_normal((d, n)) / np.sqrt(n)
    return X, U, sig


def random_csc(d, n, nnz_per_col, seed=0, rank=4):
    """CSC with `nnz_per_col` distinct sorted random rows per column; values =
    rank-`rank` u_i v_j signal on the pattern + N(0, 0.1^2)."""
    rng = np.random.default_rng(seed)
    u = rng.standard_normal((d, rank))
    v = rng.standard_normal((n, rank))
    colptr = np.arange(n + 1, dtype=np.int64) * nnz_per_col
    rows = np.empty(n * nnz_per_col, np.int32)
    vals = np.empty(n * nnz_per_col)
    for j in range(n):
        rr = np.sort(rng.choice(d, nnz_per_col, replace=False))
        rows[j * nnz_per_col:(j + 1) * nnz_per_col] = rr
        vals[j * nnz_per_col:(j + 1) * nnz_per_col] = u[rr] @ v[j] / np.sqrt(rank * n) + 0.1 * rng.standard_normal(
            nnz_per_col) / np.sqrt(n)
    return colptr, rows, vals


def csc_to_dense(d, n, colptr, rows, vals):
    X = np.zeros((d, n))
    for j in range(n):
        sl = slice(colptr[j], colptr[j + 1])
        X[rows[sl], j] = vals[sl]
    return X
