"""BASELINE.json's five configurations as seeded synthetic generators.

Dense configs are planted on the device with torch (fp64): U, V are seeded
Gaussian matrices orthonormalised by QR (BASELINE.json governs over SPEC.md's
Householder recipe), X = U diag(sigma) V^T
(+ 1e-3 G / sqrt(n)).  X is produced column-major (as the (n, d) row-major
tensor X^T) so it is borrowed by the C ABI with no copy.  torch is plumbing
here (data generation / verification), never the measured path.

Unspecified items are pinned: C2/C3 seed 2, C5 seed 5,
eps = 1e-8 for C2-C5; C4 values = rank-32 signal u_i v_j / sqrt(32) on the
pattern + N(0, 0.01^2) noise.
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np


@dataclass
class ConfigSpec:
    name: str
    d: int
    n: int
    k: int
    p: int
    eps: float
    seed: int
    rank: int
    noise: float
    sparse: bool = False
    nnz_per_col: int = 0

    def sigma(self) -> np.ndarray:
        i = np.arange(1, self.rank + 1, dtype=np.float64)
        if self.name == "C1":
            s = np.where(i <= 5, 1 - 0.01 * (i - 1), 0.0)
            s5 = 1 - 0.01 * 4
            s = np.where((i > 5) & (i <= 10), s5 - 0.001 * (i - 5), s)
            return np.where(i > 10, 0.5 * i ** -0.5, s)
        if self.name == "C2":
            return np.where(i <= 10, 1.0, np.where(i <= 20, 0.99 - (i - 11) * (0.09 / 9), 0.8 / np.maximum(i - 20, 1)))
        if self.name == "C3":
            s = np.where(i <= 16, 1.0 - (i - 1) * (0.05 / 15), 0.0)
            s = np.where((i > 16) & (i <= 32), 0.949 - (i - 17) * (0.009 / 15), s)
            return np.where(i > 32, 0.9 * np.exp(-0.05 * (i - 32)), s)
        if self.name == "C5":
            s = np.where(i <= 32, 1 - 0.002 * (i - 1), 0.0)
            s32 = 1 - 0.002 * 31
            s = np.where((i > 32) & (i <= 64), s32 - 0.0005 * (i - 32), s)
            return np.where(i > 64, 0.7 * np.maximum(i - 64, 1) ** -0.5, s)
        raise ValueError(self.name)

    def eig(self) -> np.ndarray:
        return self.sigma() ** 2

    def delta(self) -> float:
        """Gap budget: 2/3 (lambda_k - lambda_{p+1}) satisfies Delta <= gap <= 2 Delta."""
        lam = self.eig()
        return 2.0 / 3.0 * (lam[self.k - 1] - lam[self.p])

    def mu(self) -> float:
        lam = self.eig()
        tot = lam.sum() + (self.noise ** 2) * self.d
        return math.sqrt(tot / max(tot - lam[: self.k].sum(), 1e-300))


CONFIGS = {
    "C1": ConfigSpec("C1", 1000, 5000, 5, 10, 1e-6, 0, 1000, 0.0),
    "C2": ConfigSpec("C2", 4096, 100_000, 10, 20, 1e-8, 2, 256, 1e-3),
    "C3": ConfigSpec("C3", 2048, 200_000, 16, 32, 1e-8, 2, 128, 1e-3),
    "C4": ConfigSpec("C4", 50_000, 2_000_000, 8, 16, 1e-8, 3, 32, 0.01, sparse=True, nnz_per_col=20),
    "C5": ConfigSpec("C5", 8192, 1_000_000, 32, 64, 1e-8, 5, 512, 1e-3),
}


def make_dense_xt(spec: ConfigSpec, device="cuda", chunk_cols=16384):
    """Return (XT, U) with XT = X^T as a contiguous (n, d) float64 tensor."""
    import torch

    g = torch.Generator(device=device)
    g.manual_seed(spec.seed)
    f64 = torch.float64
    r = spec.rank
    U, _ = torch.linalg.qr(torch.randn(spec.d, r, generator=g, dtype=f64, device=device))
    V, _ = torch.linalg.qr(torch.randn(spec.n, r, generator=g, dtype=f64, device=device))
    sig = torch.tensor(spec.sigma(), dtype=f64, device=device)
    US = U * sig
    XT = torch.empty(spec.n, spec.d, dtype=f64, device=device)
    scale = spec.noise / math.sqrt(spec.n)
    for j0 in range(0, spec.n, chunk_cols):
        j1 = min(spec.n, j0 + chunk_cols)
        blk = V[j0:j1] @ US.T
        if spec.noise:
            blk.add_(torch.randn(j1 - j0, spec.d, generator=g, dtype=f64, device=device), alpha=scale)
        XT[j0:j1] = blk
    del V
    return XT, U


def make_sparse_csc(spec: ConfigSpec, seed_offset=0, n=None, d=None):
    """C4-style CSC (numpy): 20 distinct sorted uniform rows per column; values
    = rank-32 signal sum_l u_{i,l} v_{j,l} / sqrt(32) + N(0, noise^2).
    Vectorised: draw rows with replacement, redraw the duplicate positions of
    each sorted column until every column is distinct."""
    n = n or spec.n
    d = d or spec.d
    rng = np.random.default_rng(spec.seed + seed_offset)
    z = spec.nnz_per_col
    rows = np.sort(rng.integers(0, d, size=(n, z), dtype=np.int64), axis=1)
    while True:
        dup = np.zeros_like(rows, dtype=bool)
        dup[:, 1:] = rows[:, 1:] == rows[:, :-1]
        k = int(dup.sum())
        if k == 0:
            break
        rows[dup] = rng.integers(0, d, size=k, dtype=np.int64)
        rows.sort(axis=1)
    out = rows.astype(np.int32)
    U = rng.standard_normal((d, 32))
    vals = np.empty((n, z))
    for j0 in range(0, n, 262144):  # chunked: the (cols, z, 32) gather stays small
        j1 = min(n, j0 + 262144)
        V = rng.standard_normal((j1 - j0, 32))
        vals[j0:j1] = np.einsum("jzl,jl->jz", U[out[j0:j1]], V) / np.sqrt(32)
    vals += spec.noise * rng.standard_normal((n, z))
    colptr = np.arange(n + 1, dtype=np.int64) * z
    return colptr, out.reshape(-1), vals.reshape(-1)
