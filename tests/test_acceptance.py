"""SPEC.md acceptance criteria on the hot path, on the CPU
oracle (all seeds, `-m "not gpu"`) and on the device (`-m gpu`).

#5 Shift tuning (Alg. 6 / Lemma B): planted systems with λ_s/Δ ∈ {10, 10³, 10⁶};
   tune_shift terminates within ceil(4 log2(λ_s/Δ)) + 5 steps and ends with
   λ − λ_s ∈ [Δ/30, 2Δ/9]; 100 % of runs.  The inner solves use the CG backend
   (inverse_operator backend 1): at λ_s/Δ = 10⁶ the tuned system's condition
   number is ~10⁷, where the SVRG step size rule needs ~10⁷ epochs.
#6 Solver correctness (Theorem 2.2): SVRG and accelerated SVRG match the direct
   solve within tol = 1e-8 in the D-norm (D = λI − XXᵀ, relative to |w*|_D) on
   40 seeded systems spanning (λ − λ₁)/λ₁ ∈ {0.5, 0.05, 0.005}; ≥ 95 %.
"""
import math

import numpy as np
import pytest

from oracle_lib import default_si_config
from problems import planted_dense

RATIOS = (10.0, 1e3, 1e6)
GAPS = (0.5, 0.05, 0.005)


def planted_system(seed, d=40, n=80):
    """λ_1 = 1 exactly (σ_1 = 1), then a clear second eigenvalue and a tail."""
    sig = np.concatenate([[1.0, 0.8, 0.7], 0.5 / np.arange(1, min(d, n) - 2)])
    X, U, s = planted_dense(d, n, sigma=sig, seed=seed)
    return X, float(s[0] ** 2)


def check_tune(steps, lam, lam_s, delta):
    cap = math.ceil(4 * math.log2(lam_s / delta)) + 5
    gap = lam - lam_s
    return steps <= cap and delta / 30 <= gap <= 2 * delta / 9, (steps, cap, gap / delta)


def d_norm_rel(X, lam, w, w_star):
    D = lam * np.eye(X.shape[0]) - X @ X.T
    e = w - w_star
    return float(np.sqrt(max(np.sum(e * (D @ e)), 0.0)) / np.sqrt(np.sum(w_star * (D @ w_star))))


def systems6():
    out = []
    for i in range(40):
        g = GAPS[i % 3]
        X, l1 = planted_system(100 + i, d=30, n=3000)  # ηn grows with n: the 0.005 gap fits the epoch cap
        lam = l1 * (1 + g)
        b = np.random.default_rng(i).standard_normal((30, 1))
        out.append((X, l1, lam, b))
    return out


# ------------------------------------------------------------------ oracle (CPU)
@pytest.mark.parametrize("ratio", RATIOS)
def test_oracle_tune_shift_sweep(oracle, ratio):
    fails = []
    for seed in range(20):
        X, lam_s = planted_system(seed)
        delta = lam_s / ratio
        cfg = default_si_config(1, 2, delta=delta, seed=seed, backend=1, tol_tune=1e-10)
        rc, rep = oracle.tune_shift(oracle.dense(X), delta, cfg)
        ok, info = check_tune(rep.tune_steps, rep.lambda_, lam_s, delta) if rc == 0 else (False, rc)
        if not ok:
            fails.append((seed, info))
    assert not fails, fails


def test_oracle_solver_sweep(oracle):
    bad = []
    for i, (X, l1, lam, b) in enumerate(systems6()):
        w_star = np.linalg.solve(lam * np.eye(X.shape[0]) - X @ X.T, b)
        m = oracle.dense(X)
        rc, w, ep, _ = oracle.svrg_solve(m, lam, b, 1e-10, seed=i, hint=l1)
        e1 = d_norm_rel(X, lam, w, w_star) if rc == 0 else np.inf
        rc2, w2, ep2, _ = oracle.accsvrg_solve(m, lam, b, 1e-10, seed=i, hint=l1)
        e2 = d_norm_rel(X, lam, w2, w_star) if rc2 == 0 else np.inf
        if not (e1 <= 1e-8 and e2 <= 1e-8):
            bad.append((i, e1, e2))
    assert len(bad) <= 2, bad  # >= 95 % of 40


# ------------------------------------------------------------------ device (B200)
@pytest.mark.gpu
@pytest.mark.parametrize("ratio", RATIOS)
def test_device_tune_shift_sweep(g, oracle, ratio):
    fails = []
    for seed in range(6):
        X, lam_s = planted_system(seed)
        delta = lam_s / ratio
        st = g.tune_shift(g.DeviceMatrix.dense(X), delta,
                          g.SIConfig(k=1, p=2, delta=delta, seed=seed, backend="cg", tol_tune=1e-10))
        ok, info = check_tune(len(st.history), st.lam, lam_s, delta)
        rc, rep = oracle.tune_shift(oracle.dense(X), delta,
                                    default_si_config(1, 2, delta=delta, seed=seed, backend=1, tol_tune=1e-10))
        if not ok or rc != 0 or rep.tune_steps != len(st.history) or abs(rep.lambda_ - st.lam) > 1e-10 * st.lam:
            fails.append((seed, info, rc, rep.tune_steps, rep.lambda_, st.lam))
    assert not fails, fails


@pytest.mark.gpu
def test_device_solver_sweep(g):
    bad = []
    for i, (X, l1, lam, b) in enumerate(systems6()):
        w_star = np.linalg.solve(lam * np.eye(X.shape[0]) - X @ X.T, b)
        x = g.DeviceMatrix.dense(X)
        w = g.solve_svrg(x, lam, b, 1e-10, seed=i, lambda1_hint=l1).solution
        w2 = g.solve_accelerated_svrg(x, lam, b, 1e-10, lambda1_hint=l1, seed=i).solution
        e1, e2 = d_norm_rel(X, lam, w, w_star), d_norm_rel(X, lam, w2, w_star)
        if not (e1 <= 1e-8 and e2 <= 1e-8):
            bad.append((i, e1, e2))
    assert len(bad) <= 2, bad
