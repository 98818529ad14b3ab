"""Python mirror of the reference `gaplra` interface for the shift-and-invert
hot path, backed only by the sm_100a kernels behind include/gaplra_cuda.h.

Names, argument meaning and error types follow the reference:
  * errors.hpp:10-116        -> Error, ContractViolation, RankDeficient(column),
                                IndefiniteShift, SolverStalled(residual_history),
                                ShiftOutOfRange, ShiftTuningStalled(history)
  * SparseColumnsMatrix       -> DeviceMatrix (X resident in HBM)
  * GramOperator::apply       -> GramOperator.apply / gram_apply / gram_block
  * Rng::uniform_index stream -> index_stream
  * gaussian_init / qr_orthonormalize / orthonormality_defect / jacobi_eigh
  * SPEC.md solve_svrg, estimate_eigenvalues, tune_shift, restricted_projection,
    and Alg. 7's ShiftedInverse branch -> shift_invert.
Host blocks are numpy float64, row-major d x p (DenseMatrix layout).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from . import _native as N

GAPLRA_OK = 0


class Error(RuntimeError):
    """gaplra::Error (errors.hpp:10)."""


class ContractViolation(Error):
    pass


class RankDeficient(Error):
    def __init__(self, what, column):
        super().__init__(what)
        self.column = column


class IndefiniteShift(Error):
    pass


class SolverStalled(Error):
    def __init__(self, what, residual_history=()):
        super().__init__(what)
        self.residual_history = list(residual_history)


class ShiftOutOfRange(Error):
    pass


class ShiftTuningStalled(Error):
    def __init__(self, what, history=()):
        super().__init__(what)
        self.history = list(history)


class NoPreconditioningNeeded(Error):
    """tune_shift's guard signal."""


class NoUsableGap(Error):
    """find_gap_budget found no gap above the floor."""


class DegenerateProgress(Error):
    """approximate stopped making progress: a duplicated eigendirection or more
    intervals than target indices (errors.hpp:95-98)."""


class DeviceError(Error):
    pass


class OutOfMemory(DeviceError):
    pass


_CODES = {1: ContractViolation, 3: IndefiniteShift, 5: ShiftOutOfRange, 7: NoPreconditioningNeeded,
          8: DeviceError, 9: OutOfMemory, 10: NoUsableGap, 11: DegenerateProgress}


def _f64(a, shape=None):
    a = np.ascontiguousarray(a, dtype=np.float64)
    if shape is not None and a.shape != shape:
        raise ContractViolation(f"expected shape {shape}, got {a.shape}")
    return a


def _p(a, t=N._dp):
    return a.ctypes.data_as(t) if a is not None else None


class Context:
    """One CUDA device + stream (gaplra_ctx)."""

    def __init__(self, device: int = 0):
        self.lib = N.load()
        h = C.c_void_p()
        rc = self.lib.gaplra_ctx_create(device, C.byref(h))
        if rc != GAPLRA_OK:
            raise DeviceError(f"gaplra_ctx_create(device={device}) failed with status {rc} "
                              "(no CUDA device? the product path has no CPU fallback)")
        self.h = h
        self.device = device

    def close(self):
        if getattr(self, "h", None):
            self.lib.gaplra_ctx_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def check(self, rc, extra=None):
        if rc == GAPLRA_OK:
            return
        msg = self.lib.gaplra_last_error(self.h).decode(errors="replace")
        if rc == 2:
            raise RankDeficient(msg, extra if extra is not None else -1)
        if rc == 4:
            raise SolverStalled(msg, extra or ())
        if rc == 6:
            raise ShiftTuningStalled(msg, extra or ())
        raise _CODES.get(rc, Error)(msg)

    def set_stream(self, stream_handle: int | None):
        self.check(self.lib.gaplra_ctx_set_stream(self.h, C.c_void_p(stream_handle or 0)))

    def synchronize(self):
        self.check(self.lib.gaplra_ctx_synchronize(self.h))

    def host_syncs(self) -> int:
        """Times the host has waited on this context's stream."""
        return int(self.lib.gaplra_host_syncs(self.h))

    def ledger(self) -> dict:
        L = N.Ledger()
        self.check(self.lib.gaplra_ledger_get(self.h, C.byref(L)))
        return L.as_dict()

    def reset_ledger(self):
        self.check(self.lib.gaplra_ledger_reset(self.h))

    def enable_profiling(self, on: bool = True):
        self.check(self.lib.gaplra_profile_enable(self.h, int(on)))

    def profile(self) -> dict:
        P = N.Profile()
        self.check(self.lib.gaplra_profile_get(self.h, C.byref(P)))
        return P.as_dict()

    def reset_profile(self):
        self.check(self.lib.gaplra_profile_reset(self.h))


_DEFAULT: dict[int, Context] = {}


def default_context(device: int = 0) -> Context:
    if device not in _DEFAULT:
        _DEFAULT[device] = Context(device)
    return _DEFAULT[device]


class DeviceMatrix:
    """X in R^{d x n} resident in HBM (SparseColumnsMatrix, sparse_matrix.hpp:18-57)."""

    def __init__(self, ctx: Context, handle, keep=None):
        self.ctx, self.h, self._keep = ctx, handle, keep
        d, n, nnz, ld = C.c_int(), C.c_int(), C.c_int64(), C.c_int64()
        ctx.check(ctx.lib.gaplra_matrix_info(handle, C.byref(d), C.byref(n), C.byref(nnz), C.byref(ld)))
        self.d, self.n, self.nnz, self.ld = d.value, n.value, nnz.value, ld.value

    @classmethod
    def dense(cls, x: np.ndarray, ctx: Context | None = None):
        """Upload a host (d, n) float64 array (copied column-major)."""
        ctx = ctx or default_context()
        xf = np.asfortranarray(x, dtype=np.float64)
        h = C.c_void_p()
        ctx.check(ctx.lib.gaplra_matrix_dense(ctx.h, xf.shape[0], xf.shape[1], xf.ctypes.data, xf.shape[0], 0,
                                              C.byref(h)))
        return cls(ctx, h)

    @classmethod
    def from_host_pointer(cls, ptr: int, d: int, n: int, ldx: int, ctx: Context | None = None):
        """Copy a host column-major X (e.g. pinned memory) into HBM."""
        ctx = ctx or default_context()
        h = C.c_void_p()
        ctx.check(ctx.lib.gaplra_matrix_dense(ctx.h, d, n, C.c_void_p(ptr), ldx, 0, C.byref(h)))
        return cls(ctx, h)

    @classmethod
    def from_device(cls, ptr: int, d: int, n: int, ldx: int, ctx: Context | None = None, keep=None):
        """Borrow a device column-major X with ldx == round_up(d, 4) and zero pad
        rows (checked on the device, with finiteness); `keep` holds its owner."""
        ctx = ctx or default_context()
        h = C.c_void_p()
        ctx.check(ctx.lib.gaplra_matrix_dense(ctx.h, d, n, C.c_void_p(ptr), ldx, 1, C.byref(h)))
        return cls(ctx, h, keep)

    @classmethod
    def from_torch(cls, xt, d: int | None = None, ctx: Context | None = None):
        """Borrow a contiguous CUDA float64 tensor of shape (n, ld) holding X
        column-major (i.e. Xᵀ row-major); d defaults to ld."""
        if str(getattr(xt, "dtype", "")) != "torch.float64" or not xt.is_cuda or xt.dim() != 2 \
                or not xt.is_contiguous():
            raise ContractViolation("from_torch: need a contiguous (n, ld) float64 CUDA tensor")
        n, ld = xt.shape
        return cls.from_device(xt.data_ptr(), d or ld, n, ld, ctx=ctx, keep=xt)

    @classmethod
    def csc(cls, d, n, colptr, rowidx, val, ctx: Context | None = None):
        ctx = ctx or default_context()
        cp = np.ascontiguousarray(colptr, dtype=np.int64)
        ri = np.ascontiguousarray(rowidx, dtype=np.int32)
        v = np.ascontiguousarray(val, dtype=np.float64)
        h = C.c_void_p()
        ctx.check(ctx.lib.gaplra_matrix_csc(ctx.h, d, n, cp.ctypes.data, ri.ctypes.data, v.ctypes.data, 0,
                                            C.byref(h)))
        return cls(ctx, h)

    def close(self):
        if getattr(self, "h", None):
            self.ctx.lib.gaplra_matrix_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def gram_block(x: DeviceMatrix, w: np.ndarray, want_y: bool = False):
    """Z = X (Xᵀ W) for a d x p block (p GramOperator::apply calls in one pass)."""
    w = _f64(w)
    if w.ndim != 2 or w.shape[0] != x.d:
        raise ContractViolation("gram_block: W must be d x p")
    p = w.shape[1]
    z = np.zeros_like(w)
    y = np.zeros((x.n, p)) if want_y else None
    x.ctx.check(x.ctx.lib.gaplra_gram_block(x.ctx.h, x.h, p, _p(w), _p(z), _p(y)))
    return (z, y) if want_y else z


def gram_apply(x: DeviceMatrix, v: np.ndarray) -> np.ndarray:
    v = _f64(v)
    if v.shape != (x.d,):
        raise ContractViolation("gram_apply: vector length != row count")
    out = np.zeros(x.d)
    x.ctx.check(x.ctx.lib.gaplra_gram_apply(x.ctx.h, x.h, _p(v), _p(out)))
    return out


class GramOperator:
    """C = X Xᵀ in factored form (linear_operator.hpp:51-62)."""

    def __init__(self, x: DeviceMatrix):
        self.x = x

    def dim(self):
        return self.x.d

    def apply(self, v):
        return gram_apply(self.x, v)

    def apply_block(self, w):
        return gram_block(self.x, w)


def index_stream(seed: int, n: int, m: int, ctx: Context | None = None) -> np.ndarray:
    """Rng(seed).uniform_index(n) drawn m times, replayed on the device."""
    ctx = ctx or default_context()
    out = np.zeros(m, np.int32)
    ctx.check(ctx.lib.gaplra_index_stream(ctx.h, seed, n, m, _p(out, N._i32p)))
    return out


def gaussian_init(d: int, p: int, seed: int) -> np.ndarray:
    out = np.zeros((d, p))
    rc = N.load().gaplra_gaussian_init(d, p, seed, _p(out))
    if rc != GAPLRA_OK:
        raise ContractViolation(f"gaussian_init: requires 1 <= p <= d, got p={p}, d={d}")
    return out


def qr_orthonormalize(y: np.ndarray, ctx: Context | None = None) -> np.ndarray:
    ctx = ctx or default_context()
    y = _f64(y)
    if y.ndim != 2:
        raise ContractViolation("qr_orthonormalize: need a matrix")
    q = np.zeros_like(y)
    bad = C.c_int(-1)
    rc = ctx.lib.gaplra_qr_orthonormalize(ctx.h, y.shape[0], y.shape[1], _p(y), _p(q), C.byref(bad))
    ctx.check(rc, bad.value)
    return q


def orthonormality_defect(q: np.ndarray, ctx: Context | None = None) -> float:
    ctx = ctx or default_context()
    q = _f64(q)
    out = C.c_double()
    ctx.check(ctx.lib.gaplra_orthonormality_defect(ctx.h, q.shape[0], q.shape[1], _p(q), C.byref(out)))
    return out.value


@dataclass
class SymmetricEigen:
    values: np.ndarray
    vectors: np.ndarray


def jacobi_eigh(h: np.ndarray, ctx: Context | None = None) -> SymmetricEigen:
    ctx = ctx or default_context()
    h = _f64(h)
    if h.ndim != 2 or h.shape[0] != h.shape[1]:
        raise ContractViolation("jacobi_eigh: matrix must be square")
    n = h.shape[0]
    vals, vecs = np.zeros(n), np.zeros((n, n))
    ctx.check(ctx.lib.gaplra_jacobi_eigh(ctx.h, n, _p(h), _p(vals), _p(vecs)))
    return SymmetricEigen(vals, vecs)


def svrg_epoch(x: DeviceMatrix, w, y, c, eta, lam, stream_seed, m):
    """One stochastic epoch (lockstep parity unit)."""
    w = _f64(w).copy()
    x.ctx.check(x.ctx.lib.gaplra_svrg_epoch(x.ctx.h, x.h, w.shape[1], _p(w), _p(_f64(y)), _p(_f64(c)), eta, lam,
                                            stream_seed, m))
    return w


@dataclass
class SolverReport:
    """SPEC.md:301-304."""
    solution: np.ndarray
    epochs: int
    column_samples: int
    residual_norm: float
    residual_history: list


def solve_svrg(x: DeviceMatrix, lam: float, b: np.ndarray, tol: float, seed: int = 0, solve_id: int = 0,
               eta: float = 0.0, steps: int = 0, epoch_cap: int = 0, slack: float = 10.0,
               lambda1_hint: float = 0.0) -> SolverReport:
    """Block SVRG solve of (λI − XXᵀ)W = B."""
    b = _f64(b)
    if b.ndim == 1:
        b = b[:, None]
    p = b.shape[1]
    w = np.zeros_like(b)
    prm = N.SvrgParams(eta, steps, tol, epoch_cap, slack, seed, lambda1_hint)
    ep, hl = C.c_int(0), C.c_int(0)
    hist = np.zeros(8192)
    rc = x.ctx.lib.gaplra_svrg_solve(x.ctx.h, x.h, lam, p, _p(b), _p(w), C.byref(prm), solve_id, C.byref(ep),
                                     _p(hist), 8192, C.byref(hl))
    history = hist[:hl.value].tolist()
    x.ctx.check(rc, history)
    m = steps if steps > 0 else 2 * x.n
    return SolverReport(w, ep.value, ep.value * m, history[-1] if history else float("nan"), history)


def solve_accelerated_svrg(x: DeviceMatrix, lam: float, b: np.ndarray, tol: float, lambda1_hint: float,
                           seed: int = 0, solve_id: int = 0, epoch_cap: int = 0) -> SolverReport:
    """solve_accelerated_svrg: Catalyst outer loop around the
    block SVRG solve; needs the caller's λ₁ hint."""
    b = _f64(b)
    if b.ndim == 1:
        b = b[:, None]
    p = b.shape[1]
    w = np.zeros_like(b)
    prm = N.SvrgParams(0.0, 0, tol, epoch_cap, 10.0, seed, lambda1_hint)
    ep, hl = C.c_int(0), C.c_int(0)
    hist = np.zeros(8192)
    rc = x.ctx.lib.gaplra_accsvrg_solve(x.ctx.h, x.h, lam, p, _p(b), _p(w), C.byref(prm), solve_id, C.byref(ep),
                                        _p(hist), 8192, C.byref(hl))
    history = hist[:hl.value].tolist()
    x.ctx.check(rc, history)
    return SolverReport(w, ep.value, ep.value * 2 * x.n, history[-1] if history else float("nan"), history)


def solve_cg(x: DeviceMatrix, lam: float, b: np.ndarray, tol: float, max_iter: int = 0) -> SolverReport:
    """Block CG solve of (λI − XXᵀ)W = B; column_samples = 0
    and `epochs` counts CG iterations."""
    b = _f64(b)
    if b.ndim == 1:
        b = b[:, None]
    p = b.shape[1]
    w = np.zeros_like(b)
    it, hl = C.c_int(0), C.c_int(0)
    hist = np.zeros(8192)
    rc = x.ctx.lib.gaplra_cg_solve(x.ctx.h, x.h, lam, p, _p(b), _p(w), tol, max_iter, C.byref(it), _p(hist), 8192,
                                   C.byref(hl))
    history = hist[:hl.value].tolist()
    x.ctx.check(rc, history)
    return SolverReport(w, it.value, 0, history[-1] if history else float("nan"), history)


def error_report(x: DeviceMatrix, w: np.ndarray, iters: int = 20, seed: int = 0):
    """error_report: (‖X − WWᵀX‖_F, power-method ‖X − WWᵀX‖₂)."""
    w = _f64(w)
    if w.ndim == 1:
        w = w[:, None]
    if w.shape[0] != x.d:
        raise ContractViolation("error_report: W must be d x k")
    fr, sp = C.c_double(), C.c_double()
    x.ctx.check(x.ctx.lib.gaplra_error_report(x.ctx.h, x.h, w.shape[1], _p(w), iters, seed, C.byref(fr),
                                              C.byref(sp)))
    return fr.value, sp.value


def principal_angles(u: np.ndarray, s: np.ndarray, ctx: Context | None = None) -> np.ndarray:
    """principal_angles: cosines, descending, between span(U)
    (d x k orthonormal) and span(S) (d x p, full column rank)."""
    ctx = ctx or default_context()
    u, s = _f64(u), _f64(s)
    if u.shape[0] != s.shape[0]:
        raise ContractViolation("principal_angles: U and S need the same number of rows")
    cos = np.zeros(u.shape[1])
    ctx.check(ctx.lib.gaplra_principal_angles(ctx.h, u.shape[0], u.shape[1], _p(u), s.shape[1], _p(s), _p(cos)))
    return cos


def detect_multiplicative_gap(estimates, s: int, p: int):
    """Alg. 4: estimates = λ̂_s, λ̂_{s+1}, ...; the smallest
    global q with λ̂_{q+1} <= λ̂_q (1 − p⁻²), or None."""
    est = np.ascontiguousarray(estimates, dtype=np.float64)
    q = C.c_int(0)
    rc = N.load().gaplra_detect_multiplicative_gap(_p(est), len(est), s, p, C.byref(q))
    if rc != GAPLRA_OK:
        raise ContractViolation("detect_multiplicative_gap: bad arguments")
    return None if q.value < 0 else q.value


def detect_additive_gap(inv_estimates, s: int, k: int, delta: float, ctx: Context | None = None) -> int:
    """Alg. 5: inv_estimates = λ̃_s⁻¹, ...; q = min J or k;
    ShiftOutOfRange unless λ̃_s⁻¹ ∈ [Δ/27, Δ/5]."""
    ctx = ctx or default_context()
    inv = np.ascontiguousarray(inv_estimates, dtype=np.float64)
    q = C.c_int(0)
    ctx.check(ctx.lib.gaplra_detect_additive_gap(ctx.h, _p(inv), len(inv), s, k, delta, C.byref(q)))
    return q.value


def estimate_eigenvalues(x: DeviceMatrix, k: int, eps_prime: float, seed: int, *, inverse: bool = False,
                         lam: float = 0.0, rq_tol: float = 1e-3, tol: float = 1e-6, svrg_seed: int = 0,
                         lambda1_hint: float = 0.0):
    """Alg. 3 for any k: descending estimates of the top-k
    eigenvalues of A = XXᵀ (or of D⁻¹ with inverse=True) and the iterations."""
    prm = N.SvrgParams(0.0, 0, tol, 0, 10.0, svrg_seed, lambda1_hint)
    vals = np.zeros(k)
    it = C.c_int()
    x.ctx.check(x.ctx.lib.gaplra_estimate_eigenvalues(x.ctx.h, x.h, int(inverse), lam, k, eps_prime, seed, rq_tol,
                                                      C.byref(prm), _p(vals), C.byref(it)))
    return vals, it.value


@dataclass
class RankKProjection:
    """W (d x k orthonormal), Ritz values, errors, executed plan."""
    W: np.ndarray
    ritz: np.ndarray
    frobenius_error: float
    spectral_error: float
    plan: list
    ledger: dict
    ms: float
    delta: float = 0.0  # the gap budget used


def find_gap_budget(x: DeviceMatrix, k: int, p: int, seed: int = 0, rq_tol: float = 1e-3) -> float:
    """find_gap_budget: Δ from Alg. 3 estimates of λ_k and
    λ_{p+1} at ε′ = 1/100; NoUsableGap without a gap."""
    delta = C.c_double()
    x.ctx.check(x.ctx.lib.gaplra_find_gap_budget(x.ctx.h, x.h, k, p, seed, rq_tol, C.byref(delta)))
    return delta.value


def approximate(x: DeviceMatrix, cfg: SIConfig, error_iters: int = 20) -> RankKProjection:
    """Alg. 7: adaptive partition into PlainPower /
    ShiftedInverse intervals with deflation, then Alg. 2 on the concatenated
    basis.  cfg.delta is the gap budget (Δ <= λ_k − λ_{p+1} <= 2Δ); with
    cfg.delta <= 0 it comes from find_gap_budget."""
    w = np.zeros((x.d, cfg.k))
    ritz = np.zeros(cfg.k)
    rep = N.ApReport()
    x.ctx.check(x.ctx.lib.gaplra_approximate(x.ctx.h, x.h, C.byref(cfg.native()), _p(w), _p(ritz), C.byref(rep)))
    plan = [dict(s=rep.s[i], q=rep.q[i], strategy=("PlainPower", "ShiftedInverse")[rep.strategy[i]],
                 width=rep.width[i], iterations=rep.iterations[i], shift=rep.shift[i])
            for i in range(min(rep.n_intervals, 64))]
    fr, sp = error_report(x, w, iters=error_iters, seed=cfg.seed)
    return RankKProjection(w, ritz, fr, sp, plan, rep.ledger.as_dict(), rep.ms_total, rep.delta)


def estimate_top(x: DeviceMatrix, eps_prime: float, seed: int, *, inverse: bool = False, lam: float = 0.0,
                 rq_tol: float = 1e-3, tol: float = 1e-6, svrg_seed: int = 0, solve_counter: int = 0,
                 lambda1_hint: float = 0.0):
    """Alg. 3 (estimate_eigenvalues) for k = 1, on A = XXᵀ or D⁻¹."""
    prm = N.SvrgParams(0.0, 0, tol, 0, 10.0, svrg_seed, lambda1_hint)
    sc = C.c_int64(solve_counter)
    val, it = C.c_double(), C.c_int()
    x.ctx.check(x.ctx.lib.gaplra_estimate_top(x.ctx.h, x.h, int(inverse), lam, eps_prime, seed, rq_tol,
                                              C.byref(prm), C.byref(sc), C.byref(val), C.byref(it)))
    return val.value, it.value, sc.value


@dataclass
class SIConfig:
    """Pinned defaults of the ShiftedInverse pipeline."""
    k: int
    p: int
    eps: float = 1e-8
    mu: float = 1.0
    delta: float = 0.0
    lam: float = 0.0
    seed: int = 0
    tol_solve: float = 1e-10
    tol_tune: float = 1e-6
    conv_tol: float = 1e-9
    rq_tol: float = 1e-3
    max_outer: int = 0
    force: bool = False
    epoch_cap: int = 0
    monotone_slack: float = 10.0
    lambda1_hint: float = 0.0
    backend: str = "svrg"  # inverse_operator backend: "svrg" | "cg" | "accsvrg"

    def native(self) -> N.SiConfig:
        if self.backend not in ("svrg", "cg", "accsvrg"):
            raise ContractViolation(f"unknown solver backend {self.backend!r} (svrg | cg | accsvrg)")
        return N.SiConfig(self.k, self.p, self.eps, self.mu, self.delta, self.lam, self.seed, self.tol_solve,
                          self.tol_tune, self.conv_tol, self.rq_tol, self.max_outer, int(self.force),
                          self.epoch_cap, self.monotone_slack, self.lambda1_hint,
                          {"svrg": 0, "cg": 1, "accsvrg": 2}[self.backend])


@dataclass
class ShiftState:
    """SPEC.md:397-400."""
    lam: float
    inv_gap_estimate: float
    lambda1_hat: float
    history: list = field(default_factory=list)
    lambda1_hint: float = 0.0  # the λ₁ upper estimate the main phase sizes its SVRG step with


def _history(rep):
    return [(rep.tune_lambda[i], rep.tune_inv[i]) for i in range(min(rep.tune_steps, 64))]


def tune_shift(x: DeviceMatrix, delta: float, cfg: SIConfig) -> ShiftState:
    rep = N.SiReport()
    sc = C.c_int64(0)
    rc = x.ctx.lib.gaplra_tune_shift(x.ctx.h, x.h, delta, C.byref(cfg.native()), C.byref(sc), C.byref(rep))
    x.ctx.check(rc, _history(rep))
    h = _history(rep)
    return ShiftState(rep.lambda_, h[-1][1] if h else float("nan"), rep.lambda1_hat, h, rep.lambda1_hint)


def restricted_projection(x: DeviceMatrix, s: np.ndarray, k: int):
    """Alg. 2: W = S Û_k and the top-k Ritz values."""
    s = _f64(s)
    w = np.zeros((x.d, k))
    ritz = np.zeros(k)
    x.ctx.check(x.ctx.lib.gaplra_restricted_projection(x.ctx.h, x.h, s.shape[1], _p(s), k, _p(w), _p(ritz)))
    return w, ritz


@dataclass
class ShiftInvertResult:
    W: np.ndarray
    ritz: np.ndarray
    S: np.ndarray
    lam: float
    lambda1_hat: float
    tune_history: list
    outer_iterations: int
    outer_cap: int
    ledger: dict
    ms: dict
    lambda1_hint: float = 0.0  # step-size hint used by the subspace phase (pass it back with an explicit lam)


def shift_invert(x: DeviceMatrix, cfg: SIConfig) -> ShiftInvertResult:
    """Alg. 7's ShiftedInverse branch on I = {1..k}: tune_shift (unless cfg.lam
    is given) -> subspace_iterate(D⁻¹, p) -> restricted_projection(XXᵀ, S, k)."""
    w = np.zeros((x.d, cfg.k))
    ritz = np.zeros(cfg.k)
    s = np.zeros((x.d, cfg.p))
    rep = N.SiReport()
    rc = x.ctx.lib.gaplra_shift_invert(x.ctx.h, x.h, C.byref(cfg.native()), _p(w), _p(ritz), _p(s), C.byref(rep))
    x.ctx.check(rc, _history(rep))
    return ShiftInvertResult(w, ritz, s, rep.lambda_, rep.lambda1_hat, _history(rep), rep.outer_iterations,
                             rep.outer_cap, rep.ledger.as_dict(),
                             {"tune": rep.ms_tune, "subspace": rep.ms_subspace,
                              "rayleigh_ritz": rep.ms_rayleigh_ritz, "total": rep.ms_total}, rep.lambda1_hint)
