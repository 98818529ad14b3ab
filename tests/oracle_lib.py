"""ctypes bindings for the CPU oracle (oracle/liboracle.so) and, when built,
the reference shim (oracle/_ref/libgaplra_ref.so).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / reference arm — never by the product package.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
ORACLE_SO = ROOT / "oracle" / "liboracle.so"
REF_SO = ROOT / "oracle" / "_ref" / "libgaplra_ref.so"

_dp = C.POINTER(C.c_double)
_u64p = C.POINTER(C.c_uint64)
_i64p = C.POINTER(C.c_int64)
_i32p = C.POINTER(C.c_int32)
_ip = C.POINTER(C.c_int)


class OrcMat(C.Structure):
    _fields_ = [("kind", C.c_int), ("d", C.c_int), ("n", C.c_int), ("x", _dp),
                ("colptr", _i64p), ("rowidx", _i32p), ("val", _dp)]


class OrcSvrgParams(C.Structure):
    _fields_ = [("eta", C.c_double), ("m", C.c_int64), ("tol", C.c_double),
                ("epoch_cap", C.c_int), ("monotone_slack", C.c_double),
                ("root_seed", C.c_uint64), ("lambda1_hint", C.c_double)]


class OrcLedger(C.Structure):
    _fields_ = [(n, C.c_uint64) for n in (
        "gram_applies", "operator_applies", "qr_factorizations", "linear_solves",
        "solver_column_samples", "epochs", "outer_iterations")]


class OrcSiConfig(C.Structure):
    _fields_ = [("k", C.c_int), ("p", C.c_int), ("eps", C.c_double), ("mu", C.c_double),
                ("delta", C.c_double), ("lambda_", C.c_double), ("seed", C.c_uint64),
                ("tol_solve", C.c_double), ("tol_tune", C.c_double), ("conv_tol", C.c_double),
                ("rq_tol", C.c_double), ("max_outer", C.c_int), ("force", C.c_int),
                ("epoch_cap", C.c_int), ("monotone_slack", C.c_double), ("lambda1_hint", C.c_double),
                ("backend", C.c_int)]


class OrcSiReport(C.Structure):
    _fields_ = [("lambda_", C.c_double), ("lambda1_hat", C.c_double), ("lambda1_hint", C.c_double),
                ("tune_steps", C.c_int),
                ("tune_lambda", C.c_double * 64), ("tune_inv", C.c_double * 64),
                ("outer_iterations", C.c_int), ("outer_cap", C.c_int), ("ledger", OrcLedger)]


class OrcApReport(C.Structure):
    _fields_ = [("n_intervals", C.c_int), ("s", C.c_int * 64), ("q", C.c_int * 64), ("strategy", C.c_int * 64),
                ("width", C.c_int * 64), ("iterations", C.c_int * 64), ("shift", C.c_double * 64),
                ("ledger", OrcLedger), ("delta", C.c_double)]

    def plan(self):
        n = min(self.n_intervals, 64)
        return [dict(s=self.s[i], q=self.q[i], strategy=("PlainPower", "ShiftedInverse")[self.strategy[i]],
                     width=self.width[i], iterations=self.iterations[i], shift=self.shift[i]) for i in range(n)]


def build_oracle(ref: bool | None = None) -> None:
    """Compile oracle/liboracle.so (and oracle/_ref when /root/reference exists)."""
    subprocess.run(["make", "-s", "-C", str(ROOT / "oracle"), "liboracle.so"], check=True)
    if ref is None:
        ref = Path(os.environ.get("GAPLRA_REF_DIR", "/root/reference/proj")).exists()
    if ref:
        env = dict(os.environ)
        if "GAPLRA_REF_DIR" in env:
            env["REF"] = env["GAPLRA_REF_DIR"]
        subprocess.run(["make", "-s", "-C", str(ROOT / "oracle"), "ref"], check=True, env=env)


def _ptr(a, t=_dp):
    return a.ctypes.data_as(t) if a is not None else None


def c64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


class Oracle:
    def __init__(self, path: Path = ORACLE_SO):
        if not path.exists():
            build_oracle(ref=False)
        self.lib = L = C.CDLL(str(path))
        L.orc_derive_seed.restype = C.c_uint64
        L.orc_derive_seed.argtypes = [C.c_uint64, C.c_uint64]
        L.orc_max_col_norm2.restype = C.c_double
        L.orc_sin_theta.restype = C.c_double
        L.orc_sin_theta.argtypes = [C.c_int, C.c_int, _dp, C.c_int, _dp]
        self.nthreads = int(os.environ.get("GAPLRA_ORACLE_THREADS", os.cpu_count() or 1))

    # -- matrices ------------------------------------------------------------
    @staticmethod
    def dense(x: np.ndarray):
        """x: (d, n) float64; stored column-major (Fortran order)."""
        xf = np.asfortranarray(x, dtype=np.float64)
        m = OrcMat(0, xf.shape[0], xf.shape[1], xf.ctypes.data_as(_dp), None, None, None)
        m._keep = (xf,)
        return m

    @staticmethod
    def csc(d, n, colptr, rowidx, val):
        colptr = np.ascontiguousarray(colptr, dtype=np.int64)
        rowidx = np.ascontiguousarray(rowidx, dtype=np.int32)
        val = np.ascontiguousarray(val, dtype=np.float64)
        m = OrcMat(1, d, n, None, colptr.ctypes.data_as(_i64p), rowidx.ctypes.data_as(_i32p),
                   val.ctypes.data_as(_dp))
        m._keep = (colptr, rowidx, val)
        return m

    # -- primitives ------------------------------------------------------------
    def derive_seed(self, root, tag):
        return int(self.lib.orc_derive_seed(root, tag))

    def next_u64(self, seed, count):
        out = np.zeros(count, np.uint64)
        self.lib.orc_next_u64(C.c_uint64(seed), C.c_int64(count), _ptr(out, _u64p))
        return out

    def uniform_index(self, seed, n, count):
        out = np.zeros(count, np.uint64)
        self.lib.orc_uniform_index(C.c_uint64(seed), C.c_uint64(n), C.c_int64(count), _ptr(out, _u64p))
        return out

    def normal(self, seed, count):
        out = np.zeros(count, np.float64)
        self.lib.orc_normal(C.c_uint64(seed), C.c_int64(count), _ptr(out))
        return out

    def gaussian_init(self, d, p, seed):
        out = np.zeros((d, p))
        rc = self.lib.orc_gaussian_init(d, p, C.c_uint64(seed), _ptr(out))
        return rc, out

    def qr(self, y):
        y = c64(y)
        out = np.zeros_like(y)
        bad = C.c_int(-1)
        rc = self.lib.orc_qr(y.shape[0], y.shape[1], _ptr(y), _ptr(out), C.byref(bad))
        return rc, out, bad.value

    def jacobi(self, h):
        h = c64(h)
        n = h.shape[0]
        vals, vecs = np.zeros(n), np.zeros((n, n))
        rc = self.lib.orc_jacobi(n, _ptr(h), _ptr(vals), _ptr(vecs))
        return rc, vals, vecs

    def max_col_norm2(self, m):
        return float(self.lib.orc_max_col_norm2(C.byref(m)))

    def gram_block(self, m, w, want_y=False):
        w = c64(w)
        p = w.shape[1]
        z = np.zeros_like(w)
        y = np.zeros((m.n, p)) if want_y else None
        rc = self.lib.orc_gram_block(C.byref(m), p, _ptr(w), _ptr(z), _ptr(y), self.nthreads)
        return rc, z, y

    def svrg_epoch(self, m, w, y, cblk, eta, lam, stream_seed, steps):
        w = c64(w).copy()
        idx = np.zeros(steps, np.uint64)
        rc = self.lib.orc_svrg_epoch(C.byref(m), w.shape[1], _ptr(w), _ptr(c64(y)), _ptr(c64(cblk)),
                                     C.c_double(eta), C.c_double(lam), C.c_uint64(stream_seed),
                                     C.c_int64(steps), _ptr(idx, _u64p), self.nthreads)
        return rc, w, idx

    def svrg_solve(self, m, lam, b, tol, seed=0, solve_id=0, eta=0.0, steps=0, epoch_cap=0,
                   slack=10.0, hint=0.0):
        b = c64(b)
        w = np.zeros_like(b)
        prm = OrcSvrgParams(eta, steps, tol, epoch_cap, slack, seed, hint)
        ep, hl = C.c_int(0), C.c_int(0)
        hist = np.zeros(4096)
        rc = self.lib.orc_svrg_solve(C.byref(m), C.c_double(lam), b.shape[1], _ptr(b), _ptr(w),
                                     C.byref(prm), C.c_int64(solve_id), C.byref(ep), _ptr(hist),
                                     4096, C.byref(hl), self.nthreads)
        return rc, w, ep.value, hist[:hl.value].copy()

    def restricted_projection(self, m, s, k):
        s = c64(s)
        w = np.zeros((s.shape[0], k))
        ritz = np.zeros(k)
        rc = self.lib.orc_restricted_projection(C.byref(m), s.shape[1], _ptr(s), k, _ptr(w),
                                                _ptr(ritz), self.nthreads)
        return rc, w, ritz

    def shift_invert(self, m, cfg: OrcSiConfig):
        d = m.d
        w = np.zeros((d, cfg.k))
        ritz = np.zeros(cfg.k)
        s = np.zeros((d, cfg.p))
        rep = OrcSiReport()
        rc = self.lib.orc_shift_invert(C.byref(m), C.byref(cfg), _ptr(w), _ptr(ritz), _ptr(s),
                                       C.byref(rep), self.nthreads)
        return rc, w, ritz, s, rep

    def tune_shift(self, m, delta, cfg: OrcSiConfig):
        rep = OrcSiReport()
        sc = C.c_int64(0)
        rc = self.lib.orc_tune_shift(C.byref(m), C.c_double(delta), C.byref(cfg), C.byref(sc),
                                     C.byref(rep), self.nthreads)
        return rc, rep

    def detect_multiplicative_gap(self, est, s, p):
        est = np.ascontiguousarray(est, dtype=np.float64)
        q = self.lib.orc_detect_multiplicative_gap(_ptr(est), len(est), s, p)
        return None if q < 0 else q

    def detect_additive_gap(self, inv, s, k, delta):
        inv = np.ascontiguousarray(inv, dtype=np.float64)
        q = C.c_int(0)
        rc = self.lib.orc_detect_additive_gap(_ptr(inv), len(inv), s, k, C.c_double(delta), C.byref(q))
        return rc, q.value

    def estimate_eigenvalues(self, m, k, eps_prime, seed, *, inverse=False, lam=0.0, rq_tol=1e-3, tol=1e-6,
                             svrg_seed=0, hint=0.0):
        prm = OrcSvrgParams(0.0, 0, tol, 0, 10.0, svrg_seed, hint)
        vals = np.zeros(k)
        it = C.c_int(0)
        rc = self.lib.orc_estimate_eigenvalues(C.byref(m), int(inverse), C.c_double(lam), k, C.c_double(eps_prime),
                                               C.c_uint64(seed), C.c_double(rq_tol), C.byref(prm), _ptr(vals),
                                               C.byref(it), self.nthreads)
        return rc, vals, it.value

    def find_gap_budget(self, m, k, p, seed=0, rq_tol=1e-3):
        delta = C.c_double()
        rc = self.lib.orc_find_gap_budget(C.byref(m), k, p, C.c_uint64(seed), C.c_double(rq_tol), C.byref(delta),
                                          self.nthreads)
        return rc, delta.value

    def approximate(self, m, cfg):
        w = np.zeros((m.d, cfg.k))
        ritz = np.zeros(cfg.k)
        rep = OrcApReport()
        rc = self.lib.orc_approximate(C.byref(m), C.byref(cfg), _ptr(w), _ptr(ritz), C.byref(rep), self.nthreads)
        return rc, w, ritz, rep

    def accsvrg_solve(self, m, lam, b, tol, seed=0, solve_id=0, hint=0.0, epoch_cap=0):
        b = c64(b)
        w = np.zeros_like(b)
        prm = OrcSvrgParams(0.0, 0, tol, epoch_cap, 10.0, seed, hint)
        ep, hl = C.c_int(0), C.c_int(0)
        hist = np.zeros(8192)
        rc = self.lib.orc_accsvrg_solve(C.byref(m), C.c_double(lam), b.shape[1], _ptr(b), _ptr(w), C.byref(prm),
                                        C.c_int64(solve_id), C.byref(ep), _ptr(hist), 8192, C.byref(hl),
                                        self.nthreads)
        return rc, w, ep.value, hist[:hl.value]

    def cg_solve(self, m, lam, b, tol, max_iter=0):
        b = c64(b)
        w = np.zeros_like(b)
        it, hl = C.c_int(0), C.c_int(0)
        hist = np.zeros(8192)
        rc = self.lib.orc_cg_solve(C.byref(m), C.c_double(lam), b.shape[1], _ptr(b), _ptr(w), C.c_double(tol),
                                   max_iter, C.byref(it), _ptr(hist), 8192, C.byref(hl), self.nthreads)
        return rc, w, it.value, hist[:hl.value]

    def error_report(self, m, w, iters=20, seed=0):
        w = c64(w)
        fr, sp = C.c_double(), C.c_double()
        rc = self.lib.orc_error_report(C.byref(m), w.shape[1], _ptr(w), iters, C.c_uint64(seed), C.byref(fr),
                                       C.byref(sp))
        return rc, fr.value, sp.value

    def principal_angles(self, u, s):
        u, s = c64(u), c64(s)
        cos = np.zeros(u.shape[1])
        rc = self.lib.orc_principal_angles(u.shape[0], u.shape[1], _ptr(u), s.shape[1], _ptr(s), _ptr(cos))
        return rc, cos

    def sin_theta(self, u, q):
        u, q = c64(u), c64(q)
        return float(self.lib.orc_sin_theta(u.shape[0], u.shape[1], _ptr(u), q.shape[1], _ptr(q)))


class Reference:
    """The reference's own shipped primitives (oracle/_ref), when built."""

    def __init__(self, path: Path = REF_SO):
        self.lib = L = C.CDLL(str(path))
        L.ref_derive_seed.restype = C.c_uint64
        L.ref_derive_seed.argtypes = [C.c_uint64, C.c_uint64]

    def derive_seed(self, root, tag):
        return int(self.lib.ref_derive_seed(root, tag))

    def next_u64(self, seed, count):
        out = np.zeros(count, np.uint64)
        self.lib.ref_next_u64(C.c_uint64(seed), C.c_int64(count), _ptr(out, _u64p))
        return out

    def uniform_index(self, seed, n, count):
        out = np.zeros(count, np.uint64)
        self.lib.ref_uniform_index(C.c_uint64(seed), C.c_uint64(n), C.c_int64(count), _ptr(out, _u64p))
        return out

    def normal(self, seed, count):
        out = np.zeros(count)
        self.lib.ref_normal(C.c_uint64(seed), C.c_int64(count), _ptr(out))
        return out

    def gaussian_init(self, d, p, seed):
        out = np.zeros((d, p))
        rc = self.lib.ref_gaussian_init(d, p, C.c_uint64(seed), _ptr(out))
        return rc, out

    def qr(self, y):
        y = c64(y)
        out = np.zeros_like(y)
        bad = C.c_int(-1)
        rc = self.lib.ref_qr(y.shape[0], y.shape[1], _ptr(y), _ptr(out), C.byref(bad))
        return rc, out, bad.value

    def jacobi(self, h):
        h = c64(h)
        n = h.shape[0]
        vals, vecs = np.zeros(n), np.zeros((n, n))
        rc = self.lib.ref_jacobi(n, _ptr(h), _ptr(vals), _ptr(vecs))
        return rc, vals, vecs

    def gram_apply_dense(self, x, v):
        xf = np.asfortranarray(x, dtype=np.float64)
        out = np.zeros(x.shape[0])
        rc = self.lib.ref_gram_apply_dense(x.shape[0], x.shape[1], _ptr(xf), _ptr(c64(v)), _ptr(out))
        return rc, out

    def gram_apply_csc(self, d, n, colptr, rowidx, val, v):
        colptr = np.ascontiguousarray(colptr, dtype=np.int64)
        rowidx = np.ascontiguousarray(rowidx, dtype=np.int32)
        val = c64(val)
        out = np.zeros(d)
        rc = self.lib.ref_gram_apply_csc(d, n, _ptr(colptr, _i64p), _ptr(rowidx, _i32p), _ptr(val),
                                         _ptr(c64(v)), _ptr(out))
        return rc, out

    def svrg_epoch_dense(self, x, w, y, cblk, eta, lam, stream_seed, steps):
        xf = np.asfortranarray(x, dtype=np.float64)
        w = c64(w).copy()
        idx = np.zeros(steps, np.uint64)
        rc = self.lib.ref_svrg_epoch_dense(x.shape[0], x.shape[1], _ptr(xf), w.shape[1], _ptr(w),
                                           _ptr(c64(y)), _ptr(c64(cblk)), C.c_double(eta),
                                           C.c_double(lam), C.c_uint64(stream_seed), C.c_int64(steps),
                                           _ptr(idx, _u64p))
        return rc, w, idx


def default_si_config(k, p, *, eps=1e-8, mu=1.0, delta=0.0, lam=0.0, seed=0, tol_solve=1e-10,
                      tol_tune=1e-6, conv_tol=1e-9, rq_tol=1e-3, max_outer=0, force=0,
                      epoch_cap=0, slack=10.0, hint=0.0, backend=0):
    return OrcSiConfig(k, p, eps, mu, delta, lam, seed, tol_solve, tol_tune, conv_tol, rq_tol,
                       max_outer, force, epoch_cap, slack, hint, backend)
