"""ctypes binding of include/gaplra_cuda.h (libgaplra_cuda.so, built in-tree).

The product path has no CPU fallback: if the shared library is missing or no
CUDA device is present, loading / context creation raises.
"""
from __future__ import annotations

import ctypes as C
import os
import re
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
LIB_PATH = PKG / "libgaplra_cuda.so"
HEADER = ROOT / "include" / "gaplra_cuda.h"

_dp = C.POINTER(C.c_double)
_i32p = C.POINTER(C.c_int32)
_i64p = C.POINTER(C.c_int64)
_ip = C.POINTER(C.c_int)


class SvrgParams(C.Structure):
    _fields_ = [("eta", C.c_double), ("m", C.c_int64), ("tol", C.c_double), ("epoch_cap", C.c_int),
                ("monotone_slack", C.c_double), ("root_seed", C.c_uint64), ("lambda1_hint", C.c_double)]


class Ledger(C.Structure):
    _fields_ = [(n, C.c_uint64) for n in (
        "gram_applies", "operator_applies", "qr_factorizations", "linear_solves",
        "solver_column_samples", "epochs", "outer_iterations")]

    def as_dict(self):
        return {k: int(getattr(self, k)) for k, _ in self._fields_}


class SiConfig(C.Structure):
    _fields_ = [("k", C.c_int), ("p", C.c_int), ("eps", C.c_double), ("mu", C.c_double),
                ("delta", C.c_double), ("lambda_", C.c_double), ("seed", C.c_uint64),
                ("tol_solve", C.c_double), ("tol_tune", C.c_double), ("conv_tol", C.c_double),
                ("rq_tol", C.c_double), ("max_outer", C.c_int), ("force", C.c_int),
                ("epoch_cap", C.c_int), ("monotone_slack", C.c_double), ("lambda1_hint", C.c_double),
                ("backend", C.c_int)]


class SiReport(C.Structure):
    _fields_ = [("lambda_", C.c_double), ("lambda1_hat", C.c_double), ("lambda1_hint", C.c_double),
                ("tune_steps", C.c_int),
                ("tune_lambda", C.c_double * 64), ("tune_inv", C.c_double * 64),
                ("outer_iterations", C.c_int), ("outer_cap", C.c_int), ("ledger", Ledger),
                ("ms_tune", C.c_double), ("ms_subspace", C.c_double),
                ("ms_rayleigh_ritz", C.c_double), ("ms_total", C.c_double)]


PROF_CLASSES = ["gram", "epoch", "h_pass", "index", "qr", "anchor", "block_gram", "gram_p1", "epoch_p1",
                "block_u", "r10", "r11"]


class ApReport(C.Structure):
    _fields_ = [("n_intervals", C.c_int), ("s", C.c_int * 64), ("q", C.c_int * 64), ("strategy", C.c_int * 64),
                ("width", C.c_int * 64), ("iterations", C.c_int * 64), ("shift", C.c_double * 64),
                ("ledger", Ledger), ("ms_total", C.c_double), ("delta", C.c_double)]


class Profile(C.Structure):
    _fields_ = [("ms", C.c_double * 12), ("count", C.c_uint64 * 12), ("bytes", C.c_double * 12),
                ("flops", C.c_double * 12)]

    def as_dict(self):
        return {name: {"ms": self.ms[i], "count": int(self.count[i]), "bytes": self.bytes[i],
                       "flops": self.flops[i]} for i, name in enumerate(PROF_CLASSES[:10])}


_SIGS = {
    "gaplra_launch_count": (C.c_ulonglong, []),
    "gaplra_host_syncs": (C.c_ulonglong, [C.c_void_p]),
    "gaplra_profile_enable": (C.c_int, [C.c_void_p, C.c_int]),
    "gaplra_profile_get": (C.c_int, [C.c_void_p, C.POINTER(Profile)]),
    "gaplra_profile_reset": (C.c_int, [C.c_void_p]),
    "gaplra_version": (C.c_int, []),
    "gaplra_ctx_create": (C.c_int, [C.c_int, C.POINTER(C.c_void_p)]),
    "gaplra_ctx_destroy": (C.c_int, [C.c_void_p]),
    "gaplra_last_error": (C.c_char_p, [C.c_void_p]),
    "gaplra_ctx_set_stream": (C.c_int, [C.c_void_p, C.c_void_p]),
    "gaplra_ctx_synchronize": (C.c_int, [C.c_void_p]),
    "gaplra_ledger_get": (C.c_int, [C.c_void_p, C.POINTER(Ledger)]),
    "gaplra_ledger_reset": (C.c_int, [C.c_void_p]),
    "gaplra_matrix_dense": (C.c_int, [C.c_void_p, C.c_int, C.c_int, C.c_void_p, C.c_int64, C.c_int,
                                      C.POINTER(C.c_void_p)]),
    "gaplra_matrix_csc": (C.c_int, [C.c_void_p, C.c_int, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p,
                                    C.c_int, C.POINTER(C.c_void_p)]),
    "gaplra_matrix_destroy": (C.c_int, [C.c_void_p]),
    "gaplra_matrix_info": (C.c_int, [C.c_void_p, _ip, _ip, _i64p, _i64p]),
    "gaplra_gram_apply": (C.c_int, [C.c_void_p, C.c_void_p, _dp, _dp]),
    "gaplra_gram_block": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int, _dp, _dp, _dp]),
    "gaplra_gram_block_device": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int, C.c_void_p, C.c_int64,
                                           C.c_void_p, C.c_int64, C.c_void_p, C.c_int64]),
    "gaplra_index_stream": (C.c_int, [C.c_void_p, C.c_uint64, C.c_uint64, C.c_int64, _i32p]),
    "gaplra_gaussian_init": (C.c_int, [C.c_int, C.c_int, C.c_uint64, _dp]),
    "gaplra_qr_orthonormalize": (C.c_int, [C.c_void_p, C.c_int, C.c_int, _dp, _dp, _ip]),
    "gaplra_orthonormality_defect": (C.c_int, [C.c_void_p, C.c_int, C.c_int, _dp, _dp]),
    "gaplra_jacobi_eigh": (C.c_int, [C.c_void_p, C.c_int, _dp, _dp, _dp]),
    "gaplra_svrg_epoch": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int, _dp, _dp, _dp, C.c_double,
                                    C.c_double, C.c_uint64, C.c_int64]),
    "gaplra_svrg_solve": (C.c_int, [C.c_void_p, C.c_void_p, C.c_double, C.c_int, _dp, _dp,
                                    C.POINTER(SvrgParams), C.c_int64, _ip, _dp, C.c_int, _ip]),
    "gaplra_estimate_top": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int, C.c_double, C.c_double,
                                      C.c_uint64, C.c_double, C.POINTER(SvrgParams), _i64p, _dp, _ip]),
    "gaplra_tune_shift": (C.c_int, [C.c_void_p, C.c_void_p, C.c_double, C.POINTER(SiConfig), _i64p,
                                    C.POINTER(SiReport)]),
    "gaplra_restricted_projection": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int, _dp, C.c_int, _dp, _dp]),
    "gaplra_shift_invert": (C.c_int, [C.c_void_p, C.c_void_p, C.POINTER(SiConfig), _dp, _dp, _dp,
                                      C.POINTER(SiReport)]),
    "gaplra_detect_multiplicative_gap": (C.c_int, [_dp, C.c_int, C.c_int, C.c_int, _ip]),
    "gaplra_detect_additive_gap": (C.c_int, [C.c_void_p, _dp, C.c_int, C.c_int, C.c_int, C.c_double, _ip]),
    "gaplra_estimate_eigenvalues": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int, C.c_double, C.c_int, C.c_double,
                                              C.c_uint64, C.c_double, C.POINTER(SvrgParams), _dp, _ip]),
    "gaplra_find_gap_budget": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int, C.c_int, C.c_uint64, C.c_double, _dp]),
    "gaplra_approximate": (C.c_int, [C.c_void_p, C.c_void_p, C.POINTER(SiConfig), _dp, _dp, C.POINTER(ApReport)]),
    "gaplra_accsvrg_solve": (C.c_int, [C.c_void_p, C.c_void_p, C.c_double, C.c_int, _dp, _dp, C.POINTER(SvrgParams),
                                       C.c_int64, _ip, _dp, C.c_int, _ip]),
    "gaplra_cg_solve": (C.c_int, [C.c_void_p, C.c_void_p, C.c_double, C.c_int, _dp, _dp, C.c_double, C.c_int,
                                  _ip, _dp, C.c_int, _ip]),
    "gaplra_error_report": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int, _dp, C.c_int, C.c_uint64, _dp, _dp]),
    "gaplra_principal_angles": (C.c_int, [C.c_void_p, C.c_int, C.c_int, _dp, C.c_int, _dp, _dp]),
}


def header_symbols() -> list[str]:
    """Every entry point include/gaplra_cuda.h declares."""
    return re.findall(r"GAPLRA_API\s+(?:int|const char\*|unsigned long long)\s+(gaplra_\w+)\(", HEADER.read_text())


_LIB = None


def load(path: Path | None = None) -> C.CDLL:
    """Load libgaplra_cuda.so; raises (no CPU fallback) if it is not built."""
    global _LIB
    if _LIB is not None and path is None:
        return _LIB
    p = Path(path or os.environ.get("GAPLRA_CUDA_LIB", LIB_PATH))
    if not p.exists():
        raise ImportError(f"{p} is not built: run `python -c 'import __graft_entry__ as g; g.build()'` "
                          "(the product path has no CPU fallback)")
    lib = C.CDLL(str(p))
    for name, (res, args) in _SIGS.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    if path is None:
        _LIB = lib
    return lib
