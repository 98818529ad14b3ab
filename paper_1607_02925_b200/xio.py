"""Binary X files with a JSON spectrum sidecar.

The reference reads X only as text (Matrix Market / CSV, proj/core/src/
matrix_io.cpp:87-239); at C2–C5 sizes (3.3–65.5 GB of fp64) text IO dominates
and C5 does not fit host RAM twice.  This format is the device path's:

  <path>        raw little-endian fp64 (dense: column-major, d*n values;
                CSC: colptr int64[n+1] | rowidx int32[nnz] | val fp64[nnz])
  <path>.json   {"format": "gaplra-x/1", "kind": "dense"|"csc", "d", "n", "nnz",
                 "sha256", plus caller metadata such as the planted sigma, k, p,
                 seed, and the recipe}

`load_dense_device` streams the file to HBM in column chunks (bounded host
memory), verifying the SHA-256 on the way, and returns a DeviceMatrix that
borrows the device buffer.  The sidecar is plain JSON so the oracle and the
tests can read the planted spectrum without touching X.
"""
from __future__ import annotations

import hashlib
import json
from pathlib import Path

import numpy as np

FORMAT = "gaplra-x/1"
_CHUNK_BYTES = 256 << 20


def _sidecar(path: Path) -> Path:
    return Path(str(path) + ".json")


def save_dense(path, X: np.ndarray, **meta) -> dict:
    """Write X (d x n float64) column-major plus the sidecar; returns the sidecar."""
    path = Path(path)
    X = np.asarray(X, dtype=np.float64)
    d, n = X.shape
    h = hashlib.sha256()
    with open(path, "wb") as f:
        step = max(1, _CHUNK_BYTES // (8 * d))
        for j in range(0, n, step):
            blk = np.asfortranarray(X[:, j:j + step]).tobytes(order="F")
            h.update(blk)
            f.write(blk)
    side = {"format": FORMAT, "kind": "dense", "d": d, "n": n, "nnz": d * n, "dtype": "f64",
            "layout": "column-major", "sha256": h.hexdigest(), **meta}
    _sidecar(path).write_text(json.dumps(side, indent=1))
    return side


def save_csc(path, d: int, n: int, colptr, rowidx, val, **meta) -> dict:
    path = Path(path)
    colptr = np.ascontiguousarray(colptr, dtype=np.int64)
    rowidx = np.ascontiguousarray(rowidx, dtype=np.int32)
    val = np.ascontiguousarray(val, dtype=np.float64)
    if colptr.shape != (n + 1,) or rowidx.shape != val.shape or colptr[-1] != len(val):
        raise ValueError("save_csc: inconsistent CSC arrays")
    h = hashlib.sha256()
    with open(path, "wb") as f:
        for a in (colptr, rowidx, val):
            b = a.tobytes()
            h.update(b)
            f.write(b)
    side = {"format": FORMAT, "kind": "csc", "d": d, "n": n, "nnz": int(len(val)), "sha256": h.hexdigest(), **meta}
    _sidecar(path).write_text(json.dumps(side, indent=1))
    return side


def read_sidecar(path) -> dict:
    side = json.loads(_sidecar(Path(path)).read_text())
    if side.get("format") != FORMAT:
        raise ValueError(f"{path}: not a {FORMAT} file")
    return side


def load_dense(path, verify: bool = True) -> tuple[np.ndarray, dict]:
    """Host copy of a dense file (d x n, Fortran order) and its sidecar."""
    side = read_sidecar(path)
    if side["kind"] != "dense":
        raise ValueError(f"{path}: kind {side['kind']}, not dense")
    raw = np.fromfile(path, dtype="<f8")
    if verify and hashlib.sha256(raw.tobytes()).hexdigest() != side["sha256"]:
        raise ValueError(f"{path}: SHA-256 mismatch")
    return raw.reshape((side["d"], side["n"]), order="F"), side


def load_csc(path, verify: bool = True):
    side = read_sidecar(path)
    if side["kind"] != "csc":
        raise ValueError(f"{path}: kind {side['kind']}, not csc")
    n, nnz = side["n"], side["nnz"]
    raw = Path(path).read_bytes()
    if verify and hashlib.sha256(raw).hexdigest() != side["sha256"]:
        raise ValueError(f"{path}: SHA-256 mismatch")
    o1 = 8 * (n + 1)
    o2 = o1 + 4 * nnz
    colptr = np.frombuffer(raw[:o1], dtype="<i8")
    rowidx = np.frombuffer(raw[o1:o2], dtype="<i4")
    val = np.frombuffer(raw[o2:o2 + 8 * nnz], dtype="<f8")
    return (side["d"], n, colptr, rowidx, val), side


def load_dense_device(path, ctx=None, verify: bool = True):
    """Stream a dense file into HBM (column chunks of <= 256 MB through host
    memory) and return (DeviceMatrix borrowing the buffer, sidecar).  The
    device buffer is column-major with ld = round_up(d, 4) and zero pad rows."""
    import torch

    from .gaplra import DeviceMatrix, default_context

    side = read_sidecar(path)
    if side["kind"] != "dense":
        raise ValueError(f"{path}: kind {side['kind']}, not dense")
    d, n = side["d"], side["n"]
    ld = (d + 3) // 4 * 4
    XT = torch.zeros((n, ld), dtype=torch.float64, device="cuda")  # row j of XT = column j of X
    h = hashlib.sha256()
    step = max(1, _CHUNK_BYTES // (8 * d))
    with open(path, "rb") as f:
        for j in range(0, n, step):
            cols = min(step, n - j)
            b = f.read(8 * d * cols)
            if len(b) != 8 * d * cols:
                raise ValueError(f"{path}: truncated")
            if verify:
                h.update(b)
            blk = torch.frombuffer(bytearray(b), dtype=torch.float64).view(cols, d)
            XT[j:j + cols, :d].copy_(blk, non_blocking=False)
    if verify and h.hexdigest() != side["sha256"]:
        raise ValueError(f"{path}: SHA-256 mismatch")
    ctx = ctx or default_context()
    return DeviceMatrix.from_device(XT.data_ptr(), d, n, ld, ctx=ctx, keep=XT), side
