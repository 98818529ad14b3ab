"""Generate tests/golden/ref_vectors.json from the REFERENCE's own shipped
sources (oracle/_ref/libgaplra_ref.so = /root/reference/proj/core/src/*.cpp +
oracle/ref_shim.cpp, built by `make -C oracle ref`).  Run in the build
container (the reference is not present on the GPU box):

    python tests/golden/make_golden.py

Small inputs are stored in the fixture, so the tests never regenerate them.
"""
import json
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parent))
from oracle_lib import REF_SO, Reference, build_oracle  # noqa: E402


def hexs(a):
    return [float(x).hex() for x in np.asarray(a, dtype=np.float64).ravel()]


def main():
    if not REF_SO.exists():
        build_oracle(ref=True)
    r = Reference()
    rng = np.random.default_rng(20260101)
    out = {"source": "reference sources /root/reference/proj/core/src/*.cpp via oracle/_ref (this script)"}
    out["derive_seed"] = [[root, tag, r.derive_seed(root, tag)] for root, tag in
                          [(0, 0x6761757373), (1, 0), (2**63 + 7, 12345), (42, 0x73767267 ^ (3 << 20) ^ 5)]]
    out["next_u64"] = {str(s): [int(v) for v in r.next_u64(s, 16)] for s in (0, 1, 0x039B1995888F80DB)}
    out["uniform_index"] = [[s, n, [int(v) for v in r.uniform_index(s, n, 64)]] for s, n in
                            [(0, 5000), (7, 1), (9, 3), (11, 2_000_000), (13, 100_000), (2**40, 2**31 - 1)]]
    out["normal"] = {str(s): hexs(r.normal(s, 17)) for s in (0, 5)}
    out["gaussian_init"] = [[d, p, s, hexs(r.gaussian_init(d, p, s)[1])] for d, p, s in [(4, 2, 0), (9, 3, 77)]]
    qr = []
    for d, p in [(6, 3), (40, 5)]:
        y = rng.standard_normal((d, p))
        rc, q, bad = r.qr(y)
        qr.append({"y": hexs(y), "d": d, "p": p, "rc": rc, "q": hexs(q), "bad": bad})
    y = rng.standard_normal((8, 3))
    y[:, 2] = y[:, 0] - y[:, 1]
    rc, q, bad = r.qr(y)
    qr.append({"y": hexs(y), "d": 8, "p": 3, "rc": rc, "q": None, "bad": bad})
    out["qr"] = qr
    jac = []
    for n in (1, 3, 7, 12):
        h = rng.standard_normal((n, n))
        h = h + h.T
        rc, vals, vecs = r.jacobi(h)
        jac.append({"n": n, "h": hexs(h), "vals": hexs(vals), "vecs": hexs(vecs)})
    rc, vals, vecs = r.jacobi(np.array([[4.0, 1, 0], [1, 3, 0], [0, 0, 1]]))
    jac.append({"n": 3, "h": hexs(np.array([[4.0, 1, 0], [1, 3, 0], [0, 0, 1]])), "vals": hexs(vals),
                "vecs": hexs(vecs)})
    out["jacobi"] = jac
    x = rng.standard_normal((7, 11))
    x[2, 3] = 0.0  # exact zero: dropped by from_dense
    v = rng.standard_normal(7)
    out["gram_dense"] = {"x": hexs(x), "d": 7, "n": 11, "v": hexs(v), "out": hexs(r.gram_apply_dense(x, v)[1])}
    colptr = np.array([0, 2, 2, 5, 6], dtype=np.int64)
    rowidx = np.array([0, 4, 1, 2, 5, 3], dtype=np.int32)
    val = rng.standard_normal(6)
    v = rng.standard_normal(6)
    out["gram_csc"] = {"d": 6, "n": 4, "colptr": colptr.tolist(), "rowidx": rowidx.tolist(), "val": hexs(val),
                       "v": hexs(v), "out": hexs(r.gram_apply_csc(6, 4, colptr, rowidx, val, v)[1])}
    # one SVRG epoch built only from reference primitives (SPEC.md:362 direct form)
    d, n, p = 10, 24, 3
    x = rng.standard_normal((d, n)) / np.sqrt(n)
    w = rng.standard_normal((d, p))
    yv = x.T @ w
    cb = 1e-3 * rng.standard_normal((d, p))
    eta, lam = 0.01, 3.0
    rc, w1, idx = r.svrg_epoch_dense(x, w, yv, cb, eta, lam, 4242, 48)
    out["svrg_epoch"] = {"d": d, "n": n, "p": p, "x": hexs(x), "w": hexs(w), "y": hexs(yv), "c": hexs(cb),
                         "eta": eta, "lam": lam, "seed": 4242, "m": 48, "w_out": hexs(w1),
                         "idx": [int(i) for i in idx]}
    (HERE / "ref_vectors.json").write_text(json.dumps(out, indent=0))
    print("wrote", HERE / "ref_vectors.json")


if __name__ == "__main__":
    main()
