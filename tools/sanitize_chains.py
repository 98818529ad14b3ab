"""Race / protocol stress of every chain layout (compute-sanitizer is closed on
this GPU pool, so the evidence is behavioural): each layout's epoch is checked
against the CPU oracle, then re-run R times — alone and beside a perturbing
torch GEMM stream that shifts the CTAs' relative timing — and every re-run must
be bitwise identical to the first.  A race in the mbarrier / named-barrier /
DSMEM / L2-exchange protocols shows up as a mismatch or a hang.
    python tools/sanitize_chains.py [R]"""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))
import numpy as np
import torch

import paper_1607_02925_b200 as g
from oracle_lib import Oracle
from problems import random_csc

o = Oracle()
R = int(sys.argv[1]) if len(sys.argv) > 1 else 0
noise_stream = torch.cuda.Stream()
na = torch.randn(4096, 4096, device="cuda")


def perturb():
    with torch.cuda.stream(noise_stream):
        for _ in range(8):
            na.copy_(na @ na * 1e-3)


def stress(run, ref):
    bad = 0
    for r in range(R):
        if r % 2:
            perturb()
        if not np.array_equal(run(), ref):
            bad += 1
    return bad


LAYOUTS = [  # (d, n, p, m, what)
    (4096, 200, 1, 70, "v3 RR p=1, 16-CTA cluster x 256 rows (C2)"),
    (2048, 200, 1, 70, "v3 RR p=1, 8-CTA cluster (C3)"),
    (8192, 200, 1, 70, "v3 RR H=2 p=1, 512 rows (C5)"),
    (4096, 200, 20, 70, "v4 DSMEM, 3 groups (C2)"),
    (2048, 200, 32, 70, "v4 DSMEM, 8-CTA clusters (C3)"),
    (8192, 200, 64, 70, "v4 512 rows, L2 exchange, half-stage ring (C5)"),
    (1000, 200, 10, 70, "v3 PC<=3, d<=1024 (C1)"),
]
worst = 0.0
for d, n, p, m, what in LAYOUTS:
    rng = np.random.default_rng(d + p)
    X = rng.standard_normal((d, n)) / np.sqrt(n)
    mo = o.dense(X)
    w0 = rng.standard_normal((d, p))
    _, z, y = o.gram_block(mo, w0, want_y=True)
    lam = 1.2 * np.linalg.norm(X, 2) ** 2
    eta = 1.0 / (4.0 * (lam + n * o.max_col_norm2(mo)))
    c = eta * (z + rng.standard_normal((d, p)))
    _, wo, _ = o.svrg_epoch(mo, w0, y, c, eta, lam, 31, m)
    xm = g.DeviceMatrix.dense(X)
    m_long = 4000 if R else m
    wd = g.svrg_epoch(xm, w0, y, c, eta, lam, 31, m)
    err = float(np.abs(wd - wo).max() / np.abs(wo).max())
    worst = max(worst, err)
    bad = 0
    if R:
        ref = g.svrg_epoch(xm, w0, y, c, eta, lam, 32, m_long)
        bad = stress(lambda: g.svrg_epoch(xm, w0, y, c, eta, lam, 32, m_long), ref)
        worst = max(worst, float(bad))
    print(f"{what}: rel err {err:.2e}; {R} re-runs of m={m_long}: {bad} not bitwise identical", flush=True)
cp, ri, v = random_csc(2000, 4000, 20, seed=3)
mo = o.csc(2000, 4000, cp, ri, v)
rng = np.random.default_rng(1)
w0 = rng.standard_normal((2000, 16))
_, z, y = o.gram_block(mo, w0, want_y=True)
lam = 1.5 * float(np.sum(v * v))
eta = 1.0 / (4.0 * (lam + 4000 * o.max_col_norm2(mo)))
c = eta * (z + rng.standard_normal((2000, 16)))
_, wo, _ = o.svrg_epoch(mo, w0, y, c, eta, lam, 5, 700)
xs = g.DeviceMatrix.csc(2000, 4000, cp, ri, v)
wd = g.svrg_epoch(xs, w0, y, c, eta, lam, 5, 700)
err = float(np.abs(wd - wo).max() / np.abs(wo).max())
worst = max(worst, err)
bad = 0
if R:
    ref = g.svrg_epoch(xs, w0, y, c, eta, lam, 6, 8000)
    bad = stress(lambda: g.svrg_epoch(xs, w0, y, c, eta, lam, 6, 8000), ref)
    worst = max(worst, float(bad))
print(f"blocked sparse epoch: rel err {err:.2e}; {R} re-runs: {bad} not bitwise identical")
print("sanitize_chains", "ok" if worst <= 1e-10 else "FAIL", worst)
