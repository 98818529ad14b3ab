"""C4 at full size: one p = 16 (or argv[1]) SVRG epoch on the device, timed (no oracle)."""
import sys, time
from pathlib import Path
ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT)); sys.path.insert(0, str(ROOT / "tests"))
import numpy as np
import paper_1607_02925_b200 as g
from paper_1607_02925_b200.configs import CONFIGS, make_sparse_csc
spec = CONFIGS["C4"]
p = int(sys.argv[1]) if len(sys.argv) > 1 else 16
cp, ri, v = make_sparse_csc(spec)
x = g.DeviceMatrix.csc(spec.d, spec.n, cp, ri, v)
rng = np.random.default_rng(3)
w0 = rng.standard_normal((spec.d, p))
lam = 2030.76
nrm2 = np.add.reduceat(v * v, cp[:-1]).max()
eta = 1.0 / (4.0 * (lam + spec.n * nrm2))
y = np.zeros((spec.n, p)); c = eta * rng.standard_normal((spec.d, p))
for _ in range(2):
    t = time.time(); g.svrg_epoch(x, w0, y, c, eta, lam, 31, 2 * spec.n); print("wall_s", round(time.time() - t, 3), flush=True)
