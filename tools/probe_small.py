"""Minimal C2 epoch run for ncu: one p=20 and one p=1 solve capped at 2 epochs."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np

import paper_1607_02925_b200 as g
from paper_1607_02925_b200.configs import CONFIGS, make_dense_xt

spec = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "C2"]
XT, U = make_dense_xt(spec)
x = g.DeviceMatrix.from_device(XT.data_ptr(), spec.d, spec.n, spec.d, keep=XT)
lam = float(spec.eig()[0] + spec.delta() / 10)
rng = np.random.default_rng(0)
for p in (spec.p, 1):
    try:
        g.solve_svrg(x, lam, rng.standard_normal((spec.d, p)), 1e-12, seed=1, epoch_cap=2)
    except g.SolverStalled:
        pass
print("ok")
