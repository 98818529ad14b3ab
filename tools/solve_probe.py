"""Launch-list probe for one C2-shaped block SVRG solve (3 epochs) without the
planting launches: random device X (4096 x 100000), p = 20 (or argv[1]).
Usage (on the GPU box): ncu --metrics gpu__time_duration.sum -c N python tools/solve_probe.py [p]"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch

import paper_1607_02925_b200 as g

p = int(sys.argv[1]) if len(sys.argv) > 1 else 20
d, n = 4096, 100000
XT = torch.randn(n, d, dtype=torch.float64, device="cuda") / np.sqrt(n)
x = g.DeviceMatrix.from_device(XT.data_ptr(), d, n, d, keep=XT)
lam = 1.2 * (1.0 + np.sqrt(d / n)) ** 2  # above lambda_1 of X Xᵀ (Marchenko–Pastur edge)
B = np.random.default_rng(0).standard_normal((d, p))
try:
    g.solve_svrg(x, lam, B, 1e-14, seed=1, epoch_cap=3, lambda1_hint=lam / 1.2)
except g.SolverStalled:
    pass
torch.cuda.synchronize()
print("done")
