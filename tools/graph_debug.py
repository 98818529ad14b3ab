"""Debug probe for the device-resident epoch loop (graph mode) on small solves."""
import sys
sys.path.insert(0, '/root/repo')
sys.path.insert(0, '/root/repo/tests')
import numpy as np

import paper_1607_02925_b200 as g
from problems import planted_dense

for d, n, p in [(32, 3000, 1), (30, 3000, 1), (30, 3000, 4), (2048, 4000, 1), (2048, 4000, 20), (8192, 3000, 64)]:
    try:
        X, _, _ = planted_dense(d, n, seed=1)
        x = g.DeviceMatrix.dense(X)
        r = g.solve_svrg(x, 1.05 * np.linalg.norm(X, 2) ** 2, np.ones((d, p)), 1e-10, seed=1)
        print(d, n, p, "ok epochs", r.epochs, flush=True)
    except Exception as e:
        print(d, n, p, "ERR", e, flush=True)
