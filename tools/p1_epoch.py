"""p = 1 epoch of a dense config under the current GAPLRA_* environment: a
small-n lockstep check against the oracle at the config's d (same chain
layout), then 3 epochs of a solve at full size with the per-class times.
    GAPLRA_P1_XG=1 python tools/p1_epoch.py C2 [p]"""
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))
import numpy as np
import torch

import paper_1607_02925_b200 as g
from oracle_lib import Oracle
from paper_1607_02925_b200.configs import CONFIGS, make_dense_xt

name = sys.argv[1] if len(sys.argv) > 1 else "C2"
p = int(sys.argv[2]) if len(sys.argv) > 2 else 1
spec = CONFIGS[name]
o = Oracle()
d, n, m = spec.d, 300, 1000
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
wd = g.svrg_epoch(xm, w0, y, c, eta, lam, 31, m)
err = float(np.abs(wd - wo).max() / np.abs(wo).max())
same = all(np.array_equal(g.svrg_epoch(xm, w0, y, c, eta, lam, 31, m), wd) for _ in range(5))
XT, _ = make_dense_xt(spec)
torch.cuda.synchronize()
ctx = g.default_context()
x = g.DeviceMatrix.from_device(XT.data_ptr(), spec.d, spec.n, spec.d, ctx=ctx, keep=XT)
ctx.enable_profiling(True)
lam = float(spec.eig()[0] + spec.delta() / 10)
B = np.random.default_rng(0).standard_normal((spec.d, p))
ctx.reset_profile()
try:
    g.solve_svrg(x, lam, B, 1e-10, seed=1, epoch_cap=4)
except g.SolverStalled:
    pass
prof = {k: round(v["ms"] / v["count"], 3) for k, v in ctx.profile().items() if v["count"]}
print(json.dumps({"config": name, "p": p, "lockstep_rel_err": err, "bitwise_reruns": same, "ms_per_launch": prof}), flush=True)
assert err <= 1e-10 and same
