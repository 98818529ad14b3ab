"""Per-epoch device time of a solve at a config's epoch layout, with the
per-class split (for the side-stream scheduling variants, GAPLRA_OVERLAP).
    python tools/epoch_sched.py C5 [p ...]"""
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch

import paper_1607_02925_b200 as g
from paper_1607_02925_b200.configs import CONFIGS, make_dense_xt

spec = CONFIGS[sys.argv[1]]
ps = [int(v) for v in sys.argv[2:]] or [1, spec.p]
XT, _ = make_dense_xt(spec)
torch.cuda.synchronize()
ctx = g.default_context()
x = g.DeviceMatrix.from_device(XT.data_ptr(), spec.d, spec.n, spec.d, ctx=ctx, keep=XT)
lam = float(spec.eig()[0] * 1.04)
rng = np.random.default_rng(0)
for p in ps:
    B = rng.standard_normal((spec.d, p))
    for rep in range(2):
        ctx.enable_profiling(rep == 1)
        ctx.reset_profile()
        torch.cuda.synchronize()
        t = time.time()
        try:
            g.solve_svrg(x, lam, B, 1e-14, seed=1, epoch_cap=6)
        except g.SolverStalled:
            pass
        torch.cuda.synchronize()
        wall = time.time() - t
    prof = ctx.profile()
    ep = prof["epoch" if p > 1 else "epoch_p1"]["count"]
    out = {"cfg": spec.name, "p": p, "epochs": ep, "wall_ms_per_epoch": wall * 1e3 / max(ep, 1)}
    for k, v in prof.items():
        if v["count"]:
            out[k] = round(v["ms"] / v["count"], 3)
    print(json.dumps(out), flush=True)
