"""C4 sparse probe: plant the C4 CSC (n reducible), upload through the C ABI,
time gram passes and a 2-epoch solve at p = 16 and p = 1 with the blocked
sparse epoch (GAPLRA_SPARSE_BLOCKED=0 for the step-by-step kernel).

    python tools/sparse_probe.py [n]
"""
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np

import paper_1607_02925_b200 as g
from paper_1607_02925_b200.configs import CONFIGS, make_sparse_csc

spec = CONFIGS["C4"]
n = int(sys.argv[1]) if len(sys.argv) > 1 else spec.n
t = time.time()
cp, ri, v = make_sparse_csc(spec, n=n)
gen = time.time() - t
t = time.time()
ctx = g.default_context()
x = g.DeviceMatrix.csc(spec.d, n, cp, ri, v, ctx=ctx)
up = time.time() - t
print(json.dumps({"n": n, "nnz": int(cp[-1]), "gen_s": gen, "upload_s": up}), flush=True)
ctx.enable_profiling(True)
rng = np.random.default_rng(0)
for p in (spec.p, 1):
    W = rng.standard_normal((spec.d, p))
    g.gram_block(x, W)
    ctx.reset_profile()
    t = time.time()
    try:
        g.solve_svrg(x, 3.0, W, 1e-12, seed=1, epoch_cap=2)
    except g.SolverStalled:
        pass
    prof = {k: {"ms_per": v["ms"] / v["count"], "count": v["count"]} for k, v in ctx.profile().items() if v["count"]}
    print(json.dumps({"p": p, "wall_s": time.time() - t, "prof": prof}), flush=True)
