"""Small-n probe of a config's epoch layout (d, p from the config, n reduced):
one solve capped at 2 epochs, printing the chosen layout and per-class times."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch

import paper_1607_02925_b200 as g

d, n, p = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
gen = torch.Generator(device="cuda")
gen.manual_seed(1)
XT = torch.randn(n, d, generator=gen, dtype=torch.float64, device="cuda") / np.sqrt(n)
x = g.DeviceMatrix.from_device(XT.data_ptr(), d, n, d, keep=XT)
ctx = g.default_context()
ctx.enable_profiling(True)
W = np.random.default_rng(0).standard_normal((d, p))
t = time.time()
try:
    g.solve_svrg(x, 4.0, W, 1e-12, seed=1, epoch_cap=2)
except g.SolverStalled:
    pass
print({"d": d, "n": n, "p": p, "wall_s": round(time.time() - t, 3),
       "prof": {k: round(v["ms"] / max(v["count"], 1), 3) for k, v in ctx.profile().items() if v["count"]}}, flush=True)
