"""Time-to-ε of a config's pipeline through the public API with per-kernel
profiling off (the production path), printing host syncs; run once with
GAPLRA_GRAPH=0 (host-driven epoch loop) and once without (device-resident).
    python tools/graph_timing.py C1 [reps]"""
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch

import paper_1607_02925_b200 as g
from paper_1607_02925_b200.configs import CONFIGS, make_dense_xt

name = sys.argv[1] if len(sys.argv) > 1 else "C1"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
spec = CONFIGS[name]
XT, _ = make_dense_xt(spec)
torch.cuda.synchronize()
ctx = g.default_context()
x = g.DeviceMatrix.from_device(XT.data_ptr(), spec.d, spec.n, spec.d, ctx=ctx, keep=XT)
lam, hint = 0.0, 0.0
if name == "C1":
    lam, hint = float(spec.eig()[0] + spec.delta() / 10), float(spec.eig()[0])
cfg = g.SIConfig(k=spec.k, p=spec.p, eps=spec.eps, mu=spec.mu(), delta=spec.delta(), seed=spec.seed, lam=lam,
                 lambda1_hint=hint)
g.shift_invert(x, cfg)
out = []
for _ in range(reps):
    s0 = ctx.host_syncs()
    t = time.perf_counter()
    r = g.shift_invert(x, cfg)
    wall = time.perf_counter() - t
    out.append({"device_s": r.ms["total"] / 1e3, "wall_s": wall, "host_syncs": ctx.host_syncs() - s0,
                "epochs": r.ledger["epochs"], "solves": r.ledger["linear_solves"], "outer": r.outer_iterations})
print(json.dumps({"config": name, "runs": out}))
