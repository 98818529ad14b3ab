"""Device time of the bench step (one shift-and-invert outer iteration at the tuned shift) under the current
GAPLRA_* environment, profiling off.   python tools/step_time.py [C5] [reps]"""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch

import paper_1607_02925_b200 as g
from paper_1607_02925_b200.configs import CONFIGS, make_dense_xt

name = sys.argv[1] if len(sys.argv) > 1 else "C5"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
LAM = {"C5": (1.0416918791917118, 1.0045493671607475)}
spec = CONFIGS[name]
XT, _ = make_dense_xt(spec)
torch.cuda.synchronize()
ctx = g.default_context()
x = g.DeviceMatrix.from_device(XT.data_ptr(), spec.d, spec.n, spec.d, ctx=ctx, keep=XT)
lam, hint = LAM[name]
cfg = g.SIConfig(k=spec.k, p=spec.p, eps=spec.eps, mu=spec.mu(), delta=spec.delta(), seed=spec.seed, lam=lam,
                 lambda1_hint=hint, max_outer=1)
out = []
for _ in range(reps + 1):
    r = g.shift_invert(x, cfg)
    out.append(round(r.ms["total"], 1))
print(json.dumps({"config": name, "step_ms": out[1:], "first_ms": out[0], "epochs": r.ledger["epochs"]}))
