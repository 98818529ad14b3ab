"""Wall/device time of one SVRG solve capped at a few epochs, profiling off (production path).
    python tools/solve_time.py C5 1 [epochs]"""
import json, sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np, torch
import paper_1607_02925_b200 as g
from paper_1607_02925_b200.configs import CONFIGS, make_dense_xt
name, p = sys.argv[1], int(sys.argv[2])
cap = int(sys.argv[3]) if len(sys.argv) > 3 else 8
spec = CONFIGS[name]
XT, _ = make_dense_xt(spec); torch.cuda.synchronize()
ctx = g.default_context()
x = g.DeviceMatrix.from_device(XT.data_ptr(), spec.d, spec.n, spec.d, ctx=ctx, keep=XT)
lam = float(spec.eig()[0] + spec.delta() / 10)
B = np.random.default_rng(0).standard_normal((spec.d, p))
out = []
for _ in range(3):
    torch.cuda.synchronize(); t = time.perf_counter()
    try:
        g.solve_svrg(x, lam, B, 1e-14, seed=1, epoch_cap=cap)
    except g.SolverStalled:
        pass
    torch.cuda.synchronize(); out.append(round((time.perf_counter() - t) * 1e3, 1))
print(json.dumps({"config": name, "p": p, "epoch_cap": cap, "wall_ms": out, "syncs": ctx.host_syncs()}))
