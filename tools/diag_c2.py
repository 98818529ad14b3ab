"""Diagnose the C2 pipeline: tune_shift history, then SVRG residual histories."""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np

import paper_1607_02925_b200 as g
from paper_1607_02925_b200.configs import CONFIGS, make_dense_xt

spec = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "C2"]
XT, U = make_dense_xt(spec)
x = g.DeviceMatrix.from_device(XT.data_ptr(), spec.d, spec.n, spec.d, keep=XT)
import torch
ev = torch.linalg.eigvalsh(XT.T @ XT).flip(0)[:30].cpu().numpy()
print(json.dumps({"top_eigs": ev[:25].tolist(), "delta": spec.delta()}), flush=True)
cfg = g.SIConfig(k=spec.k, p=spec.p, eps=spec.eps, mu=spec.mu(), delta=spec.delta(), seed=spec.seed)
try:
    st = g.tune_shift(x, spec.delta(), cfg)
    print(json.dumps({"tune_lambda": st.lam, "l1hat": st.lambda1_hat, "history": st.history}), flush=True)
    lam = st.lam
except g.Error as e:
    print("tune failed", type(e).__name__, e, getattr(e, "history", None), flush=True)
    lam = float(ev[0] + spec.delta() / 10)
rng = np.random.default_rng(0)
for lam_try in (lam, float(ev[0]) + 0.05, float(ev[0]) + 0.2):
    for p in (1, spec.p):
        try:
            r = g.solve_svrg(x, lam_try, rng.standard_normal((spec.d, p)), 1e-10, seed=3)
            print(json.dumps({"lam": lam_try, "gap": lam_try - float(ev[0]), "p": p, "epochs": r.epochs,
                              "hist": [round(h, 12) for h in r.residual_history[::5]]}), flush=True)
        except g.SolverStalled as e:
            print(json.dumps({"lam": lam_try, "gap": lam_try - float(ev[0]), "p": p, "STALLED": str(e),
                              "hist": e.residual_history}), flush=True)
