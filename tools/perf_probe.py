"""GPU probe: generate a config on the device, time the units and the full
pipeline with the runtime's live CUDA-event profile.  Usage:
  python tools/perf_probe.py C2 [--pipeline] [--max-outer N]"""
import argparse
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch

import paper_1607_02925_b200 as g
from paper_1607_02925_b200.configs import CONFIGS, make_dense_xt

ap = argparse.ArgumentParser()
ap.add_argument("cfg", default="C2", nargs="?")
ap.add_argument("--pipeline", action="store_true")
ap.add_argument("--max-outer", type=int, default=0)
ap.add_argument("--solve", action="store_true")
a = ap.parse_args()
spec = CONFIGS[a.cfg]
t0 = time.time()
XT, U = make_dense_xt(spec)
if a.cfg == "C1":
    pass
torch.cuda.synchronize()
print(json.dumps({"gen_s": time.time() - t0, "cfg": a.cfg}), flush=True)
ctx = g.default_context()
x = g.DeviceMatrix.from_device(XT.data_ptr(), spec.d, spec.n, spec.d, ctx=ctx, keep=XT)
ctx.enable_profiling(True)
rng = np.random.default_rng(0)
for p in (1, spec.p):
    W = rng.standard_normal((spec.d, p))
    for _ in range(2):
        g.gram_block(x, W)
    ctx.reset_profile()
    for _ in range(5):
        g.gram_block(x, W)
    pr = ctx.profile()["gram" if p > 1 else "gram_p1"]
    t = pr["ms"] / pr["count"] / 1e3
    print(json.dumps({"unit": "gram", "p": p, "ms": t * 1e3, "GBps": pr["bytes"] / pr["count"] / t / 1e9,
                      "TFLOPs": pr["flops"] / pr["count"] / t / 1e12}), flush=True)
lam = float(spec.eig()[0] + spec.delta() / 10)
if a.solve:
    for p in (1, spec.p):
        B = rng.standard_normal((spec.d, p))
        ctx.reset_profile()
        t = time.time()
        try:
            r = g.solve_svrg(x, lam, B, 1e-10, seed=1, epoch_cap=3)
        except g.SolverStalled as e:
            pass
        prof = ctx.profile()
        out = {"unit": "solve3epochs", "p": p, "wall_s": time.time() - t}
        for k, v in prof.items():
            if v["count"]:
                tt = v["ms"] / v["count"] / 1e3
                out[k] = {"ms_per": tt * 1e3, "count": v["count"], "GBps": v["bytes"] / v["count"] / tt / 1e9,
                          "TFLOPs": v["flops"] / v["count"] / tt / 1e12}
        print(json.dumps(out), flush=True)
if a.pipeline:
    lam, hint = 0.0, 0.0
    if a.cfg == "C1":  # NoPreconditioningNeeded fires on C1: explicit shift
        lam = float(spec.eig()[0] + spec.delta() / 10)
        hint = float(spec.eig()[0])
    cfg = g.SIConfig(k=spec.k, p=spec.p, eps=spec.eps, mu=spec.mu(), delta=spec.delta(), seed=spec.seed,
                     max_outer=a.max_outer, lam=lam, lambda1_hint=hint)
    ctx.reset_profile()
    ctx.reset_ledger()
    t = time.time()
    res = g.shift_invert(x, cfg)
    wall = time.time() - t
    prof = ctx.profile()
    print(json.dumps({"pipeline_wall_s": wall, "ms": res.ms, "lam": res.lam, "tune": res.tune_history,
                      "outer": res.outer_iterations, "ledger": res.ledger, "ritz": res.ritz.tolist(),
                      "prof": {k: v for k, v in prof.items() if v["count"]}}), flush=True)
