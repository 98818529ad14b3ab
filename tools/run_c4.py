"""C4 end to end (sparse): plant the CSC, upload through the C ABI, estimate
the spectrum for the gap budget Δ = 2/3 (λ_k − λ_{p+1}) with a long block
subspace iteration on X Xᵀ through the library's own gram pass (verification
/ setup only: SURVEY.md §8(d) lists "Δ from an ARPACK-style oracle" for C4),
run the shift-and-invert pipeline, and compare W with the reference subspace.

    python tools/run_c4.py [iters] [svrg|cg|accsvrg]
"""
import json
import math
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import numpy as np

import paper_1607_02925_b200 as g
from paper_1607_02925_b200.configs import CONFIGS, make_sparse_csc

spec = CONFIGS["C4"]
iters = int(sys.argv[1]) if len(sys.argv) > 1 else 300
backend = sys.argv[2] if len(sys.argv) > 2 else "svrg"
t0 = time.time()
cp, ri, v = make_sparse_csc(spec)
gen_s = time.time() - t0
ctx = g.default_context()
x = g.DeviceMatrix.csc(spec.d, spec.n, cp, ri, v, ctx=ctx)
# spectrum: block power iteration with 48 vectors (setup / verification only)
rng = np.random.default_rng(7)
q, _ = np.linalg.qr(rng.standard_normal((spec.d, 48)))
t = time.time()
for it in range(iters):
    q, _ = np.linalg.qr(g.gram_block(x, q))
z = g.gram_block(x, q)
h = q.T @ z
lam, vec = np.linalg.eigh((h + h.T) / 2)
lam, vec = lam[::-1], vec[:, ::-1]
ref = q @ vec[:, : spec.k]
spec_s = time.time() - t
tot = float(np.sum(v * v))
delta = 2.0 / 3.0 * (lam[spec.k - 1] - lam[spec.p])
mu = math.sqrt(tot / max(tot - lam[: spec.k].sum(), 1e-300))
print(json.dumps({"spectrum_s": spec_s, "lambda_top": lam[: spec.p + 2].tolist(), "delta": delta, "mu": mu}),
      flush=True)
cfg = g.SIConfig(k=spec.k, p=spec.p, eps=spec.eps, mu=mu, delta=delta, seed=spec.seed, backend=backend)
ctx.enable_profiling(True)
ctx.reset_profile()
t = time.time()
res = g.shift_invert(x, cfg)
wall = time.time() - t
R = ref - res.W @ (res.W.T @ ref)
sin = float(np.sqrt(max(np.linalg.eigvalsh(R.T @ R).max(), 0.0)))
prof = {k: {"ms": vv["ms"], "count": vv["count"]} for k, vv in ctx.profile().items() if vv["count"]}
out = {"config": "C4", "backend": backend, "d": spec.d, "n": spec.n, "nnz": int(cp[-1]), "k": spec.k, "p": spec.p, "eps": spec.eps,
       "gen_s": gen_s, "spectrum_iters": iters, "spectrum_s": spec_s, "lambda_top": lam[: spec.p + 2].tolist(),
       "delta": delta, "mu": mu, "time_to_eps_s": res.ms["total"] / 1e3, "wall_s": wall, "ms_phases": res.ms,
       "lambda": res.lam, "tune_steps": len(res.tune_history), "outer_iterations": res.outer_iterations,
       "ledger": res.ledger, "ritz": res.ritz.tolist(),
       "ritz_max_rel_err_vs_power_iteration": float(np.max(np.abs(res.ritz - lam[: spec.k]) / lam[: spec.k])),
       "sin_theta_vs_power_iteration": sin, "profile": prof}
(ROOT / "gpurun_out").mkdir(exist_ok=True)
(ROOT / "gpurun_out" / f"config_C4_{backend}.json").write_text(json.dumps(out, indent=1))
print(json.dumps(out), flush=True)
