"""C1 time-to-ε measured for real on the CPU (the reference algorithm: oracle/,
the reference's primitives restated bit for bit + the SPEC solver) at 1 host
thread (the reference is single-threaded) and at every host thread, beside the
device pipeline on the same X bytes.  Writes gpurun_out/cpu_c1.json.
    python tools/cpu_c1.py"""
import json
import os
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))
import numpy as np
import torch

import paper_1607_02925_b200 as g
from bench import cpu_model
from oracle_lib import Oracle, default_si_config
from paper_1607_02925_b200.configs import CONFIGS, make_dense_xt

spec = CONFIGS["C1"]
XT, _ = make_dense_xt(spec)
torch.cuda.synchronize()
X = XT.cpu().numpy().T  # the device pipeline's X bytes, column-major
lam, hint = float(spec.eig()[0] + spec.delta() / 10), float(spec.eig()[0])
cfg = g.SIConfig(k=spec.k, p=spec.p, eps=spec.eps, mu=spec.mu(), delta=spec.delta(), seed=spec.seed, lam=lam,
                 lambda1_hint=hint)
x = g.DeviceMatrix.from_device(XT.data_ptr(), spec.d, spec.n, spec.d, keep=XT)
g.shift_invert(x, cfg)  # warm-up
dev = [g.shift_invert(x, cfg) for _ in range(3)]
out = {"config": "C1", "cpu_model": cpu_model(), "host_threads": os.cpu_count(),
       "device_time_to_eps_s": min(r.ms["total"] for r in dev) / 1e3, "device_outer_iterations": dev[0].outer_iterations}
o = Oracle()
m = o.dense(X)
ocfg = default_si_config(spec.k, spec.p, eps=spec.eps, mu=spec.mu(), delta=spec.delta(), lam=lam, seed=spec.seed,
                         hint=hint)
for nth in (os.cpu_count() or 1, 1):
    o.nthreads = nth
    t = time.perf_counter()
    rc, w, ritz, s, rep = o.shift_invert(m, ocfg)
    dt = time.perf_counter() - t
    out[f"cpu_time_to_eps_s_{nth}t"] = dt
    out[f"cpu_outer_iterations_{nth}t"] = rep.outer_iterations
    out["sin_theta_device_vs_cpu"] = o.sin_theta(w, dev[0].W)
    print(json.dumps(out), flush=True)
out["speedup_vs_1t"] = out["cpu_time_to_eps_s_1t"] / out["device_time_to_eps_s"]
out["speedup_vs_all_threads"] = out[f"cpu_time_to_eps_s_{os.cpu_count() or 1}t"] / out["device_time_to_eps_s"]
(ROOT / "gpurun_out").mkdir(exist_ok=True)
(ROOT / "gpurun_out" / "cpu_c1.json").write_text(json.dumps(out, indent=1))
print(json.dumps(out))
