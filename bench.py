#!/usr/bin/env python
"""bench.py — time-to-ε of the B200 shift-and-invert pipeline on BASELINE.json
config C2 (configs[1]: dense fp64 X 4096 x 100000, k = 10, p = 20, eps = 1e-8).

One "step" = one full ShiftedInverse pipeline (tune_shift -> block SVRG
subspace iteration on (λI − XXᵀ)⁻¹ -> Rayleigh–Ritz) through the C ABI
gaplra_shift_invert.  `value` is the device time of that pipeline with X
already resident in HBM (CUDA events on the launching stream, inside the
runtime); `e2e` is the same call measured end to end from pinned host X:
host->device copy of X + pipeline + device->host read of W and the Ritz values.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Multi-GPU: replicas only — every rank solves its own instance;
value is the max over ranks ("scaling": "weak").  --impl reference times the
reference CPU algorithm (oracle/, the reference's shipped primitives restated
bit-for-bit plus the SPEC-restated solver) on a bounded sample of the same
workload with all host threads, extrapolated to the full pipeline with the
pipeline's work ledger (tests/golden/c2_work_ledger.json).
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import tempfile
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

METRIC = "time-to-ε rank-k subspace; X·(XᵀW) pass GB/s and % of roofline"
LEDGER = ROOT / "tests" / "golden" / "c2_work_ledger.json"
PEAKS = ROOT / "MEASURED_PEAKS.json"
FP64_PEAK_TFLOPS = 37.14  # measured DMMA fp64 on this pool's B200 (profiles/r01_microbench.txt)
FP64_PEAK_SRC = "measured mma.sync f64 (DMMA) microbenchmark, profiles/r01_microbench.txt (nominal 37.2)"
NCU_TRAFFIC = ROOT / "profiles" / "ncu_traffic.json"


def pinned_config(spec, lam=0.0, hint=0.0):
    import paper_1607_02925_b200 as g

    return g.SIConfig(k=spec.k, p=spec.p, eps=spec.eps, mu=spec.mu(), delta=spec.delta(), seed=spec.seed,
                      lam=lam, lambda1_hint=hint)


def workload_desc(spec):
    return (f"{spec.name}: dense fp64 X {spec.d}x{spec.n} = U diag(sigma) V^T + {spec.noise:g} G/sqrt(n), "
            f"rank {spec.rank}, k={spec.k}, p={spec.p}, eps={spec.eps:g}, seed {spec.seed}")


# --------------------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi clocks + throttle reasons during the timed region."""

    def __init__(self, index):
        self.index = index
        self.tmp = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        self.proc = None

    def __enter__(self):
        q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--id={self.index}", f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=self.tmp, stderr=subprocess.DEVNULL)
        except OSError:
            self.proc = None
        return self

    def __exit__(self, *exc):
        if self.proc:
            self.proc.terminate()
            self.proc.wait(timeout=10)

    def summary(self):
        self.tmp.flush()
        rows = []
        for line in open(self.tmp.name):
            parts = [x.strip() for x in line.split(",")]
            if len(parts) >= 9:
                rows.append(parts)
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({n for r in rows for n, v in zip(names, r[5:9]) if v.lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": float(rows[0][2]) if rows[0][2].replace(".", "").isdigit() else None,
                "reasons": reasons, "samples": len(rows)}


# ------------------------------------------------------------------ CPU baseline
def cpu_unit_costs(spec, xt_host, seconds=12.0, nthreads=None):
    """Time the CPU oracle on a bounded sample of the workload: one X(XᵀW) pass
    and one SVRG step block on a column slice, for p and for p = 1.  Returns
    per-column pass cost and per-step epoch cost (seconds) per p."""
    import numpy as np

    from oracle_lib import Oracle

    o = Oracle()
    if nthreads:
        o.nthreads = nthreads
    rng = np.random.default_rng(0)
    out = {}
    budget = seconds / 4.0
    for p in (spec.p, 1):
        ncols = 512
        w = rng.standard_normal((spec.d, p))
        while True:
            xs = np.ascontiguousarray(xt_host[:ncols]).T  # d x ncols, Fortran order view
            m = o.dense(xs)
            t = time.perf_counter()
            o.gram_block(m, w)
            dt = time.perf_counter() - t
            if dt > budget / 3 or ncols >= xt_host.shape[0]:
                break
            ncols = min(xt_host.shape[0], int(ncols * max(2.0, (budget / 3) / max(dt, 1e-6))))
        pass_per_col = dt / ncols
        steps = 256
        lam = float(spec.eig()[0]) * 1.1
        _, z, y = o.gram_block(m, w, want_y=True)
        eta = 1e-4
        c = eta * z
        while True:
            t = time.perf_counter()
            o.svrg_epoch(m, w, y, c, eta, lam, 1234, steps)
            dt = time.perf_counter() - t
            if dt > budget / 3 or steps >= 1 << 20:
                break
            steps = int(steps * max(2.0, (budget / 3) / max(dt, 1e-6)))
        out[p] = {"pass_s_per_col": pass_per_col, "step_s": dt / steps, "sample_cols": ncols, "sample_steps": steps}
    return out, o.nthreads


def cpu_extrapolate(spec, units, ledger):
    """Time-to-ε of the CPU reference = Σ_class count × unit cost (same algorithm
    ⇒ same work ledger as the device run)."""
    n, m = spec.n, 2 * spec.n
    t = 0.0
    t += ledger["gram"] * n * units[spec.p]["pass_s_per_col"]
    t += ledger["gram_p1"] * n * units[1]["pass_s_per_col"]
    t += ledger["epoch"] * m * units[spec.p]["step_s"]
    t += ledger["epoch_p1"] * m * units[1]["step_s"]
    return t


def cpu_sample_desc(units, nthreads):
    p_hi = max(units)
    return (f"oracle/ (reference primitives restated bit-for-bit + SPEC solver) on {nthreads} host threads: "
            f"one X(X^T W) pass over {units[p_hi]['sample_cols']} columns and {units[p_hi]['sample_steps']} SVRG "
            f"steps at p={p_hi}, same at p=1 ({units[1]['sample_cols']} cols / {units[1]['sample_steps']} steps); "
            "time-to-eps extrapolated as sum(count x unit cost) over the pipeline's work ledger")


def load_ledger(prof=None):
    if prof:
        return {k: prof[k]["count"] for k in ("gram", "gram_p1", "epoch", "epoch_p1")}
    if LEDGER.exists():
        return json.loads(LEDGER.read_text())["counts"]
    return {"gram": 100, "gram_p1": 1600, "epoch": 900, "epoch_p1": 735}  # provisional (r01 probe)


# ----------------------------------------------------------------- rooflines
HBM_READ_GBS = 6963.0  # profiles/r01_microbench.txt: 4 GB read-only buffer


def rooflines(prof):
    peaks = json.loads(PEAKS.read_text()) if PEAKS.exists() else {}
    hbm = float(peaks.get("hbm_gbs", 6650.0))
    hbm_src = "MEASURED_PEAKS.json hbm_gbs" if "hbm_gbs" in peaks else "fallback 6.65 TB/s (B200_PROFILING.md)"
    ridge = FP64_PEAK_TFLOPS * 1e12 / (hbm * 1e9)
    traffic = json.loads(NCU_TRAFFIC.read_text()) if NCU_TRAFFIC.exists() else {}
    out = {}
    for name, v in prof.items():
        if not v["count"] or v["ms"] <= 0:
            continue
        t = v["ms"] / 1e3
        per = v["count"]
        intensity = v["flops"] / max(v["bytes"], 1.0)
        if intensity >= ridge and v["flops"] > 0:
            ach = v["flops"] / t / 1e12
            out[name] = {"bound": "tensor", "achieved": ach, "peak": FP64_PEAK_TFLOPS, "unit": "TFLOP/s",
                         "frac": ach / FP64_PEAK_TFLOPS, "peak_source": FP64_PEAK_SRC + " (fp64 pipe)",
                         "traffic": traffic.get(name), "launches": per, "ms_per_launch": v["ms"] / per,
                         "gbps": v["bytes"] / t / 1e9}
        else:
            ach = v["bytes"] / t / 1e9
            out[name] = {"bound": "hbm", "achieved": ach, "peak": hbm, "unit": "GB/s", "frac": ach / hbm,
                         "peak_source": hbm_src, "traffic": traffic.get(name), "launches": per,
                         "ms_per_launch": v["ms"] / per, "tflops": v["flops"] / t / 1e12}
            if name in ("gram_p1", "h_pass"):  # X read once, nothing comparable written
                out[name]["note"] = (f"read-only stream: hbm_gbs is a copy (read + write) figure; a 4 GB read "
                                     f"measured {HBM_READ_GBS} GB/s (profiles/r01_microbench.txt), "
                                     f"frac {ach / HBM_READ_GBS:.3f} of that")
    return out


# ------------------------------------------------------------------- our arm
def run_ours(args, rank, world, local_rank):
    import numpy as np
    import torch

    import paper_1607_02925_b200 as g
    from paper_1607_02925_b200 import _native as N
    from paper_1607_02925_b200.configs import CONFIGS, make_dense_xt

    torch.cuda.set_device(local_rank)
    spec = CONFIGS[args.config]
    dist = None
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    t0 = time.time()
    XT, _ = make_dense_xt(spec, device=f"cuda:{local_rank}")
    xt_host = torch.empty(XT.shape, dtype=torch.float64, pin_memory=True)
    xt_host.copy_(XT)
    torch.cuda.synchronize()
    gen_s = time.time() - t0
    ctx = g.Context(local_rank)
    lib = N.load()
    lam, hint = 0.0, 0.0
    if spec.name == "C1":  # NoPreconditioningNeeded fires on C1: explicit shift
        lam, hint = float(spec.eig()[0] + spec.delta() / 10), float(spec.eig()[0])
    cfg = pinned_config(spec, lam, hint)
    d, n, k = spec.d, spec.n, spec.k
    host_ptr = xt_host.data_ptr()

    def e2e_step():
        """Public API from host buffers: H2D of X, pipeline, D2H of W + ritz."""
        ts = time.perf_counter()
        x = g.DeviceMatrix.from_host_pointer(host_ptr, d, n, d, ctx=ctx)
        res = g.shift_invert(x, cfg)
        x.close()
        return res, time.perf_counter() - ts

    for _ in range(args.warmup):
        e2e_step()
    ctx.reset_profile()
    ctx.enable_profiling(True)
    launches0 = lib.gaplra_launch_count()
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    dev_s, e2e_s, results = [], [], []
    with ClockSampler(local_rank) as clk:
        for _ in range(args.steps):
            res, wall = e2e_step()
            dev_s.append(res.ms["total"] / 1e3)
            e2e_s.append(wall)
            results.append(res)
    torch.cuda.synchronize()
    launches = lib.gaplra_launch_count() - launches0
    prof = ctx.profile()
    value = sum(dev_s) / len(dev_s)
    e2e = sum(e2e_s) / len(e2e_s)
    if dist:
        from paper_1607_02925_b200.replicas import max_over_ranks

        value, e2e = max_over_ranks([value, e2e], device=f"cuda:{local_rank}")
    res = results[-1]
    # accuracy check against a dense eigendecomposition (verification only, untimed)
    check = {}
    if rank == 0:
        A = XT.T @ XT
        ev, evec = torch.linalg.eigh(A)
        ev, evec = ev.flip(0)[:k].cpu().numpy(), evec.flip(1)[:, :k].cpu().numpy()
        W = res.W
        R = evec - W @ (W.T @ evec)
        sin = float(np.sqrt(max(np.linalg.eigvalsh(R.T @ R).max(), 0.0)))
        check = {"sin_theta_vs_eigh": sin, "ritz_max_rel_err_vs_eigh": float(np.max(np.abs(res.ritz - ev) / ev)),
                 "ritz": res.ritz.tolist(), "lambda": res.lam, "tune_steps": len(res.tune_history),
                 "outer_iterations": res.outer_iterations, "ledger": res.ledger, "ms_phases": res.ms}
        del A
    if rank != 0:
        if dist:
            dist.barrier()
            dist.destroy_process_group()
        return
    rl = rooflines(prof)
    dominant = max(rl, key=lambda kk: rl[kk]["ms_per_launch"] * rl[kk]["launches"]) if rl else None
    ledger = load_ledger(prof)
    out_dir = ROOT / "gpurun_out"
    out_dir.mkdir(exist_ok=True)
    (out_dir / "bench_work_ledger.json").write_text(json.dumps(
        {"config": spec.name, "counts": ledger, "profile": prof, "ledger": res.ledger}, indent=1))
    cpu = None
    if world == 1 and not args.no_cpu:
        units, nth = cpu_unit_costs(spec, xt_host.numpy(), seconds=args.cpu_seconds)
        cpu_v = cpu_extrapolate(spec, units, ledger)
        cpu = {"value": cpu_v, "unit": "s", "cores": nth, "kind": "port", "sample": cpu_sample_desc(units, nth),
               "unit_costs": {str(kk): vv for kk, vv in units.items()}}
    line = {
        "metric": METRIC, "value": value, "unit": "s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": value * 1e3, "higher_is_better": False, "scaling": "weak", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic (seeded on-device planting with BASELINE.json's C2 recipe)",
        "config": {"workload": workload_desc(spec), "d": d, "n": n, "k": k, "p": spec.p, "eps": spec.eps,
                   "parallelism": "replicas" if world > 1 else "single-gpu",
                   "l2": "inputs larger than L2 (X = %.2f GB > 126 MB)" % (8 * d * n / 1e9)},
        "e2e": {"value": e2e, "unit": "s", "h2d_bytes_per_step": 8 * d * n, "d2h_bytes_per_step": 8 * (d * k + k)},
        "roofline": dict(rl[dominant], kernel=dominant) if dominant else None,
        "rooflines": rl,
        "cpu_baseline": cpu,
        "clocks": clk.summary(),
        "gpu_launches": int(launches),
        "check": check,
        "gen_s": gen_s,
    }
    print(json.dumps(line), flush=True)
    if dist:
        dist.barrier()
        dist.destroy_process_group()


# ------------------------------------------------------------- reference arm
def run_reference(args, rank, world):
    if rank != 0:
        return
    import numpy as np

    from paper_1607_02925_b200.configs import CONFIGS

    spec = CONFIGS[args.config]
    # a bounded sample of the workload: ncols columns of X (host, numpy; same recipe)
    rng = np.random.default_rng(spec.seed)
    ncols = 16384
    U, _ = np.linalg.qr(rng.standard_normal((spec.d, spec.rank)))
    V, _ = np.linalg.qr(rng.standard_normal((ncols, spec.rank)))
    V *= math.sqrt(ncols / spec.n)  # rows of a Haar n x r orthonormal matrix have norm^2 r/n
    xt = (V * spec.sigma()) @ U.T + spec.noise / math.sqrt(spec.n) * rng.standard_normal((ncols, spec.d))
    ledger = load_ledger()
    vals = []
    units = nth = None
    for _ in range(args.warmup + args.steps):
        units, nth = cpu_unit_costs(spec, xt, seconds=args.cpu_seconds)
        vals.append(cpu_extrapolate(spec, units, ledger))
    v = sum(vals[args.warmup:]) / max(1, args.steps)
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": "s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": v * 1e3, "higher_is_better": False, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": f"synthetic (host sample with BASELINE.json's {args.config} recipe)",
            "config": {"workload": workload_desc(spec), "d": spec.d, "n": spec.n, "k": spec.k, "p": spec.p,
                       "eps": spec.eps},
            "cpu_baseline": {"value": v, "unit": "s", "cores": nth, "kind": "port",
                             "sample": cpu_sample_desc(units, nth)},
            "e2e": {"value": v, "unit": "s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "ledger_source": str(LEDGER.relative_to(ROOT)) if LEDGER.exists() else "provisional"}
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=1)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", default="C2")
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    ap.add_argument("--no-cpu", action="store_true")
    args = ap.parse_args()
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local_rank = int(os.environ.get("LOCAL_RANK", 0))
    if args.impl == "reference":
        run_reference(args, rank, world)
    else:
        run_ours(args, rank, world, local_rank)


if __name__ == "__main__":
    main()
