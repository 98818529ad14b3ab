#!/usr/bin/env python
"""bench.py — the B200 shift-and-invert pipeline on BASELINE.json's largest
single-GPU configuration, C5 (configs[4]: dense fp64 X 8192 x 1,000,000 =
65.5 GB in HBM, k = 32, p = 64, eps = 1e-8).

A full C5 time-to-ε pipeline is minutes long, so it runs ONCE, untimed by the
step loop, in the setup (`time_to_eps` in the JSON line: device time of
tune_shift -> subspace iteration -> Rayleigh–Ritz with X resident, CUDA events
inside the runtime).  It also yields the tuned shift λ and the step-size hint.

One timed "step" = one shift-and-invert outer iteration at that λ through the
public C ABI (`gaplra_shift_invert` with the explicit λ and max_outer = 1):
the cold block SVRG solve (λI − XXᵀ)W = S⁰ at p = 64 to tol 1e-10 (its epochs:
anchor X·(XᵀW) pass, H pass, s-step block coefficients, the epoch chain), the
MGS2 QR, and Rayleigh–Ritz — the unit the C5 subspace phase repeats.
  value  = device time of the step with X resident in HBM (CUDA events);
  e2e    = the same call from pinned HOST X: H2D of X (65.5 GB) + the step +
           D2H of W and the Ritz values, wall clock.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                  [--config C5] [--no-full]

Multi-GPU: replicas only — every rank solves its own instance;
the step time is the max over ranks ("scaling": "weak").  `--impl reference`
times the reference CPU algorithm (oracle/: the reference's primitives restated
bit for bit + the SPEC-restated solver) on the host cores on a bounded sample
of the same step (same X bytes), extrapolated to the step with its work ledger
(tests/golden/<config>_step_ledger.json) and labelled so.
"""
from __future__ import annotations

import argparse
import ctypes
import json
import os
import platform
import statistics
import subprocess
import sys
import tempfile
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

METRIC = "time-to-ε rank-k subspace; X·(XᵀW) pass GB/s and % of roofline"
PEAKS = ROOT / "MEASURED_PEAKS.json"
FP64_PEAK_TFLOPS = 37.14  # measured DMMA fp64 on this pool's B200 (profiles/r01_microbench.txt)
FP64_PEAK_SRC = "measured mma.sync f64 (DMMA) microbenchmark, profiles/r01_microbench.txt (nominal 37.2)"
NCU_TRAFFIC = ROOT / "profiles" / "ncu_traffic.json"
HBM_READ_GBS = 6963.0  # profiles/r01_microbench.txt: 4 GB read-only buffer


def step_ledger_path(name):
    return ROOT / "tests" / "golden" / f"{name.lower()}_step_ledger.json"


def workload(spec):
    """The `config` dict, identical in both arms."""
    return {"workload": (f"{spec.name}: dense fp64 X {spec.d}x{spec.n} = U diag(sigma) V^T + {spec.noise:g} G/sqrt(n), "
                         f"rank {spec.rank}, k={spec.k}, p={spec.p}, eps={spec.eps:g}, seed {spec.seed}; "
                         "step = one shift-and-invert outer iteration at the tuned shift (cold block SVRG solve of "
                         f"(lambda I - X X^T) W = S0 at p={spec.p} to tol 1e-10 + MGS2 QR + Rayleigh-Ritz) through "
                         "gaplra_shift_invert(lambda, max_outer=1); full time-to-eps measured once in setup"),
            "config": spec.name, "d": spec.d, "n": spec.n, "k": spec.k, "p": spec.p, "eps": spec.eps,
            "l2": "inputs larger than L2 (X = %.1f GB > 126 MB)" % (8 * spec.d * spec.n / 1e9)}


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return platform.processor() or "unknown"


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
def cpu_unit_costs(spec, x_cols, seconds=12.0, nthreads=None):
    """Time the CPU oracle on a bounded sample of the step: one X(XᵀW) pass
    over a column slice and a run of SVRG steps, at p.  x_cols: (ncols, d)
    row-major = the first ncols columns of X, column-major.  Returns per-column
    pass cost and per-step epoch cost (seconds)."""
    import numpy as np

    from oracle_lib import Oracle

    o = Oracle()
    if nthreads:
        o.nthreads = nthreads
    rng = np.random.default_rng(0)
    budget = seconds / 2.0
    p = spec.p
    w = rng.standard_normal((spec.d, p))
    ncols = min(64, x_cols.shape[0])
    while True:
        m = o.dense(x_cols[:ncols].T)  # (d, ncols) Fortran view: no copy
        t = time.perf_counter()
        o.gram_block(m, w)
        dt = time.perf_counter() - t
        if dt > budget / 2 or ncols >= x_cols.shape[0]:
            break
        ncols = min(x_cols.shape[0], int(ncols * max(2.0, (budget / 2) / max(dt, 1e-6))))
    pass_per_col = dt / ncols
    _, z, y = o.gram_block(m, w, want_y=True)
    lam, eta = 1.05, 1e-6
    c = eta * z
    steps = 64
    while True:
        t = time.perf_counter()
        o.svrg_epoch(m, w, y, c, eta, lam, 1234, steps)
        dts = time.perf_counter() - t
        if dts > budget / 2 or steps >= 1 << 22:
            break
        steps = int(steps * max(2.0, (budget / 2) / max(dts, 1e-6)))
    return {"pass_s_per_col": pass_per_col, "step_s": dts / steps, "sample_cols": ncols, "sample_steps": steps,
            "threads": o.nthreads}


def cpu_step_seconds(spec, units, ledger):
    """The step's CPU time = (p-wide X(XᵀW) passes) x n x per-column cost + SVRG
    steps x per-step cost (identical algorithm => identical work ledger; the
    ledger equality is pinned by tests/test_gpu_fullsize.py on C1)."""
    passes = ledger["gram_applies"] / spec.p
    return passes * spec.n * units["pass_s_per_col"] + ledger["solver_column_samples"] * units["step_s"]


def cpu_baseline(spec, x_cols, ledger, seconds):
    u16 = cpu_unit_costs(spec, x_cols, seconds=seconds)
    u1 = cpu_unit_costs(spec, x_cols, seconds=seconds / 2, nthreads=1)
    v16, v1 = cpu_step_seconds(spec, u16, ledger), cpu_step_seconds(spec, u1, ledger)
    sample = (f"oracle/ (reference primitives restated bit for bit + SPEC solver), CPU '{cpu_model()}': one "
              f"X(X^T W) pass at p={spec.p} over the first {u16['sample_cols']} columns of the same X and "
              f"{u16['sample_steps']} SVRG steps at p={spec.p}, d={spec.d}, timed on {u16['threads']} threads "
              f"(columns of W split over threads); extrapolated to the step's work ledger "
              f"({ledger['gram_applies'] // spec.p} passes, {ledger['solver_column_samples']} steps)")
    return {"value": v16, "unit": "s", "cores": u16["threads"], "kind": "port", "sample": sample,
            "extrapolated": True, "cpu_model": cpu_model(), "unit_timings": {str(u16["threads"]): u16, "1": u1},
            "one_thread": {"value": v1, "cores": 1,
                           "note": "faithful to the reference, which is single-threaded (linear_operator.hpp:16-30)"}}


# ----------------------------------------------------------------- rooflines
def rooflines(prof, config="C5"):
    peaks = json.loads(PEAKS.read_text()) if PEAKS.exists() else {}
    hbm = float(peaks.get("hbm_gbs", 6650.0))
    hbm_src = "MEASURED_PEAKS.json hbm_gbs" if "hbm_gbs" in peaks else "fallback 6.65 TB/s (B200_PROFILING.md)"
    ridge = FP64_PEAK_TFLOPS * 1e12 / (hbm * 1e9)
    traffic = json.loads(NCU_TRAFFIC.read_text()).get(config, {}) if NCU_TRAFFIC.exists() else {}
    tsrc = f"{NCU_TRAFFIC.relative_to(ROOT)} [{config}]: " + traffic.get("_source", "")
    out = {}
    for name, v in prof.items():
        if not v["count"] or v["ms"] <= 0:
            continue
        t = v["ms"] / 1e3
        per = v["count"]
        intensity = v["flops"] / max(v["bytes"], 1.0)
        tr = traffic.get(name)
        if intensity >= ridge and v["flops"] > 0:
            ach = v["flops"] / t / 1e12
            out[name] = {"bound": "tensor", "achieved": ach, "peak": FP64_PEAK_TFLOPS, "unit": "TFLOP/s",
                         "frac": ach / FP64_PEAK_TFLOPS, "peak_source": FP64_PEAK_SRC + " (fp64 pipe)",
                         "traffic": tr, "traffic_source": tsrc if tr else None, "launches": per,
                         "ms_per_launch": v["ms"] / per, "algorithmic_bytes_per_launch": v["bytes"] / per,
                         "algorithmic_flops_per_launch": v["flops"] / per, "gbps": v["bytes"] / t / 1e9}
        else:
            ach = v["bytes"] / t / 1e9
            out[name] = {"bound": "hbm", "achieved": ach, "peak": hbm, "unit": "GB/s", "frac": ach / hbm,
                         "peak_source": hbm_src, "traffic": tr, "traffic_source": tsrc if tr else None,
                         "launches": per, "ms_per_launch": v["ms"] / per,
                         "algorithmic_bytes_per_launch": v["bytes"] / per, "tflops": v["flops"] / t / 1e12}
            if name in ("gram_p1", "h_pass"):  # X read once, nothing comparable written
                out[name]["note"] = (f"read-only stream: hbm_gbs is a copy (read + write) figure; a 4 GB read "
                                     f"measured {HBM_READ_GBS} GB/s (profiles/r01_microbench.txt), "
                                     f"frac {ach / HBM_READ_GBS:.3f} of that")
    return out


# ------------------------------------------------------------------- host X
def pinned_host_copy(XT):
    """Exact-size page-locked host copy of the device X (torch's pinned caching
    allocator rounds to powers of two: 65.5 GB would pin 128 GB)."""
    import numpy as np
    import torch

    host = np.empty(tuple(XT.shape), dtype=np.float64)
    rc = torch.cuda.cudart().cudaHostRegister(host.ctypes.data, host.nbytes, 0)
    if int(rc) != 0:
        raise RuntimeError(f"cudaHostRegister failed ({rc})")
    torch.from_numpy(host).copy_(XT)
    return host


def max_over_ranks(vals, dist, device):
    if not dist:
        return vals
    import torch

    t = torch.tensor(vals, dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return t.tolist()


# ------------------------------------------------------------------- our arm
def run_ours(args, rank, world, local_rank):
    import numpy as np
    import torch

    import paper_1607_02925_b200 as g
    from paper_1607_02925_b200 import _native as N
    from paper_1607_02925_b200.configs import CONFIGS, make_dense_xt

    torch.cuda.set_device(local_rank)
    dev = f"cuda:{local_rank}"
    spec = CONFIGS[args.config]
    dist = None
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    d, n, k, p = spec.d, spec.n, spec.k, spec.p
    t0 = time.time()
    XT, _ = make_dense_xt(spec, device=dev)  # (n, d) row-major = X column-major, ld = d (d % 4 == 0)
    torch.cuda.synchronize()
    gen_s = time.time() - t0
    host = pinned_host_copy(XT)
    ctx = g.Context(local_rank)
    lib = N.load()
    x_res = g.DeviceMatrix.from_device(XT.data_ptr(), d, n, d, ctx=ctx, keep=XT)

    # ---- setup: the full time-to-ε pipeline once (or tune_shift alone)
    base = g.SIConfig(k=k, p=p, eps=spec.eps, mu=spec.mu(), delta=spec.delta(), seed=spec.seed)
    full = None
    if spec.name == "C1":  # NoPreconditioningNeeded fires on C1: explicit shift
        lam, hint = float(spec.eig()[0] + spec.delta() / 10), float(spec.eig()[0])
        base.lam, base.lambda1_hint = lam, hint
    if not args.no_full:
        ctx.reset_profile()
        ctx.enable_profiling(True)
        res = g.shift_invert(x_res, base)
        ctx.enable_profiling(False)
        lam, hint = res.lam, res.lambda1_hint
        full = {"value": res.ms["total"] / 1e3, "unit": "s", "ms_phases": res.ms, "lambda": res.lam,
                "tune_steps": len(res.tune_history), "outer_iterations": res.outer_iterations, "ledger": res.ledger,
                "profile": {kk: {"ms": v["ms"], "count": v["count"]} for kk, v in ctx.profile().items() if v["count"]},
                "what": "device time of the whole pipeline (tune_shift -> subspace iteration -> Rayleigh-Ritz), "
                        "X resident, measured once in setup (not a timed step)"}
        if rank == 0:  # verification only (untimed): dense eigendecomposition of X Xᵀ
            A = XT.T @ XT
            ev, evec = torch.linalg.eigh(A)
            ev, evec = ev.flip(0)[:k].cpu().numpy(), evec.flip(1)[:, :k].cpu().numpy()
            R = evec - res.W @ (res.W.T @ evec)
            full["sin_theta_vs_eigh"] = float(np.sqrt(max(np.linalg.eigvalsh(R.T @ R).max(), 0.0)))
            full["ritz_max_rel_err_vs_eigh"] = float(np.max(np.abs(res.ritz - ev) / ev))
            del A
    elif args.lam > 0.0:
        lam, hint = args.lam, args.hint
    elif spec.name != "C1":
        st = g.tune_shift(x_res, spec.delta(), base)
        lam, hint = st.lam, st.lambda1_hint
    step_cfg = g.SIConfig(k=k, p=p, eps=spec.eps, mu=spec.mu(), delta=spec.delta(), seed=spec.seed, lam=lam,
                          lambda1_hint=hint, max_outer=1)
    x_res.close()
    del x_res, XT  # the steps upload X from the pinned host copy
    torch.cuda.empty_cache()

    def e2e_step():
        """Public C ABI from host buffers: H2D of X, one outer iteration, D2H of W + ritz."""
        ts = time.perf_counter()
        x = g.DeviceMatrix.from_host_pointer(host.ctypes.data, d, n, d, ctx=ctx)
        r = g.shift_invert(x, step_cfg)
        x.close()
        return r, time.perf_counter() - ts

    for _ in range(args.warmup):
        e2e_step()
    # the timed steps run the production path (per-kernel profiling off; the
    # epoch loop is host-driven for >= 1 TFLOP epochs, device-resident below);
    # one extra profiled step afterwards gives the
    # per-kernel-class rooflines (same kernels, host-driven epoch loop)
    ctx.enable_profiling(False)
    launches0 = lib.gaplra_launch_count()
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    dev_s, e2e_s, last = [], [], None
    with ClockSampler(local_rank) as clk:
        for _ in range(args.steps):
            last, wall = e2e_step()
            dev_s.append(last.ms["total"] / 1e3)
            e2e_s.append(wall)
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    launches = lib.gaplra_launch_count() - launches0
    ctx.reset_profile()
    ctx.enable_profiling(True)
    prof_res, _ = e2e_step()  # untimed: rooflines
    ctx.enable_profiling(False)
    prof = ctx.profile()
    value = sum(dev_s) / len(dev_s)
    e2e = sum(e2e_s) / len(e2e_s)
    value, e2e = max_over_ranks([value, e2e], dist, dev)
    if rank != 0:
        if dist:
            dist.destroy_process_group()
        return
    rl = rooflines(prof, spec.name)
    dominant = max(rl, key=lambda kk: rl[kk]["ms_per_launch"] * rl[kk]["launches"]) if rl else None
    step_ledger = last.ledger  # ONE step's counts (the report is per call)
    out_dir = ROOT / "gpurun_out"
    out_dir.mkdir(exist_ok=True)
    (out_dir / f"bench_{spec.name.lower()}_step_ledger.json").write_text(json.dumps(
        {"config": spec.name, "lambda": lam, "lambda1_hint": hint, "ledger": step_ledger,
         "source": "bench.py step (gaplra_shift_invert, explicit lambda, max_outer=1)"}, indent=1))
    cpu = None
    if world == 1 and not args.no_cpu:
        cpu = cpu_baseline(spec, host, step_ledger, args.cpu_seconds)
    torch.cuda.cudart().cudaHostUnregister(host.ctypes.data)
    line = {
        "metric": METRIC, "value": value, "unit": "s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": value * 1e3, "higher_is_better": False, "scaling": "weak", "vs_baseline": None,
        "dtype": "f64", "data": f"synthetic (seeded on-device planting with BASELINE.json's {spec.name} recipe)",
        "config": workload(spec),
        "e2e": {"value": e2e, "unit": "s", "h2d_bytes_per_step": 8 * d * n, "d2h_bytes_per_step": 8 * (d * k + k)},
        "roofline": dict(rl[dominant], kernel=dominant) if dominant else None,
        "rooflines": rl,
        "cpu_baseline": cpu,
        "clocks": clk.summary(),
        "gpu_launches": int(launches),
        "time_to_eps": full,
        "step": {"lambda": lam, "lambda1_hint": hint, "outer_iterations": last.outer_iterations,
                 "ledger": step_ledger, "ms_phases": last.ms,
                 "profiled_step_ms": prof_res.ms["total"],
                 "note": "value/e2e: the production path, no per-kernel events (epoch loop host-driven when an "
                         "epoch is >= 1 TFLOP, as at C5 p = 64; a device-resident CUDA-graph WHILE loop below "
                         "that); rooflines: one extra untimed step with per-kernel CUDA events (host-driven "
                         "loop, same kernels)"},
        "gen_s": gen_s,
    }
    print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()


# ------------------------------------------------------------- reference arm
def run_reference(args, rank, world):
    """The reference CPU algorithm on the same step: oracle/ on the host cores,
    same X bytes (planted by the same seeded torch generator; only the first
    columns are copied to the host), extrapolated with the step's ledger."""
    if rank != 0:
        return
    import numpy as np
    import torch

    from paper_1607_02925_b200.configs import CONFIGS, make_dense_xt

    spec = CONFIGS[args.config]
    led_file = step_ledger_path(spec.name)
    ledger = json.loads(led_file.read_text())["ledger"]
    if torch.cuda.is_available():
        XT, _ = make_dense_xt(spec, device="cuda")
        x_cols = XT[:65536].cpu().numpy()  # the first columns of the GPU arm's X, byte for byte
        del XT
        torch.cuda.empty_cache()
    else:  # CPU-only host: same recipe on the CPU generator (different bytes, same distribution)
        import dataclasses

        XT, _ = make_dense_xt(dataclasses.replace(spec, n=min(spec.n, 65536)), device="cpu")
        x_cols = XT.numpy()
    vals, cb = [], None
    for _ in range(args.warmup + args.steps):
        cb = cpu_baseline(spec, x_cols, ledger, args.cpu_seconds)
        vals.append(cb["value"])
    v = sum(vals[args.warmup:]) / max(1, args.steps)
    cb["value"] = v
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": "s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": v * 1e3, "higher_is_better": False, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64",
            "data": f"synthetic (seeded planting with BASELINE.json's {spec.name} recipe; same X bytes as the GPU arm)",
            "config": workload(spec), "cpu_baseline": cb,
            "e2e": {"value": v, "unit": "s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "ledger_source": str(led_file.relative_to(ROOT))}
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", default="C5")
    ap.add_argument("--cpu-seconds", type=float, default=16.0)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-full", action="store_true", help="skip the once-per-run full time-to-eps pipeline")
    ap.add_argument("--lam", type=float, default=0.0,
                    help="profiling aid: the tuned shift (with --hint), skipping tune_shift when --no-full")
    ap.add_argument("--hint", type=float, default=0.0)
    args = ap.parse_args()
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local_rank = int(os.environ.get("LOCAL_RANK", 0))
    if args.gpus != world:
        print(json.dumps({"error": f"--gpus {args.gpus} but WORLD_SIZE={world}: launch N ranks with "
                                   "torch.distributed.run --nproc-per-node N"}), flush=True)
        sys.exit(2)
    if args.warmup < 3 and args.impl == "ours":
        print("warning: fewer than 3 warm-up steps", file=sys.stderr)
    if args.impl == "reference":
        run_reference(args, rank, world)
    else:
        run_ours(args, rank, world, local_rank)


if __name__ == "__main__":
    main()
