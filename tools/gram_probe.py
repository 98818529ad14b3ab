"""GPU probe for the X·(XᵀW) pass alone: random device X (d x n), device W,
`iters` timed gram_block_device calls.  Usage:
  python tools/gram_probe.py [d] [n] [p] [iters]
Prints ms per pass, GB/s of X and TFLOP/s (4·d·n·p)."""
import ctypes as C
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch

import paper_1607_02925_b200 as g

d, n, p, iters = (int(v) for v in (sys.argv[1:] + ["4096", "100000", "20", "20"][len(sys.argv) - 1:])[:4])
ctx = g.default_context()
torch.manual_seed(0)
XT = torch.randn(n, d, dtype=torch.float64, device="cuda")  # X column-major = Xᵀ row-major
x = g.DeviceMatrix.from_device(XT.data_ptr(), d, n, d, ctx=ctx, keep=XT)
ld = 1 if p == 1 else (p + 1) // 2 * 2
W = torch.randn(d, ld, dtype=torch.float64, device="cuda")
Z = torch.zeros(d, ld, dtype=torch.float64, device="cuda")
Y = torch.zeros(n, ld, dtype=torch.float64, device="cuda")
lib = ctx.lib


def run():
    ctx.check(lib.gaplra_gram_block_device(ctx.h, x.h, p, C.c_void_p(W.data_ptr()), ld, C.c_void_p(Z.data_ptr()), ld,
                                           C.c_void_p(Y.data_ptr()), ld))


for _ in range(3):
    run()
ctx.synchronize()
ctx.enable_profiling(True)  # CUDA events on the context's launching stream
ctx.reset_profile()
for _ in range(iters):
    run()
ctx.synchronize()
pr = ctx.profile()["gram" if p > 1 else "gram_p1"]
ms = pr["ms"] / pr["count"]
zr = XT.T @ (XT @ W[:, :p])
err = (Z[:, :p] - zr).abs().max().item() / zr.abs().max().item()
print(json.dumps({"d": d, "n": n, "p": p, "ms": ms, "GBps": 8.0 * d * n / ms / 1e6,
                  "TFLOPs": 4.0 * d * n * p / ms / 1e9, "rel_err": err}), flush=True)
