"""Filter perf_probe.py --solve output: p, epoch ms per launch, chain phase cycles."""
import json
import sys

for line in sys.stdin:
    line = line.strip()
    if not line.startswith("{"):
        continue
    try:
        d = json.loads(line)
    except ValueError:
        continue
    if d.get("unit") == "solve3epochs":
        ep = d.get("epoch") or d.get("epoch_p1") or {}
        print("p", d["p"], "epoch_ms", round(ep.get("ms_per", float("nan")), 3))
    elif "epoch_phase_cycles_per_block" in d:
        print("  phases", d["epoch_phase_cycles_per_block"], "pc", d["pc"], "groups", d["groups"])
