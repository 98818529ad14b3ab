"""Aggregate an ncu --metrics gpu__time_duration.sum --csv launch list into
per-kernel launches / ms / share.  Usage: python tools/launch_shares.py in.csv [note]"""
import csv
import json
import re
import sys

rows = [r for r in csv.reader(l for l in open(sys.argv[1]) if l.startswith('"'))]
h = rows[0]
ik, iv, iu = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
agg = {}
for r in rows[1:]:
    name = re.sub(r"\(.*", "", r[ik]).replace("void ", "").replace("(anonymous namespace)::", "")
    name = re.sub(r"gaplra_cuda::|<unnamed>::|unnamed>::", "", name)
    ms = float(r[iv].replace(",", "")) * {"nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0, "ns": 1e-6, "us": 1e-3,
                                            "ms": 1.0}.get(r[iu], 1e-6)
    a = agg.setdefault(name, [0, 0.0])
    a[0] += 1
    a[1] += ms
tot = sum(v[1] for v in agg.values())
out = {"source": sys.argv[2] if len(sys.argv) > 2 else sys.argv[1], "total_ms": round(tot, 3),
       "kernels": {k: {"launches": v[0], "ms": round(v[1], 3), "share": round(v[1] / tot, 4)}
                   for k, v in sorted(agg.items(), key=lambda kv: -kv[1][1])}}
print(json.dumps(out, indent=1))
