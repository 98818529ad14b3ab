"""Summarise an `ncu --page source --csv` SASS dump: stall reasons and hottest instructions."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = next(r for r in rows if "Address" in r and "Source" in r)
data = [r for r in rows if len(r) == len(hdr) and r[0].startswith("0x")]
iS, iSrc, iEx = hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Source"), hdr.index("Instructions Executed")
f = lambda x: float(x) if x not in ("", "-") else 0.0
stall_cols = [i for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
tot = sum(f(r[iS]) for r in data) or 1
print("total samples", tot, "instructions executed", sum(f(r[iEx]) for r in data))
agg = {}
for r in data:
    for i in stall_cols:
        agg[hdr[i]] = agg.get(hdr[i], 0) + f(r[i])
print({k: round(100 * v / tot, 1) for k, v in sorted(agg.items(), key=lambda x: -x[1])[:8]})
n = int(sys.argv[2]) if len(sys.argv) > 2 else 30
for k, r in enumerate(sorted(data, key=lambda r: -f(r[iS]))[:n]):
    print(f"{int(f(r[iS])):8d} {int(f(r[iEx])):12d}  {r[iSrc][:100]}  @{r[0][-5:]}")
