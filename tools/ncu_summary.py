"""Summarise an .ncu-rep (ncu --set full) into a small JSON: per kernel the duration, DRAM bytes, pipe / issue
utilisation and the warp-stall mix.   python tools/ncu_summary.py rep.ncu-rep "note" > out.json"""
import csv
import io
import json
import subprocess
import sys

rep, note = sys.argv[1], (sys.argv[2] if len(sys.argv) > 2 else "")
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units, data = rows[0], rows[1], rows[2:]
want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "lts__t_sectors_op_read.sum", "lts__t_bytes.sum",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "launch__grid_size", "launch__block_size", "launch__registers_per_thread",
        "smsp__inst_executed.sum", "sm__cycles_elapsed.max"]
out = {"report": rep, "note": note, "kernels": []}
for r in data:
    k = {"kernel": r[hdr.index("Kernel Name")]}
    for m in want:
        if m in hdr:
            i = hdr.index(m)
            k[m] = {"value": r[i], "unit": units[i]}
    st = {}
    for i, h in enumerate(hdr):
        if h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("_not_issued"):
            try:
                st[h.replace("smsp__pcsamp_warps_issue_stalled_", "")] = float(r[i].replace(",", ""))
            except ValueError:
                pass
    tot = sum(st.values()) or 1.0
    k["stall_pct"] = {a: round(100 * b / tot, 1) for a, b in sorted(st.items(), key=lambda kv: -kv[1])[:8]}
    out["kernels"].append(k)
print(json.dumps(out, indent=1))
