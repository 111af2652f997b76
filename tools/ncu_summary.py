"""Summarise one kernel of an `ncu --set full` capture into profiles/*.json.

    python tools/ncu_summary.py gpurun_out/prof_c1_cur.ncu-rep profiles/r01_rsolve_c1_ncu_full.json
"""
import csv
import io
import json
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
        "smsp__inst_executed.sum", "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
        "launch__shared_mem_per_block_dynamic", "sm__cycles_elapsed.avg.per_second"]

rep, out = sys.argv[1], sys.argv[2]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units, vals = rows[0], rows[1], rows[2]
col = {h: i for i, h in enumerate(hdr)}
res = {"Kernel Name": vals[col["Kernel Name"]]}
for k in KEYS:
    if k in col:
        res[k] = f"{vals[col[k]]} {units[col[k]]}".strip()
stalls = {}
for h, i in col.items():
    if h.startswith("smsp__average_warps_issue_stalled_") and h.endswith("_per_issue_active.ratio"):
        try:
            v = float(vals[i].replace(",", ""))
        except ValueError:
            continue
        if v >= 0.2:
            stalls[h[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]] = round(v, 3)
res["stall_cycles_per_issued_instruction"] = dict(sorted(stalls.items(), key=lambda x: -x[1]))
json.dump(res, open(out, "w"), indent=1)
print(json.dumps(res, indent=1))
