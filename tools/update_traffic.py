"""Refresh profiles/ncu_traffic.json from `ncu --set full` raw CSV exports:
dram bytes (read + write) per launch and the headline pipe metrics of each
hot kernel. Usage: python tools/update_traffic.py KERNEL=RAW_CSV[:ENTRIES] ..."""
import csv
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
KEYS = {"duration": "gpu__time_duration.sum",
        "alu_pipe_pct": "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
        "fma_pipe_pct": "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "lsu_pipe_pct": "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
        "issue_pct": "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "regs": "launch__registers_per_thread",
        "warps_active_pct": "sm__warps_active.avg.pct_of_peak_sustained_active",
        "stall_no_instruction": "smsp__average_warps_issue_stalled_no_instruction_per_issue_active.ratio",
        "stall_math_pipe": "smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio"}

path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
db = json.load(open(path))
for arg in sys.argv[1:]:
    kernel, spec = arg.split("=", 1)
    src, _, entries = spec.partition(":")
    rows = list(csv.reader(open(os.path.join(ROOT, src))))
    r, u = dict(zip(rows[0], rows[2])), dict(zip(rows[0], rows[1]))
    val = lambda k: float(r[k].replace(",", "")) * SCALE.get(u[k], 1)
    e = db.setdefault(kernel, {})
    e["dram_bytes"] = int(val("dram__bytes_read.sum") + val("dram__bytes_write.sum"))
    if entries:
        e["entries"] = int(entries)
    e["ncu"] = {k: f"{r[m]} {u[m]}" for k, m in KEYS.items() if m in r}
    e["source"] = src
json.dump(db, open(path, "w"), indent=1)
print(json.dumps(db, indent=1))
