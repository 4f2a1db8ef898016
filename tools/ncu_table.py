"""Summarise an ncu --csv metrics dump: one line per kernel launch (first of each name)."""
import collections
import csv
import re
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr, data = None, collections.OrderedDict()
for r in rows:
    if r and r[0] == "ID":
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        data.setdefault((d["ID"], d["Kernel Name"]), {})[d["Metric Name"]] = d["Metric Value"]


def short(m):
    m = m.replace("smsp__average_warps_issue_stalled_", "st_").replace("_per_issue_active.ratio", "")
    m = m.replace(".avg.pct_of_peak_sustained_active", "%").replace("sm__inst_executed_pipe_", "")
    return m.replace("smsp__", "").replace("gpu__time_duration.sum", "ns")


for (i, k), d in data.items():
    k = re.sub(r"\(.*", "", k).replace("void ", "").replace("poslo_gpu::<unnamed>::", "")
    print(f"{i:>3} {k[:40]:40s} " + " ".join(f"{short(m)}={float(v.replace(',', '')):.4g}" for m, v in d.items()))
