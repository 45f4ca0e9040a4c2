"""Per-kernel stall breakdown (cycles per issued instruction) from an `ncu --page raw --csv`
export: python profiles/stalls.py raw.csv[.gz]"""
import csv
import gzip
import io
import sys

path = sys.argv[1]
f = io.TextIOWrapper(gzip.open(path)) if path.endswith(".gz") else open(path)
rows = list(csv.reader(f))
h = rows[0]
ki = h.index("Kernel Name")
pre = "smsp__average_warps_issue_stalled_"
st = [i for i, c in enumerate(h) if c.startswith(pre) and c.endswith("_per_issue_active.ratio")]
extra = {c: h.index(c) for c in ("sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
                                 "sass__inst_executed_local_loads", "gpu__time_duration.sum",
                                 "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum") if c in h}
seen = set()
for r in rows[2:]:
    k = r[ki].split("<")[0].split("(")[0].replace("void ", "").replace("rtnb::", "")
    if k in seen:
        continue
    seen.add(k)
    vals = sorted(((float(r[i].replace(",", "") or 0), h[i][len(pre):].replace("_per_issue_active.ratio", ""))
                   for i in st), reverse=True)[:6]
    ex = {c.split("__")[1].split(".")[0]: r[i] for c, i in extra.items()}
    print(f"{k:14s}", " ".join(f"{n}={v:.2f}" for v, n in vals), ex)
