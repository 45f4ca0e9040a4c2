"""Summarise ncu outputs into profiles/ (run here, on the CPU box).

  python profiles/summarize.py launches <launches.csv>        # per-kernel share of the step
  python profiles/summarize.py full <report.ncu-rep> [cfg]    # key metrics per kernel + dram bytes
"""
import collections
import csv
import io
import json
import os
import re
import subprocess
import sys

KEYS = ["Duration", "DRAM Throughput", "Memory Throughput", "L2 Cache Throughput", "L1/TEX Cache Throughput",
        "Compute (SM) Throughput", "Achieved Occupancy", "Theoretical Occupancy", "Registers Per Thread",
        "Grid Size", "Block Size", "Dynamic Shared Memory Per Block", "Executed Ipc Active", "Issue Slots Busy",
        "No Eligible", "Waves Per SM", "dram__bytes_read.sum", "dram__bytes_write.sum"]


def short(name):
    n = re.sub(r"<.*", "", name).replace("void ", "").replace("rtnb::", "")
    return n.split("(")[0].replace("(anonymous namespace)::", "")


def launches(path):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hi]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    tot, cnt = collections.defaultdict(float), collections.Counter()
    for r in rows[hi + 1:]:
        if len(r) <= vi:
            continue
        v = float(r[vi].replace(",", ""))
        v *= {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}.get(r[ui], 1.0)
        tot[short(r[ki])] += v
        cnt[short(r[ki])] += 1
    T = sum(tot.values())
    out = {"launches": sum(cnt.values()), "total_us": T, "kernels": {}}
    for k in sorted(tot, key=lambda k: -tot[k]):
        out["kernels"][k] = {"n": cnt[k], "avg_us": tot[k] / cnt[k], "share": tot[k] / T}
    return out


def full(path):
    txt = subprocess.run(["ncu", "-i", path, "--page", "details", "--csv"], capture_output=True, text=True).stdout
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    res = collections.OrderedDict()
    rows = list(csv.reader(io.StringIO(txt)))
    h = rows[0]
    ki, mi, vi, ui, ii = (h.index(x) for x in ("Kernel Name", "Metric Name", "Metric Value", "Metric Unit", "ID"))
    for r in rows[1:]:
        if r[mi] in KEYS:
            d = res.setdefault(r[ii], {"kernel": short(r[ki])})
            d.setdefault(r[mi], f"{r[vi]} {r[ui]}".strip())
    rr = list(csv.reader(io.StringIO(raw)))
    if rr:
        hh = rr[0]
        cols = {k: hh.index(k) for k in ("ID", "dram__bytes_read.sum", "dram__bytes_write.sum") if k in hh}
        units = rr[1] if len(rr) > 1 else []
        for r in rr[2:]:
            if "ID" not in cols or r[cols["ID"]] not in res:
                continue
            for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
                if k in cols:
                    res[r[cols["ID"]]][k] = f"{r[cols[k]]} {units[cols[k]] if units else ''}".strip()
    return res


def to_bytes(s):
    v, _, u = s.partition(" ")
    return float(v.replace(",", "")) * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3,
                                        "MB": 1e6, "GB": 1e9}.get(u.strip(), 1)


if __name__ == "__main__":
    mode, path = sys.argv[1], sys.argv[2]
    if mode == "launches":
        print(json.dumps(launches(path), indent=1))
    else:
        res = full(path)
        print(json.dumps(res, indent=1))
        if len(sys.argv) > 3:
            cfg = sys.argv[3]
            summ = os.path.join(os.path.dirname(os.path.abspath(__file__)), "ncu_summary.json")
            try:
                allsum = json.load(open(summ))
            except (OSError, ValueError):
                allsum = {}
            entry = allsum.setdefault(cfg, {})
            for d in res.values():
                if "dram__bytes_read.sum" in d:
                    entry[d["kernel"]] = {"dram_bytes_per_launch": to_bytes(d["dram__bytes_read.sum"]) +
                                          to_bytes(d.get("dram__bytes_write.sum", "0 byte")),
                                          "duration": d.get("Duration")}
            json.dump(allsum, open(summ, "w"), indent=1)
