#!/usr/bin/env python3
"""Summarise ncu CSV launch lists into profiles/*.json.

    python tools/ncu_summary.py gpurun_out/launches_cfg5.csv profiles/r01_cfg5_launches.json \
        [--alg-bytes full_aa=80966451200 ...]

Per kernel: launches, mean gpu__time_duration, mean dram read+write bytes per
launch and the implied DRAM GB/s (cold-cache, serialised: compare shares, not
absolutes, with the bench's CUDA-event numbers).
"""
import csv
import json
import sys
from collections import defaultdict


def parse(path):
    rows = list(csv.reader(open(path)))
    start = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    hdr = rows[start]
    ix = {k: j for j, k in enumerate(hdr)}
    per = defaultdict(dict)
    names = {}
    for r in rows[start + 1:]:
        if len(r) < len(hdr):
            continue
        kid = int(r[ix["ID"]])
        names[kid] = r[ix["Kernel Name"]]
        v = r[ix["Metric Value"]].replace(",", "")
        try:
            per[kid][r[ix["Metric Name"]]] = float(v)
        except ValueError:
            pass
    return names, per


def short(name):
    n = name.split("(")[0]
    n = n.replace("void ", "").replace("lbmgpu::", "")
    return n


def summarise(path):
    names, per = parse(path)
    agg = defaultdict(lambda: {"launches": 0, "ns": 0.0, "rd": 0.0, "wr": 0.0})
    for kid, m in per.items():
        a = agg[short(names[kid])]
        a["launches"] += 1
        a["ns"] += m.get("gpu__time_duration.sum", 0.0)
        a["rd"] += m.get("dram__bytes_read.sum", 0.0)
        a["wr"] += m.get("dram__bytes_write.sum", 0.0)
    out = {}
    total = sum(a["ns"] for a in agg.values()) or 1.0
    for k, a in agg.items():
        n = a["launches"]
        b = (a["rd"] + a["wr"]) / n
        out[k] = {"launches": n, "mean_ns": a["ns"] / n, "share_of_listed": a["ns"] / total,
                  "dram_read_bytes_per_launch": a["rd"] / n,
                  "dram_write_bytes_per_launch": a["wr"] / n,
                  "dram_bytes_per_launch": b,
                  "dram_GBps": b / (a["ns"] / n) if a["ns"] else None}
    return out


if __name__ == "__main__":
    src, dst = sys.argv[1], sys.argv[2]
    s = summarise(src)
    json.dump({"source": src, "kernels": s}, open(dst, "w"), indent=1)
    for k, v in sorted(s.items(), key=lambda kv: -kv[1]["mean_ns"] * kv[1]["launches"]):
        print(f"{k:60s} n={v['launches']:3d} {v['mean_ns'] / 1e3:10.1f} us "
              f"{v['dram_bytes_per_launch'] / 1e9:8.3f} GB {v['dram_GBps'] or 0:8.1f} GB/s")
