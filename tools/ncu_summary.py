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


# ncu kernel name (without "void lbmgpu::" and arguments) -> the bench's
# kernel-stats row of the BASELINE configs' default kernels
BENCH_ROWS = {
    "k_full_aa_even<1, 0, 128, 4>": "full_aa_even_soa",
    "k_full_aa_odd<1, 0, 128, 4>": "full_aa_odd_soa",
    "k_list_aa_even<1, 0>": "list_aa_even_soa",
    "k_list_aa_odd<1, 0>": "list_aa_odd_soa",
    "k_list_pull<1, 1, 0>": "list_pull_soa",
    "k_list_pull<1, 0, 0>": "list_pull_stream_soa",
    "k_list_collide<1>": "list_collide_soa",
    "k_full_fused<1, 0, 160, 4>": "full_push_soa_fused",   # push kind (LBMGPU_PUSH_AS_PULL=0)
    "k_full_fused<1, 1, 160, 4>": "full_push_soa_fused",   # push in pull order (default)
}
# sweeps of the cfg-1 fused launch captured with --steps 20: the push kind
# runs 20, the push in pull order 21 (collide pass + 19 pulls + stream pass)
FUSED_SWEEPS = {"k_full_fused<1, 0, 160, 4>": 20, "k_full_fused<1, 1, 160, 4>": 21}


def build(outdir, dst, sha_file):
    """profiles/ncu_summary.json from the launch lists tools/gpu_ncu_summary.sh
    captured (gpurun_out/ncu_cfg{1..5}.csv), stamped with the csrc content
    hash the capture ran (bench.py drops roofline.traffic when it differs)."""
    sha = open(sha_file).read().strip()
    out = {"csrc_sha16": sha,
           "source": "tools/gpu_ncu_summary.sh: ncu --metrics gpu__time_duration.sum,"
                     "dram__bytes_read.sum,dram__bytes_write.sum --clock-control none, "
                     "bench.py --config C --steps 2 --warmup 1 (cfg 1: --steps 20 --warmup 0), 1x B200",
           "kernels": {}, "configs": {}}
    for cid in ("1", "2", "3", "4", "5"):
        path = f"{outdir}/ncu_cfg{cid}.csv"
        try:
            s = summarise(path)
        except (OSError, StopIteration):
            continue
        rows = {}
        for k, v in s.items():
            row = BENCH_ROWS.get(k)
            if row is None:
                continue
            rec = {"ncu_kernel": k, "launches": v["launches"], "ncu_mean_ns": v["mean_ns"],
                   "dram_read_bytes_per_launch": v["dram_read_bytes_per_launch"],
                   "dram_write_bytes_per_launch": v["dram_write_bytes_per_launch"],
                   "dram_bytes_per_launch": v["dram_bytes_per_launch"]}
            if row.endswith("_fused"):
                # cfg 1 is captured with --steps 20 --warmup 0: one fused
                # launch of 20 (21) sweeps; the bench counts sweeps as launches
                sw = FUSED_SWEEPS.get(k, 20)
                rec["sweeps_per_launch"] = sw
                for key in ("dram_read_bytes_per_launch", "dram_write_bytes_per_launch",
                            "dram_bytes_per_launch"):
                    rec[key] /= sw
                rec["note"] = (f"per sweep of the {sw}-sweep fused launch; the lattice is "
                               "L2-resident, the DRAM bytes are mostly write-back")
            rows[row] = rec
        if cid == "5":
            out["kernels"] = rows
        else:
            out["configs"][cid] = rows
    json.dump(out, open(dst, "w"), indent=1)
    return out


if __name__ == "__main__":
    if sys.argv[1] == "build":
        o = build(sys.argv[2], sys.argv[3], sys.argv[4])
        print(json.dumps(o, indent=1)[:3000])
        sys.exit(0)
    src, dst = sys.argv[1], sys.argv[2]
    s = summarise(src)
    json.dump({"source": src, "kernels": s}, open(dst, "w"), indent=1)
    for k, v in sorted(s.items(), key=lambda kv: -kv[1]["mean_ns"] * kv[1]["launches"]):
        print(f"{k:60s} n={v['launches']:3d} {v['mean_ns'] / 1e3:10.1f} us "
              f"{v['dram_bytes_per_launch'] / 1e9:8.3f} GB {v['dram_GBps'] or 0:8.1f} GB/s")
