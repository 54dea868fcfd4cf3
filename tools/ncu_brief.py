"""Brief of one ncu report: duration, DRAM bytes, instructions, stall samples,
occupancy (python tools/ncu_brief.py report.ncu-rep [kernel-regex])."""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
args = ["ncu", "-i", rep, "--page", "raw", "--csv"]
if len(sys.argv) > 2:
    args += ["-k", "regex:" + sys.argv[2]]
out = subprocess.run(args, capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = rows[0]
for v in rows[2:]:
    d = dict(zip(h, v))
    print(d.get("Kernel Name", "")[:100])
    for k in ("gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
              "smsp__inst_executed.sum", "sm__warps_active.avg.pct_of_peak_sustained_active",
              "lts__t_sectors_srcunit_tex_op_read.sum", "lts__t_sectors_srcunit_tex_op_write.sum",
              "smsp__issue_active.avg.pct_of_peak_sustained_active",
              "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
              "launch__registers_per_thread", "launch__occupancy_limit_shared_mem"):
        if k in d:
            print(f"  {k:60s} {d[k]}")
    st = {k.replace("smsp__pcsamp_warps_issue_stalled_", ""): float(x)
          for k, x in d.items()
          if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued")
          and x.replace(".", "", 1).isdigit()}
    tot = sum(st.values()) or 1
    print("  stalls:", ", ".join(f"{k} {100 * x / tot:.0f}%" for k, x in
                                 sorted(st.items(), key=lambda kv: -kv[1])[:8]))
