"""Stall-reason and throughput summary of an ncu report: python tools/ncu_stalls.py rep.ncu-rep"""
import csv
import subprocess
import sys

out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(out.splitlines()))
h, v = r[0], r[2] if len(r) > 2 else r[1]
d = dict(zip(h, v))
st = [(k, float(x.replace(",", "") or 0)) for k, x in d.items()
      if "pcsamp_warps_issue_stalled" in k and not k.endswith("not_issued")]
tot = sum(x for _, x in st)
for k, x in sorted(st, key=lambda kv: -kv[1])[:12]:
    print(f"{k.replace('smsp__pcsamp_warps_issue_stalled_', ''):28s} {100 * x / tot:5.1f}%")
for k in ["gpu__time_duration.sum", "smsp__inst_executed.sum", "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
          "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
          "sm__warps_active.avg.pct_of_peak_sustained_active", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
          "dram__throughput.avg.pct_of_peak_sustained_elapsed", "launch__registers_per_thread"]:
    print(f"{k:60s} {d.get(k)}")
