"""Summarise an ncu --page raw --csv dump: stalls, pipes, memory."""
import csv
import re
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr, units = rows[0], rows[1]
for vals in rows[2:]:
    d = {h: (v, u) for h, v, u in zip(hdr, vals, units)}

    def f(k):
        try:
            return float(d[k][0].replace(",", ""))
        except Exception:
            return 0.0

    print("kernel:", d.get("Kernel Name", ("?",))[0][:80])
    for k in ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_bytes.sum",
              "smsp__inst_executed.sum", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
              "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
              "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
              "smsp__cycles_active.avg", "sm__cycles_elapsed.avg",
              "launch__registers_per_thread", "sm__warps_active.avg.pct_of_peak_sustained_active"]:
        if k in d:
            print(f"  {k:60s} {d[k][0]:>20s} {d[k][1]}")
    st = [(k, f(k)) for k in d if re.search(r"smsp__average_warp_latency_issue_stalled_[a-z_]+\.ratio$", k)
          or re.search(r"smsp__pcsamp_warps_issue_stalled_[a-z_]+$", k)]
    tot = sum(v for k, v in st if "pcsamp" in k) or 1
    print("  stall samples (pcsamp):")
    for k, v in sorted(st, key=lambda x: -x[1])[:14]:
        if "pcsamp" in k:
            print(f"    {k.replace('smsp__pcsamp_warps_issue_stalled_', ''):40s} {100 * v / tot:6.1f}%")
    pipes = [(k, f(k)) for k in d if re.search(r"sm__inst_executed_pipe_[a-z_0-9]+\.avg\.pct_of_peak_sustained_active$", k)]
    print("  pipe utilisation (% of peak):")
    for k, v in sorted(pipes, key=lambda x: -x[1])[:8]:
        print(f"    {k.replace('sm__inst_executed_pipe_', '').replace('.avg.pct_of_peak_sustained_active', ''):40s} {v:6.1f}")
