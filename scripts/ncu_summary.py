"""Summarise an ncu report: duration, DRAM, issue, stalls (development helper)."""
import csv, subprocess, sys
rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = rows[0]
for vals in rows[2:]:
    d = dict(zip(hdr, vals))
    print("----", d.get("Kernel Name", "")[:60], d.get("gpu__time_duration.sum"), "ms")
    for k in ["dram__bytes_read.sum", "dram__bytes_write.sum", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
              "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
              "smsp__inst_executed.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
              "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread"]:
        if k in d:
            print(f"  {k} = {d[k]}")
    st = [(h, v) for h, v in d.items() if h.startswith("smsp__average_warps_issue_stalled_") and h.endswith("_per_issue_active.ratio")]
    st = sorted(st, key=lambda x: -float(x[1] or 0))
    print("  stalls:", " ".join(f"{h.replace('smsp__average_warps_issue_stalled_','').replace('_per_issue_active.ratio','')}={float(v):.2f}" for h, v in st[:8]))
