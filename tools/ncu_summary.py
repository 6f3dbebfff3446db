"""Key counters of the first kernel in an ncu report (raw page).
usage: python tools/ncu_summary.py report.ncu-rep"""
import csv
import io
import subprocess
import sys

out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h, units, v = rows[0], rows[1], rows[2]
want = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_bytes.sum",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__inst_executed.sum",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "smsp__warps_active.avg.per_cycle_active", "launch__registers_per_thread",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "sm__cycles_elapsed.avg.per_second"]
for w in want:
    if w in h:
        i = h.index(w)
        print(f"{w:60s} {v[i]} {units[i]}")
st = [(h[i], float(v[i].replace(",", ""))) for i in range(len(h))
      if h[i].startswith("smsp__pcsamp_warps_issue_stalled") and not h[i].endswith("not_issued")
      and v[i].replace(",", "").replace(".", "").isdigit()]
tot = sum(x for _, x in st) or 1
for name, x in sorted(st, key=lambda kv: -kv[1])[:10]:
    print(f"  {name[33:]:40s} {x / tot * 100:5.1f}%")
