"""Sum ncu per-line instruction / stall shares over named line ranges.
usage: python tools/ncu_phases.py report.ncu-rep name:lo-hi ..."""
import re
import subprocess
import sys

out = subprocess.run([sys.executable, __file__.replace("ncu_phases", "ncu_lines"), sys.argv[1], "100000"],
                     capture_output=True, text=True).stdout
ph = []
for a in sys.argv[2:]:
    name, r = a.split(":")
    lo, hi = r.split("-")
    ph.append((name, int(lo), int(hi)))
acc = {n: [0.0, 0.0] for n, _, _ in ph}
acc["other"] = [0.0, 0.0]
for line in out.splitlines():
    m = re.match(r"L\s*(\d+)\s+([\d.]+)% smp\s+([\d.]+)% ins", line)
    if not m:
        if line.startswith("total"):
            print(line)
        continue
    ln, s, e = int(m.group(1)), float(m.group(2)), float(m.group(3))
    for n, lo, hi in ph:
        if lo <= ln <= hi:
            acc[n][0] += s
            acc[n][1] += e
            break
    else:
        acc["other"][0] += s
        acc["other"][1] += e
for n, (s, e) in acc.items():
    print(f"{n:10s} stall {s:5.1f}%  instr {e:5.1f}%")
