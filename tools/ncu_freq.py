"""Instructions per unit of work by execution-frequency class: SASS instructions of an ncu
report grouped by (executions / units), e.g. per warp-step of the sampler.
usage: python tools/ncu_freq.py report.ncu-rep units [min_share]"""
import collections
import csv
import io
import subprocess
import sys

rep, units = sys.argv[1], float(sys.argv[2])
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[1]
iA, iS, iE = hdr.index("Address"), hdr.index("Source"), hdr.index("Instructions Executed")
iW = hdr.index("Warp Stall Sampling (All Samples)")
cls = collections.OrderedDict()
tot = 0
totw = 0
for r in rows[2:]:
    if len(r) < len(hdr) or not r[iE]:
        continue
    e = int(r[iE])
    w = int(r[iW] or 0)
    tot += e
    totw += w
    f = round(e / units, 3)
    c = cls.setdefault(f, [0, 0, r[iA], r[iS]])
    c[0] += 1
    c[1] += w
print(f"total {tot / units:.1f} instr/unit  ({tot:.4e})")
for f, (k, w, a, s) in sorted(cls.items(), key=lambda t: -t[0] * t[1][0]):
    if f * k < 2:
        continue
    print(f"freq {f:8.3f} x {k:5d} instrs = {f * k:7.1f}/unit  stall {100 * w / max(totw, 1):5.1f}%  first {a[-5:]} {s.strip()[:50]}")
