"""SASS-level view of an ncu report: instructions executed and shared-memory bank-conflict
wavefronts per SASS instruction, heaviest first (or a listing of an address range).
usage: python tools/ncu_sass.py report.ncu-rep [top|lo-hi] [--conflicts]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
arg = sys.argv[2] if len(sys.argv) > 2 else "40"
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[1]
iA, iS, iE = hdr.index("Address"), hdr.index("Source"), hdr.index("Instructions Executed")
iX = hdr.index("L1 Wavefronts Shared Excessive")
iW = hdr.index("Warp Stall Sampling (All Samples)")
recs = []
for r in rows[2:]:
    if len(r) < len(hdr):
        continue
    try:
        recs.append((int(r[iA], 16), r[iS], int(r[iE] or 0), int(r[iX] or 0), int(r[iW] or 0)))
    except ValueError:
        continue
tot = sum(x[2] for x in recs) or 1
totx = sum(x[3] for x in recs) or 1
print(f"total instr {tot:.4e}  excessive smem wavefronts {totx:.4e}")
if "-" in arg:
    lo, hi = (int(v, 16) for v in arg.split("-"))
    for a, s, e, x, w in recs:
        if lo <= a <= hi:
            print(f"{a:6x} {100*e/tot:5.2f}% x{x:>10d} w{w:>6d}  {s}")
else:
    key = 3 if "--conflicts" in sys.argv else 2
    for a, s, e, x, w in sorted(recs, key=lambda t: -t[key])[: int(arg)]:
        print(f"{a:6x} {100*e/tot:5.2f}% x{x:>10d} w{w:>6d}  {s}")
