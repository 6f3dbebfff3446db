"""SASS opcode mix of an ncu report (source page), per `unit` work items.
usage: python tools/ncu_ops.py report.ncu-rep units [top]"""
import collections
import csv
import io
import subprocess
import sys

out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
units = float(sys.argv[2])
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
for hi, r in enumerate(rows):
    if "Source" in r and "Instructions Executed" in r:
        break
h = rows[hi]
i_src, i_ex = h.index("Source"), h.index("Instructions Executed")
tot, byop = 0, collections.Counter()
for r in rows[hi + 1:]:
    try:
        n = int(r[i_ex])
    except (ValueError, IndexError):
        continue
    t = r[i_src].split()
    if not t:
        continue
    op = t[1] if t[0].startswith("@") else t[0]
    byop[op.split(".")[0]] += n
    tot += n
print(f"total {tot:.4e} = {tot / units:.1f} per unit")
print(" ".join(f"{k}:{v / units:.1f}" for k, v in byop.most_common(top)))
