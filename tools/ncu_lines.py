"""Per-source-line summary of an ncu report (the correlated cuda,sass source page): warp
stall samples and executed warp instructions per CUDA line, heaviest first.
usage: python tools/ncu_lines.py report.ncu-rep [top]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = None
agg = {}
cur = None
stall_cols = []
for r in rows:
    if len(r) > 3 and r[0] == "Line No":
        hdr = r
        iW = hdr.index("Warp Stall Sampling (All Samples)")
        iE = hdr.index("Instructions Executed")
        stall_cols = [(i, c) for i, c in enumerate(hdr) if c.startswith("stall_") and "Not Issued" not in c]
        continue
    if hdr is None or len(r) < len(hdr):
        continue
    if r[0]:  # a cuda line row (aggregate of its sass)
        try:
            w = int(r[iW] or 0)
            e = int(r[iE] or 0)
        except ValueError:
            continue
        st = {c: int(r[i] or 0) for i, c in stall_cols if (r[i] or "0").isdigit()}
        key = int(r[0])
        a = agg.setdefault(key, [0, 0, r[1][:90], {}])
        a[0] += w
        a[1] += e
        for c, v in st.items():
            a[3][c] = a[3].get(c, 0) + v
tot_w = sum(a[0] for a in agg.values()) or 1
tot_e = sum(a[1] for a in agg.values()) or 1
print(f"total stall samples {tot_w}, warp instructions {tot_e:.4e}")
for ln, (w, e, src, st) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
    topst = sorted(st.items(), key=lambda kv: -kv[1])[:3]
    print(f"L{ln:5d} {w / tot_w * 100:5.1f}% smp {e / tot_e * 100:5.1f}% ins  {src:90s} " +
          " ".join(f"{c[6:]}={v}" for c, v in topst))
