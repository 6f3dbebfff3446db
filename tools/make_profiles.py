"""Summaries committed under profiles/ from the raw ncu outputs in gpurun_out/.

  python tools/make_profiles.py LAUNCH_CSV STEP_LAUNCHES_JSON  NCU_REP SAMPLER_SUMMARY_JSON
  python tools/make_profiles.py --kernel NCU_REP OUT_JSON "description" ALGORITHMIC_BYTES "command"
  python tools/make_profiles.py --launches LAUNCH_CSV OUT_JSON "command"   (whole run, per kernel)

LAUNCH_CSV : `ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file ...
             python tools/profile_step.py` (two C2 steps; the second is summarised)
NCU_REP    : `ncu --set full --import-source on --clock-control none -k regex:sb_batch -c 1
             -o ... python tools/profile_sampler.py dsb`
"""
import csv
import io
import json
import subprocess
import sys

METRICS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
           "sm__throughput.avg.pct_of_peak_sustained_elapsed", "smsp__issue_active.avg.pct_of_peak_sustained_active",
           "sm__inst_executed.avg.per_cycle_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
           "launch__registers_per_thread", "launch__grid_size", "launch__block_size", "smsp__inst_executed.sum",
           "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
           "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
           "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
           "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "sm__cycles_elapsed.avg.per_second",
           "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
           "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio",
           "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio",
           "smsp__average_warps_issue_stalled_not_selected_per_issue_active.ratio",
           "smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio",
           "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
           "smsp__average_warps_issue_stalled_mio_throttle_per_issue_active.ratio",
           "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
           "dram__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_bytes.sum"]


def launches(path, out):
    rows = [r for r in csv.reader(open(path)) if r]
    hdr_i = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr = rows[hdr_i]
    ki, mi, vi = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
    recs = [(r[ki], float(r[vi].replace(",", ""))) for r in rows[hdr_i + 1:]
            if len(r) > vi and r[mi] == "gpu__time_duration.sum"]
    half = len(recs) // 2  # two identical steps: keep the second
    step = recs[half:]
    tot = sum(v for _, v in step)
    agg = {}
    for k, v in step:
        name = k.split("(")[0].replace("void ", "").replace("momc_b200::", "").replace("(anonymous namespace)::", "")
        agg[name] = agg.get(name, 0.0) + v
    unit = "us" if tot > 1000 else "ms"
    data = {"source": "ncu --metrics gpu__time_duration.sum --clock-control none (cold-cache, serialised launches; "
                      "compare shares, not absolutes)",
            "command": "python tools/profile_step.py (2 device-resident C2 steps; second step summarised)",
            "launches_per_step": len(step), "total_kernel_ns": tot,
            "kernels": [{"kernel": k, "ns": v, "share": v / tot} for k, v in sorted(agg.items(), key=lambda x: -x[1])]}
    json.dump(data, open(out, "w"), indent=1)
    print(f"{out}: {len(step)} launches, top {data['kernels'][0]['kernel']} {data['kernels'][0]['share']:.3f}")


def whole_run(path, out, command):
    rows = [r for r in csv.reader(open(path)) if r]
    hdr_i = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr = rows[hdr_i]
    ki, mi, vi = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
    recs = [(r[ki], float(r[vi].replace(",", ""))) for r in rows[hdr_i + 1:]
            if len(r) > vi and r[mi] == "gpu__time_duration.sum"]
    tot = sum(v for _, v in recs)
    agg = {}
    for k, v in recs:
        name = k.split("(")[0].replace("void ", "").replace("momc_b200::", "").replace("(anonymous namespace)::", "")
        a = agg.setdefault(name, [0.0, 0])
        a[0] += v
        a[1] += 1
    data = {"source": "ncu --metrics gpu__time_duration.sum --clock-control none (cold-cache, serialised launches; "
                      "compare shares, not absolutes)", "command": command, "launches": len(recs),
            "total_kernel_ns": tot,
            "kernels": [{"kernel": k, "ns": a[0], "launches": a[1], "share": a[0] / tot}
                        for k, a in sorted(agg.items(), key=lambda x: -x[1][0])]}
    json.dump(data, open(out, "w"), indent=1)
    print(f"{out}: {len(recs)} launches, top {data['kernels'][0]['kernel']} {data['kernels'][0]['share']:.3f}")


def sampler(rep, out, desc=None, alg_bytes=8 * 1000120, command=None):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    d = dict(zip(rows[0], rows[2]))
    units = dict(zip(rows[0], rows[1]))
    m = {}
    for k in METRICS:
        if k in d:
            try:
                m[k] = float(d[k].replace(",", ""))
            except ValueError:
                pass
    def to_bytes(k):
        u = units.get(k, "byte").lower()
        scale = {"byte": 1, "kbyte": 1e3, "mbyte": 1e6, "gbyte": 1e9}.get(u, 1)
        return m.get(k, 0.0) * scale
    dram = to_bytes("dram__bytes_read.sum") + to_bytes("dram__bytes_write.sum")
    data = {"kernel": desc or "sb_batch_kernel<42,4,1,3,true,128,4> (dSB, heavy-hex K=4, 220 x 4546 = 1,000,120 samples)",
            "source": f"ncu --set full --import-source on --clock-control none, "
                      f"{command or 'python tools/profile_sampler.py dsb'} ({rep})",
            "metrics": m, "units": {k: units.get(k, "") for k in m},
            "dram_bytes_per_launch": dram, "algorithmic_bytes_per_launch": alg_bytes}
    json.dump(data, open(out, "w"), indent=1)
    print(f"{out}: {m.get('gpu__time_duration.sum')} {units.get('gpu__time_duration.sum')}, dram {dram:.0f} B")


if __name__ == "__main__":
    if sys.argv[1] == "--kernel":
        sampler(sys.argv[2], sys.argv[3], sys.argv[4], float(sys.argv[5]), sys.argv[6])
    elif sys.argv[1] == "--launches":
        whole_run(sys.argv[2], sys.argv[3], sys.argv[4])
    else:
        launches(sys.argv[1], sys.argv[2])
        sampler(sys.argv[3], sys.argv[4])
