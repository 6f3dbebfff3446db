"""Per-run cost of the streaming check (momc_b200_stream_step after sampling: one collapse +
front over the run's pool and the running archive, plus the HV when the value set changed),
K=4 C2 shape, runs_per_step=1. Prints mean / median pareto_filtering_s over runs 5..N."""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2604_26477_b200 import api  # noqa: E402
from paper_2604_26477_b200.instances import load_heavy_hex  # noqa: E402

N = int(sys.argv[1]) if len(sys.argv) > 1 else 60
g = np.load(os.path.join(ROOT, "tests", "golden", "heavyhex42_k4_exact.npz"))
r = [float(x) for x in g["reference"]]
s = api.Session(0)
s.set_instance(load_heavy_hex(4))
s.set_weights(api.build_weights(4, resolution=13))
cfg = api.SolverConfig(variant=api.SolverVariant.discrete_sb, batch_size=4546, seed=7)
per_run = s.num_blocks(cfg, 1)
s.running_reset()
filt, samp, F = [], [], []
for run in range(N):
    hv, f, rep = s.stream_step(cfg, run + 1, run * per_run, (run + 1) * per_run, r)
    filt.append(rep["pareto_filtering_s"] * 1e3)
    samp.append(rep["sampling_s"] * 1e3)
    F.append(f)
print(json.dumps({"runs": N, "check_ms_mean": float(np.mean(filt[5:])), "check_ms_median": float(np.median(filt[5:])),
                  "check_ms_max": float(np.max(filt[5:])), "sampling_ms_mean": float(np.mean(samp[5:])),
                  "archive_final": F[-1], "hv_final": hv}))
