"""C1 throughput on one GPU: 42-node heavy-hex K=3, bSB, 190 weights (H=21) x batch 3000 =
570,000 samples, seed 7, through the resident pipeline (sample -> filter -> r -> HV), with
two warm-up calls; prints the mean step and stage times of 10 calls."""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2604_26477_b200 import api  # noqa: E402
from paper_2604_26477_b200.instances import load_heavy_hex  # noqa: E402

s = api.Session(0)
s.set_instance(load_heavy_hex(3))
s.set_weights(api.build_weights(3, resolution=21))
cfg = api.SolverConfig(variant=api.SolverVariant.ballistic_sb, batch_size=3000, seed=7)
for _ in range(2):
    s.pipeline(cfg, 1, 0, -1, True, 4096)
reps = [s.pipeline(cfg, 1, 0, -1, True, 4096) for _ in range(10)]
e2e = float(np.mean([r["end_to_end_s"] for r in reps]))
samp = float(np.mean([r["sampling_s"] for r in reps]))
print(json.dumps({"workload": "C1: heavy-hex 42, K=3, bSB, 190 x 3000", "samples": reps[-1]["pool_size"],
                  "step_s": e2e, "samples_per_s": reps[-1]["pool_size"] / e2e, "sampling_s": samp,
                  "sampling_samples_per_s": reps[-1]["pool_size"] / samp, "archive": reps[-1]["archive_size"],
                  "hv": reps[-1]["hv"], "pareto_filtering_s": float(np.mean([r["pareto_filtering_s"] for r in reps]))}))
