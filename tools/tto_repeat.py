"""Sequential streaming time-to-optimal (K=4, C2 shape) repeated in one process: first-call
costs show up as a slower first repetition."""
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2604_26477_b200 import api, streaming  # noqa: E402
from paper_2604_26477_b200.instances import load_heavy_hex  # noqa: E402

R = int(sys.argv[1]) if len(sys.argv) > 1 else 2
g = np.load(os.path.join(ROOT, "tests", "golden", "heavyhex42_k4_exact.npz"))
r = [float(x) for x in g["reference"]]
inst = load_heavy_hex(4)
w = api.build_weights(4, resolution=13)
cfg = api.SolverConfig(variant=api.SolverVariant.discrete_sb, batch_size=4546, seed=7)
out = []
for rep in range(3):
    s = api.Session(0)
    s.set_instance(inst)
    s.set_weights(w)
    s.pipeline(cfg, 1, 0, s.num_blocks(cfg, 1), do_hv=False)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    res = streaming.time_to_target(s, cfg, r, float(g["hv_star"]), 300, runs_per_step=R)
    out.append(round(time.perf_counter() - t0, 4))
    del s
print(json.dumps({"runs_per_step": R, "seconds": out}))
