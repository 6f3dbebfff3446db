"""Per-run wall-time breakdown of the sequential streaming loop (K=4, C2 shape)."""
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2604_26477_b200 import api, streaming  # noqa: E402
from paper_2604_26477_b200 import distributed as mdist  # noqa: E402
from paper_2604_26477_b200.instances import load_heavy_hex  # noqa: E402


def main():
    k = 4
    g = np.load(os.path.join(ROOT, "tests", "golden", f"heavyhex42_k{k}_exact.npz"))
    r = [float(x) for x in g["reference"]]
    inst = load_heavy_hex(k)
    w = api.build_weights(k, resolution=13)
    cfg = api.SolverConfig(variant=api.SolverVariant.discrete_sb, batch_size=4546, seed=7)
    dev = torch.device("cuda", 0)
    s = api.Session(0)
    s.set_instance(inst)
    s.set_weights(w)
    per_run = s.num_blocks(cfg, 1)
    s.pipeline(cfg, 1, 0, per_run, do_hv=False)
    torch.cuda.synchronize()
    T = {"pipeline": 0.0, "sampling": 0.0, "filter_in_pipeline": 0.0, "front_copy": 0.0, "merge": 0.0, "hv": 0.0}
    running = None
    runs = 30
    t00 = time.perf_counter()
    for run in range(runs):
        t0 = time.perf_counter()
        rep = s.pipeline(cfg, run + 1, run * per_run, (run + 1) * per_run, do_hv=False)
        t1 = time.perf_counter()
        T["pipeline"] += t1 - t0
        T["sampling"] += rep["sampling_s"]
        T["filter_in_pipeline"] += rep["pareto_filtering_s"]
        mine = streaming._packed_front(s, dev)
        t2 = time.perf_counter()
        T["front_copy"] += t2 - t1
        if running is not None:
            rows = torch.cat([running, mine], dim=0)
            mdist.merge_on_device(s, rows[:, :k].contiguous().view(torch.float64), rows[:, k:].contiguous())
            running = streaming._packed_front(s, dev)
        else:
            running = mine
        t3 = time.perf_counter()
        T["merge"] += t3 - t2
        s.archive_hypervolume(r)
        T["hv"] += time.perf_counter() - t3
    total = time.perf_counter() - t00
    print(json.dumps({"per_run_ms": {k2: round(v / runs * 1e3, 3) for k2, v in T.items()},
                      "total_per_run_ms": round(total / runs * 1e3, 3)}))


if __name__ == "__main__":
    main()
