"""Streaming time-to-optimal-hypervolume on one GPU.

Run after run (run r = the r-th replica of the C1/C2 pool: same lattice and batch, RNG key
run_key(seed, r)), the run's archive is merged into the running archive on the device and
its HV at the frozen reference point is compared with HV* of the exact front
(tests/golden/heavyhex42_k{k}_exact.npz, tools/exact_front.py). Prints the trace and the
first run whose running archive reaches HV* exactly."""
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2604_26477_b200 import api  # noqa: E402
from paper_2604_26477_b200.instances import load_heavy_hex  # noqa: E402


def main():
    k = int(sys.argv[1]) if len(sys.argv) > 1 else 4
    max_runs = int(sys.argv[2]) if len(sys.argv) > 2 else 200
    g = np.load(os.path.join(ROOT, "tests", "golden", f"heavyhex42_k{k}_exact.npz"))
    r = [float(x) for x in g["reference"]]
    hv_star = float(g["hv_star"])
    exact = {tuple(v) for v in g["values"]}
    inst = load_heavy_hex(k)
    H = 21 if k == 3 else 13
    batch = 3000 if k == 3 else 4546
    variant = api.SolverVariant.ballistic_sb if k == 3 else api.SolverVariant.discrete_sb
    s = api.Session(0)
    s.set_instance(inst)
    s.set_weights(api.build_weights(k, resolution=H))
    cfg = api.SolverConfig(variant=variant, batch_size=batch, seed=7)
    from paper_2604_26477_b200 import streaming
    rps = 2 if k == 4 else 1  # runs per C-ABI call, as bench.py (TTO_RUNS_PER_STEP)
    streaming.time_to_target(s, cfg, r, hv_star, 2 * rps, runs_per_step=rps)  # warm-up (allocations, plans)
    trace = []
    res = streaming.time_to_target(s, cfg, r, hv_star, max_runs, trace=trace, runs_per_step=rps)
    reached = res["runs"] if res["reached"] else None
    arc = s.archive(with_configs=False)
    missing = [list(x) for x in exact - {tuple(v) for v in arc.values}]
    print(json.dumps({"k": k, "hv_star": hv_star, "reached_at_run": reached, "result": res, "final": trace[-1], "missing_front_points": len(missing),
                      "missing_sample": missing[:10],
                      "trace": trace[:: max(1, len(trace) // 40)]}))


if __name__ == "__main__":
    main()
