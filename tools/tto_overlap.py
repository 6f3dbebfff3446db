"""Sequential vs overlapped streaming time-to-optimal (K=4, C2 shape) on one GPU."""
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


def main():
    k = 4
    g = np.load(os.path.join(ROOT, "tests", "golden", f"heavyhex42_k{k}_exact.npz"))
    r = [float(x) for x in g["reference"]]
    target = float(g["hv_star"])
    inst = load_heavy_hex(k)
    w = api.build_weights(k, resolution=13)
    cfg = api.SolverConfig(variant=api.SolverVariant.discrete_sb, batch_size=4546, seed=7)
    dev = torch.device("cuda", 0)
    out = {}
    for it, S in enumerate((1, 1, 2, 2, 3)):
        sessions = [api.Session(0) for _ in range(S)]
        for s in sessions:
            s.set_instance(inst)
            s.set_weights(w)
            s.pipeline(cfg, 1, 0, s.num_blocks(cfg, 1), do_hv=False)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        if S == 1:
            res = streaming.time_to_target(sessions[0], cfg, r, target, 300, device=dev, runs_per_step=[1, 2][it])
        else:
            merger = api.Session(0)
            merger.set_instance(inst)
            res = streaming.time_to_target_overlapped(sessions, merger, cfg, r, target, 300,
                                                      runs_per_step=[0, 0, 1, 2, 2][it])
        res["wall"] = time.perf_counter() - t0
        out[f"{it}:sessions{S}:R{[1, 2, 1, 2, 2][it]}"] = {"seconds": round(res["seconds"], 4), "runs": res["runs"]}
        del sessions
    print(json.dumps(out))


if __name__ == "__main__":
    main()
