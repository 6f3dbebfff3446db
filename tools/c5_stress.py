"""C5 Pareto stress on one GPU: heavy-hex K=4 dSB, 220 x 4546 x runs (runs=100 -> 1.0e8
samples) through the full pipeline; prints stage timings, archive size and HV (the
best-found HV* for the C2 reference point)."""
import json
import os
import sys
import time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2604_26477_b200 import api
from paper_2604_26477_b200.instances import load_heavy_hex

runs = int(sys.argv[1]) if len(sys.argv) > 1 else 100
s = api.Session(0)
inst = load_heavy_hex(4)
s.set_instance(inst)
s.set_weights(api.build_weights(4, resolution=13))
cfg = api.SolverConfig(variant=api.SolverVariant.discrete_sb, batch_size=4546, seed=7)
g = np.load(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden",
                         "c2_heavyhex_k4_dsb.npz"))
r = g["reference"].tolist()
s.pipeline(cfg, runs, 0, -1, True, 4096, fixed_reference=r)  # warm-up: pool-sized buffers, plans
t0 = time.perf_counter()
rep = s.pipeline(cfg, runs, 0, -1, True, 4096, fixed_reference=r)
wall = time.perf_counter() - t0
arc = s.archive()
out = {"runs": runs, "samples": rep["pool_size"], "wall_s": wall, "sampling_s": rep["sampling_s"],
       "pareto_filtering_s": rep["pareto_filtering_s"], "unique_configs": rep["unique_configs"],
       "unique_vectors": rep["unique_vectors"], "archive": rep["archive_size"], "hv_at_c2_reference": rep["hv"],
       "front_method": rep["front_method"], "stages": {k: rep[k] for k in ("dedup_s", "eval_s", "collapse_s",
                                                                          "front_s", "order_s", "hv_s")}}
print(json.dumps(out))
np.savez_compressed(f"gpurun_out/c5_archive_runs{runs}.npz", values=arc.values.astype(np.int32), words=arc.configs,
                    reference=np.array(r), hv=rep["hv"])
