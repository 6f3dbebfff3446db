"""Quick sampler throughput probe (device events), C2 shape: heavy-hex K=4, 220 weights, dSB."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2604_26477_b200 import api
from paper_2604_26477_b200.instances import load_heavy_hex

s = api.Session(0)
for k, H, var, batch in ((4, 13, api.SolverVariant.discrete_sb, 4546), (3, 21, api.SolverVariant.ballistic_sb, 3000)):
    inst = load_heavy_hex(k)
    w = api.build_weights(k, resolution=H)
    s.set_instance(inst); s.set_weights(w)
    cfg = api.SolverConfig(variant=var, batch_size=batch, seed=7)
    for rep in range(3):
        t = s.sample(cfg, 1)
    M = len(w) * batch
    print(f"K={k} {var.name}: {M} samples in {t*1e3:.3f} ms -> {M/t:.4e} samples/s", flush=True)
