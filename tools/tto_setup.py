import os, sys, time
sys.path.insert(0, "/root/repo")
import numpy as np, torch
from paper_2604_26477_b200 import api
from paper_2604_26477_b200.instances import load_heavy_hex
g = np.load("/root/repo/tests/golden/heavyhex42_k4_exact.npz")
r = [float(x) for x in g["reference"]]
inst = load_heavy_hex(4); w = api.build_weights(4, resolution=13)
cfg = api.SolverConfig(variant=api.SolverVariant.discrete_sb, batch_size=4546, seed=7)
s = api.Session(0); s.set_instance(inst); s.set_weights(w); s.pipeline(cfg, 1, 0, s.num_blocks(cfg, 1), do_hv=False)
torch.cuda.synchronize()
for it in range(3):
    t0 = time.perf_counter(); s.set_instance(inst); t1 = time.perf_counter(); s.set_weights(w); t2 = time.perf_counter()
    per_run = s.num_blocks(cfg, 1); s.running_reset()
    ts = []
    for run in range(4):
        a = time.perf_counter(); s.stream_step(cfg, run + 1, run * per_run, (run + 1) * per_run, r); ts.append((time.perf_counter() - a) * 1e3)
    print(f"set_instance {1e3*(t1-t0):.2f} ms set_weights {1e3*(t2-t1):.2f} ms steps {['%.2f' % x for x in ts]}")
