"""One C4-shaped fused dense sampler launch (N=2000, K=3, dSB, H=12) for ncu: a warm-up
sample, then the profiled sample and one tensor-core evaluate_cuts over the pool.
C4_BATCH sets the trajectories per weight (default 1000), C4_WEIGHTS the weight count."""
import os
import sys
import time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2604_26477_b200 import api

batch = int(os.environ.get("C4_BATCH", "1000"))
nw = int(os.environ.get("C4_WEIGHTS", "55"))
s = api.Session(0)
inst = s.generate_uniform_instance(2000, 1.0, 3, 3)
w = api.build_weights(3, resolution=12)[:nw]
s.set_weights(w)
cfg = api.SolverConfig(variant=api.SolverVariant.discrete_sb, batch_size=batch, seed=3,
                       alpha=float(os.environ.get("C4_ALPHA", "0.15")))
s.sample(cfg, 1)
t0 = time.perf_counter()
sec = s.sample(cfg, 1)
wall = time.perf_counter() - t0
pool = s.pool(stamps=False)
t1 = time.perf_counter()
api.evaluate_cuts(inst, pool.words, session=s)
t_eval = time.perf_counter() - t1
print(f"path {s.sampler_path()} samples {pool.size()} sampling {sec:.4f} s wall {wall:.4f} s "
      f"({pool.size() / sec:.3e} samples/s) eval (host round trip) {t_eval:.4f} s")
