"""Two device-resident C2 pipeline steps (for the ncu launch list: the second step's
kernel shares are the committed evidence; no timing is taken from an ncu run)."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2604_26477_b200 import api
from paper_2604_26477_b200.instances import load_heavy_hex

s = api.Session(0)
s.set_instance(load_heavy_hex(4))
s.set_weights(api.build_weights(4, resolution=13))
cfg = api.SolverConfig(variant=api.SolverVariant.discrete_sb, batch_size=4546, seed=7)
for step in range(2):
    l0 = s.launches()
    rep = s.pipeline(cfg, 1, 0, -1, True, 4096)
    print(f"step {step}: launches {s.launches() - l0} hv {rep['hv']} archive {rep['archive_size']}", flush=True)
