"""One sampler launch of the C2 shape (for ncu). argv[1]: dsb|bsb"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2604_26477_b200 import api
from paper_2604_26477_b200.instances import load_heavy_hex
var = sys.argv[1] if len(sys.argv) > 1 else "dsb"
k, H, batch = (4, 13, 4546) if var == "dsb" else (3, 21, 3000)
s = api.Session(0)
s.set_instance(load_heavy_hex(k)); s.set_weights(api.build_weights(k, resolution=H))
t = s.sample(api.SolverConfig(variant=api.parse_variant(var), batch_size=batch, seed=7), 1)
print(f"{var}: {t*1e3:.3f} ms")
