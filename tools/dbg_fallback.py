import sys; sys.path.insert(0,'.')
from paper_2604_26477_b200 import api
from paper_2604_26477_b200.instances import load_heavy_hex
s=api.Session(0); s.set_instance(load_heavy_hex(4)); s.set_weights(api.build_weights(4,resolution=13))
s.sample(api.SolverConfig(variant=api.SolverVariant.discrete_sb,batch_size=4546,seed=7),1)
v=s.fallback_blocks(); print('fallbacks', v & ((1<<40)-1), 'reasons', bin(v>>40))
