"""Probe: does the CUPTI range profiler (libmomc_b200_prof.so) see torch kernels and the momc
sampler kernel?"""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2604_26477_b200 import api
from paper_2604_26477_b200.instances import load_heavy_hex

lib = ctypes.CDLL(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "paper_2604_26477_b200", "libmomc_b200_prof.so"))
lib.momc_prof_error.restype = ctypes.c_char_p
x = torch.ones(1 << 24, device="cuda:0")
s = api.Session(0)
s.set_instance(load_heavy_hex(4))
s.set_weights(api.build_weights(4, resolution=13))
cfg = api.SolverConfig(variant=api.SolverVariant.discrete_sb, batch_size=4546, seed=7)
s.sample(cfg, 1)
for name, fn, sub in (("torch", lambda: x.mul_(2.0), "elementwise"), ("momc", lambda: s.sample(cfg, 1), "sb_batch")):
    # user range, user replay
    torch.cuda.synchronize()
    rc = lib.momc_prof_begin_mode(0, 1)
    print(name, "user begin", rc, lib.momc_prof_error())
    for p in range(8):
        lib.momc_prof_pass_begin()
        fn()
        torch.cuda.synchronize()
        done = lib.momc_prof_pass_end()
        print("  pass", p, "done", done, lib.momc_prof_error())
        if done != 0:
            break
    rd, wr, n = ctypes.c_double(0), ctypes.c_double(0), ctypes.c_int(0)
    rc = lib.momc_prof_end(sub.encode(), ctypes.byref(rd), ctypes.byref(wr), ctypes.byref(n))
    print(name, "user end", rc, rd.value, wr.value, n.value, lib.momc_prof_error()[:400])
    torch.cuda.synchronize()
    rc = lib.momc_prof_begin(0)
    print(name, "begin", rc, lib.momc_prof_error())
    fn()
    torch.cuda.synchronize()
    rd, wr, n = ctypes.c_double(0), ctypes.c_double(0), ctypes.c_int(0)
    rc = lib.momc_prof_end(sub.encode(), ctypes.byref(rd), ctypes.byref(wr), ctypes.byref(n))
    print(name, "end", rc, rd.value, wr.value, n.value, lib.momc_prof_error()[:400])
