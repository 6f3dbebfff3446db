"""Exact Pareto fronts of the 42-node heavy-hex instances on one GPU.

Prints the front size, the exact reference point, HV* at the bench's frozen reference point
(the sampled r clamped under the exact front) and the wall time; with --save [DIR] writes
(DIR, default tests/golden)/heavyhex42_k{3,4}_exact.npz (front values + owners, r, HV*), which the bench
uses as its time-to-optimal target."""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2604_26477_b200 import api  # noqa: E402
from paper_2604_26477_b200.instances import load_heavy_hex  # noqa: E402


def main():
    save = "--save" in sys.argv
    outdir = sys.argv[sys.argv.index("--save") + 1] if save and len(sys.argv) > sys.argv.index("--save") + 1 \
        else os.path.join(ROOT, "tests", "golden")
    s = api.Session(0)
    out = {}
    for k in (3, 4):
        inst = load_heavy_hex(k)
        api.brute_force_pareto(inst, session=s)  # warm-up (module load, pools)
        t0 = time.perf_counter()
        exact, r_exact = api.brute_force_pareto(inst, session=s, with_reference=True)
        dt = time.perf_counter() - t0
        r_s = api.reference_point_sampled(inst, 4096, 7, session=s)
        r = api.clamp_reference(r_s, exact)
        hv = api.hypervolume(exact, r, session=s)
        out[f"k{k}"] = {"front": exact.size(), "seconds": dt, "reference_exact": r_exact,
                        "reference_sampled": r_s, "reference_frozen": r, "hv_star": hv}
        if save:
            np.savez_compressed(os.path.join(outdir, f"heavyhex42_k{k}_exact.npz"),
                                values=exact.values, words=exact.configs, reference=np.array(r),
                                reference_exact=np.array(r_exact), hv_star=hv)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
