"""Generates the committed golden fixtures from the reference itself (run here, where
/root/reference exists; the fixtures travel to the GPU box, the reference does not).

  c1_heavyhex_k3_bsb.npz  C1: 42-node heavy-hex K=3, bSB, 190 weights (H=21) x 3000, seed 7
  c2_heavyhex_k4_dsb.npz  C2: 42-node heavy-hex K=4, dSB, 220 weights (H=13) x 4546, seed 7
Each holds the pool fold, the reference archive (values + lex-smallest configs), the
sampled reference point (reference_point_sampled(inst, 4096, 7) clamped under the
archive) and the exact hypervolume, all computed by oracle/_ref/libmomc_ref.so.
Usage: python tests/golden/make_golden.py [c1|c2|all]
"""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from oracle.refbind import RefLib, make_cfg, pool_fold  # noqa: E402
from paper_2604_26477_b200.instances import ensure_heavy_hex  # noqa: E402

CASES = {
    "c1": dict(k=3, H=21, variant="bsb", batch=3000, file="c1_heavyhex_k3_bsb.npz"),
    "c2": dict(k=4, H=13, variant="dsb", batch=4546, file="c2_heavyhex_k4_dsb.npz"),
}


def make(name):
    c = CASES[name]
    R = RefLib()
    path = ensure_heavy_hex(c["k"])
    inst = R.instance_load(path)
    nums = R.das_dennis(c["k"], c["H"])
    cfg = make_cfg(c["variant"], batch_size=c["batch"], seed=7, threads=os.cpu_count() or 8)
    t = time.time()
    words = R.run_sampler(inst, nums, c["H"], cfg, 1)["words"]
    ts = time.time() - t
    t = time.time()
    arc = R.filter_pool(inst, words)
    tf = time.time() - t
    r = R.reference_point_sampled(inst, 4096, 7)
    r = np.minimum(r, arc.values.min(axis=0))
    t = time.time()
    hv = R.hypervolume(arc.values, r)
    th = time.time() - t
    out = os.path.join(os.path.dirname(os.path.abspath(__file__)), c["file"])
    np.savez_compressed(out, k=c["k"], H=c["H"], variant=c["variant"], batch=c["batch"], seed=7,
                        pool_size=words.shape[0], pool_fold=np.uint64(pool_fold(words)),
                        archive_values=arc.values.astype(np.int32), archive_words=arc.words, reference=r, hv=hv,
                        cpu_seconds=np.array([ts, tf, th]))
    print(f"{name}: pool {words.shape[0]} fold {pool_fold(words):#x} archive {arc.values.shape[0]} hv {hv} "
          f"(sample {ts:.1f}s filter {tf:.1f}s hv {th:.1f}s) -> {out}")


if __name__ == "__main__":
    which = sys.argv[1] if len(sys.argv) > 1 else "all"
    for nm in (CASES if which == "all" else [which]):
        make(nm)
