"""C4 at its full size (N = 2000 dense, 1,999,000 edges, K = 3, dSB, 55 weights x 3000 =
165,000 samples): size-independent properties of the tensor-core path where the CPU
reference cannot run the whole workload (it samples ~140 samples/s):

* determinism: the same configuration sampled twice gives the same pool, word for word;
* block equivalence (the sharding contract): the two halves of the block range
  sampled separately give the rows of the whole-range pool;
* the archive is mutually non-dominated and its values equal evaluate_cuts of its configs
  (the int8-GEMM evaluation is exact);
* the HV at the sampled reference is positive and reproducible.
"""
import numpy as np
import pytest

from paper_2604_26477_b200 import api

pytestmark = pytest.mark.gpu


def test_c4_full_size_properties():
    s = api.Session(0)
    inst = s.generate_uniform_instance(2000, 1.0, 3, 3)
    assert inst.num_edges() == 1999000
    w = api.build_weights(3, resolution=12)
    assert len(w) == 55
    s.set_weights(w)
    cfg = api.SolverConfig(variant=api.SolverVariant.discrete_sb, batch_size=3000, seed=3)

    rep1 = s.pipeline(cfg, 1, 0, -1, True, 1000)
    p1 = s.pool(stamps=False).words.copy()
    a1 = s.archive()
    rep2 = s.pipeline(cfg, 1, 0, -1, True, 1000)
    p2 = s.pool(stamps=False).words
    assert p1.shape == (165000, 32)
    assert np.array_equal(p1, p2)
    assert rep1["hv"] == rep2["hv"] > 0

    total = s.num_blocks(cfg, 1)
    chunks = total // len(w)
    half = (len(w) // 2) * chunks  # a weight boundary: rows [0, 27 x 3000)
    s.sample(cfg, 1, 0, half)
    lo = s.pool(stamps=False).words[: (len(w) // 2) * 3000].copy()
    s.sample(cfg, 1, half, total)
    hi = s.pool(stamps=False).words[(len(w) // 2) * 3000:].copy()
    assert np.array_equal(np.concatenate([lo, hi]), p1)

    vals = a1.values
    assert vals.shape[0] == rep1["archive_size"] > 0
    ge = (vals[:, None, :] >= vals[None, :, :]).all(axis=2)
    gt = (vals[:, None, :] > vals[None, :, :]).any(axis=2)
    dominated = (ge & gt).any(axis=0)  # column j dominated by some row i
    assert not dominated.any()
    assert np.array_equal(api.evaluate_cuts(inst, a1.configs, session=s), vals)
