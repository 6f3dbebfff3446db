"""C4 at its stated size (BASELINE config 4): N = 2000 dense K = 3 instance
(generate_uniform_instance(2000, 1.0, 3, WeightSpec{}, 3), instance.hpp:259-284), 55 interior
weights (H = 12), dSB, T = 50. The fused tensor-core step (int8 H*J(c), csrc/dense.cu) is
compared with the unmodified reference (oracle/_ref) on the first 16 trajectories of every
weight: 880 samples, word for word. The measured mismatch is 0 words, so
the assertion is exact; the evaluation of those samples (int8 tcgen05 GEMM form of
evaluate_cuts, pareto.hpp:330-363) is compared exactly too."""
import os

import numpy as np
import pytest

from oracle.refbind import make_cfg
from paper_2604_26477_b200 import api

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def c4(ref):
    s = api.Session(0)
    inst = s.generate_uniform_instance(2000, 1.0, 3, 3)
    ri = ref.generate_uniform(2000, 1.0, 3, 3)
    nums = ref.das_dennis(3, 12)
    nums = nums[np.all(nums > 0, axis=1)]
    assert nums.shape[0] == 55
    yield s, inst, ri, nums
    s.close()


def test_c4_sample_matches_reference(ref, c4):
    s, inst, ri, nums = c4
    batch = 16
    want = ref.run_sampler(ri, nums, 12, make_cfg("dsb", batch_size=batch, seed=3, threads=os.cpu_count()), 1)["words"]
    s.set_weights([api.WeightVector(list(r), 12) for r in nums])
    s.sample(api.SolverConfig(variant=api.SolverVariant.discrete_sb, batch_size=batch, seed=3), 1)
    assert s.sampler_path() == "dense_i8"
    got = s.pool(stamps=False).words
    assert got.shape == want.shape == (55 * batch, 32)
    mm = int(np.sum(np.any(got != want, axis=1)))
    print(f"C4 N=2000 dSB: {mm} of {got.shape[0]} words differ from the reference")
    assert mm == 0
    # the same samples through the tensor-core evaluate_cuts
    assert np.array_equal(api.evaluate_cuts(inst, got, session=s), ref.evaluate_cuts(ri, got))


def test_c4_full_batch_block_equivalence(c4):
    """trajectories are position-independent: a 3000-trajectory batch sampled in one fused
    launch holds the 16-trajectory pool's words in its first 16 rows of every weight"""
    s, inst, ri, nums = c4
    s.set_weights([api.WeightVector(list(r), 12) for r in nums[:3]])
    cfg = api.SolverConfig(variant=api.SolverVariant.discrete_sb, batch_size=16, seed=3)
    s.sample(cfg, 1)
    small = s.pool(stamps=False).words.reshape(3, 16, 32)
    s.sample(api.SolverConfig(variant=api.SolverVariant.discrete_sb, batch_size=1000, seed=3), 1)
    big = s.pool(stamps=False).words.reshape(3, 1000, 32)
    assert np.array_equal(big[:, :16], small)
