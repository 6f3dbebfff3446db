"""GPU parity of the SB sampler (solver.hpp:439-529) against the reference and its oracle.

Arithmetic is FP64 in the reference's order on both sides, so the expected result is
bit-identical packed spins and every comparison asserts zero differing words (printing the
count). DESIGN.md §3 states the only unreproduced primitives (CUDA log / exp in the
ziggurat's rare wedge / tail branches); they have never produced a differing word.
"""
import numpy as np
import pytest

from oracle.refbind import make_cfg, pool_fold
from paper_2604_26477_b200 import api
from paper_2604_26477_b200.api import InvalidArgument, MomcRuntimeError, SolverConfig, SolverVariant
from paper_2604_26477_b200.instances import load_heavy_hex

pytestmark = pytest.mark.gpu

MAX_WORD_MISMATCH = 0  # bit-exact pools


def inst_from_ref(ri):
    ei, ej, w = ri.edges()
    return api.MultiObjectiveInstance.from_arrays(ri.n, ri.k, ei, ej, w)


def weights_of(nums, H):
    return [api.WeightVector(list(r), H) for r in nums]


def cfg_of(variant="bsb", **kw):
    v = {"bsb": SolverVariant.ballistic_sb, "dsb": SolverVariant.discrete_sb, "simcim": SolverVariant.simcim}[variant]
    return SolverConfig(variant=v, **kw)


def mismatch(a, b):
    """fraction of differing pool rows, printed as a count"""
    diff = int(np.count_nonzero(np.any(a != b, axis=1)))
    print(f"{diff} of {a.shape[0]} pool rows differ")
    return diff / max(a.shape[0], 1)


@pytest.mark.parametrize("variant,fold", [("bsb", 0x4C640870582EDE16), ("dsb", 0x4572BF3D54216F62)])
def test_readme_config_pool_fold(ref, session, variant, fold):
    """README config (proj/README.md:56-77) -> SURVEY Appendix A pool folds, bit-exact."""
    ri = ref.generate_uniform(10, 0.5, 3, 54)
    inst = inst_from_ref(ri)
    nums = ref.das_dennis(3, 12)
    pool = api.run_sampler(inst, weights_of(nums, 12), cfg_of(variant, batch_size=500, seed=54), 1, session=session)
    assert pool.size() == 27500
    assert pool_fold(pool.words) == fold
    if variant == "bsb":
        w = pool.words[:, 0]
        assert [int(w[i]) for i in range(8)] == [0x2E1, 0x2E1, 0x11F, 0x2E1, 0x2B2, 0x11E, 0x2B2, 0x14D]
        assert int(w[500]) == 0x2B2 and int(w[27499]) == 0x0E5


@pytest.mark.parametrize("variant", ["bsb", "dsb", "simcim"])
@pytest.mark.parametrize("n,density,k,seed", [(2, 1.0, 2, 3), (4, 1.0, 3, 1), (10, 0.8, 2, 3), (20, 0.5, 3, 40),
                                              (33, 0.3, 3, 5), (42, 0.2, 4, 6), (64, 0.1, 2, 8), (70, 0.5, 2, 6)])
def test_pool_matches_reference(ref, session, variant, n, density, k, seed):
    ri = ref.generate_uniform(n, density, k, seed)
    inst = inst_from_ref(ri)
    H = 5 if k == 2 else 4
    nums = ref.das_dennis(k, H)
    batch = 300 if n <= 64 else 40
    c = make_cfg(variant, batch_size=batch, seed=seed + 11, threads=8)
    expect = ref.run_sampler(ri, nums, H, c, 2)["words"]
    pool = api.run_sampler(inst, weights_of(nums, H), cfg_of(variant, batch_size=batch, seed=seed + 11), 2,
                           session=session)
    assert pool.words.shape == expect.shape
    assert mismatch(pool.words, expect) == MAX_WORD_MISMATCH


@pytest.mark.parametrize("variant", ["bsb", "dsb", "simcim"])
@pytest.mark.parametrize("dt,a0", [(0.5, 1.0), (1.0, 0.8), (0.7, 1.3)])
def test_non_unit_time_step_matches_reference(ref, session, variant, dt, a0):
    """dt != 1 or dt*a0 != 1 takes the general update (the unit-dt specialisation skips the
    exact products dt*d and dt*a0*y only when both are 1)"""
    ri = ref.generate_uniform(42, 0.2, 3, 9)
    inst = inst_from_ref(ri)
    nums = ref.das_dennis(3, 4)
    c = make_cfg(variant, batch_size=200, seed=21, threads=8, dt=dt, a0=a0)
    expect = ref.run_sampler(ri, nums, 4, c, 1)["words"]
    pool = api.run_sampler(inst, weights_of(nums, 4), cfg_of(variant, batch_size=200, seed=21, dt=dt, a0=a0), 1,
                           session=session)
    assert mismatch(pool.words, expect) == MAX_WORD_MISMATCH


@pytest.mark.parametrize("variant", ["bsb", "dsb"])
def test_heavy_hex_k4_matches_reference(ref, session, variant):
    inst = load_heavy_hex(4)
    ri = ref.instance_load("data/heavyhex42_k4_seed7.txt")
    nums = ref.das_dennis(4, 13)
    assert nums.shape[0] == 220
    c = make_cfg(variant, batch_size=129, seed=7, threads=8)  # ragged 128-chunk tail
    expect = ref.run_sampler(ri, nums, 13, c, 1)["words"]
    pool = api.run_sampler(inst, weights_of(nums, 13), cfg_of(variant, batch_size=129, seed=7), 1, session=session)
    mm = mismatch(pool.words, expect)
    print(f"heavy-hex K=4 {variant}: {mm * 100:.4f}% words differ")
    assert mm == MAX_WORD_MISMATCH


def test_noiseless_and_zero_init(ref, session):
    ri = ref.generate_uniform(12, 0.7, 3, 21)
    inst = inst_from_ref(ri)
    nums = ref.das_dennis(3, 5)
    for alpha, init in ((0.0, 0.1), (0.0, 0.0), (0.3, 0.0)):
        c = make_cfg("bsb", batch_size=64, seed=3, alpha=alpha, init_scale=init, threads=4)
        expect = ref.run_sampler(ri, nums, 5, c, 1)["words"]
        pool = api.run_sampler(inst, weights_of(nums, 5),
                               cfg_of("bsb", batch_size=64, seed=3, alpha=alpha, init_scale=init), 1, session=session)
        assert np.array_equal(pool.words, expect)


def test_scalarize_matches_reference(ref, session):
    ri = ref.generate_uniform(30, 0.4, 3, 77)
    inst = inst_from_ref(ri)
    session.set_instance(inst)
    nums = ref.das_dennis(3, 7)
    session.set_weights(weights_of(nums, 7))
    for l in (0, 5, nums.shape[0] - 1):
        J, c0 = session.coupling(l)
        Jr, c0r = ref.scalarize(ri, nums[l], 7)
        assert np.array_equal(J, Jr)
        assert c0 == c0r


def test_scalarize_large_matches_reference(ref, session):
    """the grid-wide scalarisation kernels (nnz x L > 2^20): n=400 dense, 36 weights"""
    ri = ref.generate_uniform(400, 0.9, 3, 78, kind="real", lo=-1.0, hi=1.0)
    inst = inst_from_ref(ri)
    session.set_instance(inst)
    nums = ref.das_dennis(3, 7)
    session.set_weights(weights_of(nums, 7))
    for l in (0, 11, nums.shape[0] - 1):
        J, c0 = session.coupling(l)
        Jr, c0r = ref.scalarize(ri, nums[l], 7)
        assert np.array_equal(J, Jr)
        assert c0 == c0r


def test_degenerate_coupling_is_usage_error(session):
    inst = api.MultiObjectiveInstance(3, 2, [(0, 1, [1.0, -1.0])])
    with pytest.raises(InvalidArgument, match="degenerate scalarized coupling"):
        api.run_sampler(inst, [api.WeightVector([1, 1], 2)], SolverConfig(batch_size=4), 1, session=session)


def test_numerical_failure_reports_step(session):
    inst = api.MultiObjectiveInstance(3, 2, [(0, 1, [1.0, 1.0]), (1, 2, [float("nan"), 1.0])])
    with pytest.raises(MomcRuntimeError, match=r"numerical failure at step 1 \(run 0, weight 0\)"):
        api.run_sampler(inst, [api.WeightVector([1, 1], 2)], SolverConfig(batch_size=8), 1, session=session)


def test_config_validation_messages(session):
    inst = api.MultiObjectiveInstance(2, 1, [(0, 1, [1.0])])
    with pytest.raises(InvalidArgument, match="n_iterations must be >= 1"):
        api.run_sampler(inst, [api.WeightVector([1], 1)], SolverConfig(n_iterations=0), 1, session=session)
    with pytest.raises(InvalidArgument, match="runs must be >= 1"):
        api.run_sampler(inst, [api.WeightVector([1], 1)], SolverConfig(), 0, session=session)
    with pytest.raises(InvalidArgument, match="at least one weight vector"):
        api.run_sampler(inst, [], SolverConfig(), 1, session=session)


@pytest.mark.parametrize("variant", ["dsb", "bsb", "simcim"])
def test_register_path_fallback_blocks_are_identical(session, variant):
    """blocks re-run on the exact sequential path (the register path's overflow fallback)
    produce the same words as the register path (MOMC_TEST_FORCE_FALLBACK re-runs every
    3rd block)"""
    import os
    from paper_2604_26477_b200.instances import load_heavy_hex
    inst = load_heavy_hex(4)
    s = session
    s.set_instance(inst)
    s.set_weights(api.build_weights(4, resolution=5))
    cfg = SolverConfig(variant=api.parse_variant(variant), batch_size=300, seed=11)
    s.sample(cfg, 1)
    a = s.pool(stamps=False).words.copy()
    before = s.fallback_blocks() & ((1 << 40) - 1)
    os.environ["MOMC_TEST_FORCE_FALLBACK"] = "3"
    try:
        s.sample(cfg, 1)
    finally:
        del os.environ["MOMC_TEST_FORCE_FALLBACK"]
    b = s.pool(stamps=False).words
    assert (s.fallback_blocks() & ((1 << 40) - 1)) > before
    assert np.array_equal(a, b)


@pytest.mark.parametrize("variant", ["dsb", "bsb", "simcim"])
def test_batch_kernel_sequential_streams_are_identical(session, variant):
    """noise streams resolved on the batch kernel's in-kernel sequential path (seq_resolve,
    taken by streams that need more than 56 words) give the same words as the walk
    (MOMC_TEST_SEQ_STREAMS=3 sends every 3rd (trajectory, step) stream there)"""
    import os
    from paper_2604_26477_b200.instances import load_heavy_hex
    inst = load_heavy_hex(4)
    s = session
    s.set_instance(inst)
    s.set_weights(api.build_weights(4, resolution=5))
    cfg = SolverConfig(variant=api.parse_variant(variant), batch_size=300, seed=12)
    s.sample(cfg, 1)
    a = s.pool(stamps=False).words.copy()
    os.environ["MOMC_TEST_SEQ_STREAMS"] = "3"
    try:
        s.sample(cfg, 1)
    finally:
        del os.environ["MOMC_TEST_SEQ_STREAMS"]
    b = s.pool(stamps=False).words
    diff = int(np.count_nonzero(a != b))
    print(f"{variant}: {diff} of {a.size} words differ with every 3rd stream resolved sequentially")
    assert diff == 0
