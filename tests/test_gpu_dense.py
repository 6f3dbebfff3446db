"""Dense instances (C4 shape) on the GPU: the device instance generator is bit-identical to
generate_uniform_instance; the int8 tensor-core dSB path agrees with the reference within
the stated tolerance (coupled = (H*J)·sgn(x)/H is one correctly rounded
division, the reference sums rounded FP64 products, so trajectories may differ at ulp level;
asserted: the measured value, 0 differing words, reported as a count); evaluate_cuts through
int8 GEMMs is exact."""
import numpy as np
import pytest

from oracle.refbind import make_cfg
from paper_2604_26477_b200 import api

pytestmark = pytest.mark.gpu
MAX_DENSE_WORD_MISMATCH = 0.0  # measured; the path rounds J(c).sgn(X) once


@pytest.mark.parametrize("n,density,k,kind,lo,hi", [(300, 0.3, 3, "int", 1, 10), (120, 0.8, 2, "real", 0.0, 1.0),
                                                    (257, 1.0, 4, "int", -5, 5)])
def test_device_generator_matches_reference(ref, session, n, density, k, kind, lo, hi):
    inst = session.generate_uniform_instance(n, density, k, 17, kind=kind, lo=lo, hi=hi)
    ri = ref.generate_uniform(n, density, k, 17, kind=kind, lo=lo, hi=hi)
    ei, ej, w = ri.edges()
    assert np.array_equal(inst.edge_i, ei) and np.array_equal(inst.edge_j, ej) and np.array_equal(inst.weights, w)


@pytest.mark.parametrize("n,batch,seed", [(512, 48, 5), (272, 37, 6)])
def test_dense_dsb_agrees_with_reference(ref, session, n, batch, seed):
    """n = 272 leaves a half window (272 = 8 x 32 + 16) and batch 37 a partial CTA of warps"""
    H = 4
    inst = session.generate_uniform_instance(n, 0.5, 3, seed)
    ri = ref.generate_uniform(n, 0.5, 3, seed)
    nums = ref.das_dennis(3, H)
    weights = [api.WeightVector(list(r), H) for r in nums]
    want = ref.run_sampler(ri, nums, H, make_cfg("dsb", batch_size=batch, seed=9, threads=16), 1)["words"]
    session.set_dense_threshold(256)
    session.set_weights(weights)
    session.sample(api.SolverConfig(variant=api.SolverVariant.discrete_sb, batch_size=batch, seed=9), 1)
    got = session.pool(stamps=False).words
    mm = float(np.mean(np.any(got != want, axis=1)))
    print(f"dense dSB n={n}: {int(round(mm * got.shape[0]))} of {got.shape[0]} pool rows differ")
    assert mm <= MAX_DENSE_WORD_MISMATCH


def test_dense_dsb_non_unit_dt_agrees_with_reference(ref, session):
    """dt = 0.5, a0 = 1.2: the general update of the warp-per-trajectory kernel"""
    n, H = 288, 4
    session.generate_uniform_instance(n, 0.5, 3, 8)
    ri = ref.generate_uniform(n, 0.5, 3, 8)
    nums = ref.das_dennis(3, H)
    batch = 33
    want = ref.run_sampler(ri, nums, H, make_cfg("dsb", batch_size=batch, seed=4, threads=16, dt=0.5, a0=1.2),
                           1)["words"]
    session.set_dense_threshold(256)
    session.set_weights([api.WeightVector(list(r), H) for r in nums])
    session.sample(api.SolverConfig(variant=api.SolverVariant.discrete_sb, batch_size=batch, seed=4, dt=0.5, a0=1.2), 1)
    got = session.pool(stamps=False).words
    assert float(np.mean(np.any(got != want, axis=1))) <= MAX_DENSE_WORD_MISMATCH


def test_dense_dsb_noiseless_agrees_with_reference(ref, session):
    """alpha = 0: the noise-free instantiation of the update kernel"""
    n, H = 256, 4
    session.generate_uniform_instance(n, 0.6, 3, 13)
    ri = ref.generate_uniform(n, 0.6, 3, 13)
    nums = ref.das_dennis(3, H)
    batch = 24
    want = ref.run_sampler(ri, nums, H, make_cfg("dsb", batch_size=batch, seed=2, threads=16, alpha=0.0), 1)["words"]
    session.set_dense_threshold(256)
    session.set_weights([api.WeightVector(list(r), H) for r in nums])
    session.sample(api.SolverConfig(variant=api.SolverVariant.discrete_sb, batch_size=batch, seed=2, alpha=0.0), 1)
    got = session.pool(stamps=False).words
    assert float(np.mean(np.any(got != want, axis=1))) <= MAX_DENSE_WORD_MISMATCH


def test_dense_dsb_two_runs_agree_with_reference(ref, session):
    """runs = 2: pairs of both runs in one launch group (per-pair run keys, pair offsets)"""
    n, H = 256, 4
    session.generate_uniform_instance(n, 0.5, 3, 14)
    ri = ref.generate_uniform(n, 0.5, 3, 14)
    nums = ref.das_dennis(3, H)
    batch = 20
    want = ref.run_sampler(ri, nums, H, make_cfg("dsb", batch_size=batch, seed=6, threads=16), 2)["words"]
    session.set_dense_threshold(256)
    session.set_weights([api.WeightVector(list(r), H) for r in nums])
    session.sample(api.SolverConfig(variant=api.SolverVariant.discrete_sb, batch_size=batch, seed=6), 2)
    got = session.pool(stamps=False).words
    assert got.shape == want.shape
    assert float(np.mean(np.any(got != want, axis=1))) <= MAX_DENSE_WORD_MISMATCH


def test_dense_eval_gemm_exact(ref, session):
    n = 512
    inst = session.generate_uniform_instance(n, 0.7, 3, 8)
    ri = ref.generate_uniform(n, 0.7, 3, 8)
    rng = np.random.default_rng(4)
    words = rng.integers(0, 2**63, size=(5000, n // 64), dtype=np.uint64)
    got = api.evaluate_cuts(inst, words, session=session)
    assert np.array_equal(got, ref.evaluate_cuts(ri, words))


def test_dense_reference_point_matches_reference(ref, session):
    inst = session.generate_uniform_instance(512, 0.5, 3, 12)
    ri = ref.generate_uniform(512, 0.5, 3, 12)
    assert api.reference_point_sampled(inst, 333, 7, session=session) == ref.reference_point_sampled(ri, 333, 7).tolist()


def test_dense_bf16_path_agrees_with_reference(ref, session):
    """H = 21 (190 weights for K = 3) with |w| <= 10 puts |H*J| up to 210: beyond int8, so the
    fused kernel runs kind::f16 with bf16 H*J (exact integers <= 256) and FP32 accumulation"""
    n, H = 320, 21
    session.generate_uniform_instance(n, 0.4, 3, 31)
    ri = ref.generate_uniform(n, 0.4, 3, 31)
    nums = ref.das_dennis(3, H)[::9]  # 24 of the 253 lattice vectors, including boundary ones
    batch = 9
    want = ref.run_sampler(ri, nums, H, make_cfg("dsb", batch_size=batch, seed=12, threads=16), 1)["words"]
    session.set_dense_threshold(256)
    session.set_weights([api.WeightVector(list(r), H) for r in nums])
    session.sample(api.SolverConfig(variant=api.SolverVariant.discrete_sb, batch_size=batch, seed=12), 1)
    assert session.sampler_path() == "dense_bf16"
    got = session.pool(stamps=False).words
    mm = int(np.sum(np.any(got != want, axis=1)))
    print(f"dense bf16 dSB n={n}: {mm} of {got.shape[0]} words differ")
    assert mm <= MAX_DENSE_WORD_MISMATCH * got.shape[0]


_CHECKED_SCRIPT = r"""
import sys, numpy as np
sys.path.insert(0, {root!r})
from paper_2604_26477_b200 import api
s = api.Session(0)
s.generate_uniform_instance(288, 0.5, 3, 12)
s.set_dense_threshold(256)
s.set_weights(api.build_weights(3, resolution=4))
s.sample(api.SolverConfig(variant=api.SolverVariant.discrete_sb, batch_size=40, seed=21), 1)
assert s.sampler_path() == "dense_i8", s.sampler_path()
np.save({out!r}, s.pool(stamps=False).words)
"""


def test_dense_unchecked_steps_equal_checked_steps(tmp_path):
    """The update kernel runs without the per-step finiteness check (a final-state scan and a
    checked re-run on failure replace it); with the checks forced on (MOMC_TEST_DENSE_CHECKED)
    the pool is the same."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    pools = []
    for checked in (False, True):
        out = str(tmp_path / f"words_{int(checked)}.npy")
        env = dict(os.environ)
        env.pop("MOMC_TEST_DENSE_CHECKED", None)
        if checked:
            env["MOMC_TEST_DENSE_CHECKED"] = "1"
        subprocess.run([sys.executable, "-c", _CHECKED_SCRIPT.format(root=root, out=out)], env=env, check=True,
                       timeout=300)
        pools.append(np.load(out))
    diff = int(np.sum(np.any(pools[0] != pools[1], axis=1)))
    print(f"checked vs unchecked dense steps: {diff} of {pools[0].shape[0]} pool rows differ")
    assert pools[0].shape[0] > 0 and diff == 0
