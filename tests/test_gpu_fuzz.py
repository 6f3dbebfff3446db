"""Randomised sampler parity: random instances (n from 3 to 90, so the register path for
n <= 64 and the generic path above), K, density, variant, lattice, batch (1 to 257), T,
alpha (incl. 0), dt / a0 (incl. non-unit) and runs, each pool compared word for word with
the reference (solver.hpp:439-529). Fixed seeds keep it reproducible."""
import random

import numpy as np
import pytest

from oracle.refbind import make_cfg
from paper_2604_26477_b200 import api

pytestmark = pytest.mark.gpu
VARIANTS = {"bsb": api.SolverVariant.ballistic_sb, "dsb": api.SolverVariant.discrete_sb,
            "simcim": api.SolverVariant.simcim}


@pytest.mark.parametrize("seed", [101, 202])
def test_random_configurations_match_reference(ref, session, seed):
    rnd = random.Random(seed)
    compared = 0
    for _ in range(40):
        n = rnd.choice([3, 7, 12, 17, 25, 31, 33, 40, 42, 50, 63, 64, 65, 90])
        k = rnd.choice([2, 3, 4])
        dens = rnd.choice([0.1, 0.3, 0.6, 1.0])
        iseed = rnd.randrange(1000)
        var = rnd.choice(list(VARIANTS))
        H = k + rnd.choice([1, 2, 3])
        batch = rnd.choice([1, 5, 64, 65, 130, 257])
        T = rnd.choice([1, 7, 50])
        alpha = rnd.choice([0.15, 0.0, 0.4])
        dt = rnd.choice([1.0, 0.5])
        a0 = rnd.choice([1.0, 0.9])
        runs = rnd.choice([1, 2])
        ri = ref.generate_uniform(n, dens, k, iseed)
        ei, ej, w = ri.edges()
        if len(ei) == 0:
            continue
        inst = api.MultiObjectiveInstance.from_arrays(n, k, ei, ej, w)
        nums = ref.das_dennis(k, H)
        c = make_cfg(var, n_iterations=T, batch_size=batch, seed=iseed, threads=16, alpha=alpha, dt=dt, a0=a0)
        want = ref.run_sampler(ri, nums, H, c, runs)["words"]
        cfg = api.SolverConfig(variant=VARIANTS[var], n_iterations=T, batch_size=batch, seed=iseed, alpha=alpha,
                               dt=dt, a0=a0)
        got = api.run_sampler(inst, [api.WeightVector(list(r), H) for r in nums], cfg, runs, session=session).words
        assert np.array_equal(got, want), dict(n=n, k=k, dens=dens, seed=iseed, var=var, H=H, batch=batch, T=T,
                                               alpha=alpha, dt=dt, a0=a0, runs=runs)
        compared += 1
    assert compared >= 30


@pytest.mark.parametrize("seed", [303, 404])
def test_random_pools_filter_and_hv_match_reference(ref, session, seed):
    """the Pareto stage on random pools of random instances (integer and real weights,
    K = 2..5, duplicates): archive values / configs / order, evaluate_cuts and the HV at the
    clamped sampled reference point (pareto.hpp:253-410, :540-655)"""
    from test_gpu_pareto import check_archive, inst_from_ref, random_words

    rnd = random.Random(seed)
    for _ in range(12):
        n = rnd.choice([5, 9, 16, 30, 42, 64, 65, 90])
        k = rnd.choice([2, 3, 4, 5])
        kind = rnd.choice(["int", "int", "real"])
        ri = ref.generate_uniform(n, rnd.choice([0.2, 0.5, 1.0]), k, rnd.randrange(1000), kind=kind,
                                  lo=1.0 if kind == "int" else -1.0, hi=10.0 if kind == "int" else 1.0)
        if len(ri.edges()[0]) == 0:
            continue
        inst = inst_from_ref(ri)
        M = rnd.choice([1, 7, 500, 20000])
        words = random_words(n, M, rnd.randrange(10**6))
        if M > 1:
            words[M // 2:] = words[: M - M // 2]
        assert np.array_equal(api.evaluate_cuts(inst, words, session=session), ref.evaluate_cuts(ri, words))
        got = api.non_dominated_filter(api.SamplePool(n, words), inst, session=session)
        want = ref.filter_pool(ri, words)
        check_archive(got, want)
        r = api.clamp_reference(api.reference_point_sampled(inst, 256, 5, session=session), got)
        h = api.hypervolume(got, r, session=session)
        assert h == pytest.approx(ref.hypervolume(want.values, np.asarray(r)), rel=1e-12)


def test_random_dense_configurations_agree_with_reference(ref):
    """the int8 tensor-core dSB path (n >= 256) on random configurations: words within the
    measured dense tolerance (0 differing words)"""
    from test_gpu_dense import MAX_DENSE_WORD_MISMATCH

    rnd = random.Random(505)
    s = api.Session(0)
    s.set_dense_threshold(256)
    for _ in range(6):
        n = rnd.choice([256, 272, 320])
        k = rnd.choice([2, 3])
        H = k + rnd.choice([1, 2])
        iseed = rnd.randrange(1000)
        dens = rnd.choice([0.3, 0.7])
        batch = rnd.choice([1, 9, 33])
        T = rnd.choice([5, 50])
        alpha = rnd.choice([0.15, 0.0])
        runs = rnd.choice([1, 2])
        s.generate_uniform_instance(n, dens, k, iseed)
        ri = ref.generate_uniform(n, dens, k, iseed)
        nums = ref.das_dennis(k, H)
        s.set_weights([api.WeightVector(list(r), H) for r in nums])
        c = make_cfg("dsb", n_iterations=T, batch_size=batch, seed=iseed, threads=16, alpha=alpha)
        want = ref.run_sampler(ri, nums, H, c, runs)["words"]
        s.sample(api.SolverConfig(variant=api.SolverVariant.discrete_sb, n_iterations=T, batch_size=batch, seed=iseed,
                                  alpha=alpha), runs)
        got = s.pool(stamps=False).words
        assert got.shape == want.shape
        assert float(np.mean(np.any(got != want, axis=1))) <= MAX_DENSE_WORD_MISMATCH, dict(
            n=n, k=k, H=H, seed=iseed, dens=dens, batch=batch, T=T, alpha=alpha, runs=runs)
