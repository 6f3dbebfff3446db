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
