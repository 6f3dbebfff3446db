"""The streaming merge (momc_b200_stream_step: each run's pool filtered together with the running
archive) against one non-dominated filter over all those runs' pool at once: the same value
vectors and the same lex-smallest configurations (pareto.hpp:370-410; the merge law
filter(A U B) = filter(filter(A) U B), test_pareto.cpp:115-125). K=4 dSB packs its cut values
into one 64-bit key, so it takes the fused pass with the archive rows inserted into the
collapse table; the K=3 bSB case checks the same law on the second shape."""
import numpy as np
import pytest

from paper_2604_26477_b200 import api
from paper_2604_26477_b200.instances import load_heavy_hex

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("k, res, variant, batch, runs", [
    (4, 13, api.SolverVariant.discrete_sb, 300, 5),
    (3, 21, api.SolverVariant.ballistic_sb, 200, 4),
])
def test_running_archive_equals_one_filter(k, res, variant, batch, runs):
    inst = load_heavy_hex(k)
    w = api.build_weights(k, resolution=res)
    cfg = api.SolverConfig(variant=variant, batch_size=batch, seed=11)
    s = api.Session(0)
    s.set_instance(inst)
    s.set_weights(w)
    per_run = s.num_blocks(cfg, 1)
    s.running_reset()
    sizes = []
    for run in range(runs):
        _, F, _ = s.stream_step(cfg, run + 1, run * per_run, (run + 1) * per_run)
        sizes.append(F)
    s.running_to_archive()
    got = s.archive()

    ref = api.Session(0)
    pool = api.run_sampler(inst, w, cfg, runs, session=ref)
    want = api.non_dominated_filter(pool, inst, session=ref)
    print(f"K={k}: running sizes {sizes}, one-filter archive {want.values.shape[0]}")
    assert got.values.shape == want.values.shape
    assert np.array_equal(got.values, want.values)
    mism = int(np.sum(np.any(got.configs != want.configs, axis=1)))
    print(f"K={k}: {mism} differing configs of {want.values.shape[0]}")
    assert mism == 0


def test_running_archive_hv_matches_archive_hv():
    """The HV returned by each streaming step equals the HV of that step's one-shot archive."""
    inst = load_heavy_hex(4)
    w = api.build_weights(4, resolution=13)
    cfg = api.SolverConfig(variant=api.SolverVariant.discrete_sb, batch_size=300, seed=5)
    s = api.Session(0)
    s.set_instance(inst)
    s.set_weights(w)
    per_run = s.num_blocks(cfg, 1)
    r = [-60.0, -70.0, -70.0, -70.0]
    s.running_reset()
    ref = api.Session(0)
    for run in range(3):
        hv, _, _ = s.stream_step(cfg, run + 1, run * per_run, (run + 1) * per_run, r)
        pool = api.run_sampler(inst, w, cfg, run + 1, session=ref)
        arc = api.non_dominated_filter(pool, inst, session=ref)
        assert hv == api.hypervolume(arc, r, session=ref)
