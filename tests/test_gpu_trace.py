"""GPU samples_to_reach (pareto.hpp:763-781) and convergence_trace (pareto.hpp:716-757)
against the reference on the same pools: identical counts, HV values and elapsed times."""
import numpy as np
import pytest

from oracle.refbind import make_cfg
from paper_2604_26477_b200 import api
from paper_2604_26477_b200.api import InvalidArgument

pytestmark = pytest.mark.gpu


def inst_from_ref(ri):
    ei, ej, w = ri.edges()
    return api.MultiObjectiveInstance.from_arrays(ri.n, ri.k, ei, ej, w)


def readme_pool(ref):
    ri = ref.generate_uniform(10, 0.5, 3, 54)
    nums = ref.das_dennis(3, 12)
    words = ref.run_sampler(ri, nums, 12, make_cfg("bsb", batch_size=500, seed=54, threads=8), 1)["words"]
    return ri, inst_from_ref(ri), words


def test_samples_to_reach_readme(ref, session):
    """proj/README.md:64-77: samples_to_optimal = 6054 at r = 0 and hv_max = 1141902."""
    ri, inst, words = readme_pool(ref)
    pool = api.SamplePool(10, words)
    r = [0.0, 0.0, 0.0]
    assert api.samples_to_reach(pool, inst, r, 1141902.0, session=session) == 6054
    for target in (1.0, 5e5, 1141000.0, 1141901.5, 1141902.0, 1141903.0, 2e6):
        assert api.samples_to_reach(pool, inst, r, target, session=session) == ref.samples_to_reach(ri, words, r, target)


def test_samples_to_reach_heavy_hex(ref, session):
    from paper_2604_26477_b200.instances import ensure_heavy_hex
    ri = ref.instance_load(ensure_heavy_hex(3))
    inst = inst_from_ref(ri)
    nums = ref.das_dennis(3, 21)
    words = ref.run_sampler(ri, nums, 21, make_cfg("bsb", batch_size=40, seed=7, threads=8), 1)["words"]
    pool = api.SamplePool(42, words)
    r = list(ref.reference_point_sampled(ri, 1000, 7))
    arc = ref.filter_pool(ri, words)
    r = list(np.minimum(r, arc.values.min(axis=0)))
    full = ref.hypervolume(arc.values, r)
    for target in (full * 0.5, full * 0.99, full, full + 1):
        assert api.samples_to_reach(pool, inst, r, target, session=session) == ref.samples_to_reach(ri, words, r, target)


@pytest.mark.parametrize("checkpoints", [1, 7, 40])
def test_convergence_trace_matches_reference(ref, session, checkpoints):
    ri, inst, words = readme_pool(ref)
    rng = np.random.default_rng(checkpoints)
    stamps = rng.integers(0, 2000, size=words.shape[0]).astype(np.int64) * 1000  # many ties
    pool = api.SamplePool(10, words, stamps=stamps)
    got = api.convergence_trace(pool, inst, [0.0, 0.0, 0.0], checkpoints, session=session)
    el, hv, sm = ref.convergence_trace(ri, words, stamps, [0.0, 0.0, 0.0], checkpoints)
    assert [p.samples for p in got] == sm.tolist()
    assert [p.hv for p in got] == hv.tolist()
    assert [p.elapsed_s for p in got] == el.tolist()


def test_trace_errors(session, ref):
    ri, inst, words = readme_pool(ref)
    with pytest.raises(InvalidArgument, match="checkpoints must be >= 1"):
        api.convergence_trace(api.SamplePool(10, words), inst, [0, 0, 0], 0, session=session)
    with pytest.raises(InvalidArgument, match="empty pool"):
        api.samples_to_reach(api.SamplePool(10), inst, [0, 0, 0], 1.0, session=session)
