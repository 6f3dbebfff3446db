"""One context reused across instances, lattices and paths must give the same results as a
fresh context for each (guards every cache keyed on the instance or the lattice: the dense
H*J(c), the int8 weight layers, padded rows, cut packing)."""
import numpy as np
import pytest

from paper_2604_26477_b200 import api
from paper_2604_26477_b200.instances import load_heavy_hex

pytestmark = pytest.mark.gpu


def _dense_run(s, seed, H):
    s.generate_uniform_instance(256, 0.5, 3, seed)
    s.set_dense_threshold(256)
    s.set_weights(api.build_weights(3, resolution=H))
    rep = s.pipeline(api.SolverConfig(variant=api.SolverVariant.discrete_sb, batch_size=24, seed=seed), 1, 0, -1,
                     True, 256)
    return s.pool(stamps=False).words.copy(), s.archive().values.copy(), rep["hv"]


def _hh_run(s, k, variant):
    s.set_instance(load_heavy_hex(k))
    s.set_weights(api.build_weights(k, resolution=5 if k == 4 else 7))
    rep = s.pipeline(api.SolverConfig(variant=variant, batch_size=70, seed=3), 1, 0, -1, True, 512)
    return s.pool(stamps=False).words.copy(), s.archive().values.copy(), rep["hv"]


def test_context_reuse_matches_fresh_contexts():
    plan = [("dense", 31, 4), ("hh", 4, api.SolverVariant.discrete_sb), ("dense", 32, 4), ("dense", 32, 5),
            ("hh", 3, api.SolverVariant.ballistic_sb), ("dense", 31, 4), ("hh", 4, api.SolverVariant.simcim)]
    shared = api.Session(0)
    for kind, a, b in plan:
        run = _dense_run if kind == "dense" else _hh_run
        got = run(shared, a, b)
        want = run(api.Session(0), a, b)
        for g, w in zip(got, want):
            assert np.array_equal(np.asarray(g), np.asarray(w)), (kind, a, b)


def test_streaming_and_enumeration_after_other_work():
    """the running archive and the enumerator on a context that sampled other instances first"""
    from paper_2604_26477_b200 import streaming

    def stream(s):
        s.set_instance(load_heavy_hex(3))
        s.set_weights(api.build_weights(3, resolution=7))
        cfg = api.SolverConfig(variant=api.SolverVariant.ballistic_sb, batch_size=60, seed=9)
        res = streaming.time_to_target(s, cfg, [-60.0, -60.0, -60.0], None, 3)
        return res["hv"], s.archive().values.copy()

    shared = api.Session(0)
    _dense_run(shared, 33, 4)
    _hh_run(shared, 4, api.SolverVariant.discrete_sb)
    hv_a, arc_a = stream(shared)
    hv_b, arc_b = stream(api.Session(0))
    assert hv_a == hv_b and np.array_equal(arc_a, arc_b)

    g = api.Session(0).generate_uniform_instance(16, 0.6, 2, 5)
    fresh = api.brute_force_pareto(g, session=api.Session(0))
    shared.generate_uniform_instance(16, 0.6, 2, 5)
    again = api.brute_force_pareto(g, session=shared)
    assert np.array_equal(fresh.values, again.values) and np.array_equal(fresh.configs, again.configs)
