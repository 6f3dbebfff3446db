"""GPU exhaustive enumeration: brute_force_pareto (oracle.hpp:25-77) and
reference_point_exact (pareto.hpp:603-617) on the device, bit-exact against the reference
at n <= 22 (values, lex-min owner configurations, order), and beyond the reference's cap on
the 42-node heavy-hex instances, where the exact front must dominate every sampled archive."""
import os

import numpy as np
import pytest

from paper_2604_26477_b200 import api
from paper_2604_26477_b200.api import InvalidArgument
from paper_2604_26477_b200.instances import load_heavy_hex

pytestmark = pytest.mark.gpu
GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def inst_from_ref(ri):
    ei, ej, w = ri.edges()
    return api.MultiObjectiveInstance.from_arrays(ri.n, ri.k, ei, ej, w)


def ladder(ref, n, k, seed, rungs_every=3):
    """two chains joined by rungs: small separators, so the split path is exercised"""
    half = n // 2
    edges = [(i, i + 1) for i in range(half - 1)] + [(half + i, half + i + 1) for i in range(n - half - 1)]
    edges += [(i, half + i) for i in range(0, min(half, n - half), rungs_every)]
    edges = sorted(set(edges))
    rng = np.random.default_rng(seed)
    w = rng.integers(-10, 11, size=(len(edges), k)).astype(np.float64)
    ei = np.array([e[0] for e in edges], np.int32)
    ej = np.array([e[1] for e in edges], np.int32)
    return ref.instance_new(n, k, ei, ej, w)


def check_same(got, want):
    assert got.values.shape == want.values.shape
    assert np.array_equal(got.values, want.values)
    assert np.array_equal(got.configs, want.words)


@pytest.mark.parametrize("n,density,k,seed", [(8, 0.5, 2, 1), (12, 0.4, 3, 2), (16, 0.3, 4, 3), (18, 0.25, 3, 4),
                                              (20, 0.2, 4, 5), (22, 0.15, 3, 6)])
def test_brute_force_random_graphs_match_reference(ref, session, n, density, k, seed):
    ri = ref.generate_uniform(n, density, k, seed, kind="int", lo=-10.0, hi=10.0)
    inst = inst_from_ref(ri)
    got, r = api.brute_force_pareto(inst, session=session, with_reference=True)
    check_same(got, ref.brute_force_pareto(ri))
    assert r == list(ref.reference_point_exact(ri))
    assert api.reference_point_exact(inst, session=session) == r


@pytest.mark.parametrize("n,k,seed", [(14, 3, 11), (20, 4, 12), (22, 2, 13)])
def test_brute_force_separable_graphs_match_reference(ref, session, n, k, seed):
    ri = ladder(ref, n, k, seed)
    inst = inst_from_ref(ri)
    got, r = api.brute_force_pareto(inst, session=session, with_reference=True)
    check_same(got, ref.brute_force_pareto(ri))
    assert r == list(ref.reference_point_exact(ri))


def test_brute_force_positive_weights_and_readme(ref, session):
    ri = ref.generate_uniform(10, 0.5, 3, 54)  # README instance (U{1..10})
    inst = inst_from_ref(ri)
    got, r = api.brute_force_pareto(inst, session=session, with_reference=True)
    want = ref.brute_force_pareto(ri)
    check_same(got, want)
    assert r == [0.0, 0.0, 0.0]
    assert api.hypervolume(got, r, session=session) == 1141902.0  # proj/README.md:76


def test_brute_force_rejects_real_weights(ref, session):
    ri = ref.generate_uniform(10, 0.5, 3, 1, kind="real", lo=0.0, hi=1.0)
    with pytest.raises(InvalidArgument, match="integer weights"):
        api.brute_force_pareto(inst_from_ref(ri), session=session)


@pytest.mark.parametrize("k", [3, 4])
def test_brute_force_heavy_hex_42_dominates_sampled(session, k):
    """n = 42 is past the reference's cap: check the exact front against everything the
    sampler finds and against its own invariants."""
    inst = load_heavy_hex(k)
    exact, r_exact = api.brute_force_pareto(inst, session=session, with_reference=True)
    F = exact.size()
    assert F > 0
    # owners: s_0 = +1, values are the owners' cut values, order lex-descending
    assert np.all(exact.configs[:, 0] & np.uint64(1))
    assert np.array_equal(api.evaluate_cuts(inst, exact.configs, session=session), exact.values)
    rows = [tuple(v) for v in exact.values]
    assert rows == sorted(rows, reverse=True)
    # no entry dominates another
    v = exact.values
    for i in range(0, F, max(1, F // 200)):
        ge = np.all(v >= v[i], axis=1) & np.any(v > v[i], axis=1)
        assert not ge.any()
    # every sampled archive point is weakly dominated by an exact front point
    H = 21 if k == 3 else 13
    weights = api.build_weights(k, resolution=H)
    cfg = api.SolverConfig(variant=api.SolverVariant.discrete_sb if k == 4 else api.SolverVariant.ballistic_sb,
                           batch_size=2000, seed=7)
    pool = api.run_sampler(inst, weights, cfg, 1, session=session)
    sampled = api.non_dominated_filter(pool, inst, session=session)
    for row in sampled.values:
        assert np.any(np.all(v >= row, axis=1))
    r = api.clamp_reference(api.reference_point_sampled(inst, 4096, 7, session=session), exact)
    assert api.hypervolume(exact, r, session=session) >= api.hypervolume(sampled, r, session=session)
    assert all(a <= b for a, b in zip(r_exact, np.min(exact.values, axis=0)))
    if k == 4:  # best found over the 1e8-sample C5 run (profiles/r01_c5_stress.json)
        g = np.load(os.path.join(GOLDEN, "c2_heavyhex_k4_dsb.npz"))
        r2 = [float(x) for x in g["reference"]]
        assert api.hypervolume(exact, api.clamp_reference(r2, exact), session=session) >= 735896509.0


def test_streaming_reaches_exact_front_k3(session):
    """C1 shape: the streaming run (run after run, merged on the device) reaches HV* of the
    exact front, and the running archive is then the exact front itself."""
    import torch
    from paper_2604_26477_b200 import streaming
    inst = load_heavy_hex(3)
    g = np.load(os.path.join(GOLDEN, "heavyhex42_k3_exact.npz"))
    s = api.Session(0)
    s.set_instance(inst)
    s.set_weights(api.build_weights(3, resolution=21))
    cfg = api.SolverConfig(variant=api.SolverVariant.ballistic_sb, batch_size=3000, seed=7)
    trace = []
    res = streaming.time_to_target(s, cfg, [float(x) for x in g["reference"]], float(g["hv_star"]), 16,
                                   device=torch.device("cuda", 0), trace=trace)
    assert res["reached"], trace
    # the overlapped stream (2 sampling contexts + 1 merging context) gives the same result
    ov = [api.Session(0) for _ in range(2)]
    for o in ov:
        o.set_instance(inst)
        o.set_weights(api.build_weights(3, resolution=21))
    merger = api.Session(0)
    merger.set_instance(inst)
    res2 = streaming.time_to_target_overlapped(ov, merger, cfg, [float(x) for x in g["reference"]],
                                               float(g["hv_star"]), 16)
    assert (res2["runs"], res2["hv"], res2["archive"]) == (res["runs"], res["hv"], res["archive"])
    assert np.array_equal(merger.archive().values, s.archive().values)
    arc = s.archive()
    assert np.array_equal(arc.values, g["values"])
    # owners are the lex-smallest *sampled* configs (either sign of s_0), the exact front's
    # are the lex-smallest with s_0 = +1 (oracle.hpp:34): both evaluate to the same vectors
    assert np.array_equal(api.evaluate_cuts(inst, arc.configs, session=s), g["values"])
    hvs = [t["hv"] for t in trace]
    assert hvs == sorted(hvs)
