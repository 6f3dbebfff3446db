"""GPU parity of the Pareto stage (pareto.hpp) against the reference: evaluation, the
pool filter (dedup + collapse onto the lex-smallest config + front + archive order), the
objective-only filter, hypervolume, the sampled reference point and the bench pipeline.
Integer weights make every value exact, so all comparisons are bit-exact."""
import os

import numpy as np
import pytest

from oracle.refbind import make_cfg, pool_fold
from paper_2604_26477_b200 import api
from paper_2604_26477_b200.api import InvalidArgument, ObjectiveVector, ParetoArchive, Sense, SolverConfig
from paper_2604_26477_b200.instances import load_heavy_hex

pytestmark = pytest.mark.gpu
GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def inst_from_ref(ri):
    ei, ej, w = ri.edges()
    return api.MultiObjectiveInstance.from_arrays(ri.n, ri.k, ei, ej, w)


def random_words(n, M, seed):
    rng = np.random.default_rng(seed)
    wpc = (n + 63) // 64
    w = rng.integers(0, 2**63, size=(M, wpc), dtype=np.uint64) ^ rng.integers(0, 2, size=(M, wpc), dtype=np.uint64) << 63
    if n % 64:
        w[:, -1] &= np.uint64((1 << (n % 64)) - 1)
    return w


@pytest.mark.parametrize("n,density,k,kind", [(10, 0.5, 3, "int"), (42, 0.2, 4, "int"), (70, 0.3, 2, "int"),
                                              (12, 0.6, 3, "real")])
def test_evaluate_cuts_matches_reference(ref, session, n, density, k, kind):
    ri = ref.generate_uniform(n, density, k, 5, kind=kind, lo=(1.0 if kind == "int" else 0.0),
                              hi=(10.0 if kind == "int" else 1.0))
    inst = inst_from_ref(ri)
    words = random_words(n, 3000, 1)
    got = api.evaluate_cuts(inst, words, session=session)
    assert np.array_equal(got, ref.evaluate_cuts(ri, words))


def check_archive(got, want):
    assert got.values.shape == want.values.shape
    assert np.array_equal(got.values, want.values)
    if want.words.size:
        assert np.array_equal(got.configs, want.words)


def test_filter_readme_pool(ref, session):
    ri = ref.generate_uniform(10, 0.5, 3, 54)
    inst = inst_from_ref(ri)
    nums = ref.das_dennis(3, 12)
    words = ref.run_sampler(ri, nums, 12, make_cfg("bsb", batch_size=500, seed=54, threads=8), 1)["words"]
    got = api.non_dominated_filter(api.SamplePool(10, words), inst, session=session)
    want = ref.filter_pool(ri, words)
    assert got.size() == 14
    check_archive(got, want)
    assert list(got.values[0]) == [110.0, 93.0, 85.0] and int(got.configs[0, 0]) == 0x2B2
    assert api.hypervolume(got, [0, 0, 0], session=session) == 1141902.0


@pytest.mark.parametrize("n,density,k,seed,M", [(20, 0.5, 2, 3, 20000), (20, 0.5, 3, 4, 50000),
                                                (16, 0.7, 4, 5, 60000), (30, 0.3, 5, 6, 40000),
                                                (70, 0.2, 3, 7, 30000)])
def test_filter_random_pools(ref, session, n, density, k, seed, M):
    ri = ref.generate_uniform(n, density, k, seed)
    inst = inst_from_ref(ri)
    words = random_words(n, M, seed)
    words[M // 2:] = words[: M - M // 2]  # duplicates
    got = api.non_dominated_filter(api.SamplePool(n, words), inst, session=session)
    check_archive(got, ref.filter_pool(ri, words))


def test_filter_real_weights(ref, session):
    ri = ref.generate_uniform(14, 0.6, 3, 9, kind="real", lo=0.0, hi=1.0)
    inst = inst_from_ref(ri)
    words = random_words(14, 20000, 2)
    got = api.non_dominated_filter(api.SamplePool(14, words), inst, session=session)
    check_archive(got, ref.filter_pool(ri, words))


def test_filter_dedup_table_redo(ref, session):
    """the staged path's dedup starts with an L2-sized key table and redoes the dedup at full
    size when it fills; forced here with a 1024-slot first table (MOMC_TEST_DEDUP_SLOTS), the
    archive must still equal the reference's (real weights take the staged path)"""
    ri = ref.generate_uniform(14, 0.6, 3, 9, kind="real", lo=0.0, hi=1.0)
    inst = inst_from_ref(ri)
    words = random_words(14, 20000, 3)
    os.environ["MOMC_TEST_DEDUP_SLOTS"] = "1024"
    try:
        got = api.non_dominated_filter(api.SamplePool(14, words), inst, session=session)
    finally:
        del os.environ["MOMC_TEST_DEDUP_SLOTS"]
    check_archive(got, ref.filter_pool(ri, words))


def test_filter_lex_tiebreak(ref, session):
    """test_pareto.cpp:160-176: equal vectors keep the lexicographically smallest config."""
    inst = api.MultiObjectiveInstance(4, 2, [(0, 1, [1.0, 1.0]), (2, 3, [1.0, 1.0])])
    ri = ref.instance_new(4, 2, [0, 2], [1, 3], [[1.0, 1.0], [1.0, 1.0]])
    words = np.array([[0b1010], [0b0101], [0b0110], [0b1001], [0b0000]], dtype=np.uint64)
    got = api.non_dominated_filter(api.SamplePool(4, words), inst, session=session)
    check_archive(got, ref.filter_pool(ri, words))
    assert list(got.config(0)) == [-1, 1, -1, 1]  # smallest of the four (2,2) configs


def grid_vectors(M, k, seed):
    rng = np.random.default_rng(seed)
    return np.floor(rng.random((M, k)) * 40.0) / 4.0  # acceptance.cpp:173-188 style ties


@pytest.mark.parametrize("k", [1, 2, 3, 4, 5])
def test_filter_values_matches_reference(ref, session, k):
    vals = grid_vectors(5000, k, 10 + k)
    got = api.non_dominated_filter([ObjectiveVector(v) for v in vals], session=session)
    want = ref.filter_values(vals)
    assert np.array_equal(got.values, want.values)


@pytest.mark.parametrize("k,V", [(3, 60000), (4, 40000)])
def test_filter_values_sieve_matches_reference(ref, session, k, V):
    """continuous values: the compressed grid does not fit (> 32768 distinct per axis), so
    the sieve (front of the largest-sum sample kills, pairwise on the survivors) runs"""
    rng = np.random.default_rng(V + k)
    vals = rng.normal(size=(V, k)) + rng.normal(size=(V, 1))  # correlated: a non-trivial front
    got = api.non_dominated_filter([ObjectiveVector(list(v), Sense.cut) for v in vals], session=session)
    want = ref.filter_values(vals)
    assert np.array_equal(got.values, want.values)


@pytest.mark.parametrize("k,V", [(2, 20000), (3, 8000)])
def test_filter_values_grid_with_large_axes_matches_reference(ref, session, k, V):
    """continuous values with more than 2048 (but at most 32768) distinct values per axis: the
    compressed grid still fits, and its axes are ordered by the radix-sort branch"""
    rng = np.random.default_rng(3 * V + k)
    vals = rng.normal(size=(V, k)) + rng.normal(size=(V, 1))
    got = api.non_dominated_filter([ObjectiveVector(list(v), Sense.cut) for v in vals], session=session)
    want = ref.filter_values(vals)
    print(f"K={k}, V={V}: front {want.values.shape[0]}")
    assert np.array_equal(got.values, want.values)


def test_filter_values_hamiltonian_sense(ref, session):
    vals = grid_vectors(3000, 3, 77)
    got = api.non_dominated_filter([ObjectiveVector(v, Sense.hamiltonian) for v in vals], session=session)
    want = ref.filter_values(vals, sense="hamiltonian")
    assert np.array_equal(got.values, want.values)


def test_filter_example_front(session):
    """test_pareto.cpp:52-65: {(1,2),(2,1),(1,1)} -> {(2,1),(1,2)}."""
    got = api.non_dominated_filter([ObjectiveVector([1, 2]), ObjectiveVector([2, 1]), ObjectiveVector([1, 1])],
                                   session=session)
    assert got.values.tolist() == [[2.0, 1.0], [1.0, 2.0]]


def arch(vals):
    return ParetoArchive(np.asarray(vals, np.float64))


def test_hypervolume_worked_examples(session):
    """test_hypervolume.cpp:36-80"""
    hv = lambda v, r: api.hypervolume(arch(v), r, session=session)  # noqa: E731
    assert hv([[10, 5], [5, 10]], [0, 0]) == 75.0
    assert hv([[10, 5], [5, 10], [8, 8]], [0, 0]) == 84.0
    assert hv([[3, 4]], [1, 1]) == 6.0
    assert hv([[2, 3, 4]], [0, 0, 0]) == 24.0
    assert hv([[2, 3, 4, 5]], [1, 1, 1, 1]) == 24.0
    assert hv([[7], [3], [5]], [2]) == 5.0
    assert hv([[3, 2, 1], [1, 2, 3], [2, 2, 2]], [0, 0, 0]) == 12.0
    assert hv([[3, 2, 1], [1, 2, 3], [2, 2, 2], [1, 1, 1], [2, 2, 2]], [0, 0, 0]) == 12.0
    assert hv([[10, 5], [0, 20]], [0, 0]) == 50.0
    with pytest.raises(InvalidArgument, match="empty archive"):
        api.hypervolume(ParetoArchive(np.zeros((0, 2))), [0, 0], session=session)
    with pytest.raises(InvalidArgument, match=r"not dominated by archive entry 0 \(objective 0\)"):
        hv([[1, 2]], [2, 0])


@pytest.mark.parametrize("k", [2, 3, 4, 5])
def test_hypervolume_random_fronts(ref, session, k):
    for seed in range(4):
        front = ref.filter_values(grid_vectors(400, k, 100 * k + seed)).values
        r = np.full(k, -1.0)
        got = api.hypervolume(arch(front), r, session=session)
        want = ref.hypervolume(front, r)
        assert got == pytest.approx(want, rel=1e-12)


def test_hypervolume_integer_front_exact(ref, session):
    rng = np.random.default_rng(3)
    front = ref.filter_values(rng.integers(-300, 300, size=(20000, 4)).astype(np.float64)).values
    r = front.min(axis=0) - 3
    assert api.hypervolume(arch(front), r, session=session) == ref.hypervolume(front, r)


def test_reference_point_sampled_matches_reference(ref, session):
    ri = ref.instance_load("data/heavyhex42_k4_seed7.txt")
    inst = load_heavy_hex(4)
    for count, seed in ((1000, 7), (4096, 7), (17, 123)):
        assert api.reference_point_sampled(inst, count, seed, session=session) == \
            ref.reference_point_sampled(ri, count, seed).tolist()


def test_bench_readme_config(ref, session):
    """proj/README.md:64-77 with the exact reference point (0,0,0): archive 14, hv 1141902."""
    ri = ref.generate_uniform(10, 0.5, 3, 54)
    inst = inst_from_ref(ri)
    w = api.build_weights(3, 55)
    res = api.bench(inst, w, SolverConfig(batch_size=500, seed=54), 1, fixed_reference=[0, 0, 0], session=session)
    assert res.report["pool_size"] == 27500
    assert res.report["archive_size"] == 14
    assert res.report["hv"] == 1141902.0
    assert pool_fold(res.pool.words) == 0x4C640870582EDE16


@pytest.mark.parametrize("case", ["c1_heavyhex_k3_bsb", "c2_heavyhex_k4_dsb"])
def test_full_size_pipeline_matches_reference_golden(session, case):
    """C1 / C2 at full size: pool, archive (values + configs) and HV bit-equal to the
    reference's (tests/golden/make_golden.py)."""
    g = np.load(os.path.join(GOLDEN, case + ".npz"))
    k, H = int(g["k"]), int(g["H"])
    inst = load_heavy_hex(k)
    w = api.build_weights(k, resolution=H)
    cfg = SolverConfig(variant=api.parse_variant(str(g["variant"])), batch_size=int(g["batch"]), seed=7)
    res = api.bench(inst, w, cfg, 1, ref_count=4096, session=session)
    assert res.report["pool_size"] == int(g["pool_size"])
    assert pool_fold(res.pool.words) == int(g["pool_fold"])
    assert np.array_equal(res.archive.values, g["archive_values"].astype(np.float64))
    assert np.array_equal(res.archive.configs, g["archive_words"])
    assert res.report["reference"] == g["reference"].tolist()
    assert res.report["hv"] == float(g["hv"])


def test_pipeline_order_overlap_joins_on_error():
    """momc_b200_pipeline orders the archive on a side stream beside the HV. When the HV raises
    (a fixed reference not dominated by the archive) the order is still joined: the archive
    read afterwards is the complete ordered one, equal to a plain filter of the same pool, and
    the context keeps working."""
    from paper_2604_26477_b200.instances import load_heavy_hex
    inst = load_heavy_hex(4)
    w = api.build_weights(4, resolution=13)
    cfg = api.SolverConfig(variant=api.SolverVariant.discrete_sb, batch_size=300, seed=3)
    s = api.Session(0)
    s.set_instance(inst)
    s.set_weights(w)
    with pytest.raises(InvalidArgument, match="not dominated by archive entry"):
        s.pipeline(cfg, 1, 0, s.num_blocks(cfg, 1), fixed_reference=[1e9, 1e9, 1e9, 1e9])
    got = s.archive()
    ref = api.Session(0)
    want = api.non_dominated_filter(api.run_sampler(inst, w, cfg, 1, session=ref), inst, session=ref)
    assert np.array_equal(got.values, want.values) and np.array_equal(got.configs, want.configs)
    rep = s.pipeline(cfg, 1, 0, s.num_blocks(cfg, 1))
    assert rep["hv"] == api.hypervolume(want, rep["reference"], session=ref)
    assert rep["order_s"] > 0
