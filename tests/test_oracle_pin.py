"""Pins the CPU oracles (CPU only): the C restatement (oracle/momc_oracle.c) against the
unmodified reference compiled with the Eigen shim (oracle/_ref/libmomc_ref.so), and both
against the reference's own golden vectors / known answers."""
import os

import numpy as np
import pytest

from oracle.refbind import make_cfg, pool_fold

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def inst_tuple(ri):
    ei, ej, w = ri.edges()
    return (ri.n, ri.k, ei, ej, w)


@pytest.mark.parametrize("lib", ["ref", "orc"])
def test_philox_known_answers(request, lib):
    """test_rng.cpp:14-27"""
    L = request.getfixturevalue(lib)
    assert L.philox(0, [0, 0, 0, 0]).tolist() == [0x6627E8D5, 0xE169C58D, 0xBC57AC4C, 0x9B00DBD8]
    assert L.philox(0xFFFFFFFFFFFFFFFF, [0xFFFFFFFF] * 4).tolist() == [0x408F276D, 0x41C83B0E, 0xA20BC7C6, 0x6D5451FD]
    pi_key = 0xA4093822 | (0x299F31D0 << 32)
    assert L.philox(pi_key, [0x243F6A88, 0x85A308D3, 0x13198A2E, 0x03707344]).tolist() == \
        [0xD16CFE09, 0x94FDCCEB, 0x5001E420, 0x24126EA1]


def test_keys_tags_and_tables(ref, orc):
    assert ref.run_key(54, 0) == orc.run_key(54, 0) == 0x326A9F7808F64370
    for tag, step in ((1, 0), (3, 17), (8, 0), (3, 0x3FFFFFF)):
        assert ref.tag_word(tag, step) == orc.tag_word(tag, step)
    for a, b in zip(ref.ziggurat_tables(), orc.ziggurat_tables()):
        assert np.array_equal(a, b)


def test_noise_golden_vector(ref, orc):
    """first normals of (seed 54, run 0, weight 0, trajectory 0, step 0)."""
    key = ref.run_key(54, 0)
    want = [0.65025771496111984, 0.70798024355005751, 1.4312023647046184, 1.5694745382996151]
    assert ref.stream_normals(key, 0, 0, ref.tag_word(3, 0), 4).tolist() == want
    assert orc.stream_normals(key, 0, 0, orc.tag_word(3, 0), 4).tolist() == want


def test_streams_agree_at_length(ref, orc):
    key = ref.derive_key(99, 5)
    for ids in ((0, 0, 0), (3, 41, ref.tag_word(3, 7)), (219, 4545, ref.tag_word(3, 49))):
        assert np.array_equal(ref.stream_u32(key, *ids, 997), orc.stream_u32(key, *ids, 997))
        assert np.array_equal(ref.stream_normals(key, *ids, 20000), orc.stream_normals(key, *ids, 20000))


def test_init_state_golden(ref):
    """init x/y of (run 0, weight 0, trajectory 0) in the README config."""
    x, y = ref.init_state(make_cfg(), 10, 1, ref.run_key(54, 0), 0, 0)
    assert x[0, :3].tolist() == [0.08392249308096103, -0.013113623729995118, 0.05484339978717441]
    assert y[0, :3].tolist() == [-0.069778551787939833, 0.0074215326993339438, -0.0044465427655931309]


def test_lattice_counts(ref, orc):
    """test_weights.cpp:37-102 / acceptance criterion 2"""
    assert ref.das_dennis(3, 21, interior=False).shape[0] == 253
    assert ref.das_dennis(4, 13, interior=False).shape[0] == 560
    assert ref.das_dennis(3, 21).shape[0] == 190
    assert ref.das_dennis(4, 13).shape[0] == 220
    assert ref.das_dennis(3, 12).shape[0] == 55
    for k, h in ((3, 21), (4, 13), (3, 12), (2, 7)):
        assert np.array_equal(ref.das_dennis(k, h), orc.das_dennis(k, h))
        assert np.array_equal(ref.das_dennis(k, h, False), orc.das_dennis(k, h, False))
    assert ref.resolution_for_interior_count(3, 190) == orc.resolution_for_interior_count(3, 190) == 21
    assert ref.resolution_for_interior_count(4, 220) == orc.resolution_for_interior_count(4, 220) == 13


def test_scalarize(ref, orc):
    ri = ref.generate_uniform(10, 0.5, 3, 54)
    nums = ref.das_dennis(3, 12)
    J, c0 = ref.scalarize(ri, nums[0], 12)
    assert c0 == 0.024390243902439025  # w[0] = (10,1,1)/12, c0 = 1/41
    for l in range(nums.shape[0]):
        Jr, cr = ref.scalarize(ri, nums[l], 12)
        Jo, co = orc.scalarize(inst_tuple(ri), nums[l], 12)
        assert np.array_equal(Jr, Jo) and cr == co


@pytest.mark.parametrize("variant,fold", [("bsb", 0x4C640870582EDE16), ("dsb", 0x4572BF3D54216F62)])
def test_readme_pool_folds(ref, orc, variant, fold):
    ri = ref.generate_uniform(10, 0.5, 3, 54)
    nums = ref.das_dennis(3, 12)
    cfg = make_cfg(variant, batch_size=500, seed=54, threads=os.cpu_count() or 4)
    wr = ref.run_sampler(ri, nums, 12, cfg, 1)["words"]
    wo = orc.run_sampler(inst_tuple(ri), nums, 12, cfg, 1)
    assert pool_fold(wr) == pool_fold(wo) == fold
    if variant == "bsb":
        assert [int(v) for v in wr[:8, 0]] == [0x2E1, 0x2E1, 0x11F, 0x2E1, 0x2B2, 0x11E, 0x2B2, 0x14D]
        assert int(wr[500, 0]) == 0x2B2 and int(wr[27499, 0]) == 0x0E5


@pytest.mark.parametrize("variant", ["bsb", "dsb", "simcim"])
@pytest.mark.parametrize("n,density,k", [(4, 1.0, 2), (20, 0.5, 3), (70, 0.3, 2)])
def test_restatement_pools_match_reference(ref, orc, variant, n, density, k):
    ri = ref.generate_uniform(n, density, k, n + k)
    nums = ref.das_dennis(k, 4)
    cfg = make_cfg(variant, batch_size=700, n_iterations=20, seed=n, threads=os.cpu_count() or 4)
    assert np.array_equal(ref.run_sampler(ri, nums, 4, cfg, 2)["words"], orc.run_sampler(inst_tuple(ri), nums, 4, cfg, 2))


def test_readme_bench_report(ref):
    """proj/README.md:64-77, reproduced by the shim build of the reference."""
    rep = ref.bench(make_cfg("bsb", batch_size=500, seed=54, threads=os.cpu_count() or 4), n=10, density=0.5, k=3,
                    instance_seed=54, weight_count=55)
    assert (rep["pool_size"], rep["archive_size"], rep["hv"], rep["hv_max"], rep["samples_to_optimal"]) == \
        ("27500", "14", "1141902", "1141902", "6054")


def test_filters_and_hv_match_reference(ref, orc):
    ri = ref.generate_uniform(18, 0.5, 4, 11)
    rng = np.random.default_rng(0)
    words = rng.integers(0, 1 << 18, size=(30000, 1)).astype(np.uint64)
    a = ref.filter_pool(ri, words)
    v, c = orc.filter_pool(inst_tuple(ri), words)
    assert np.array_equal(a.values, v) and np.array_equal(a.words, c)
    assert np.array_equal(ref.evaluate_cuts(ri, words[:500]), orc.evaluate_cuts(inst_tuple(ri), words[:500]))
    assert np.array_equal(ref.cut_values(ri, words[:500]), orc.cut_values(inst_tuple(ri), words[:500]))
    r = v.min(axis=0) - 1
    assert ref.hypervolume(a.values, r) == orc.hypervolume(v, r)
    vals = np.floor(rng.random((4000, 3)) * 40) / 4
    assert np.array_equal(ref.filter_values(vals).values, orc.filter_values(vals))
    assert ref.reference_point_sampled(ri, 1000, 7).tolist() == orc.reference_point_sampled(inst_tuple(ri), 1000, 7).tolist()


def test_hypervolume_worked_examples(ref, orc):
    """test_hypervolume.cpp:36-80"""
    for L in (ref, orc):
        hv = lambda v, r: L.hypervolume(np.array(v, np.float64), np.array(r, np.float64))  # noqa: E731
        assert hv([[10, 5], [5, 10]], [0, 0]) == 75.0
        assert hv([[10, 5], [5, 10], [8, 8]], [0, 0]) == 84.0
        assert hv([[2, 3, 4, 5]], [1, 1, 1, 1]) == 24.0
        assert hv([[3, 2, 1], [1, 2, 3], [2, 2, 2]], [0, 0, 0]) == 12.0
        assert hv([[3, 2, 1], [1, 2, 3], [2, 2, 2], [1, 1, 1], [2, 2, 2]], [0, 0, 0]) == 12.0


def test_c1_golden_fixture(ref, orc):
    """The committed C1 fixture (tests/golden/make_golden.py) against the C restatement."""
    from paper_2604_26477_b200.instances import ensure_heavy_hex
    g = np.load(os.path.join(GOLDEN, "c1_heavyhex_k3_bsb.npz"))
    ri = ref.instance_load(ensure_heavy_hex(3))
    nums = ref.das_dennis(3, 21)
    words = orc.run_sampler(inst_tuple(ri), nums, 21, make_cfg("bsb", batch_size=3000, seed=7), 1,
                            threads=os.cpu_count() or 4)
    assert pool_fold(words) == int(g["pool_fold"])
    v, c = orc.filter_pool(inst_tuple(ri), words)
    assert np.array_equal(v, g["archive_values"].astype(np.float64)) and np.array_equal(c, g["archive_words"])
    assert orc.hypervolume(v, g["reference"]) == float(g["hv"])
