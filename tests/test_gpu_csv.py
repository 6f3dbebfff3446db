"""Pool CSV (solver.hpp:357-432) with the record rows formatted / parsed on the device:
byte-identical to the reference's writer, identical loads, the reference's messages."""
import numpy as np
import pytest

from oracle.refbind import RefError, make_cfg
from paper_2604_26477_b200 import api, csvio
from paper_2604_26477_b200.api import MomcRuntimeError

pytestmark = pytest.mark.gpu


def _pool(rng, M, n):
    wpc = (n + 63) // 64
    words = rng.integers(0, 2**63, size=(M, wpc), dtype=np.uint64) | (
        rng.integers(0, 2, size=(M, wpc), dtype=np.uint64) << np.uint64(63))
    if n % 64:
        words[:, -1] &= np.uint64((1 << (n % 64)) - 1)
    rec = np.stack([rng.integers(0, 5, M), rng.integers(0, 300, M), rng.integers(0, 2**32, M)], 1).astype(np.uint32)
    stamps = rng.integers(-10**12, 10**15, M).astype(np.int64)
    stamps[:3] = [0, -1, 2**63 - 1][:M]
    p = api.SamplePool(n, words, stamps=stamps, records=rec)
    p.model_construction_seconds = 4.6e-05
    p.sampling_seconds = 0.142
    return p


@pytest.mark.parametrize("M,n", [(1, 1), (1000, 42), (5000, 70), (300, 128), (20000, 2000)])
def test_pool_csv_matches_reference(ref, session, tmp_path, M, n):
    pool = _pool(np.random.default_rng(M), M, n)
    mine, theirs = tmp_path / "mine.csv", tmp_path / "ref.csv"
    csvio.save_pool_csv(pool, mine, session=session)
    ref.save_pool_csv(theirs, pool.words, pool.records, pool.stamps, n, pool.model_construction_seconds,
                      pool.sampling_seconds)
    assert mine.read_bytes() == theirs.read_bytes()
    got = csvio.load_pool_csv(theirs, session=session)
    assert got == pool
    assert got.model_construction_seconds == pool.model_construction_seconds
    assert got.sampling_seconds == pool.sampling_seconds


def test_pool_csv_round_trip_sampler(ref, session, tmp_path):
    """test_solver.cpp:377-392 shape: a sampled pool round-trips (records, stamps, timings)."""
    ri = ref.generate_uniform(70, 0.5, 2, 6)
    ei, ej, w = ri.edges()
    inst = api.MultiObjectiveInstance.from_arrays(70, 2, ei, ej, w)
    weights = api.interior_filter(api.das_dennis(2, 3))
    pool = api.run_sampler(inst, weights, api.SolverConfig(batch_size=30, n_iterations=4), 2, session=session)
    p = tmp_path / "pool.csv"
    csvio.save_pool_csv(pool, p, session=session)
    loaded = csvio.load_pool_csv(p, session=session)
    assert loaded == pool and api.same_samples(loaded, pool)
    assert loaded.sampling_seconds == pool.sampling_seconds


GOOD_ROW = "1,2,3,4,000000000000002a\n"
BAD = [
    ("", ":1: malformed pool header"),
    ("# pool n=0 model_construction_s=0 sampling_s=0\n", ":1: malformed pool header"),
    ("# pool n=3 model_construction_s=0\n", ":1: malformed pool header"),
    ("# pool n=6 model_construction_s=0 sampling_s=0\n", ":2: missing column header"),
    ("# pool n=6 model_construction_s=0 sampling_s=0\nh\n" + GOOD_ROW + "1,2,3,4\n", ":4: malformed pool record"),
    ("# pool n=6 model_construction_s=0 sampling_s=0\nh\n" + GOOD_ROW + "1,2,3,4,\n", ":4: malformed pool record"),
    ("# pool n=6 model_construction_s=0 sampling_s=0\nh\n\n" + "1,x,3,4,000000000000002a\n", ":4: malformed pool record"),
    ("# pool n=6 model_construction_s=0 sampling_s=0\nh\n" + "1,2,3,99999999999999999999,000000000000002a\n",
     ":3: malformed pool record"),
    ("# pool n=6 model_construction_s=0 sampling_s=0\nh\n" + GOOD_ROW * 3 + "1,2,3,4,2a\n", ":6: bad spin field width"),
    ("# pool n=6 model_construction_s=0 sampling_s=0\nh\n" + "1,2,3,4,000000000000002a\r\n", ":3: bad spin field width"),
]


@pytest.mark.parametrize("text,msg", BAD)
def test_pool_csv_errors_match_reference(ref, session, tmp_path, text, msg):
    p = tmp_path / "bad.csv"
    p.write_text(text)
    with pytest.raises(RefError) as want:
        ref.load_pool_csv(p)
    with pytest.raises(MomcRuntimeError) as got:
        csvio.load_pool_csv(p, session=session)
    assert str(got.value) == str(want.value) == f"{p}{msg}"


def test_pool_csv_lenient_fields_match_reference(ref, session, tmp_path):
    """stoul / stoll leniency: whitespace, '+', trailing garbage, negative wrap, empty lines,
    no final newline, junk hex digits."""
    rows = [" 7,+2,3x,-5,000000000000002a", "", "-1,0,4294967297,  12,zzzzzzzzzzzzzzzz", "0,0,0,0,ffffffffffffffff"]
    p = tmp_path / "odd.csv"
    p.write_text("# pool n=64 model_construction_s=  1.5 sampling_s=2e-3\nx\n" + "\n".join(rows))
    want = ref.load_pool_csv(p)
    got = csvio.load_pool_csv(p, session=session)
    assert np.array_equal(got.records, want["rec3"]) and np.array_equal(got.stamps, want["stamps"])
    assert np.array_equal(got.words, want["words"])
    assert got.model_construction_seconds == want["mc"] and got.sampling_seconds == want["ss"]
