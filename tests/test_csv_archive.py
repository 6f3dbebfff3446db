"""Archive / trace CSV (pareto.hpp:787-897), host side: byte-identical files to the
reference's writer, identical loads, the reference's error messages."""
import os

import numpy as np
import pytest

from oracle.refbind import RefError
from paper_2604_26477_b200 import csvio
from paper_2604_26477_b200.api import InvalidArgument, MomcRuntimeError, ParetoArchive, TracePoint


def _archive(rng, F, k, n, with_cfg=True):
    vals = np.round(rng.normal(size=(F, k)) * 50) + np.where(rng.random((F, k)) < 0.2, 0.25, 0.0)
    wpc = (n + 63) // 64
    words = rng.integers(0, 2**63, size=(F, wpc), dtype=np.uint64) if with_cfg and n else None
    if words is not None and n % 64:
        words[:, -1] &= np.uint64((1 << (n % 64)) - 1)
    a = ParetoArchive(vals, words, n if words is not None else 0)
    a.filtering_seconds = 0.001234
    return a


@pytest.mark.parametrize("F,k,n,with_cfg,ref_pt", [(20, 3, 42, True, [-1.5, 0, 2]), (5, 2, 70, True, []),
                                                     (7, 4, 0, False, [1e-4, 2, 3, 4]), (0, 0, 0, False, [])])
def test_archive_csv_matches_reference(ref, tmp_path, F, k, n, with_cfg, ref_pt):
    rng = np.random.default_rng(F + k)
    a = _archive(rng, F, k, n, with_cfg)
    a.reference = list(ref_pt)
    mine, theirs = tmp_path / "mine.csv", tmp_path / "ref.csv"
    csvio.save_archive_csv(a, mine)
    ref.save_archive_csv(theirs, a.values.reshape(F, k), a.configs, n, a.filtering_seconds, ref_pt)
    assert mine.read_bytes() == theirs.read_bytes()
    got = csvio.load_archive_csv(theirs)
    want = ref.load_archive_csv(theirs)
    assert np.array_equal(got.values.reshape(want["values"].shape), want["values"])
    assert got.reference == want["reference"] and got.filtering_seconds == want["fs"]
    if with_cfg and F:
        assert np.array_equal(got.configs, want["words"])


BAD = [
    ("", "1: malformed archive header"),
    ("# pool n=3\n", "1: malformed archive header"),
    ("# archive k=2 n=0\n", "1: malformed archive header"),
    ("# archive k=2 n=0 filtering_s=0\n", "2: missing column header"),
    ("# archive k=2 n=0 filtering_s=0\nc1,c2,spins\n1,2\n", "3: malformed archive row"),
    ("# archive k=2 n=4 filtering_s=0\nc1,c2,spins\n\n1,2,0f\n", "4: bad spin field width"),
]


@pytest.mark.parametrize("text,msg", BAD)
def test_archive_csv_errors_match_reference(ref, tmp_path, text, msg):
    p = tmp_path / "bad.csv"
    p.write_text(text)
    with pytest.raises(RefError) as want:
        ref.load_archive_csv(p)
    assert str(want.value).endswith(msg) or msg in str(want.value)
    with pytest.raises(MomcRuntimeError) as got:
        csvio.load_archive_csv(p)
    assert str(got.value) == str(want.value) if hasattr(want.value, "args") else True
    assert str(got.value) == f"{p}:{msg}"


def test_archive_csv_stod_error(tmp_path):
    p = tmp_path / "bad.csv"
    p.write_text("# archive k=2 n=0 filtering_s=0\nc1,c2,spins\nx,2,-\n")
    with pytest.raises(InvalidArgument, match="stod"):
        csvio.load_archive_csv(p)


def test_missing_file():
    with pytest.raises(MomcRuntimeError, match="cannot open /nonexistent/x.csv"):
        csvio.load_archive_csv("/nonexistent/x.csv")


def test_trace_csv(tmp_path):
    p = tmp_path / "t.csv"
    csvio.save_trace_csv([TracePoint(0.5, 12.0, 3), TracePoint(1e-05, 1141902.0, 27500)], p)
    assert p.read_text() == "elapsed_s,hv,samples\n0.5,12,3\n1e-05,1141902,27500\n"
