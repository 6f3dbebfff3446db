"""Host-side mirror of the reference interface (CPU only): validation messages, text I/O,
lattices and config checks behave like proj/include/momc (test_instance.cpp,
test_weights.cpp, test_solver.cpp)."""
import os

import numpy as np
import pytest

from paper_2604_26477_b200 import api
from paper_2604_26477_b200.api import InvalidArgument, MomcRuntimeError
from paper_2604_26477_b200.instances import ensure_heavy_hex, heavy_hex_edges, heavy_hex_instance


def test_instance_validation_messages():
    """instance.hpp:104-123"""
    with pytest.raises(InvalidArgument, match="vertex count must be positive"):
        api.MultiObjectiveInstance(0, 1, [])
    with pytest.raises(InvalidArgument, match="objective count must be positive"):
        api.MultiObjectiveInstance(3, 0, [])
    with pytest.raises(InvalidArgument, match="self-loop edge"):
        api.MultiObjectiveInstance(3, 1, [(1, 1, [1.0])])
    with pytest.raises(InvalidArgument, match="0 <= i < j < n"):
        api.MultiObjectiveInstance(3, 1, [(2, 1, [1.0])])
    with pytest.raises(InvalidArgument, match="exactly K weights"):
        api.MultiObjectiveInstance(3, 2, [(0, 1, [1.0])])
    with pytest.raises(InvalidArgument, match="duplicate edge"):
        api.MultiObjectiveInstance(3, 1, [(0, 1, [1.0]), (0, 1, [2.0])])


def test_instance_io_round_trip_and_reference_parse(tmp_path, ref):
    inst = heavy_hex_instance(4)
    p = tmp_path / "hh.txt"
    api.save_instance(inst, p)
    assert api.load_instance(p) == inst
    ri = ref.instance_load(str(p))
    ei, ej, w = ri.edges()
    assert np.array_equal(ei, inst.edge_i) and np.array_equal(ej, inst.edge_j) and np.array_equal(w, inst.weights)


@pytest.mark.parametrize("text,msg", [
    ("", "1: malformed header: empty file"),
    ("3 1\n", "1: malformed header: expected 'n K m'"),
    ("3 1 1 9\n0 1 1\n", "1: malformed header: trailing tokens"),
    ("3 1 2\n0 1 1\n", "3: unexpected end of file"),
    ("3 1 1\n0 x 1\n", "2: malformed edge line"),
    ("3 1 1\n1 1 1\n", "2: self-loop"),
    ("3 1 1\n0 5 1\n", "2: vertex index out of range"),
    ("3 1 1\n2 1 1\n", "2: edge endpoints must satisfy i < j"),
    ("3 1 2\n0 1 1\n0 1 2\n", "3: duplicate edge"),
    ("3 2 1\n0 1 1\n", "2: expected 2 weights"),
    ("3 1 1\n0 1 1 2\n", "2: expected exactly 1 weights"),
])
def test_load_instance_errors_match_reference(tmp_path, ref, text, msg):
    """instance.hpp:486-530 (test_instance.cpp:202-228): same line-numbered messages."""
    p = tmp_path / "bad.txt"
    p.write_text(text)
    with pytest.raises(MomcRuntimeError) as e:
        api.load_instance(p)
    assert str(e.value) == f"{p}:{msg}"
    from oracle.refbind import RefError
    with pytest.raises(RefError) as e2:
        ref.instance_load(str(p))
    assert str(e2.value) == str(e.value)


def test_heavy_hex_graph():
    edges = heavy_hex_edges()
    assert len(edges) == 45
    deg = np.zeros(42, int)
    for i, j in edges:
        assert 0 <= i < j < 42
        deg[i] += 1
        deg[j] += 1
    assert deg.max() == 3 and deg.min() >= 1
    inst = heavy_hex_instance(4)
    assert (inst.weights > 0).any() and (inst.weights < 0).any()  # mixed sign
    assert api.load_instance(ensure_heavy_hex(4)) == inst


def test_lattices_match_reference(ref):
    for k, h in ((2, 5), (3, 12), (3, 21), (4, 13)):
        lat = api.das_dennis(k, h)
        assert np.array_equal(np.array([[w.numerator(q) for q in range(k)] for w in lat]),
                              ref.das_dennis(k, h, interior=False))
        inner = api.interior_filter(lat)
        assert np.array_equal(np.array([[w.numerator(q) for q in range(k)] for w in inner]), ref.das_dennis(k, h))
    assert api.resolution_for_interior_count(3, 190) == 21
    assert len(api.build_weights(4, 220)) == 220
    with pytest.raises(InvalidArgument, match="at least two objectives"):
        api.das_dennis(1, 3)
    with pytest.raises(InvalidArgument, match="sum to the resolution"):
        api.WeightVector([1, 1], 3)
    with pytest.raises(InvalidArgument, match="non-negative"):
        api.WeightVector([-1, 4], 3)
    w = api.WeightVector([10, 1, 1], 12)
    assert w[0] == 10 / 12 and w.is_interior()


def test_solver_config_validation():
    """solver.hpp:57-66 / test_solver.cpp:52-73"""
    cfg = api.SolverConfig()
    cfg.validate()
    for field, val, msg in (("n_iterations", 0, "n_iterations must be >= 1"), ("dt", 0.0, "dt must be positive"),
                            ("a0", 0.0, "a0 must be positive"), ("alpha", -0.1, "alpha must be non-negative"),
                            ("batch_size", 0, "batch_size must be >= 1"),
                            ("init_scale", -1.0, "init_scale must be non-negative"),
                            ("threads", -1, "threads must be non-negative")):
        c = api.SolverConfig(**{field: val})
        with pytest.raises(InvalidArgument, match=msg):
            c.validate()
    assert api.parse_variant("dsb") == api.SolverVariant.discrete_sb
    with pytest.raises(InvalidArgument, match="unknown solver variant: gsb"):
        api.parse_variant("gsb")
    assert api.pump_schedule(25, 50) == 0.5
    with pytest.raises(InvalidArgument):
        api.pump_schedule(51, 50)


def test_sample_pool_records_and_packing():
    words = np.array([[0b101], [0b010], [0b111], [0b000]], dtype=np.uint64)
    pool = api.SamplePool(3, words, runs=2, weights=1, batch=2, stamps=np.arange(4))
    assert pool.size() == 4 and pool.words_per_config() == 1
    assert pool.record(3).run == 1 and pool.record(3).trajectory == 1 and pool.record(3).timestamp_ns == 3
    assert pool.config(0).tolist() == [1, -1, 1]
    assert api.same_samples(pool, api.SamplePool(3, words.copy(), 2, 1, 2))


def test_archive_reference_validation():
    a = api.ParetoArchive(np.array([[3.0, 4.0], [5.0, 1.0]]))
    a.set_reference([0.0, 0.0])
    with pytest.raises(InvalidArgument, match=r"archive entry 1 \(objective 1\)"):
        a.validate_reference([0.0, 2.0])
    assert api.clamp_reference([4.0, 0.5], a) == [3.0, 0.5]


def test_product_fails_loudly_without_gpu():
    """There is no CPU fallback: without a B200 the session cannot be created."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2604_26477_b200 import _lib
    if not os.path.exists(_lib.LIB_PATH):
        with pytest.raises(ImportError):
            api.Session(0)
        return
    with pytest.raises(MomcRuntimeError, match="no CUDA device"):
        api.Session(0)


def test_format_number_matches_to_chars():
    """format_number (instance.hpp:462-470) against libstdc++ std::to_chars output
    (tests/golden/make_to_chars.py)."""
    import os
    g = np.load(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "to_chars_vectors.npz"))
    from paper_2604_26477_b200.api import _to_chars_shortest, format_number
    for v, t in zip(g["values"].tolist(), g["text"].tolist()):
        assert _to_chars_shortest(v) == t, v
    assert format_number(3.0) == "3" and format_number(-12.0) == "-12" and format_number(1e15) == "1e+15"
    assert format_number(0.142) == "0.142" and format_number(1e-4) == "1e-04"
