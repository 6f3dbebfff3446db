"""generate_correlated_instance (instance.hpp:364-458) and measured_correlation
(instance.hpp:338-357) on the device: bit-identical instances and correlations; the
acceptance criterion-4 workload (acceptance.cpp:128-151: n=200, rho=-0.92, 55 x 3000 SimCIM/
dSB samples end to end) through the device bench."""
import numpy as np
import pytest

from paper_2604_26477_b200 import api
from paper_2604_26477_b200.api import InvalidArgument

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("n,density,rho,seed", [(10, 1.0, -0.92, 5), (30, 0.5, -0.5, 1), (200, 1.0, -0.92, 42),
                                                (64, 0.3, -0.2, 9)])
def test_correlated_instance_matches_reference(ref, session, n, density, rho, seed):
    got = session.generate_correlated_instance(n, density, rho, seed)
    want = ref.generate_correlated(n, density, rho, seed)
    ei, ej, w = want.edges()
    assert np.array_equal(got.edge_i, ei) and np.array_equal(got.edge_j, ej)
    assert np.array_equal(got.weights, np.asarray(w).reshape(-1, 3))
    assert session.measured_correlation() == ref.measured_correlation(want)
    assert session.measured_correlation(500, 3) == ref.measured_correlation(want, 500, 3)
    assert abs(session.measured_correlation() - rho) < 0.05


def test_correlated_errors(ref, session):
    with pytest.raises(InvalidArgument, match=r"target correlation must lie in \(-1, 0\)"):
        session.generate_correlated_instance(10, 1.0, 0.3, 1)
    with pytest.raises(InvalidArgument, match="vertex count must be at least 4"):
        session.generate_correlated_instance(3, 1.0, -0.5, 1)
    with pytest.raises(InvalidArgument, match="correlation measure requires K=3"):
        api.measured_correlation(api.MultiObjectiveInstance(4, 2, [(0, 1, [1, 2])]), session=session)


def test_acceptance_end_to_end_bound(session):
    """acceptance.cpp:128-151: bench(n=200, d=1.0, K=3, rho=-0.92, seed 42, 55 weights, runs 1,
    sampled:4096) -> pool 165,000, archive >= 1, end-to-end < 60 s (here: well under 1 s)."""
    inst = session.generate_correlated_instance(200, 1.0, -0.92, 42)
    weights = api.build_weights(3, count=55)
    cfg = api.SolverConfig(variant=api.SolverVariant.ballistic_sb, seed=42)
    res = api.bench(inst, weights, cfg, 1, ref_count=4096, session=session)
    rep = res.report
    assert rep["pool_size"] == 55 * 3000 and rep["archive_size"] >= 1
    assert rep["model_construction_s"] > 0 and rep["sampling_s"] > 0 and rep["pareto_filtering_s"] > 0
    assert rep["end_to_end_s"] >= 0.95 * (rep["model_construction_s"] + rep["sampling_s"] + rep["pareto_filtering_s"])
    assert rep["end_to_end_s"] < 60.0
