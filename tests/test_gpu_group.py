"""Device groups through the C-ABI (momc_b200_group_*): the sharded pool, the merged archive
and the bench report of a group equal one context's, which equal the reference's
(solver.hpp:455-522 task pool replaced by per-device shards; pareto.hpp:370-410 merge law).
On a one-GPU box the members share device 0 and the fronts travel by peer copy; the NCCL
transport needs distinct devices."""
import numpy as np
import pytest

from paper_2604_26477_b200 import api
from paper_2604_26477_b200.instances import load_heavy_hex

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def setup():
    inst = load_heavy_hex(4)
    w = api.build_weights(4, resolution=13)
    cfg = api.SolverConfig(variant=api.SolverVariant.discrete_sb, batch_size=257, seed=5)
    return inst, w, cfg


@pytest.mark.parametrize("members", [2, 3, 5])
def test_group_pool_archive_bench_equal_single(setup, members):
    inst, w, cfg = setup
    g = api.DeviceGroup([0] * members)
    assert g.size() == members and g.transport() == "copy"
    s = api.Session(0)
    one = api.run_sampler(inst, w, cfg, 2, session=s)
    many = g.run_sampler(inst, w, cfg, 2)
    diff = int(np.count_nonzero(np.any(one.words != many.words, axis=1)))
    print(f"{members} members: {diff} of {one.words.shape[0]} pool rows differ")
    assert diff == 0
    a = api.non_dominated_filter(one, inst, session=s)
    b = g.non_dominated_filter(many, inst)
    assert np.array_equal(a.values, b.values) and np.array_equal(a.configs, b.configs)
    r1 = api.bench(inst, w, cfg, 2, ref_count=4096, session=s)
    r2 = g.bench(inst, w, cfg, 2, ref_count=4096)
    assert r1.report["hv"] == r2.report["hv"] and r1.report["reference"] == r2.report["reference"]
    assert np.array_equal(r1.pool.words, r2.pool.words)
    assert np.array_equal(r1.archive.values, r2.archive.values)
    assert np.array_equal(r1.archive.configs, r2.archive.configs)


def test_group_single_device_and_env(setup, monkeypatch):
    inst, w, cfg = setup
    monkeypatch.setenv("MOMC_GPUS", "1")
    g = api.DeviceGroup()
    assert g.size() == 1 and g.transport() == "single"
    r = g.bench(inst, w, cfg, 1, ref_count=4096)
    r0 = api.bench(inst, w, cfg, 1, ref_count=4096, session=api.Session(0))
    assert r.report["hv"] == r0.report["hv"]
    monkeypatch.setenv("MOMC_GPUS", "0,0")
    assert api.DeviceGroup().transport() == "copy"
    monkeypatch.setenv("MOMC_GPUS", "0,")
    with pytest.raises(api.InvalidArgument, match="MOMC_GPUS: empty device entry"):
        api.DeviceGroup()


def test_group_nccl_transport_one_rank(setup, monkeypatch):
    """the NCCL code path (dlopen'd libnccl, ncclCommInitAll, padded ncclAllGather of the
    packed fronts, unpack, merge) as a one-rank group on one GPU"""
    inst, w, cfg = setup
    monkeypatch.setenv("MOMC_GROUP_TRANSPORT", "nccl")
    g = api.DeviceGroup([0])
    assert g.transport() == "nccl"
    s = api.Session(0)
    r1 = api.bench(inst, w, cfg, 1, ref_count=4096, session=s)
    r2 = g.bench(inst, w, cfg, 1, ref_count=4096)
    assert r1.report["hv"] == r2.report["hv"]
    assert np.array_equal(r1.archive.values, r2.archive.values)
    assert np.array_equal(r1.archive.configs, r2.archive.configs)
    b = g.non_dominated_filter(r1.pool, inst)
    assert np.array_equal(r1.archive.values, b.values) and np.array_equal(r1.archive.configs, b.configs)
