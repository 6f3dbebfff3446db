"""The multi-GPU merge on one device: every shard of the flattened (run, weight, chunk)
blocks is sampled and filtered separately, the shard archives (values + configs) are
concatenated the way distributed.gather_fronts returns them, and merged with the device
filter (momc_b200_filter_values_dev). The result must equal the single-pass archive."""
import numpy as np
import pytest
import torch

from paper_2604_26477_b200 import api
from paper_2604_26477_b200 import distributed as mdist
from paper_2604_26477_b200.instances import load_heavy_hex

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("world", [2, 3, 8])
def test_shard_merge_equals_single_device(session, world):
    inst = load_heavy_hex(4)
    session.set_instance(inst)
    session.set_weights(api.build_weights(4, resolution=13))
    cfg = api.SolverConfig(variant=api.SolverVariant.discrete_sb, batch_size=1000, seed=11)
    runs = 2
    rep = session.pipeline(cfg, runs, 0, -1, do_hv=True, ref_count=4096)
    whole = session.archive()
    total = session.num_blocks(cfg, runs)
    dev = torch.device("cuda", 0)
    vs, ws = [], []
    for rank in range(world):
        b0, b1 = mdist.shard_range(total, world, rank)
        session.pipeline(cfg, runs, b0, b1, do_hv=False)
        v, w = mdist.local_archive_tensors(session, dev)
        vs.append(v.clone())
        ws.append(w.clone())
    av, aw = torch.cat(vs), torch.cat(ws)
    mdist.merge_on_device(session, av, aw)
    merged = session.archive()
    assert np.array_equal(merged.values, whole.values)
    assert np.array_equal(merged.configs, whole.configs)
    r = api.clamp_reference(api.reference_point_sampled(inst, 4096, cfg.seed, session=session), merged)
    assert session.archive_hypervolume(r) == rep["hv"]
