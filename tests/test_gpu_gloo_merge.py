"""The N > 1 path with the package's own device filter (gloo, world_size 2, both ranks on
cuda:0; neither rank's kernels wait on the other's): each rank samples its block share,
filters it to a local front on the device, the fronts are all-gathered
(distributed.allgather_rows) and merged by momc_b200_filter_values_dev; the merged archive
equals one device's archive of the whole pool, which is the reference's (merge law of
test_pareto.cpp:115-125 with the lex-min owner). The streaming time-to-target run at world 2
reaches the same archive and HV as at world 1."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _setup():
    from paper_2604_26477_b200 import api
    from paper_2604_26477_b200.instances import load_heavy_hex
    inst = load_heavy_hex(4)
    w = api.build_weights(4, resolution=13)
    cfg = api.SolverConfig(variant=api.SolverVariant.discrete_sb, batch_size=300, seed=13)
    return api, inst, w, cfg


def _worker(rank, world, port, out_dir):
    import sys
    sys.path.insert(0, ROOT)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import torch
    from paper_2604_26477_b200 import distributed as mdist
    from paper_2604_26477_b200 import streaming
    api, inst, w, cfg = _setup()
    dev = torch.device("cuda", 0)
    s = api.Session(0)
    s.set_instance(inst)
    s.set_weights(w)
    runs = 3
    b0, b1 = mdist.shard_range(s.num_blocks(cfg, runs), world, rank)
    s.pipeline(cfg, runs, b0, b1, do_hv=False)
    vals, words = mdist.local_archive_tensors(s, dev)
    av, aw = mdist.gather_fronts(vals, words)
    mdist.merge_on_device(s, av, aw)
    arc = s.archive()
    g = np.load(os.path.join(ROOT, "tests", "golden", "heavyhex42_k4_exact.npz"))
    r = [float(x) for x in g["reference"]]
    res = streaming.time_to_target(s, cfg, r, None, 5, world, rank, dev)
    if rank == 0:
        np.savez(os.path.join(out_dir, "merge.npz"), v=arc.values, w=arc.configs, tv=s.archive().values,
                 thv=res["hv"], truns=res["runs"])
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_device_merge_equals_one_device(tmp_path):
    mp.start_processes(_worker, args=(2, _free_port(), str(tmp_path)), nprocs=2, start_method="spawn")
    d = np.load(tmp_path / "merge.npz")
    import sys
    sys.path.insert(0, ROOT)
    from paper_2604_26477_b200 import streaming
    api, inst, w, cfg = _setup()
    s = api.Session(0)
    s.set_instance(inst)
    s.set_weights(w)
    s.pipeline(cfg, 3, 0, -1, do_hv=False)
    one = s.archive()
    assert np.array_equal(d["v"], one.values)
    assert np.array_equal(d["w"], one.configs)
    g = np.load(os.path.join(ROOT, "tests", "golden", "heavyhex42_k4_exact.npz"))
    res = streaming.time_to_target(s, cfg, [float(x) for x in g["reference"]], None, 5)
    assert int(d["truns"]) == res["runs"] == 5
    assert float(d["thv"]) == res["hv"]
    assert np.array_equal(d["tv"], s.archive().values)
