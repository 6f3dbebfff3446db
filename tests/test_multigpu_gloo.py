"""N > 1 path on the CPU (gloo, world_size 2): block sharding, the variable-size all-gather
of local fronts, and the merge law filter(A u B) = filter(filter(A) u filter(B))
(test_pareto.cpp:115-125) with the lex-smallest-config collapse, using the reference as the
filter (the CUDA merge kernel itself is covered by tests/test_gpu_*)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2604_26477_b200.distributed import allgather_rows, gather_fronts, shard_range

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_shard_range_partitions():
    for total in (0, 1, 7, 1980, 15620):
        for world in (1, 2, 3, 8):
            parts = [shard_range(total, world, r) for r in range(world)]
            assert parts[0][0] == 0 and parts[-1][1] == total
            assert all(a[1] == b[0] for a, b in zip(parts, parts[1:]))
            sizes = [e - b for b, e in parts]
            assert max(sizes) - min(sizes) <= 1


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out_dir):
    import sys
    sys.path.insert(0, ROOT)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle.refbind import RefLib
    R = RefLib()
    ri = R.generate_uniform(18, 0.5, 3, 21)
    rng = np.random.default_rng(5)
    pool = rng.integers(0, 1 << 18, size=(20000, 1)).astype(np.uint64)
    b, e = shard_range(pool.shape[0], world, rank)
    local = R.filter_pool(ri, pool[b:e])
    vals = torch.from_numpy(local.values.copy())
    words = torch.from_numpy(local.words.view(np.int64).copy())
    av, aw = gather_fronts(vals, words)
    # variable-size gather of plain rows too
    rows = allgather_rows(torch.full((rank + 2, 3), float(rank)))
    assert rows.shape[0] == sum(r + 2 for r in range(world))
    merged = R.filter_pool(ri, aw.numpy().view(np.uint64))
    if rank == 0:
        whole = R.filter_pool(ri, pool)
        np.savez(os.path.join(out_dir, "merge.npz"), mv=merged.values, mw=merged.words, wv=whole.values,
                 ww=whole.words, gathered=av.shape[0])
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_front_merge_equals_single_filter(tmp_path):
    pytest.importorskip("torch.distributed")
    if not dist.is_available():
        pytest.skip("torch.distributed unavailable")
    mp.start_processes(_worker, args=(2, _free_port(), str(tmp_path)), nprocs=2, start_method="spawn")
    d = np.load(tmp_path / "merge.npz")
    assert np.array_equal(d["mv"], d["wv"])
    assert np.array_equal(d["mw"], d["ww"])  # lex-smallest configs survive the merge
    assert int(d["gathered"]) >= d["wv"].shape[0]
