"""Multi-GPU sharding of the hot path: one process per GPU.

Every (run, weight, trajectory) RNG stream is position-independent (solver.hpp:86-94), so
any partition of the flattened (run, weight, chunk) blocks reproduces the single-device
pool bit-for-bit. Each rank samples its contiguous block range, filters it to a local
front on its GPU, and the local fronts (values + lex-smallest configs) are all-gathered
with NCCL (torch.distributed) and merged by the same device filter on every rank. The
merge law filter(A u B) = filter(filter(A) u filter(B)) (test_pareto.cpp:115-125) plus the
lex-min collapse rule make the merged archive equal to the single-device one.
"""
from __future__ import annotations

import numpy as np
import torch
import torch.distributed as dist


def shard_range(total: int, world: int, rank: int) -> tuple[int, int]:
    """Balanced contiguous [begin, end) share of `total` blocks for `rank`."""
    if world < 1 or rank < 0 or rank >= world:
        raise ValueError("bad world/rank")
    base, rem = divmod(total, world)
    begin = rank * base + min(rank, rem)
    return begin, begin + base + (1 if rank < rem else 0)


def allgather_rows(local: torch.Tensor, group=None) -> torch.Tensor:
    """All-gather a variable number of rows (dim 0) across ranks; returns the concatenation
    in rank order. Sizes first, then one padded collective. (gloo: through host memory.)"""
    if local.is_cuda and dist.get_backend(group) == "gloo":
        return allgather_rows(local.cpu(), group).to(local.device)
    world = dist.get_world_size(group)
    n = torch.tensor([local.shape[0]], dtype=torch.int64, device=local.device)
    sizes = [torch.zeros_like(n) for _ in range(world)]
    dist.all_gather(sizes, n, group=group)
    sizes = [int(s.item()) for s in sizes]
    cap = max(max(sizes), 1)
    pad = torch.zeros((cap,) + tuple(local.shape[1:]), dtype=local.dtype, device=local.device)
    pad[: local.shape[0]] = local
    bufs = [torch.empty_like(pad) for _ in range(world)]
    dist.all_gather(bufs, pad, group=group)
    return torch.cat([b[:s] for b, s in zip(bufs, sizes)], dim=0)


def gather_fronts(vals: torch.Tensor, words: torch.Tensor, group=None):
    """All-gather local archives: float64 values (F x K) and packed configs (F x wpc,
    carried as int64 bit patterns because NCCL has no uint64)."""
    return allgather_rows(vals, group), allgather_rows(words, group)


def merge_on_device(session, vals: torch.Tensor, words: torch.Tensor) -> int:
    """Filter the gathered fronts into the session's resident archive (CUDA)."""
    torch.cuda.current_stream(vals.device).synchronize()
    K = vals.shape[1]
    wpc = words.shape[1]
    return session.merge_device(vals.data_ptr(), words.data_ptr(), wpc, vals.shape[0], K)


def local_archive_tensors(session, device) -> tuple[torch.Tensor, torch.Tensor]:
    """Device-to-device copy of the session's resident archive into torch tensors."""
    F = session.archive_size()
    K = session.inst.k()
    wpc = (session.inst.n() + 63) // 64
    vals = torch.empty((max(F, 1), K), dtype=torch.float64, device=device)[:F]
    words = torch.empty((max(F, 1), wpc), dtype=torch.int64, device=device)[:F]
    if F:
        session.archive_copy_device(vals.data_ptr(), words.data_ptr())
    return vals, words


def numpy_words(t: torch.Tensor) -> np.ndarray:
    return t.detach().cpu().numpy().view(np.uint64)
