"""Streaming time-to-optimal-hypervolume (SURVEY.md §8d "time-to-optimal", §8f #2).

The reference measures time-to-optimal offline: `samples_to_reach` (pareto.hpp:763-781)
replays a finished pool until the running archive's HV reaches a target. On the device the
natural unit is a *run* (solver.hpp:481-527: every run is the full lattice x batch with its
own RNG key run_key(seed, run)), so the stream is: sample run r -> local front -> merge into
the running archive (device filter, lex-min owners) -> HV at the frozen reference point ->
stop when HV equals the target. With N ranks, round q samples runs q*N .. q*N+N-1 (run
q*N+rank on rank `rank`), the per-run fronts are all-gathered (NCCL) and every rank merges
the same rows, so every rank holds the same running archive and takes the same decision
without another collective.
"""
from __future__ import annotations

import time

import torch

from . import distributed as mdist


def _packed_front(session, device):
    """resident archive -> one int64 tensor [F, K + wpc] (values as bit patterns)"""
    vals, words = mdist.local_archive_tensors(session, device)
    return torch.cat([vals.view(torch.int64), words], dim=1)


def time_to_target(session, cfg, reference, hv_target: float, max_runs: int, world: int = 1, rank: int = 0,
                   device=None, trace: list | None = None) -> dict:
    """Runs rounds until the running archive's HV at `reference` equals `hv_target` (exact
    arithmetic for integer weights) or `max_runs` runs are spent. Returns the number of
    runs / samples used, the wall time (device-synchronised, this rank) and the final HV.
    The caller times the whole call as the end-to-end figure (model build included: every
    round re-scalarises its weight blocks, pipeline.hpp:337-341)."""
    device = device or torch.device("cuda", torch.cuda.current_device())
    k = session.inst.k()
    per_run = session.num_blocks(cfg, 1)
    samples_per_run = session.L * cfg.batch_size
    running = None
    hv = 0.0
    runs_done = 0
    t0 = time.perf_counter()
    rounds = (max_runs + world - 1) // world
    for q in range(rounds):
        run = q * world + rank
        session.pipeline(cfg, run + 1, run * per_run, (run + 1) * per_run, do_hv=False)
        mine = _packed_front(session, device)
        rows = mdist.allgather_rows(mine) if world > 1 else mine
        if running is not None:
            rows = torch.cat([running, rows], dim=0)
        if world > 1 or running is not None:
            vals = rows[:, :k].contiguous().view(torch.float64)
            words = rows[:, k:].contiguous()
            mdist.merge_on_device(session, vals, words)
            running = _packed_front(session, device)
        else:
            running = rows
        runs_done = (q + 1) * world
        hv = session.archive_hypervolume(reference)
        if trace is not None:
            trace.append({"runs": runs_done, "samples": runs_done * samples_per_run, "archive": int(running.shape[0]),
                          "hv": hv, "wall_s": time.perf_counter() - t0})
        if hv == hv_target:
            break
    torch.cuda.synchronize(device)
    return {"reached": hv == hv_target, "runs": runs_done, "samples": runs_done * samples_per_run,
            "seconds": time.perf_counter() - t0, "hv": hv, "archive": int(running.shape[0]) if running is not None else 0}


def time_to_target_overlapped(sessions: list, cfg, reference, hv_target: float, max_runs: int, device=None,
                              trace: list | None = None) -> dict:
    """One GPU, several sessions (contexts: own stream + buffers) in host threads: run r is
    sampled by session r % S while the previous run's front is filtered / merged on another
    session's stream, so the Pareto stage hides under the next run's sampler. Merges happen
    strictly in run order, so the result (runs, samples, archive, HV) equals the sequential
    stream's; only the wall time differs."""
    import threading

    device = device or torch.device("cuda", torch.cuda.current_device())
    S = len(sessions)
    per_run = sessions[0].num_blocks(cfg, 1)
    samples_per_run = sessions[0].L * cfg.batch_size
    st = {"next": 0, "running": None, "hv": 0.0, "done": False, "runs": 0, "error": None}
    cv = threading.Condition()
    t0 = time.perf_counter()

    def worker(w):
        s = sessions[w]
        try:
            torch.cuda.set_device(device)
            for run in range(w, max_runs, S):
                with cv:
                    if st["done"]:
                        return
                s.pipeline(cfg, run + 1, run * per_run, (run + 1) * per_run, do_hv=False)
                mine = _packed_front(s, device)
                with cv:
                    while st["next"] != run and not st["done"]:
                        cv.wait()
                    if st["done"]:
                        return
                    if st["running"] is not None:
                        rows = torch.cat([st["running"], mine], dim=0)
                        k = s.inst.k()
                        mdist.merge_on_device(s, rows[:, :k].contiguous().view(torch.float64), rows[:, k:].contiguous())
                        st["running"] = _packed_front(s, device)
                    else:
                        st["running"] = mine
                    st["hv"] = s.archive_hypervolume(reference)
                    st["runs"] = run + 1
                    if trace is not None:
                        trace.append({"runs": run + 1, "samples": (run + 1) * samples_per_run,
                                      "archive": int(st["running"].shape[0]), "hv": st["hv"],
                                      "wall_s": time.perf_counter() - t0})
                    st["next"] = run + 1
                    if st["hv"] == hv_target:
                        st["done"] = True
                    cv.notify_all()
        except BaseException as ex:  # surface worker errors in the caller
            with cv:
                st["error"] = ex
                st["done"] = True
                cv.notify_all()

    threads = [threading.Thread(target=worker, args=(w,)) for w in range(S)]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    if st["error"] is not None:
        raise st["error"]
    torch.cuda.synchronize(device)
    return {"reached": st["hv"] == hv_target, "runs": st["runs"], "samples": st["runs"] * samples_per_run,
            "seconds": time.perf_counter() - t0, "hv": st["hv"],
            "archive": int(st["running"].shape[0]) if st["running"] is not None else 0}
