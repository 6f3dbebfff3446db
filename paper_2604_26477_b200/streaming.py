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


def _reached(hv: float, hv_target) -> bool:
    """samples_to_reach's stopping rule (pareto.hpp:771-779): hv >= target - 1e-9 max(1, |target|).
    hv_target None (or +inf) never stops: the stream spends max_runs."""
    if hv_target is None or hv_target == float("inf"):
        return False
    return hv >= hv_target - 1e-9 * max(1.0, abs(hv_target))


def _packed_front(session, device):
    """resident archive -> one int64 tensor [F, K + wpc] (values as bit patterns)"""
    vals, words = mdist.local_archive_tensors(session, device)
    return torch.cat([vals.view(torch.int64), words], dim=1)


def time_to_target(session, cfg, reference, hv_target, max_runs: int, world: int = 1, rank: int = 0,
                   device=None, trace: list | None = None, runs_per_step: int = 1) -> dict:
    """Runs rounds until the running archive's HV at `reference` reaches `hv_target` (the
    reference's tolerance, `_reached`; None = never) or `max_runs` runs are spent. Returns the number of
    runs / samples used, the wall time (device-synchronised, this rank) and the final HV.
    The caller times the whole call as the end-to-end figure (model build included: the
    weight blocks are scalarised once, on the first round, pipeline.hpp:337-341; later rounds
    reuse the resident J(c)). The last round samples only the runs left below max_runs.

    One GPU: one C-ABI call per run (momc_b200_stream_step: sample -> front -> merge into the
    context's running archive -> HV). N ranks: each rank's run front is all-gathered (NCCL)
    and merged into every rank's running archive (momc_b200_running_merge_values).
    `runs_per_step` runs are sampled per call (one launch, one merge, one HV check), so the
    check happens every runs_per_step x world runs."""
    device = device or torch.device("cuda", torch.cuda.current_device())
    k = session.inst.k()
    per_run = session.num_blocks(cfg, 1)
    samples_per_run = session.L * cfg.batch_size
    session.running_reset()
    hv, F, runs_done = 0.0, 0, 0
    t0 = time.perf_counter()
    R = max(1, int(runs_per_step))
    rounds = (max_runs + world * R - 1) // (world * R)
    for q in range(rounds):
        # round q covers runs [q*world*R, min((q+1)*world*R, max_runs)); rank r takes its R-slice
        lo, hi = q * world * R, min((q + 1) * world * R, max_runs)
        run = min(lo + rank * R, hi)  # this rank's first run of the round
        run_end = min(run + R, hi)
        if world == 1:
            hv, F, _ = session.stream_step(cfg, run_end, run * per_run, run_end * per_run, reference)
        else:
            if run_end > run:
                session.stream_step(cfg, run_end, run * per_run, run_end * per_run, None, merge=False)
                front = _packed_front(session, device)
            else:  # the last round left this rank no run: contribute an empty front
                front = torch.empty((0, k + (session.inst.n() + 63) // 64), dtype=torch.int64, device=device)
            rows = mdist.allgather_rows(front)
            vals = rows[:, :k].contiguous().view(torch.float64)
            words = rows[:, k:].contiguous()
            torch.cuda.current_stream(device).synchronize()
            hv, F = session.running_merge_values(vals.data_ptr(), words.data_ptr(), words.shape[1], vals.shape[0], k,
                                                 reference)
        runs_done = hi
        if trace is not None:
            trace.append({"runs": runs_done, "samples": runs_done * samples_per_run, "archive": F, "hv": hv,
                          "wall_s": time.perf_counter() - t0})
        if _reached(hv, hv_target):
            break
    torch.cuda.synchronize(device)
    session.running_to_archive()
    return {"reached": _reached(hv, hv_target), "runs": runs_done, "samples": runs_done * samples_per_run,
            "seconds": time.perf_counter() - t0, "hv": hv, "archive": F}


def time_to_target_overlapped(sessions: list, merger, cfg, reference, hv_target, max_runs: int,
                              trace: list | None = None, runs_per_step: int = 1) -> dict:
    """One GPU, several sampling contexts in host threads plus one merging context: run r is
    sampled and filtered by sessions[r % S] (the register sampler on its low-priority stream)
    while earlier runs' fronts are merged into `merger`'s running archive on its own stream.
    Merges happen strictly in run order, so runs / samples / archive / HV equal the sequential
    stream's; only the wall time differs. Step k samples runs [k R, (k+1) R) (R = runs_per_step)
    in one launch on sessions[k % S] and is merged (one merge, one HV check) after step k - 1."""
    import threading

    S = len(sessions)
    k = sessions[0].inst.k()
    wpc = (sessions[0].inst.n() + 63) // 64
    per_run = sessions[0].num_blocks(cfg, 1)
    samples_per_run = sessions[0].L * cfg.batch_size
    merger.running_reset()
    st = {"next": 0, "hv": 0.0, "F": 0, "done": False, "runs": 0, "error": None}
    cv = threading.Condition()
    t0 = time.perf_counter()

    R = max(1, int(runs_per_step))
    steps = (max_runs + R - 1) // R

    def worker(w):
        s = sessions[w]
        try:
            for step in range(w, steps, S):
                with cv:
                    if st["done"]:
                        return
                run, run_end = step * R, min((step + 1) * R, max_runs)
                s.stream_step(cfg, run_end, run * per_run, run_end * per_run, None, merge=False)
                with cv:
                    while st["next"] != step and not st["done"]:
                        cv.wait()
                    if st["done"]:
                        return
                    v, wd, F = s.archive_device_ptrs()
                    st["hv"], st["F"] = merger.running_merge_values(v, wd, wpc, F, k, reference)
                    st["runs"] = run_end
                    if trace is not None:
                        trace.append({"runs": run_end, "samples": run_end * samples_per_run, "archive": st["F"],
                                      "hv": st["hv"], "wall_s": time.perf_counter() - t0})
                    st["next"] = step + 1
                    if _reached(st["hv"], hv_target):
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
    merger.running_to_archive()
    return {"reached": _reached(st["hv"], hv_target), "runs": st["runs"], "samples": st["runs"] * samples_per_run,
            "seconds": time.perf_counter() - t0, "hv": st["hv"], "archive": st["F"]}
