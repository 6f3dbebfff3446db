"""The multi-rank bench path (shard runs, all-gather fronts, merge, streaming
time-to-optimal) run as 2 ranks on the one GPU of this box over gloo: a functional check of
the N>1 code path only (no timing is taken from it; the ranks' kernels never wait on each
other, they only meet in the host collectives)."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_bench_two_ranks_functional():
    env = dict(os.environ, MOMC_BENCH_DEVICE="0", MOMC_DIST_BACKEND="gloo")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", "29531", os.path.join(ROOT, "bench.py"), "--gpus", "2",
           "--steps", "1", "--warmup", "3", "--no-cpu-baseline"]
    out = subprocess.run(cmd, capture_output=True, text=True, env=env, timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, out.stdout[-2000:]
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["config"]["runs"] == 2
    assert d["config"]["samples_per_step"] == 2 * 1000120
    # two runs merged over the ranks: the archive grows past the single run's 9,821 points
    assert d["archive_size"] > 9821
    tto = d["time_to_optimal"]
    assert tto["k4"]["reached"] and tto["k4"]["hv"] == tto["k4"]["hv_star"]
    assert tto["k3"]["reached"] and tto["k3"]["runs"] % 2 == 0
    # e2e through the public API with host buffers on every rank (not a copy of the device time)
    e = d["e2e"]
    assert e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] >= 1000120 * 8
    assert e["value"] > 0 and e["ms_per_step"] != d["ms_per_step"]
