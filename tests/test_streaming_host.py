"""Host logic of streaming.time_to_target (no GPU): the reference's stopping rule
(samples_to_reach, pareto.hpp:771-779: hv >= target - 1e-9 max(1, |target|)) and the run
accounting when max_runs is not a multiple of world x runs_per_step."""
import pytest
import torch

from paper_2604_26477_b200 import streaming


class _Inst:
    def k(self):
        return 3

    def n(self):
        return 10


class FakeSession:
    """stream_step's contract: sample runs' blocks [b0, b1) and return (hv, F, report);
    here hv grows by one per run sampled."""

    def __init__(self):
        self.inst = _Inst()
        self.L = 5
        self.calls = []
        self.total_runs = 0

    def num_blocks(self, cfg, runs):
        return 2 * runs

    def running_reset(self):
        self.total_runs = 0

    def running_to_archive(self):
        pass

    def stream_step(self, cfg, runs, b0, b1, reference, merge=True):
        assert b1 > b0 and b1 <= self.num_blocks(cfg, runs)
        self.calls.append((runs, b0, b1))
        self.total_runs += (b1 - b0) // 2
        return float(self.total_runs), 1, {}


class Cfg:
    batch_size = 7


@pytest.fixture(autouse=True)
def _no_cuda_sync(monkeypatch):
    monkeypatch.setattr(torch.cuda, "synchronize", lambda *a, **k: None)


def test_reached_rule():
    assert streaming._reached(10.0, 10.0)
    assert streaming._reached(11.0, 10.0)  # passed between checks
    assert streaming._reached(1e12 - 1e-4, 1e12)  # within 1e-9 relative
    assert not streaming._reached(9.99, 10.0)
    assert not streaming._reached(1e30, None)
    assert not streaming._reached(1e30, float("inf"))


def test_stops_when_target_passed():
    s = FakeSession()
    res = streaming.time_to_target(s, Cfg(), [0, 0, 0], 4.5, 100, device="cpu", runs_per_step=2)
    # checks at 2, 4, 6 runs: 6 >= 4.5 stops (the old equality rule ran all 100)
    assert res["reached"] and res["runs"] == 6 and res["samples"] == 6 * 5 * 7


def test_no_target_spends_max_runs_exactly():
    s = FakeSession()
    res = streaming.time_to_target(s, Cfg(), [0, 0, 0], None, 7, device="cpu", runs_per_step=3)
    assert not res["reached"]
    assert res["runs"] == 7 and s.total_runs == 7
    assert s.calls[-1] == (7, 12, 14)  # the last round samples only run 6
