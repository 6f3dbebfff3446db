"""Host-side mirror of the reference's C++ interface for the hot path (proj/include/momc).

Same names, argument meaning and error behaviour as the reference, on top of the C-ABI
(include/momc_b200.h):

  reference (file:line)                              here
  MultiObjectiveInstance  instance.hpp:102-172      MultiObjectiveInstance
  load_instance / save_instance  instance.hpp:473-530  load_instance / save_instance
  WeightVector / das_dennis / interior_filter /
    resolution_for_interior_count  weights.hpp:26-117  same names
  SolverVariant / SolverConfig  solver.hpp:26-67    SolverVariant / SolverConfig
  SamplePool  solver.hpp:258-338                    SamplePool
  run_sampler  solver.hpp:439-529                   run_sampler (CUDA)

``std::invalid_argument`` maps to :class:`InvalidArgument` (a ValueError), any other
reference exception to :class:`MomcRuntimeError` (a RuntimeError).
"""
from __future__ import annotations

import ctypes as C
import enum
import math
import os
from dataclasses import dataclass, field

import numpy as np

from . import _lib


class InvalidArgument(ValueError):
    """std::invalid_argument in the reference (CLI exit code 2, cli.hpp:335-356)."""


class MomcRuntimeError(RuntimeError):
    """std::runtime_error in the reference (CLI exit code 1)."""


def _raise(code: int, err) -> None:
    if code == 0:
        return
    msg = err.value.decode(errors="replace") if hasattr(err, "value") else str(err)
    if code == 2:
        raise InvalidArgument(msg)
    raise MomcRuntimeError(msg)


def _errbuf():
    return C.create_string_buffer(2048)


# ----------------------------------------------------------------------------- instance
@dataclass
class Edge:
    """instance.hpp:24-28"""

    i: int
    j: int
    w: list


class MultiObjectiveInstance:
    """instance.hpp:102-172: one graph, K weight layers, validated on construction."""

    def __init__(self, n: int, k: int, edges):
        if n < 1:
            raise InvalidArgument("vertex count must be positive")
        if k < 1:
            raise InvalidArgument("objective count must be positive")
        ei, ej, w = [], [], []
        seen = set()
        for e in edges:
            i, j, ww = (e.i, e.j, e.w) if isinstance(e, Edge) else e
            if i == j:
                raise InvalidArgument("self-loop edge")
            if i < 0 or j < 0 or i >= n or j >= n or i >= j:
                raise InvalidArgument("edge endpoints must satisfy 0 <= i < j < n")
            if len(ww) != k:
                raise InvalidArgument("every edge must carry exactly K weights")
            if (i, j) in seen:
                raise InvalidArgument("duplicate edge")
            seen.add((i, j))
            ei.append(i)
            ej.append(j)
            w.append([float(x) for x in ww])
        self._n, self._k = int(n), int(k)
        self.edge_i = np.asarray(ei, dtype=np.int32)
        self.edge_j = np.asarray(ej, dtype=np.int32)
        self.weights = np.asarray(w, dtype=np.float64).reshape(len(ei), k)

    @classmethod
    def from_arrays(cls, n, k, edge_i, edge_j, w) -> "MultiObjectiveInstance":
        w = np.asarray(w, dtype=np.float64).reshape(-1, k)
        return cls(n, k, [(int(a), int(b), list(c)) for a, b, c in zip(edge_i, edge_j, w)])

    def n(self) -> int:
        return self._n

    def k(self) -> int:
        return self._k

    def num_edges(self) -> int:
        return int(self.edge_i.shape[0])

    def edges(self):
        return [Edge(int(a), int(b), list(c)) for a, b, c in zip(self.edge_i, self.edge_j, self.weights)]

    def layer_sum(self, layer: int) -> float:
        """instance.hpp:131-137 (edge order)."""
        if layer < 0 or layer >= self._k:
            raise InvalidArgument("layer out of range")
        s = 0.0
        for v in self.weights[:, layer].tolist():
            s += v
        return s

    def view(self):
        """momc_instance_view over this instance's arrays (keeps them alive via self)."""
        v = _lib.InstanceViewC()
        v.n, v.k, v.m = self._n, self._k, self.num_edges()
        self._keep = (np.ascontiguousarray(self.edge_i), np.ascontiguousarray(self.edge_j),
                      np.ascontiguousarray(self.weights))
        v.edge_i = self._keep[0].ctypes.data_as(_lib.i32p)
        v.edge_j = self._keep[1].ctypes.data_as(_lib.i32p)
        v.w = self._keep[2].ctypes.data_as(_lib.dp)
        return v

    def __eq__(self, other):
        return (isinstance(other, MultiObjectiveInstance) and self._n == other._n and self._k == other._k
                and np.array_equal(self.edge_i, other.edge_i) and np.array_equal(self.edge_j, other.edge_j)
                and np.array_equal(self.weights, other.weights))


def format_number(v: float) -> str:
    """instance.hpp:462-470: integers verbatim, reals as the shortest round-trip form."""
    if v == math.floor(v) and abs(v) < 1e15:
        return str(int(v))
    return repr(float(v))


def save_instance(inst: MultiObjectiveInstance, path) -> None:
    """instance.hpp:473-484 text format: header "n K m", then "i j w1 .. wK"."""
    with open(path, "w") as fh:
        fh.write(f"{inst.n()} {inst.k()} {inst.num_edges()}\n")
        for a, b, ws in zip(inst.edge_i.tolist(), inst.edge_j.tolist(), inst.weights.tolist()):
            fh.write(f"{a} {b} " + " ".join(format_number(x) for x in ws) + "\n")


def load_instance(path) -> MultiObjectiveInstance:
    """instance.hpp:486-530, with the reference's line-numbered messages."""
    path = str(path)
    try:
        fh = open(path)
    except OSError:
        raise MomcRuntimeError(f"cannot open {path}")

    def fail(line, msg):
        raise MomcRuntimeError(f"{path}:{line}: {msg}")

    with fh:
        text = fh.read()
    lines = text.split("\n")
    if text.endswith("\n"):
        lines = lines[:-1]  # std::getline reports EOF after a trailing newline
    if not lines:
        fail(1, "malformed header: empty file")
    head = lines[0].split()
    try:
        n, k, m = int(head[0]), int(head[1]), int(head[2])
    except (ValueError, IndexError):
        fail(1, "malformed header: expected 'n K m'")
    if n < 1 or k < 1 or m < 0:
        fail(1, "malformed header: expected 'n K m'")
    if len(head) > 3:
        fail(1, "malformed header: trailing tokens")
    ei, ej, ws = [], [], []
    seen = set()
    for e in range(m):
        ln = e + 2
        if e + 1 >= len(lines):
            fail(ln, "unexpected end of file")
        tok = lines[e + 1].split()
        try:
            i, j = int(tok[0]), int(tok[1])
        except (ValueError, IndexError):
            fail(ln, "malformed edge line")
        if i == j:
            fail(ln, "self-loop")
        if i < 0 or j < 0 or i >= n or j >= n:
            fail(ln, "vertex index out of range")
        if i > j:
            fail(ln, "edge endpoints must satisfy i < j")
        if (i, j) in seen:
            fail(ln, "duplicate edge")
        seen.add((i, j))
        if len(tok) < 2 + k:
            fail(ln, f"expected {k} weights")
        try:
            w = [float(x) for x in tok[2:2 + k]]
        except ValueError:
            fail(ln, f"expected {k} weights")
        if len(tok) > 2 + k:
            fail(ln, f"expected exactly {k} weights")
        ei.append(i)
        ej.append(j)
        ws.append(w)
    return MultiObjectiveInstance(n, k, list(zip(ei, ej, ws)))


# ----------------------------------------------------------------------------- weights
class WeightVector:
    """weights.hpp:26-70: numerators summing to the resolution H."""

    def __init__(self, numerators, resolution: int):
        if resolution < 1:
            raise InvalidArgument("lattice resolution must be positive")
        nums = [int(v) for v in numerators]
        if any(v < 0 for v in nums):
            raise InvalidArgument("weight numerators must be non-negative")
        if len(nums) < 1 or sum(nums) != resolution:
            raise InvalidArgument("weight numerators must sum to the resolution")
        self._num = nums
        self._h = int(resolution)

    def size(self):
        return len(self._num)

    def resolution(self):
        return self._h

    def numerator(self, k):
        return self._num[k]

    def __getitem__(self, k):
        return self._num[k] / self._h

    def components(self):
        return [v / self._h for v in self._num]

    def is_interior(self):
        return all(v != 0 for v in self._num)

    def __eq__(self, o):
        return isinstance(o, WeightVector) and self._num == o._num and self._h == o._h

    def __repr__(self):
        return f"WeightVector({self._num}, {self._h})"


def binomial(n: int, k: int) -> int:
    if k < 0 or k > n:
        return 0
    return math.comb(n, k)


def das_dennis(k: int, h: int):
    """weights.hpp:75-96: lex-descending lattice, |result| = C(H+K-1, K-1)."""
    if k < 2:
        raise InvalidArgument("lattice needs at least two objectives")
    if h < 1:
        raise InvalidArgument("lattice resolution must be positive")
    out = []
    num = [0] * k

    def rec(pos, rem):
        if pos == k - 1:
            num[pos] = rem
            out.append(WeightVector(list(num), h))
            return
        for v in range(rem, -1, -1):
            num[pos] = v
            rec(pos + 1, rem - v)

    rec(0, h)
    return out


def interior_filter(lattice):
    """weights.hpp:100-107"""
    return [w for w in lattice if w.is_interior()]


def resolution_for_interior_count(k: int, count: int) -> int:
    """weights.hpp:110-117"""
    if k < 2 or count < 1:
        raise InvalidArgument("need k >= 2 and count >= 1")
    for h in range(k, 100000):
        if binomial(h - 1, k - 1) >= count:
            return h
    raise InvalidArgument("requested interior count is out of range")


def build_weights(k: int, count: int = 55, resolution: int = 0):
    """pipeline.hpp:64-78 WeightSelection -> interior lattice."""
    h = resolution if resolution > 0 else resolution_for_interior_count(k, count)
    return interior_filter(das_dennis(k, h))


def _weights_array(weights, k):
    if len(weights) == 0:
        raise InvalidArgument("run_sampler needs at least one weight vector")
    H = weights[0].resolution()
    for w in weights:
        if w.size() != k:
            raise InvalidArgument("weight vector length does not match objective count")
        if w.resolution() != H:
            raise InvalidArgument("all weight vectors must share one resolution")
    nums = np.asarray([[w.numerator(q) for q in range(k)] for w in weights], dtype=np.int32)
    return nums, H


# ----------------------------------------------------------------------------- solver
class SolverVariant(enum.IntEnum):
    """solver.hpp:26"""

    ballistic_sb = 0
    discrete_sb = 1
    simcim = 2


def parse_variant(name: str) -> SolverVariant:
    """solver.hpp:38-44"""
    table = {"bsb": SolverVariant.ballistic_sb, "dsb": SolverVariant.discrete_sb, "simcim": SolverVariant.simcim}
    if name not in table:
        raise InvalidArgument("unknown solver variant: " + name)
    return table[name]


@dataclass
class SolverConfig:
    """solver.hpp:46-67 (defaults T=50, dt=1, a0=1, alpha=0.15, batch=3000, init_scale=0.1)."""

    variant: SolverVariant = SolverVariant.ballistic_sb
    n_iterations: int = 50
    dt: float = 1.0
    a0: float = 1.0
    alpha: float = 0.15
    batch_size: int = 3000
    init_scale: float = 0.1
    seed: int = 0
    threads: int = 1

    def validate(self):
        if self.n_iterations < 1:
            raise InvalidArgument("n_iterations must be >= 1")
        if not self.dt > 0.0:
            raise InvalidArgument("dt must be positive")
        if not self.a0 > 0.0:
            raise InvalidArgument("a0 must be positive")
        if self.alpha < 0.0:
            raise InvalidArgument("alpha must be non-negative")
        if self.batch_size < 1:
            raise InvalidArgument("batch_size must be >= 1")
        if self.init_scale < 0.0:
            raise InvalidArgument("init_scale must be non-negative")
        if self.threads < 0:
            raise InvalidArgument("threads must be non-negative")

    def c(self) -> _lib.SolverCfgC:
        v = parse_variant(self.variant) if isinstance(self.variant, str) else SolverVariant(self.variant)
        return _lib.SolverCfgC(int(v), self.n_iterations, self.dt, self.a0, self.alpha, self.batch_size,
                               self.init_scale, self.seed, self.threads)


def pump_schedule(t: int, total: int) -> float:
    """solver.hpp:70-76 (a0 is not applied)."""
    if total < 1 or t < 0 or t > total:
        raise InvalidArgument("pump schedule requires 0 <= t <= total")
    return t / total


@dataclass
class SampleRecord:
    """solver.hpp:246-253"""

    run: int
    weight: int
    trajectory: int
    timestamp_ns: int = 0


class SamplePool:
    """solver.hpp:258-338: packed spins in canonical (run, weight, trajectory) order."""

    def __init__(self, n: int, words=None, runs: int = 0, weights: int = 0, batch: int = 0, stamps=None):
        if n < 1:
            raise InvalidArgument("pool spin count must be positive")
        self._n = n
        wpc = (n + 63) // 64
        self.words = (np.zeros((0, wpc), np.uint64) if words is None
                      else np.ascontiguousarray(words, np.uint64).reshape(-1, wpc))
        self.runs, self.L, self.batch = runs, weights, batch
        self.stamps = stamps
        self.model_construction_seconds = 0.0
        self.sampling_seconds = 0.0

    def n(self):
        return self._n

    def size(self):
        return int(self.words.shape[0])

    def __len__(self):
        return self.size()

    def empty(self):
        return self.size() == 0

    def words_per_config(self):
        return (self._n + 63) // 64

    def record(self, i: int) -> SampleRecord:
        per_run = self.L * self.batch
        run, rem = divmod(i, per_run)
        l, t = divmod(rem, self.batch)
        ts = int(self.stamps[i]) if self.stamps is not None else 0
        return SampleRecord(run, l, t, ts)

    def config(self, i: int) -> np.ndarray:
        w = self.words[i]
        return np.array([1 if (int(w[b // 64]) >> (b % 64)) & 1 else -1 for b in range(self._n)], dtype=np.int8)

    def packed_words(self) -> np.ndarray:
        return self.words.reshape(-1)


def same_samples(a: SamplePool, b: SamplePool) -> bool:
    """solver.hpp:316-327"""
    return (a.n() == b.n() and a.size() == b.size() and (a.runs, a.L, a.batch) == (b.runs, b.L, b.batch)
            and np.array_equal(a.words, b.words))


# ----------------------------------------------------------------------------- device session
class Session:
    """One momc_ctx: a device, a stream and the resident instance / weights / pool."""

    def __init__(self, device: int = 0):
        self.lib = _lib.load()
        h = _lib.vp()
        err = _errbuf()
        _raise(self.lib.momc_b200_ctx_create(device, C.byref(h), err, 2048), err)
        self.h = h
        self.device = device
        self.inst = None

    def close(self):
        if getattr(self, "h", None):
            self.lib.momc_b200_ctx_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def launches(self) -> int:
        return int(self.lib.momc_b200_ctx_launches(self.h))

    def stream(self) -> int:
        return int(self.lib.momc_b200_ctx_stream(self.h) or 0)

    def sync(self):
        err = _errbuf()
        _raise(self.lib.momc_b200_ctx_sync(self.h, err, 2048), err)

    def set_instance(self, inst: MultiObjectiveInstance):
        err = _errbuf()
        v = inst.view()
        _raise(self.lib.momc_b200_set_instance(self.h, C.byref(v), err, 2048), err)
        self.inst = inst

    def set_weights(self, weights):
        nums, H = _weights_array(weights, self.inst.k())
        err = _errbuf()
        _raise(self.lib.momc_b200_set_weights(self.h, nums.ctypes.data_as(_lib.i32p), nums.shape[0], H, err, 2048),
               err)
        self.L = nums.shape[0]

    def coupling(self, l: int):
        n = self.inst.n()
        J = np.zeros((n, n), np.float64)
        c0 = C.c_double()
        err = _errbuf()
        _raise(self.lib.momc_b200_get_coupling(self.h, l, J.ctypes.data_as(_lib.dp), C.byref(c0), err, 2048), err)
        return J, c0.value

    def sample(self, config: SolverConfig, runs: int = 1, block_begin: int = 0, block_end: int = -1) -> float:
        config.validate()
        cfg = config.c()
        secs = np.zeros(1, np.float64)
        err = _errbuf()
        _raise(self.lib.momc_b200_sample(self.h, C.byref(cfg), runs, block_begin, block_end,
                                         secs.ctypes.data_as(_lib.dp), err, 2048), err)
        self._pool_geom = (runs, self.L, config.batch_size)
        return float(secs[0])

    def pool(self, stamps: bool = True) -> SamplePool:
        M = int(self.lib.momc_b200_pool_size(self.h))
        n = self.inst.n()
        wpc = (n + 63) // 64
        words = np.zeros((M, wpc), np.uint64)
        st = np.zeros(M, np.int64) if stamps else None
        err = _errbuf()
        _raise(self.lib.momc_b200_pool_get(self.h, words.ctypes.data_as(_lib.u64p),
                                           st.ctypes.data_as(_lib.i64p) if stamps else None, err, 2048), err)
        runs, L, batch = self._pool_geom
        return SamplePool(n, words, runs, L, batch, st)

    def pool_device_ptr(self) -> int:
        return int(self.lib.momc_b200_pool_device(self.h) or 0)


_default_session = None


def default_session() -> Session:
    global _default_session
    if _default_session is None:
        _default_session = Session(int(os.environ.get("MOMC_DEVICE", "0")))
    return _default_session


def run_sampler(inst: MultiObjectiveInstance, weights, config: SolverConfig, runs: int,
                session: Session | None = None) -> SamplePool:
    """solver.hpp:439-529 on the GPU; records keep canonical order, stamps per 128-chunk."""
    config.validate()
    if len(weights) == 0:
        raise InvalidArgument("run_sampler needs at least one weight vector")
    if runs < 1:
        raise InvalidArgument("runs must be >= 1")
    s = session or default_session()
    nums, H = _weights_array(weights, inst.k())
    L = nums.shape[0]
    M = runs * L * config.batch_size
    wpc = (inst.n() + 63) // 64
    words = np.zeros((M, wpc), np.uint64)
    stamps = np.zeros(M, np.int64)
    secs = np.zeros(2, np.float64)
    cfg = config.c()
    v = inst.view()
    err = _errbuf()
    rc = s.lib.momc_b200_run_sampler(s.h, C.byref(v), nums.ctypes.data_as(_lib.i32p), L, H, C.byref(cfg), runs,
                                     words.ctypes.data_as(_lib.u64p), stamps.ctypes.data_as(_lib.i64p),
                                     secs.ctypes.data_as(_lib.dp), err, 2048)
    _raise(rc, err)
    s.inst = inst
    s.L = L
    s._pool_geom = (runs, L, config.batch_size)
    pool = SamplePool(inst.n(), words, runs, L, config.batch_size, stamps)
    pool.model_construction_seconds = float(secs[0])
    pool.sampling_seconds = float(secs[1])
    return pool
