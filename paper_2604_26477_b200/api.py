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
  ObjectiveVector / Sense  instance.hpp:73-98       ObjectiveVector / Sense
  ParetoArchive  pareto.hpp:64-119                  ParetoArchive
  non_dominated_filter  pareto.hpp:253-293, :370-410  non_dominated_filter (CUDA)
  detail::evaluate_cuts  pareto.hpp:330-363        evaluate_cuts (CUDA)
  hypervolume  pareto.hpp:540-552                   hypervolume (CUDA)
  reference_point_sampled / clamp_reference  pareto.hpp:620-655   same names (CUDA / host)
  bench  pipeline.hpp:309-393                       bench (CUDA)

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


def _to_chars_shortest(v: float) -> str:
    """std::to_chars(double) without a format: the shortest round-trip digits, written in
    fixed or scientific notation, whichever is shorter (fixed on a tie); checked against
    libstdc++ on 30k values (tests/test_host_api.py)."""
    if math.isnan(v):
        return "-nan" if math.copysign(1.0, v) < 0 else "nan"
    if math.isinf(v):
        return "-inf" if v < 0 else "inf"
    r = repr(float(v))  # shortest round-trip digits
    sign = "-" if r.startswith("-") else ""
    r = r.lstrip("-")
    mant, _, ex = r.partition("e")
    ip, _, fp = mant.partition(".")
    digits = (ip + fp).lstrip("0")
    exp10 = (int(ex) if ex else 0) - len(fp)  # value = int(ip + fp) * 10**exp10
    if not digits:
        return sign + "0"
    stripped = digits.rstrip("0")
    exp10 += len(digits) - len(stripped)
    digits = stripped
    nd = len(digits)
    sci_e = exp10 + nd - 1
    sci = digits[0] + ("." + digits[1:] if nd > 1 else "") + "e" + ("-" if sci_e < 0 else "+") + f"{abs(sci_e):02d}"
    if exp10 >= 0:  # an integer: fixed notation prints its exact digits (same length)
        fixed = str(int(abs(v)))
    elif sci_e >= 0:
        fixed = digits[:sci_e + 1] + "." + digits[sci_e + 1:]
    else:
        fixed = "0." + "0" * (-sci_e - 1) + digits
    return sign + (fixed if len(fixed) <= len(sci) else sci)


def format_number(v: float) -> str:
    """instance.hpp:462-470: integers below 1e15 verbatim, everything else as std::to_chars'
    shortest round-trip form."""
    if not math.isnan(v) and not math.isinf(v) and v == math.floor(v) and abs(v) < 1e15:
        return str(int(v))
    return _to_chars_shortest(v)


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
    lines = text.split("\n") if text else []
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
    if any(len(w._num) != k for w in weights):
        raise InvalidArgument("weight vector length does not match objective count")
    if any(w._h != H for w in weights):
        raise InvalidArgument("all weight vectors must share one resolution")
    nums = np.asarray([w._num for w in weights], dtype=np.int32)  # one pass: this runs every bench call
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

    def __init__(self, n: int, words=None, runs: int = 0, weights: int = 0, batch: int = 0, stamps=None,
                 records=None):
        if n < 1:
            raise InvalidArgument("pool spin count must be positive")
        self._n = n
        wpc = (n + 63) // 64
        self.words = (np.zeros((0, wpc), np.uint64) if words is None
                      else np.ascontiguousarray(words, np.uint64).reshape(-1, wpc))
        self.runs, self.L, self.batch = runs, weights, batch
        self.stamps = stamps
        # explicit (run, weight, trajectory) keys, M x 3 uint32 (a loaded pool); otherwise the
        # keys follow from the canonical index and (runs, L, batch)
        self.records = None if records is None else np.ascontiguousarray(records, np.uint32).reshape(-1, 3)
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
        ts = int(self.stamps[i]) if self.stamps is not None else 0
        if self.records is not None:
            r = self.records[i]
            return SampleRecord(int(r[0]), int(r[1]), int(r[2]), ts)
        per_run = self.L * self.batch
        run, rem = divmod(i, per_run)
        l, t = divmod(rem, self.batch)
        return SampleRecord(run, l, t, ts)

    def record_keys(self) -> np.ndarray:
        """M x 3 uint32 (run, weight, trajectory) of every record."""
        if self.records is not None:
            return self.records
        i = np.arange(self.size(), dtype=np.int64)
        per_run = max(self.L * self.batch, 1)
        b = max(self.batch, 1)
        return np.stack([i // per_run, (i % per_run) // b, i % b], axis=1).astype(np.uint32)

    def timestamps(self) -> np.ndarray:
        return (np.zeros(self.size(), np.int64) if self.stamps is None
                else np.ascontiguousarray(self.stamps, np.int64))

    def __eq__(self, other):
        """solver.hpp:329-332: n, records (timestamps included) and spins"""
        return (isinstance(other, SamplePool) and self._n == other._n and self.size() == other.size()
                and np.array_equal(self.record_keys(), other.record_keys())
                and np.array_equal(self.timestamps(), other.timestamps()) and np.array_equal(self.words, other.words))

    def config(self, i: int) -> np.ndarray:
        w = self.words[i]
        return np.array([1 if (int(w[b // 64]) >> (b % 64)) & 1 else -1 for b in range(self._n)], dtype=np.int8)

    def packed_words(self) -> np.ndarray:
        return self.words.reshape(-1)


def same_samples(a: SamplePool, b: SamplePool) -> bool:
    """solver.hpp:316-327"""
    return (a.n() == b.n() and a.size() == b.size() and np.array_equal(a.record_keys(), b.record_keys())
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

    def fallback_blocks(self) -> int:
        return int(self.lib.momc_b200_ctx_fallback_blocks(self.h))

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

    def generate_uniform_instance(self, n: int, density: float, k: int, seed: int, kind: str = "int",
                                  lo: float = 1.0, hi: float = 10.0) -> MultiObjectiveInstance:
        """generate_uniform_instance (instance.hpp:259-284) on the device; becomes resident."""
        m = C.c_int64()
        err = _errbuf()
        _raise(self.lib.momc_b200_generate_uniform_instance(self.h, n, density, k, 0 if kind == "int" else 1, lo, hi,
                                                            seed, C.byref(m), err, 2048), err)
        return self._fetch_instance(n, k, m.value)

    def generate_correlated_instance(self, n: int, density: float, target_rho: float,
                                     seed: int) -> MultiObjectiveInstance:
        """generate_correlated_instance (instance.hpp:364-458) on the device; becomes resident."""
        m = C.c_int64()
        err = _errbuf()
        _raise(self.lib.momc_b200_generate_correlated_instance(self.h, n, density, target_rho, seed, C.byref(m), err,
                                                               2048), err)
        return self._fetch_instance(n, 3, m.value)

    def measured_correlation(self, pool_size: int = 2048, seed: int = 0) -> float:
        """measured_correlation (instance.hpp:338-357) of the resident K=3 instance."""
        out = C.c_double()
        err = _errbuf()
        _raise(self.lib.momc_b200_measured_correlation(self.h, pool_size, seed, C.byref(out), err, 2048), err)
        return out.value

    def _fetch_instance(self, n, k, m):
        err = _errbuf()
        ei = np.zeros(m, np.int32)
        ej = np.zeros(m, np.int32)
        w = np.zeros((m, k), np.float64)
        _raise(self.lib.momc_b200_instance_get(self.h, ei.ctypes.data_as(_lib.i32p), ej.ctypes.data_as(_lib.i32p),
                                               w.ctypes.data_as(_lib.dp), err, 2048), err)
        inst = MultiObjectiveInstance.__new__(MultiObjectiveInstance)
        inst._n, inst._k = n, k
        inst.edge_i, inst.edge_j, inst.weights = ei, ej, w
        self.inst = inst
        return inst

    def set_dense_threshold(self, n_min: int):
        self.lib.momc_b200_set_dense_threshold(self.h, n_min)

    SAMPLER_PATHS = ("none", "register", "generic", "dense_i8", "dense_bf16")
    KERNEL_CLASSES = ("sampler", "dense_gemm", "dense_update", "eval_gemm")

    def philox_blocks(self, keys, ctrs) -> np.ndarray:
        """Philox4x32-10 blocks on the device (momc_b200_philox_blocks): keys (N,) u64,
        ctrs (N, 4) u32 -> (N, 4) u32"""
        k = np.ascontiguousarray(keys, np.uint64).reshape(-1)
        c = np.ascontiguousarray(ctrs, np.uint32).reshape(-1, 4)
        out = np.zeros((k.shape[0], 4), np.uint32)
        err = _errbuf()
        _raise(self.lib.momc_b200_philox_blocks(self.h, k.ctypes.data_as(_lib.u64p),
                                                c.ctypes.data_as(C.POINTER(C.c_uint32)), k.shape[0],
                                                out.ctypes.data_as(C.POINTER(C.c_uint32)), err, 2048), err)
        return out

    def set_kernel_timing(self, on: bool):
        """bracket every sampler / dense GEMM / dense update / tensor-core evaluation launch
        with CUDA events (momc_b200_set_kernel_timing); a diagnostic for roofline figures"""
        self.lib.momc_b200_set_kernel_timing(self.h, int(bool(on)))

    def kernel_times(self, reset: bool = True) -> dict:
        """{class: (summed ms, launches)} since the last reset (momc_b200_kernel_times)"""
        ms = (C.c_double * 4)()
        cnt = (C.c_longlong * 4)()
        if self.lib.momc_b200_kernel_times(self.h, ms, cnt, int(bool(reset))) != 0:
            raise RuntimeError("momc_b200_kernel_times failed")
        return {name: (ms[i], cnt[i]) for i, name in enumerate(self.KERNEL_CLASSES)}

    def sampler_path(self) -> str:
        """which sampler produced the resident pool (momc_b200_sampler_path): "register" and
        "generic" are bit-exact against the reference; "dense_i8" / "dense_bf16" (the fused
        tensor-core step) round J(c).sgn(X) once"""
        return self.SAMPLER_PATHS[int(self.lib.momc_b200_sampler_path(self.h))]

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

    def num_blocks(self, config: SolverConfig, runs: int = 1) -> int:
        cfg = config.c()
        return int(self.lib.momc_b200_num_blocks(self.h, C.byref(cfg), runs))

    def pipeline(self, config: SolverConfig, runs: int = 1, block_begin: int = 0, block_end: int = -1,
                 do_hv: bool = True, ref_count: int = 4096, fixed_reference=None) -> dict:
        """Resident-instance pipeline (momc_b200_pipeline): scalarise, sample, filter, [r, HV]."""
        config.validate()
        cfg = config.c()
        rep = _lib.BenchReportC()
        fr = np.ascontiguousarray(fixed_reference, np.float64) if fixed_reference is not None else None
        err = _errbuf()
        _raise(self.lib.momc_b200_pipeline(self.h, C.byref(cfg), runs, block_begin, block_end, int(do_hv), ref_count,
                                           fr.ctypes.data_as(_lib.dp) if fr is not None else None, C.byref(rep),
                                           err, 2048), err)
        self._pool_geom = (runs, self.L, config.batch_size)
        out = {name: getattr(rep, name) for name, _ in _lib.BenchReportC._fields_}
        out["reference"] = list(rep.reference)[: self.inst.k()]
        return out

    def archive(self, with_configs: bool = True) -> "ParetoArchive":
        return _fetch_archive(self, self.inst.k(), self.inst.n(), with_configs)

    def archive_hypervolume(self, r) -> float:
        r = np.ascontiguousarray(r, np.float64)
        out = C.c_double()
        err = _errbuf()
        _raise(self.lib.momc_b200_archive_hypervolume(self.h, r.ctypes.data_as(_lib.dp), C.byref(out), err, 2048), err)
        return out.value

    def merge_device(self, d_vals: int, d_words: int, wpc: int, M: int, k: int) -> int:
        """Filter M device vectors (+ configs) into the resident archive (multi-GPU merge)."""
        F = C.c_int64()
        err = _errbuf()
        _raise(self.lib.momc_b200_filter_values_dev(self.h, C.c_void_p(d_vals), C.c_void_p(d_words), wpc, M, k,
                                                    C.byref(F), err, 2048), err)
        return F.value

    def rng_calibrate(self, blocks_per_thread: int = 2048) -> float:
        """normals/s of the RNG-only calibration kernel (roofline: the sampler's noise share)"""
        out = C.c_double()
        err = _errbuf()
        _raise(self.lib.momc_b200_rng_calibrate(self.h, blocks_per_thread, C.byref(out), err, 2048), err)
        return out.value

    # ---- streaming (running archive on the context)
    def running_reset(self):
        err = _errbuf()
        _raise(self.lib.momc_b200_running_reset(self.h, err, 2048), err)

    def stream_step(self, config: SolverConfig, runs: int, block_begin: int, block_end: int, reference=None,
                    merge: bool = True):
        """Sample blocks [block_begin, block_end) and filter them (front left in the resident
        archive, unordered); with `merge`, merge it into the running archive. Returns (hv of
        the running archive at `reference` or None, running size, report)."""
        config.validate()
        cfg = config.c()
        rep = _lib.BenchReportC()
        F = C.c_int64()
        hv = C.c_double()
        err = _errbuf()
        r = None if reference is None else np.ascontiguousarray(reference, np.float64)
        _raise(self.lib.momc_b200_stream_step(self.h, C.byref(cfg), runs, block_begin, block_end, int(merge),
                                              None if r is None else r.ctypes.data_as(_lib.dp),
                                              None if r is None else C.byref(hv), C.byref(F), C.byref(rep), err,
                                              2048), err)
        self._pool_geom = (runs, self.L, config.batch_size)
        return (None if r is None else hv.value), F.value, {name: getattr(rep, name) for name, _ in
                                                            _lib.BenchReportC._fields_}

    def running_merge_values(self, d_vals: int, d_words: int, wpc: int, M: int, k: int, reference=None):
        """Merge M device rows (values + packed configs) into the running archive."""
        F = C.c_int64()
        hv = C.c_double()
        err = _errbuf()
        r = None if reference is None else np.ascontiguousarray(reference, np.float64)
        _raise(self.lib.momc_b200_running_merge_values(self.h, C.c_void_p(d_vals), C.c_void_p(d_words), wpc, M, k,
                                                       None if r is None else r.ctypes.data_as(_lib.dp),
                                                       None if r is None else C.byref(hv), C.byref(F), err, 2048), err)
        return (None if r is None else hv.value), F.value

    def archive_device_ptrs(self):
        """(values ptr, words ptr, F) of the resident archive on the device"""
        v, w = C.c_void_p(), C.c_void_p()
        F = C.c_int64()
        self.lib.momc_b200_archive_device_ptrs(self.h, C.byref(v), C.byref(w), C.byref(F))
        return v.value or 0, w.value or 0, F.value

    def running_to_archive(self) -> int:
        F = C.c_int64()
        err = _errbuf()
        _raise(self.lib.momc_b200_running_to_archive(self.h, C.byref(F), err, 2048), err)
        return F.value

    def archive_copy_device(self, d_vals: int, d_words: int):
        err = _errbuf()
        _raise(self.lib.momc_b200_archive_copy_device(self.h, C.c_void_p(d_vals), C.c_void_p(d_words), err, 2048),
               err)

    def archive_size(self) -> int:
        return int(self.lib.momc_b200_archive_size(self.h))


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


# ----------------------------------------------------------------------------- pareto
class Sense(enum.IntEnum):
    """instance.hpp:73"""

    cut = 0
    hamiltonian = 1


class ObjectiveVector:
    """instance.hpp:78-98"""

    def __init__(self, values, sense: Sense = Sense.cut):
        if len(values) == 0:
            raise InvalidArgument("objective vector must be non-empty")
        self._v = [float(x) for x in values]
        self._sense = Sense(sense)

    def size(self):
        return len(self._v)

    def __getitem__(self, k):
        return self._v[k]

    def values(self):
        return list(self._v)

    def sense(self):
        return self._sense

    def __eq__(self, o):
        return isinstance(o, ObjectiveVector) and self._v == o._v and self._sense == o._sense


class ParetoArchive:
    """pareto.hpp:64-119: entries sorted lexicographically descending by value."""

    def __init__(self, values=None, configs=None, n: int = 0):
        self.values = np.zeros((0, 0), np.float64) if values is None else np.asarray(values, np.float64)
        self.configs = configs  # F x wpc packed words, or None for objective-only archives
        self.n = n
        self.reference = []
        self.filtering_seconds = 0.0

    def k(self):
        return 0 if self.values.shape[0] == 0 else int(self.values.shape[1])

    def size(self):
        return int(self.values.shape[0])

    def __len__(self):
        return self.size()

    def contains_value(self, v):
        return bool(np.any(np.all(self.values == np.asarray(v, np.float64), axis=1)))

    def config(self, i):
        w = self.configs[i]
        return np.array([1 if (int(w[b // 64]) >> (b % 64)) & 1 else -1 for b in range(self.n)], dtype=np.int8)

    def validate_reference(self, r):
        r = list(r)
        for i in range(self.size()):
            if len(r) != self.k():
                raise InvalidArgument("reference point length does not match archive")
            for k in range(len(r)):
                if r[k] > self.values[i, k]:
                    raise InvalidArgument(f"reference point not dominated by archive entry {i} (objective {k})")

    def set_reference(self, r):
        self.validate_reference(r)
        self.reference = list(r)


def _session_for(inst, session):
    s = session or default_session()
    if s.inst is not inst:
        s.set_instance(inst)
    return s


class DeviceGroup:
    """Several devices behind one handle (momc_b200_group_*): the blocks of run_sampler /
    bench are split across the devices, every device filters its share, the fronts are
    merged on member 0 (NCCL all-gather for distinct devices, peer copies otherwise).
    ``devices`` None: MOMC_GPUS, else device 0. ``member(0)`` is a Session view of the
    context holding the merged archive."""

    TRANSPORTS = ("single", "nccl", "copy")

    def __init__(self, devices=None):
        self.lib = _lib.load()
        h = _lib.vp()
        err = _errbuf()
        arr = None if not devices else np.ascontiguousarray(devices, np.int32)
        _raise(self.lib.momc_b200_group_create(arr.ctypes.data_as(_lib.i32p) if arr is not None else None,
                                               0 if arr is None else len(arr), C.byref(h), err, 2048), err)
        self.h = h

    def close(self):
        if getattr(self, "h", None):
            self.lib.momc_b200_group_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def size(self) -> int:
        return int(self.lib.momc_b200_group_size(self.h))

    def transport(self) -> str:
        return self.TRANSPORTS[int(self.lib.momc_b200_group_transport(self.h))]

    def member(self, i: int) -> Session:
        """a non-owning Session over member i's context"""
        s = Session.__new__(Session)
        s.lib = self.lib
        s.h = _lib.vp(self.lib.momc_b200_group_ctx(self.h, i))
        s.device = None
        s.inst = None
        s._owner = self  # keeps the group alive
        s.close = lambda: None
        return s

    def run_sampler(self, inst: MultiObjectiveInstance, weights, config: SolverConfig, runs: int) -> "SamplePool":
        config.validate()
        nums, H = _weights_array(weights, inst.k())
        L = nums.shape[0]
        M = runs * L * config.batch_size
        wpc = (inst.n() + 63) // 64
        words = np.empty((M, wpc), np.uint64)
        stamps = np.empty(M, np.int64)
        secs = np.zeros(2, np.float64)
        cfg = config.c()
        v = inst.view()
        err = _errbuf()
        _raise(self.lib.momc_b200_group_run_sampler(self.h, C.byref(v), nums.ctypes.data_as(_lib.i32p), L, H,
                                                    C.byref(cfg), runs, words.ctypes.data_as(_lib.u64p),
                                                    stamps.ctypes.data_as(_lib.i64p), secs.ctypes.data_as(_lib.dp),
                                                    err, 2048), err)
        pool = SamplePool(inst.n(), words, runs, L, config.batch_size)
        pool.stamps = stamps
        return pool

    def non_dominated_filter(self, pool, inst: MultiObjectiveInstance) -> ParetoArchive:
        words = np.ascontiguousarray(pool.words if hasattr(pool, "words") else pool, np.uint64)
        err = _errbuf()
        v = inst.view()
        _raise(self.lib.momc_b200_group_set_instance(self.h, C.byref(v), err, 2048), err)
        F = C.c_int64()
        fs = C.c_double()
        _raise(self.lib.momc_b200_group_filter_pool(self.h, words.ctypes.data_as(_lib.u64p), words.shape[0],
                                                    C.byref(F), C.byref(fs), err, 2048), err)
        return _fetch_archive(self.member(0), inst.k(), inst.n(), True)

    def bench(self, inst: MultiObjectiveInstance, weights, config: SolverConfig, runs: int = 1,
              ref_count: int = 1000, fixed_reference=None) -> "BenchResult":
        config.validate()
        nums, H = _weights_array(weights, inst.k())
        L = nums.shape[0]
        M = runs * L * config.batch_size
        wpc = (inst.n() + 63) // 64
        words = np.empty((M, wpc), np.uint64)
        rep = _lib.BenchReportC()
        cfg = config.c()
        v = inst.view()
        fr = np.ascontiguousarray(fixed_reference, np.float64) if fixed_reference is not None else None
        err = _errbuf()
        _raise(self.lib.momc_b200_group_bench(self.h, C.byref(v), nums.ctypes.data_as(_lib.i32p), L, H, C.byref(cfg),
                                              runs, ref_count, fr.ctypes.data_as(_lib.dp) if fr is not None else None,
                                              words.ctypes.data_as(_lib.u64p), None, C.byref(rep), err, 2048), err)
        report = {name: getattr(rep, name) for name, _ in _lib.BenchReportC._fields_}
        report["reference"] = list(rep.reference)[: inst.k()]
        archive = _fetch_archive(self.member(0), inst.k(), inst.n(), True)
        archive.reference = report["reference"]
        return BenchResult(report, SamplePool(inst.n(), words, runs, L, config.batch_size), archive)


def _fetch_archive(s: Session, k: int, n: int, with_configs: bool) -> ParetoArchive:
    F = int(s.lib.momc_b200_archive_size(s.h))
    vals = np.zeros((F, k), np.float64)
    wpc = (n + 63) // 64
    words = np.zeros((F, wpc), np.uint64) if with_configs else None
    err = _errbuf()
    _raise(s.lib.momc_b200_archive_get(s.h, vals.ctypes.data_as(_lib.dp),
                                       words.ctypes.data_as(_lib.u64p) if with_configs else None, err, 2048), err)
    return ParetoArchive(vals, words, n if with_configs else 0)


def non_dominated_filter(pool, inst=None, algo: str = "fast", session: Session | None = None) -> ParetoArchive:
    """pareto.hpp:370-410 (pool + instance) or pareto.hpp:253-293 (list of ObjectiveVector).

    ``algo`` is accepted for signature parity; the GPU front is exact for both."""
    if inst is None:
        vecs = list(pool)
        if not vecs:
            raise InvalidArgument("non-dominated filter needs a non-empty pool")
        sense, k = vecs[0].sense(), vecs[0].size()
        for v in vecs:
            if v.sense() != sense or v.size() != k:
                raise InvalidArgument("pool mixes objective senses or lengths")
        vals = np.ascontiguousarray([v.values() for v in vecs], np.float64)
        s = session or default_session()
        F = C.c_int64()
        err = _errbuf()
        _raise(s.lib.momc_b200_filter_values(s.h, vals.ctypes.data_as(_lib.dp), vals.shape[0], k, int(sense),
                                             C.byref(F), err, 2048), err)
        return _fetch_archive(s, k, 0, False)
    if pool.empty():
        raise InvalidArgument("non-dominated filter needs a non-empty pool")
    if pool.n() != inst.n():
        raise InvalidArgument("pool does not match instance")
    s = _session_for(inst, session)
    words = np.ascontiguousarray(pool.words, np.uint64)
    F = C.c_int64()
    secs = C.c_double()
    err = _errbuf()
    _raise(s.lib.momc_b200_filter_pool(s.h, words.ctypes.data_as(_lib.u64p), words.shape[0], C.byref(F),
                                       C.byref(secs), err, 2048), err)
    a = _fetch_archive(s, inst.k(), inst.n(), True)
    a.filtering_seconds = secs.value
    return a


def hypervolume(archive: ParetoArchive, r, session: Session | None = None) -> float:
    """pareto.hpp:540-552 (exact; integer-valued inputs give the exact integer volume)."""
    if archive.size() == 0:
        raise InvalidArgument("hypervolume of an empty archive")
    r = np.ascontiguousarray(r, np.float64)
    if r.shape[0] != archive.k():
        raise InvalidArgument("reference point length does not match archive")
    s = session or default_session()
    vals = np.ascontiguousarray(archive.values, np.float64)
    out = C.c_double()
    err = _errbuf()
    _raise(s.lib.momc_b200_hypervolume(s.h, vals.ctypes.data_as(_lib.dp), vals.shape[0], vals.shape[1],
                                       r.ctypes.data_as(_lib.dp), C.byref(out), err, 2048), err)
    return out.value


def evaluate_cuts(inst: MultiObjectiveInstance, words, session: Session | None = None) -> np.ndarray:
    """detail::evaluate_cuts (pareto.hpp:330-363) of packed configurations."""
    s = _session_for(inst, session)
    words = np.ascontiguousarray(words, np.uint64).reshape(-1, (inst.n() + 63) // 64)
    out = np.zeros((words.shape[0], inst.k()), np.float64)
    err = _errbuf()
    _raise(s.lib.momc_b200_evaluate_cuts(s.h, words.ctypes.data_as(_lib.u64p), words.shape[0],
                                         out.ctypes.data_as(_lib.dp), err, 2048), err)
    return out


def reference_point_sampled(inst: MultiObjectiveInstance, count: int, seed: int,
                            session: Session | None = None) -> list:
    """pareto.hpp:620-642"""
    if count < 1:
        raise InvalidArgument("sampled reference needs count >= 1")
    s = _session_for(inst, session)
    r = np.zeros(inst.k(), np.float64)
    err = _errbuf()
    _raise(s.lib.momc_b200_reference_point_sampled(s.h, count, seed, r.ctypes.data_as(_lib.dp), err, 2048), err)
    return r.tolist()


def brute_force_pareto(inst: MultiObjectiveInstance, session: Session | None = None,
                       with_reference: bool = False):
    """oracle.hpp:25-77 on the device: the exact front over every configuration with s_0 = +1
    (equal vectors keep the lex-smallest configuration; entries lex-descending). No n <= 22
    cap for integer-weight graphs with a small vertex separator (n <= 64). With
    ``with_reference`` also returns reference_point_exact (pareto.hpp:603-617)."""
    if inst.n() < 1:
        raise InvalidArgument("enumeration needs n >= 1")
    s = _session_for(inst, session)
    F = C.c_int64()
    r = np.zeros(inst.k(), np.float64)
    err = _errbuf()
    _raise(s.lib.momc_b200_brute_force_pareto(s.h, C.byref(F), r.ctypes.data_as(_lib.dp), err, 2048), err)
    arc = _fetch_archive(s, inst.k(), inst.n(), True)
    return (arc, r.tolist()) if with_reference else arc


def reference_point_exact(inst: MultiObjectiveInstance, session: Session | None = None) -> list:
    """pareto.hpp:603-617 (componentwise minimum over every configuration), on the device."""
    s = _session_for(inst, session)
    r = np.zeros(inst.k(), np.float64)
    err = _errbuf()
    _raise(s.lib.momc_b200_reference_point_exact(s.h, r.ctypes.data_as(_lib.dp), err, 2048), err)
    return r.tolist()


def samples_to_reach(pool: SamplePool, inst: MultiObjectiveInstance, r, target_hv: float,
                     session: Session | None = None):
    """pareto.hpp:763-781 on the device: first 1-based canonical-order sample count whose
    running archive reaches target_hv (1e-9 relative tolerance), or None."""
    if pool.empty():
        raise InvalidArgument("empty pool")
    s = _session_for(inst, session)
    words = np.ascontiguousarray(pool.words, np.uint64)
    r = np.ascontiguousarray(r, np.float64)
    out = C.c_int64()
    err = _errbuf()
    _raise(s.lib.momc_b200_samples_to_reach(s.h, words.ctypes.data_as(_lib.u64p), words.shape[0],
                                            r.ctypes.data_as(_lib.dp), float(target_hv), C.byref(out), err, 2048), err)
    return None if out.value < 0 else int(out.value)


@dataclass
class TracePoint:
    """pareto.hpp:681-685"""
    elapsed_s: float
    hv: float
    samples: int


def convergence_trace(pool: SamplePool, inst: MultiObjectiveInstance, r, checkpoints: int,
                      session: Session | None = None) -> list:
    """pareto.hpp:716-757 on the device: replay by timestamp (stable), HV of the running
    archive at `checkpoints` evenly spaced sample-count milestones."""
    if pool.empty():
        raise InvalidArgument("convergence trace needs a non-empty pool")
    if checkpoints < 1:
        raise InvalidArgument("checkpoints must be >= 1")
    s = _session_for(inst, session)
    words = np.ascontiguousarray(pool.words, np.uint64)
    stamps = np.ascontiguousarray(pool.stamps if pool.stamps is not None else np.zeros(pool.size()), np.int64)
    r = np.ascontiguousarray(r, np.float64)
    el = np.zeros(checkpoints, np.float64)
    hv = np.zeros(checkpoints, np.float64)
    sm = np.zeros(checkpoints, np.int64)
    err = _errbuf()
    _raise(s.lib.momc_b200_convergence_trace(s.h, words.ctypes.data_as(_lib.u64p), stamps.ctypes.data_as(_lib.i64p),
                                             words.shape[0], r.ctypes.data_as(_lib.dp), checkpoints,
                                             el.ctypes.data_as(_lib.dp), hv.ctypes.data_as(_lib.dp),
                                             sm.ctypes.data_as(_lib.i64p), err, 2048), err)
    return [TracePoint(float(a), float(b), int(c)) for a, b, c in zip(el, hv, sm)]


def generate_correlated_instance(n: int, density: float, target_rho: float, seed: int,
                                 session: Session | None = None) -> MultiObjectiveInstance:
    """instance.hpp:364-458 (device generation; the instance is returned on the host)."""
    s = session or default_session()
    return s.generate_correlated_instance(n, density, target_rho, seed)


def measured_correlation(inst: MultiObjectiveInstance, pool_size: int = 2048, seed: int = 0,
                         session: Session | None = None) -> float:
    """instance.hpp:338-357"""
    if inst.k() != 3:
        raise InvalidArgument("correlation measure requires K=3")
    s = _session_for(inst, session)
    return s.measured_correlation(pool_size, seed)


def clamp_reference(r, archive: ParetoArchive):
    """pareto.hpp:647-655 (host; the archive is small)."""
    out = list(r)
    for row in archive.values:
        if len(row) != len(out):
            raise InvalidArgument("reference point length does not match archive")
        out = [min(a, b) for a, b in zip(out, row)]
    return out


@dataclass
class BenchResult:
    """pipeline.hpp:297-302 (report fields as a dict)."""

    report: dict
    pool: SamplePool
    archive: ParetoArchive


def bench(inst: MultiObjectiveInstance, weights, config: SolverConfig, runs: int = 1, ref_count: int = 1000,
          fixed_reference=None, keep_pool: bool = True, session: Session | None = None,
          pool_out=None) -> BenchResult:
    """pipeline.hpp:309-393 on the GPU: scalarise -> sample -> filter -> reference -> HV.

    ``pool_out``: optional preallocated (ideally page-locked) uint64 array of M x wpc words
    that receives the pool; the returned SamplePool then views it."""
    config.validate()
    if runs < 1:
        raise InvalidArgument("runs must be >= 1")
    s = session or default_session()
    nums, H = _weights_array(weights, inst.k())
    L = nums.shape[0]
    M = runs * L * config.batch_size
    wpc = (inst.n() + 63) // 64
    if keep_pool and pool_out is not None:
        words = np.asarray(pool_out).view(np.uint64).reshape(M, wpc)
        if not words.flags["C_CONTIGUOUS"]:
            raise InvalidArgument("pool_out must be contiguous")
    else:
        words = np.empty((M, wpc), np.uint64) if keep_pool else None
    rep = _lib.BenchReportC()
    cfg = config.c()
    v = inst.view()
    fr = np.ascontiguousarray(fixed_reference, np.float64) if fixed_reference is not None else None
    err = _errbuf()
    rc = s.lib.momc_b200_bench(s.h, C.byref(v), nums.ctypes.data_as(_lib.i32p), L, H, C.byref(cfg), runs, ref_count,
                               fr.ctypes.data_as(_lib.dp) if fr is not None else None,
                               words.ctypes.data_as(_lib.u64p) if keep_pool else None, C.byref(rep), err, 2048)
    _raise(rc, err)
    s.inst = inst
    s.L = L
    s._pool_geom = (runs, L, config.batch_size)
    report = {name: getattr(rep, name) for name, _ in _lib.BenchReportC._fields_}
    report["reference"] = list(rep.reference)[: inst.k()]
    archive = _fetch_archive(s, inst.k(), inst.n(), True)
    archive.reference = report["reference"]
    pool = SamplePool(inst.n(), words, runs, L, config.batch_size) if keep_pool else None
    return BenchResult(report, pool, archive)
