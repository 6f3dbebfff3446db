"""Synthetic instances of the BASELINE configs, written in the reference
text format (instance.hpp:473-484) so both the reference and this package read them
through load_instance.

* 42-node heavy-hex (C1-C3, C5): 3 rows x 12-node chains + 6 bridge nodes (cols 0,4,8
  between rows 0-1; cols 2,6,10 between rows 1-2): 42 nodes / 45 edges, max degree 3.
  Integer weights U{-10..10} per layer from Stream(derive_key(seed, 0x68687878), i, j,
  tag_word(edge_weight)) drawn with WeightSpec::uniform_int (instance.hpp:230-235).
  Mixed sign is required: heavy-hex is bipartite, so all-positive weights give a 1-point
  front.

The host-side Philox here is only for generating these small inputs; the sampler's RNG
runs on the device (csrc/rng.cuh).
"""
from __future__ import annotations

import os

from .api import MultiObjectiveInstance, load_instance, save_instance

M64 = (1 << 64) - 1
HEAVY_HEX_CONTEXT = 0x68687878
TAG_EDGE_WEIGHT = 5


def _mix64(z: int) -> int:
    z ^= z >> 30
    z = (z * 0xBF58476D1CE4E5B9) & M64
    z ^= z >> 27
    z = (z * 0x94D049BB133111EB) & M64
    z ^= z >> 31
    return z


def derive_key(seed: int, ctx: int) -> int:
    """rng.hpp:54-57"""
    return _mix64((seed + 0x9E3779B97F4A7C15) & M64) ^ _mix64((ctx * 0x9E3779B97F4A7C15 + 1) & M64)


def philox(key: int, ctr):
    """rng.hpp:22-38"""
    c0, c1, c2, c3 = ctr
    k0, k1 = key & 0xFFFFFFFF, key >> 32
    for _ in range(10):
        p0 = 0xD2511F53 * c0
        p1 = 0xCD9E8D57 * c2
        c0, c1, c2, c3 = ((p1 >> 32) ^ c1 ^ k0) & 0xFFFFFFFF, p1 & 0xFFFFFFFF, ((p0 >> 32) ^ c3 ^ k1) & 0xFFFFFFFF, \
            p0 & 0xFFFFFFFF
        k0 = (k0 + 0x9E3779B9) & 0xFFFFFFFF
        k1 = (k1 + 0xBB67AE85) & 0xFFFFFFFF
    return [c0, c1, c2, c3]


class Stream:
    """rng.hpp:105-192 (u32/u64/below only)."""

    def __init__(self, key, id_hi, id_mid, id_lo):
        self.key = key
        self.ctr = [0, id_lo, id_mid, id_hi]
        self.buf = []

    def next_u32(self):
        if not self.buf:
            self.buf = philox(self.key, self.ctr)
            self.ctr[0] += 1
        return self.buf.pop(0)

    def next_u64(self):
        lo = self.next_u32()
        hi = self.next_u32()
        return lo | (hi << 32)

    def next_below(self, bound):
        return (self.next_u64() * bound) >> 64


def tag_word(tag: int, step: int = 0) -> int:
    return (tag << 26) | (step & 0x03FFFFFF)


def heavy_hex_edges():
    """The 42-node / 45-edge heavy-hex graph, edges (i<j) sorted by (i, j)."""
    edges = []
    for r in range(3):
        for c in range(11):
            edges.append((12 * r + c, 12 * r + c + 1))
    for b, c in zip((36, 37, 38), (0, 4, 8)):
        edges.append((c, b))
        edges.append((12 + c, b))
    for b, c in zip((39, 40, 41), (2, 6, 10)):
        edges.append((12 + c, b))
        edges.append((24 + c, b))
    return sorted((min(a, b), max(a, b)) for a, b in edges)


def heavy_hex_instance(k: int, seed: int = 7, lo: int = -10, hi: int = 10) -> MultiObjectiveInstance:
    key = derive_key(seed, HEAVY_HEX_CONTEXT)
    span = hi - lo + 1
    out = []
    for i, j in heavy_hex_edges():
        s = Stream(key, i, j, tag_word(TAG_EDGE_WEIGHT))
        out.append((i, j, [float(lo + s.next_below(span)) for _ in range(k)]))
    return MultiObjectiveInstance(42, k, out)


DATA = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "data")


def heavy_hex_path(k: int) -> str:
    return os.path.join(DATA, f"heavyhex42_k{k}_seed7.txt")


def ensure_heavy_hex(k: int) -> str:
    path = heavy_hex_path(k)
    if not os.path.exists(path):
        os.makedirs(DATA, exist_ok=True)
        save_instance(heavy_hex_instance(k), path)
    return path


def load_heavy_hex(k: int) -> MultiObjectiveInstance:
    return load_instance(ensure_heavy_hex(k))
