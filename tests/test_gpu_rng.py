"""Device Philox4x32-10 against the reference's published known-answer vectors
(proj/tests/test_rng.cpp:14-27) and against the package's host restatement on random
counters; the routine is the one every sampler kernel calls (csrc/rng.cuh)."""
import numpy as np
import pytest

from paper_2604_26477_b200 import api
from paper_2604_26477_b200.instances import philox

pytestmark = pytest.mark.gpu

KAT = [  # test_rng.cpp:17-26
    (0, (0, 0, 0, 0), (0x6627E8D5, 0xE169C58D, 0xBC57AC4C, 0x9B00DBD8)),
    (0xFFFFFFFFFFFFFFFF, (0xFFFFFFFF,) * 4, (0x408F276D, 0x41C83B0E, 0xA20BC7C6, 0x6D5451FD)),
    (0xA4093822 | (0x299F31D0 << 32), (0x243F6A88, 0x85A308D3, 0x13198A2E, 0x03707344),
     (0xD16CFE09, 0x94FDCCEB, 0x5001E420, 0x24126EA1)),
]


def test_device_philox_known_answers():
    s = api.Session(0)
    out = s.philox_blocks([k for k, _, _ in KAT], [c for _, c, _ in KAT])
    for (k, c, want), got in zip(KAT, out):
        assert tuple(int(x) for x in got) == want, (hex(k), c)


def test_device_philox_matches_host_restatement():
    rng = np.random.default_rng(3)
    keys = rng.integers(0, 2**63, 257, dtype=np.uint64) * np.uint64(2) + rng.integers(0, 2, 257, dtype=np.uint64)
    ctrs = rng.integers(0, 2**32, (257, 4), dtype=np.uint64).astype(np.uint32)
    got = api.Session(0).philox_blocks(keys, ctrs)
    for i in range(257):
        assert tuple(int(x) for x in got[i]) == tuple(philox(int(keys[i]), [int(x) for x in ctrs[i]])), i
