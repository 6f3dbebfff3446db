"""The package's host Philox restatement (instances.philox, used for host-side instance
generation and the smoke check) against the reference's known-answer vectors
(proj/tests/test_rng.cpp:14-27). CPU only."""
from paper_2604_26477_b200.instances import philox


def test_host_philox_known_answers():
    assert philox(0, [0, 0, 0, 0]) == [0x6627E8D5, 0xE169C58D, 0xBC57AC4C, 0x9B00DBD8]
    assert philox(0xFFFFFFFFFFFFFFFF, [0xFFFFFFFF] * 4) == [0x408F276D, 0x41C83B0E, 0xA20BC7C6, 0x6D5451FD]
    assert philox(0xA4093822 | (0x299F31D0 << 32), [0x243F6A88, 0x85A308D3, 0x13198A2E, 0x03707344]) == \
        [0xD16CFE09, 0x94FDCCEB, 0x5001E420, 0x24126EA1]
