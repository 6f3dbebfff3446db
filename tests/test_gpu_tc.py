"""Hand-written tcgen05 int8 blocks (csrc/tc_i8.cuh) against a host int32 reference."""
import ctypes as C

import numpy as np
import pytest

from paper_2604_26477_b200 import api

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("K,seed", [(128, 1), (256, 2), (2048, 3)])
def test_tc_i8_gemm_exact(session, K, seed):
    rng = np.random.default_rng(seed)
    A = rng.integers(-127, 128, size=(128, K), dtype=np.int8)
    B = rng.integers(-127, 128, size=(128, K), dtype=np.int8)
    D = np.zeros((128, 128), np.int32)
    err = C.create_string_buffer(2048)
    rc = session.lib.momc_b200_tc_i8_selftest(session.h, A.ctypes.data, B.ctypes.data, K, D.ctypes.data, err, 2048)
    assert rc == 0, err.value
    want = A.astype(np.int64) @ B.astype(np.int64).T
    assert np.array_equal(D.astype(np.int64), want)


def test_rng_calibration_rate(session):
    """calib.cu: the noise-only microkernel behind roofline.rng_calibration runs and reports
    a rate in a plausible band for one B200 (measured 1.0e12 normals/s)"""
    nps = session.rng_calibrate(256)
    assert 1e11 < nps < 1e13
