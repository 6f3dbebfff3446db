"""C++ drop-in parity on the GPU: tests/cpp/dropin_test.cpp runs the reference (CPU, shim
build) and momc::b200 (CUDA) through the same C++ signatures and compares pools
(same_samples), archives (values + configs), reference points, cut values and HV."""
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "tests", "cpp", "_bin", "dropin_test")


def test_cpp_dropin_matches_reference():
    if not os.path.exists(BIN):
        pytest.skip("dropin_test not built (tests/cpp/build_dropin.sh needs /root/reference)")
    res = subprocess.run([BIN, os.path.join(ROOT, "data", "heavyhex42_k4_seed7.txt")], capture_output=True, text=True,
                         timeout=600, cwd=ROOT)
    print(res.stdout, res.stderr)
    assert res.returncode == 0 and "PASSED" in res.stdout
