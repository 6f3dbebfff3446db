"""The C-ABI library loads and exports every symbol include/momc_b200.h declares (CPU only:
no compute calls)."""
import ctypes
import os
import re

import pytest

from paper_2604_26477_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    text = open(os.path.join(ROOT, "include", "momc_b200.h")).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(momc_b200_\w+)\s*\(", text)))


def test_header_declares_the_api():
    syms = declared_symbols()
    for must in ("momc_b200_ctx_create", "momc_b200_run_sampler", "momc_b200_filter_pool", "momc_b200_hypervolume",
                 "momc_b200_bench", "momc_b200_evaluate_cuts", "momc_b200_reference_point_sampled"):
        assert must in syms


def test_library_exports_every_declared_symbol():
    if not os.path.exists(_lib.LIB_PATH):
        pytest.skip("libmomc_b200.so not built (run __graft_entry__.build())")
    lib = ctypes.CDLL(_lib.LIB_PATH)
    missing = [s for s in declared_symbols() if not hasattr(lib, s)]
    assert not missing, missing


def test_binding_covers_header():
    bound = {name for name, _, _ in _lib.SIGNATURES}
    assert set(declared_symbols()) <= bound


def test_cpp_dropin_header_present():
    hpp = os.path.join(ROOT, "include", "momc_b200", "momc_b200.hpp")
    assert os.path.exists(hpp)
    text = open(hpp).read()
    for fn in ("run_sampler", "non_dominated_filter", "hypervolume", "evaluate_cuts", "reference_point_sampled"):
        assert fn in text
