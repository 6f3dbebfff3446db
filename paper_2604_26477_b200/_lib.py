"""ctypes loader of the in-tree CUDA library (libmomc_b200.so) and its C-ABI signatures.

There is no CPU fallback: importing the product API without the built library, or
creating a context without a B200, raises.
"""
from __future__ import annotations

import ctypes as C
import os

PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(PKG, "libmomc_b200.so")

u32p = C.POINTER(C.c_uint32)
u64p = C.POINTER(C.c_uint64)
i64p = C.POINTER(C.c_int64)
i32p = C.POINTER(C.c_int32)
dp = C.POINTER(C.c_double)
vp = C.c_void_p


class SolverCfgC(C.Structure):
    """momc_solver_cfg (include/momc_b200.h) == momc::SolverConfig (solver.hpp:46-67)."""

    _fields_ = [
        ("variant", C.c_int),
        ("n_iterations", C.c_int),
        ("dt", C.c_double),
        ("a0", C.c_double),
        ("alpha", C.c_double),
        ("batch_size", C.c_int),
        ("init_scale", C.c_double),
        ("seed", C.c_uint64),
        ("threads", C.c_int),
    ]


class BenchReportC(C.Structure):
    """momc_bench_report (include/momc_b200.h)."""

    _fields_ = [
        ("model_construction_s", C.c_double),
        ("sampling_s", C.c_double),
        ("pareto_filtering_s", C.c_double),
        ("end_to_end_s", C.c_double),
        ("pool_size", C.c_int64),
        ("unique_configs", C.c_int64),
        ("unique_vectors", C.c_int64),
        ("archive_size", C.c_int64),
        ("hv", C.c_double),
        ("reference", C.c_double * 16),
        ("dedup_s", C.c_double),
        ("eval_s", C.c_double),
        ("collapse_s", C.c_double),
        ("front_s", C.c_double),
        ("order_s", C.c_double),
        ("reference_s", C.c_double),
        ("hv_s", C.c_double),
        ("front_method", C.c_int),
        ("sampler_path", C.c_int),
    ]


class InstanceViewC(C.Structure):
    """momc_instance_view (include/momc_b200.h)."""

    _fields_ = [
        ("n", C.c_int),
        ("k", C.c_int),
        ("m", C.c_int),
        ("edge_i", i32p),
        ("edge_j", i32p),
        ("w", dp),
    ]


# (name, restype, argtypes) for every symbol declared in include/momc_b200.h
SIGNATURES = [
    ("momc_b200_ctx_create", C.c_int, [C.c_int, C.POINTER(vp), C.c_char_p, C.c_size_t]),
    ("momc_b200_ctx_destroy", None, [vp]),
    ("momc_b200_ctx_sync", C.c_int, [vp, C.c_char_p, C.c_size_t]),
    ("momc_b200_ctx_stream", vp, [vp]),
    ("momc_b200_ctx_launches", C.c_longlong, [vp]),
    ("momc_b200_ctx_fallback_blocks", C.c_longlong, [vp]),
    ("momc_b200_set_instance", C.c_int, [vp, C.POINTER(InstanceViewC), C.c_char_p, C.c_size_t]),
    ("momc_b200_generate_uniform_instance", C.c_int, [vp, C.c_int, C.c_double, C.c_int, C.c_int, C.c_double,
                                                      C.c_double, C.c_uint64, i64p, C.c_char_p, C.c_size_t]),
    ("momc_b200_instance_get", C.c_int, [vp, i32p, i32p, dp, C.c_char_p, C.c_size_t]),
    ("momc_b200_set_dense_threshold", C.c_int, [vp, C.c_int]),
    ("momc_b200_sampler_path", C.c_int, [vp]),
    ("momc_b200_set_kernel_timing", C.c_int, [vp, C.c_int]),
    ("momc_b200_philox_blocks", C.c_int, [vp, u64p, C.POINTER(C.c_uint32), C.c_size_t, C.POINTER(C.c_uint32),
                                          C.c_char_p, C.c_size_t]),
    ("momc_b200_group_create", C.c_int, [i32p, C.c_int, C.POINTER(vp), C.c_char_p, C.c_size_t]),
    ("momc_b200_group_destroy", None, [vp]),
    ("momc_b200_group_size", C.c_int, [vp]),
    ("momc_b200_group_ctx", vp, [vp, C.c_int]),
    ("momc_b200_group_transport", C.c_int, [vp]),
    ("momc_b200_group_set_instance", C.c_int, [vp, C.POINTER(InstanceViewC), C.c_char_p, C.c_size_t]),
    ("momc_b200_group_set_weights", C.c_int, [vp, i32p, C.c_int, C.c_int, C.c_char_p, C.c_size_t]),
    ("momc_b200_group_run_sampler", C.c_int, [vp, C.POINTER(InstanceViewC), i32p, C.c_int, C.c_int,
                                              C.POINTER(SolverCfgC), C.c_int, u64p, i64p, dp, C.c_char_p, C.c_size_t]),
    ("momc_b200_group_filter_pool", C.c_int, [vp, u64p, C.c_size_t, i64p, dp, C.c_char_p, C.c_size_t]),
    ("momc_b200_group_bench", C.c_int, [vp, C.POINTER(InstanceViewC), i32p, C.c_int, C.c_int, C.POINTER(SolverCfgC),
                                        C.c_int, C.c_int, dp, u64p, i64p, C.POINTER(BenchReportC), C.c_char_p,
                                        C.c_size_t]),
    ("momc_b200_kernel_times", C.c_int, [vp, dp, C.POINTER(C.c_longlong), C.c_int]),
    ("momc_b200_set_weights", C.c_int, [vp, i32p, C.c_int, C.c_int, C.c_char_p, C.c_size_t]),
    ("momc_b200_get_coupling", C.c_int, [vp, C.c_int, dp, dp, C.c_char_p, C.c_size_t]),
    ("momc_b200_sample", C.c_int, [vp, C.POINTER(SolverCfgC), C.c_int, C.c_longlong, C.c_longlong, dp,
                                   C.c_char_p, C.c_size_t]),
    ("momc_b200_pool_size", C.c_longlong, [vp]),
    ("momc_b200_pool_get", C.c_int, [vp, u64p, i64p, C.c_char_p, C.c_size_t]),
    ("momc_b200_pool_device", vp, [vp]),
    ("momc_b200_run_sampler", C.c_int, [vp, C.POINTER(InstanceViewC), i32p, C.c_int, C.c_int,
                                        C.POINTER(SolverCfgC), C.c_int, u64p, i64p, dp, C.c_char_p, C.c_size_t]),
    ("momc_b200_filter", C.c_int, [vp, i64p, dp, C.c_char_p, C.c_size_t]),
    ("momc_b200_filter_pool", C.c_int, [vp, u64p, C.c_size_t, i64p, dp, C.c_char_p, C.c_size_t]),
    ("momc_b200_filter_values", C.c_int, [vp, dp, C.c_size_t, C.c_int, C.c_int, i64p, C.c_char_p, C.c_size_t]),
    ("momc_b200_filter_values_dev", C.c_int, [vp, vp, vp, C.c_int, C.c_size_t, C.c_int, i64p, C.c_char_p,
                                              C.c_size_t]),
    ("momc_b200_archive_size", C.c_int64, [vp]),
    ("momc_b200_archive_get", C.c_int, [vp, dp, u64p, C.c_char_p, C.c_size_t]),
    ("momc_b200_archive_copy_device", C.c_int, [vp, vp, vp, C.c_char_p, C.c_size_t]),
    ("momc_b200_hypervolume", C.c_int, [vp, dp, C.c_int64, C.c_int, dp, dp, C.c_char_p, C.c_size_t]),
    ("momc_b200_archive_hypervolume", C.c_int, [vp, dp, dp, C.c_char_p, C.c_size_t]),
    ("momc_b200_evaluate_cuts", C.c_int, [vp, u64p, C.c_size_t, dp, C.c_char_p, C.c_size_t]),
    ("momc_b200_reference_point_sampled", C.c_int, [vp, C.c_int, C.c_uint64, dp, C.c_char_p, C.c_size_t]),
    ("momc_b200_clamp_reference", C.c_int, [vp, dp, C.c_char_p, C.c_size_t]),
    ("momc_b200_brute_force_pareto", C.c_int, [vp, C.POINTER(C.c_int64), dp, C.c_char_p, C.c_size_t]),
    ("momc_b200_reference_point_exact", C.c_int, [vp, dp, C.c_char_p, C.c_size_t]),
    ("momc_b200_generate_correlated_instance", C.c_int, [vp, C.c_int, C.c_double, C.c_double, C.c_uint64, i64p,
                                                         C.c_char_p, C.c_size_t]),
    ("momc_b200_measured_correlation", C.c_int, [vp, C.c_int, C.c_uint64, dp, C.c_char_p, C.c_size_t]),
    ("momc_b200_tc_i8_selftest", C.c_int, [vp, C.c_void_p, C.c_void_p, C.c_int, C.c_void_p, C.c_char_p, C.c_size_t]),
    ("momc_b200_rng_calibrate", C.c_int, [vp, C.c_int, dp, C.c_char_p, C.c_size_t]),
    ("momc_b200_running_reset", C.c_int, [vp, C.c_char_p, C.c_size_t]),
    ("momc_b200_stream_step", C.c_int, [vp, C.POINTER(SolverCfgC), C.c_int, C.c_longlong, C.c_longlong, C.c_int, dp,
                                        dp, i64p, C.POINTER(BenchReportC), C.c_char_p, C.c_size_t]),
    ("momc_b200_archive_device_ptrs", C.c_int, [vp, C.POINTER(C.c_void_p), C.POINTER(C.c_void_p), i64p]),
    ("momc_b200_running_merge_values", C.c_int, [vp, C.c_void_p, C.c_void_p, C.c_int, C.c_size_t, C.c_int, dp, dp,
                                                 i64p, C.c_char_p, C.c_size_t]),
    ("momc_b200_running_to_archive", C.c_int, [vp, i64p, C.c_char_p, C.c_size_t]),
    ("momc_b200_format_pool_rows", C.c_int, [vp, u32p, u32p, u32p, i64p, u64p, C.c_size_t, C.c_int, C.c_char_p,
                                             C.c_size_t, C.POINTER(C.c_size_t), C.c_char_p, C.c_size_t]),
    ("momc_b200_parse_pool_rows", C.c_int, [vp, C.c_char_p, C.c_size_t, C.c_int, C.c_int, C.c_char_p,
                                            C.POINTER(C.c_size_t), C.c_char_p, C.c_size_t]),
    ("momc_b200_parsed_pool_get", C.c_int, [vp, u32p, u32p, u32p, i64p, u64p, C.c_char_p, C.c_size_t]),
    ("momc_b200_samples_to_reach", C.c_int, [vp, u64p, C.c_size_t, dp, C.c_double, C.POINTER(C.c_int64),
                                             C.c_char_p, C.c_size_t]),
    ("momc_b200_convergence_trace", C.c_int, [vp, u64p, C.POINTER(C.c_int64), C.c_size_t, dp, C.c_int, dp, dp,
                                              C.POINTER(C.c_int64), C.c_char_p, C.c_size_t]),
    ("momc_b200_bench", C.c_int, [vp, C.POINTER(InstanceViewC), i32p, C.c_int, C.c_int, C.POINTER(SolverCfgC),
                                  C.c_int, C.c_int, dp, u64p, C.POINTER(BenchReportC), C.c_char_p, C.c_size_t]),
    ("momc_b200_pipeline", C.c_int, [vp, C.POINTER(SolverCfgC), C.c_int, C.c_longlong, C.c_longlong, C.c_int,
                                     C.c_int, dp, C.POINTER(BenchReportC), C.c_char_p, C.c_size_t]),
    ("momc_b200_num_blocks", C.c_longlong, [vp, C.POINTER(SolverCfgC), C.c_int]),
]

_lib = None


def load():
    """Load libmomc_b200.so (raises if it has not been built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} not built: run `python -c 'import __graft_entry__ as g; g.build()'` "
                          "(the momc_b200 path has no CPU fallback)")
    lib = C.CDLL(LIB_PATH)
    for name, res, args in SIGNATURES:
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib
