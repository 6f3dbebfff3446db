"""ctypes binding of the CPU checker libraries — TEST INFRASTRUCTURE ONLY.

``oracle/_ref/libmomc_ref.so`` is the UNMODIFIED reference (``/root/reference/proj/include``)
compiled against ``oracle/eigen_shim`` by ``oracle/build_ref.sh``; ``RefLib`` wraps its
C-ABI (``oracle/ref_capi.cpp``). Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s reference / cpu_baseline legs may import this module; the product
package never does.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF_SO = os.path.join(HERE, "_ref", "libmomc_ref.so")

_u32p = C.POINTER(C.c_uint32)
_u64p = C.POINTER(C.c_uint64)
_i64p = C.POINTER(C.c_int64)
_ip = C.POINTER(C.c_int)
_dp = C.POINTER(C.c_double)


class CfgC(C.Structure):
    """Mirror of ``momc::SolverConfig`` (solver.hpp:46) as passed across the C-ABI."""

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


VARIANTS = {"bsb": 0, "dsb": 1, "simcim": 2}


def make_cfg(variant="bsb", n_iterations=50, dt=1.0, a0=1.0, alpha=0.15, batch_size=3000,
             init_scale=0.1, seed=0, threads=1) -> CfgC:
    v = VARIANTS[variant] if isinstance(variant, str) else int(variant)
    return CfgC(v, n_iterations, dt, a0, alpha, batch_size, init_scale, seed, threads)


def _p(a, t):
    return a.ctypes.data_as(t)


class RefError(Exception):
    def __init__(self, code, msg):
        super().__init__(msg)
        self.code = code


@dataclass
class RefArchive:
    values: np.ndarray  # F x K float64, lexicographically descending
    words: np.ndarray  # F x wpc uint64 (empty for objective-only archives)
    filtering_seconds: float


class RefLib:
    """The reference compiled with the shim (cpu_baseline kind "reference")."""

    def __init__(self, path: str = REF_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing: run oracle/build_ref.sh (needs /root/reference)")
        L = self.lib = C.CDLL(path)
        L.momcref_philox.argtypes = [C.c_uint64, _u32p, _u32p]
        L.momcref_derive_key.restype = C.c_uint64
        L.momcref_derive_key.argtypes = [C.c_uint64, C.c_uint64]
        L.momcref_run_key.restype = C.c_uint64
        L.momcref_run_key.argtypes = [C.c_uint64, C.c_uint32]
        L.momcref_tag_word.restype = C.c_uint32
        L.momcref_tag_word.argtypes = [C.c_uint32, C.c_uint32]
        for nm in ("momcref_stream_u32",):
            getattr(L, nm).argtypes = [C.c_uint64, C.c_uint32, C.c_uint32, C.c_uint32, C.c_int, _u32p]
        L.momcref_stream_normals.argtypes = [C.c_uint64, C.c_uint32, C.c_uint32, C.c_uint32, C.c_int, _dp]
        L.momcref_stream_symmetric.argtypes = [C.c_uint64, C.c_uint32, C.c_uint32, C.c_uint32, C.c_double,
                                               C.c_int, _dp]
        L.momcref_ziggurat_tables.argtypes = [_u32p, _dp, _dp]
        L.momcref_resolution_for_interior_count.argtypes = [C.c_int, C.c_int, C.c_char_p, C.c_size_t]
        L.momcref_das_dennis.restype = C.c_longlong
        L.momcref_das_dennis.argtypes = [C.c_int, C.c_int, C.c_int, _ip, C.c_longlong, C.c_char_p, C.c_size_t]
        L.momcref_instance_new.restype = C.c_void_p
        L.momcref_instance_new.argtypes = [C.c_int, C.c_int, C.c_int, _ip, _ip, _dp, C.c_char_p, C.c_size_t]
        L.momcref_instance_load.restype = C.c_void_p
        L.momcref_instance_load.argtypes = [C.c_char_p, C.c_char_p, C.c_size_t]
        L.momcref_instance_generate_uniform.restype = C.c_void_p
        L.momcref_instance_generate_uniform.argtypes = [C.c_int, C.c_double, C.c_int, C.c_int, C.c_double,
                                                        C.c_double, C.c_uint64, C.c_char_p, C.c_size_t]
        L.momcref_instance_generate_correlated.restype = C.c_void_p
        L.momcref_instance_generate_correlated.argtypes = [C.c_int, C.c_double, C.c_double, C.c_uint64, C.c_char_p,
                                                           C.c_size_t]
        L.momcref_measured_correlation.argtypes = [C.c_void_p, C.c_int, C.c_uint64, _dp, C.c_char_p, C.c_size_t]
        L.momcref_instance_dims.argtypes = [C.c_void_p, _ip, _ip, _ip]
        L.momcref_instance_edges.argtypes = [C.c_void_p, _ip, _ip, _dp]
        L.momcref_instance_save.argtypes = [C.c_void_p, C.c_char_p, C.c_char_p, C.c_size_t]
        L.momcref_instance_free.argtypes = [C.c_void_p]
        L.momcref_cut_values.argtypes = [C.c_void_p, _u64p, C.c_size_t, _dp, C.c_char_p, C.c_size_t]
        L.momcref_scalarize.argtypes = [C.c_void_p, _ip, C.c_int, _dp, _dp, C.c_char_p, C.c_size_t]
        L.momcref_integrate_block.argtypes = [_dp, C.c_int, C.c_double, C.POINTER(CfgC), C.c_uint64, C.c_uint32,
                                              C.c_uint32, C.c_int, _dp, _dp, C.c_char_p, C.c_size_t]
        L.momcref_init_state.argtypes = [C.POINTER(CfgC), C.c_int, C.c_int, C.c_uint64, C.c_uint32, C.c_uint32,
                                         _dp, _dp, C.c_char_p, C.c_size_t]
        L.momcref_run_sampler.argtypes = [C.c_void_p, _ip, C.c_int, C.c_int, C.POINTER(CfgC), C.c_int, _u64p,
                                          _u32p, _i64p, _dp, C.c_char_p, C.c_size_t]
        L.momcref_filter_pool.restype = C.c_void_p
        L.momcref_filter_pool.argtypes = [C.c_void_p, _u64p, C.c_size_t, C.c_int, C.c_char_p, C.c_size_t]
        L.momcref_filter_values.restype = C.c_void_p
        L.momcref_filter_values.argtypes = [_dp, C.c_size_t, C.c_int, C.c_int, C.c_int, C.c_char_p, C.c_size_t]
        L.momcref_brute_force_pareto.restype = C.c_void_p
        L.momcref_brute_force_pareto.argtypes = [C.c_void_p, C.c_char_p, C.c_size_t]
        L.momcref_archive_dims.argtypes = [C.c_void_p, C.POINTER(C.c_longlong), _ip, _ip]
        L.momcref_archive_get.argtypes = [C.c_void_p, _dp, _u64p, _dp]
        L.momcref_archive_free.argtypes = [C.c_void_p]
        L.momcref_hypervolume.argtypes = [_dp, C.c_longlong, C.c_int, _dp, C.c_int, _dp, C.c_char_p, C.c_size_t]
        L.momcref_evaluate_cuts.argtypes = [C.c_void_p, _u64p, C.c_size_t, _dp, C.c_char_p, C.c_size_t]
        L.momcref_reference_point_sampled.argtypes = [C.c_void_p, C.c_int, C.c_uint64, _dp, C.c_char_p,
                                                      C.c_size_t]
        L.momcref_reference_point_exact.argtypes = [C.c_void_p, _dp, C.c_char_p, C.c_size_t]
        L.momcref_samples_to_reach.argtypes = [C.c_void_p, _u64p, C.c_size_t, _dp, C.c_double,
                                               C.POINTER(C.c_longlong), C.c_char_p, C.c_size_t]
        L.momcref_convergence_trace.argtypes = [C.c_void_p, _u64p, C.POINTER(C.c_longlong), C.c_size_t, _dp, C.c_int,
                                                _dp, _dp, C.POINTER(C.c_longlong), C.c_char_p, C.c_size_t]
        L.momcref_save_pool_csv.argtypes = [_u64p, C.POINTER(C.c_uint32), C.POINTER(C.c_longlong), C.c_size_t, C.c_int,
                                            C.c_double, C.c_double, C.c_char_p, C.c_char_p, C.c_size_t]
        L.momcref_load_pool_csv.argtypes = [C.c_char_p, C.POINTER(C.c_size_t), C.POINTER(C.c_int), _dp, _dp, _u64p,
                                            C.POINTER(C.c_uint32), C.POINTER(C.c_longlong), C.c_size_t, C.c_char_p,
                                            C.c_size_t]
        L.momcref_save_archive_csv.argtypes = [_dp, _u64p, C.c_size_t, C.c_int, C.c_int, C.c_double, _dp, C.c_int,
                                               C.c_char_p, C.c_char_p, C.c_size_t]
        L.momcref_load_archive_csv.argtypes = [C.c_char_p, C.POINTER(C.c_size_t), C.POINTER(C.c_int),
                                               C.POINTER(C.c_int), _dp, C.POINTER(C.c_int), _dp, _dp, _u64p,
                                               C.POINTER(C.c_ubyte), C.c_size_t, C.c_char_p, C.c_size_t]
        L.momcref_bench.argtypes = [C.c_char_p, C.c_int, C.c_double, C.c_int, C.c_uint64, C.POINTER(CfgC), C.c_int,
                                    C.c_int, C.c_int, C.c_char_p, C.c_int, C.c_char_p, C.c_size_t, C.c_char_p,
                                    C.c_size_t]

    # --------------------------------------------------------------- helpers
    @staticmethod
    def _err():
        return C.create_string_buffer(1024)

    @staticmethod
    def _check(rc, err):
        if rc != 0:
            raise RefError(rc, err.value.decode())

    # --------------------------------------------------------------- rng
    def philox(self, key: int, ctr) -> np.ndarray:
        c = np.asarray(ctr, dtype=np.uint32)
        out = np.zeros(4, dtype=np.uint32)
        self.lib.momcref_philox(key, _p(c, _u32p), _p(out, _u32p))
        return out

    def derive_key(self, seed, ctx) -> int:
        return int(self.lib.momcref_derive_key(seed, ctx))

    def run_key(self, seed, run) -> int:
        return int(self.lib.momcref_run_key(seed, run))

    def tag_word(self, tag, step=0) -> int:
        return int(self.lib.momcref_tag_word(tag, step))

    def stream_u32(self, key, hi, mid, lo, count) -> np.ndarray:
        out = np.zeros(count, dtype=np.uint32)
        self.lib.momcref_stream_u32(key, hi, mid, lo, count, _p(out, _u32p))
        return out

    def stream_normals(self, key, hi, mid, lo, count) -> np.ndarray:
        out = np.zeros(count, dtype=np.float64)
        self.lib.momcref_stream_normals(key, hi, mid, lo, count, _p(out, _dp))
        return out

    def stream_symmetric(self, key, hi, mid, lo, h, count) -> np.ndarray:
        out = np.zeros(count, dtype=np.float64)
        self.lib.momcref_stream_symmetric(key, hi, mid, lo, h, count, _p(out, _dp))
        return out

    def ziggurat_tables(self):
        kn = np.zeros(128, np.uint32)
        wn = np.zeros(128, np.float64)
        fn = np.zeros(128, np.float64)
        self.lib.momcref_ziggurat_tables(_p(kn, _u32p), _p(wn, _dp), _p(fn, _dp))
        return kn, wn, fn

    # --------------------------------------------------------------- weights
    def resolution_for_interior_count(self, k, count) -> int:
        err = self._err()
        h = self.lib.momcref_resolution_for_interior_count(k, count, err, 1024)
        if h < 0:
            raise RefError(-h, err.value.decode())
        return h

    def das_dennis(self, k, h, interior=True) -> np.ndarray:
        err = self._err()
        n = self.lib.momcref_das_dennis(k, h, int(interior), None, 0, err, 1024)
        if n < 0:
            raise RefError(-n, err.value.decode())
        out = np.zeros((n, k), dtype=np.int32)
        self.lib.momcref_das_dennis(k, h, int(interior), _p(out, _ip), n, err, 1024)
        return out

    # --------------------------------------------------------------- instances
    def instance_new(self, n, k, ei, ej, w) -> "RefInstance":
        ei = np.ascontiguousarray(ei, np.int32)
        ej = np.ascontiguousarray(ej, np.int32)
        w = np.ascontiguousarray(w, np.float64).reshape(-1)
        err = self._err()
        h = self.lib.momcref_instance_new(n, k, len(ei), _p(ei, _ip), _p(ej, _ip), _p(w, _dp), err, 1024)
        if not h:
            raise RefError(2, err.value.decode())
        return RefInstance(self, h)

    def instance_load(self, path) -> "RefInstance":
        err = self._err()
        h = self.lib.momcref_instance_load(str(path).encode(), err, 1024)
        if not h:
            raise RefError(1, err.value.decode())
        return RefInstance(self, h)

    def generate_uniform(self, n, density, k, seed, kind="int", lo=1.0, hi=10.0) -> "RefInstance":
        err = self._err()
        h = self.lib.momcref_instance_generate_uniform(n, density, k, 0 if kind == "int" else 1, lo, hi, seed,
                                                       err, 1024)
        if not h:
            raise RefError(2, err.value.decode())
        return RefInstance(self, h)

    def generate_correlated(self, n, density, rho, seed) -> "RefInstance":
        err = self._err()
        h = self.lib.momcref_instance_generate_correlated(n, density, rho, seed, err, 1024)
        if not h:
            raise RefError(2, err.value.decode())
        return RefInstance(self, h)

    def measured_correlation(self, inst, pool_size=2048, seed=0) -> float:
        out = C.c_double()
        err = self._err()
        self._check(self.lib.momcref_measured_correlation(inst.h, pool_size, seed, C.byref(out), err, 1024), err)
        return out.value

    # --------------------------------------------------------------- solver
    def scalarize(self, inst, nums, H):
        nums = np.ascontiguousarray(nums, np.int32)
        J = np.zeros((inst.n, inst.n), dtype=np.float64)  # column-major -> transpose below
        c0 = C.c_double()
        err = self._err()
        self._check(self.lib.momcref_scalarize(inst.h, _p(nums, _ip), H, _p(J, _dp), C.byref(c0), err, 1024), err)
        return J.T.copy(), c0.value

    def integrate_block(self, J, c0, cfg: CfgC, key, weight, traj, count):
        n = J.shape[0]
        Jc = np.asfortranarray(J, dtype=np.float64)
        x = np.zeros((count, n), np.float64)
        y = np.zeros((count, n), np.float64)
        err = self._err()
        rc = self.lib.momcref_integrate_block(Jc.ctypes.data_as(_dp), n, c0, C.byref(cfg), key, weight, traj,
                                              count, _p(x, _dp), _p(y, _dp), err, 1024)
        self._check(rc, err)
        return x, y  # row c = trajectory c (column-major n x count)

    def init_state(self, cfg, n, count, key, weight, traj):
        x = np.zeros((count, n), np.float64)
        y = np.zeros((count, n), np.float64)
        err = self._err()
        self._check(self.lib.momcref_init_state(C.byref(cfg), n, count, key, weight, traj, _p(x, _dp), _p(y, _dp),
                                                err, 1024), err)
        return x, y

    def run_sampler(self, inst, nums, H, cfg: CfgC, runs=1, records=False):
        nums = np.ascontiguousarray(nums, np.int32)
        L = nums.shape[0]
        M = runs * L * cfg.batch_size
        wpc = (inst.n + 63) // 64
        words = np.zeros((M, wpc), np.uint64)
        rec = np.zeros((M, 3), np.uint32) if records else None
        stamps = np.zeros(M, np.int64) if records else None
        t = np.zeros(2, np.float64)
        err = self._err()
        rc = self.lib.momcref_run_sampler(inst.h, _p(nums, _ip), L, H, C.byref(cfg), runs, _p(words, _u64p),
                                          _p(rec, _u32p) if records else None,
                                          _p(stamps, _i64p) if records else None, _p(t, _dp), err, 1024)
        self._check(rc, err)
        out = {"words": words, "model_construction_seconds": t[0], "sampling_seconds": t[1]}
        if records:
            out["records"] = rec
            out["stamps"] = stamps
        return out

    # --------------------------------------------------------------- pareto
    def _archive(self, h) -> RefArchive:
        F = C.c_longlong()
        k = C.c_int()
        n = C.c_int()
        self.lib.momcref_archive_dims(h, C.byref(F), C.byref(k), C.byref(n))
        wpc = (n.value + 63) // 64 if n.value else 0
        vals = np.zeros((F.value, k.value), np.float64)
        words = np.zeros((F.value, wpc), np.uint64)
        fs = C.c_double()
        self.lib.momcref_archive_get(h, _p(vals, _dp), _p(words, _u64p) if wpc else None, C.byref(fs))
        self.lib.momcref_archive_free(h)
        return RefArchive(vals, words, fs.value)

    def filter_pool(self, inst, words, algo="fast") -> RefArchive:
        words = np.ascontiguousarray(words, np.uint64)
        err = self._err()
        h = self.lib.momcref_filter_pool(inst.h, _p(words, _u64p), words.shape[0], 0 if algo == "fast" else 1,
                                         err, 1024)
        if not h:
            raise RefError(2, err.value.decode())
        return self._archive(h)

    def filter_values(self, vals, sense="cut", algo="fast") -> RefArchive:
        vals = np.ascontiguousarray(vals, np.float64)
        err = self._err()
        h = self.lib.momcref_filter_values(_p(vals, _dp), vals.shape[0], vals.shape[1], 0 if sense == "cut" else 1,
                                           0 if algo == "fast" else 1, err, 1024)
        if not h:
            raise RefError(2, err.value.decode())
        return self._archive(h)

    def brute_force_pareto(self, inst) -> RefArchive:
        err = self._err()
        h = self.lib.momcref_brute_force_pareto(inst.h, err, 1024)
        if not h:
            raise RefError(2, err.value.decode())
        return self._archive(h)

    HV_ALGOS = {None: -1, "sweep": 0, "dimension_sweep": 1, "recursive": 2, "inclusion_exclusion": 3}

    def hypervolume(self, vals, r, algo=None) -> float:
        vals = np.ascontiguousarray(vals, np.float64)
        r = np.ascontiguousarray(r, np.float64)
        out = C.c_double()
        err = self._err()
        rc = self.lib.momcref_hypervolume(_p(vals, _dp), vals.shape[0], vals.shape[1], _p(r, _dp),
                                          self.HV_ALGOS[algo], C.byref(out), err, 1024)
        self._check(rc, err)
        return out.value

    def evaluate_cuts(self, inst, words) -> np.ndarray:
        words = np.ascontiguousarray(words, np.uint64)
        out = np.zeros((words.shape[0], inst.k), np.float64)
        err = self._err()
        self._check(self.lib.momcref_evaluate_cuts(inst.h, _p(words, _u64p), words.shape[0], _p(out, _dp), err,
                                                   1024), err)
        return out

    def cut_values(self, inst, words) -> np.ndarray:
        words = np.ascontiguousarray(words, np.uint64)
        out = np.zeros((words.shape[0], inst.k), np.float64)
        err = self._err()
        self._check(self.lib.momcref_cut_values(inst.h, _p(words, _u64p), words.shape[0], _p(out, _dp), err, 1024),
                    err)
        return out

    def reference_point_sampled(self, inst, count, seed) -> np.ndarray:
        r = np.zeros(inst.k, np.float64)
        err = self._err()
        self._check(self.lib.momcref_reference_point_sampled(inst.h, count, seed, _p(r, _dp), err, 1024), err)
        return r

    def reference_point_exact(self, inst) -> np.ndarray:
        r = np.zeros(inst.k, np.float64)
        err = self._err()
        self._check(self.lib.momcref_reference_point_exact(inst.h, _p(r, _dp), err, 1024), err)
        return r

    def samples_to_reach(self, inst, words, r, target):
        words = np.ascontiguousarray(words, np.uint64)
        r = np.ascontiguousarray(r, np.float64)
        out = C.c_longlong()
        err = self._err()
        self._check(self.lib.momcref_samples_to_reach(inst.h, _p(words, _u64p), words.shape[0], _p(r, _dp), target,
                                                      C.byref(out), err, 1024), err)
        return None if out.value < 0 else out.value

    def save_pool_csv(self, path, words, rec3, stamps, n, mc, ss):
        words = np.ascontiguousarray(words, np.uint64)
        rec3 = np.ascontiguousarray(rec3, np.uint32)
        stamps = np.ascontiguousarray(stamps, np.int64)
        err = self._err()
        self._check(self.lib.momcref_save_pool_csv(_p(words, _u64p), _p(rec3, C.POINTER(C.c_uint32)),
                                                   _p(stamps, C.POINTER(C.c_longlong)), stamps.shape[0], n, mc, ss,
                                                   str(path).encode(), err, 1024), err)

    def load_pool_csv(self, path):
        M, n, mc, ss = C.c_size_t(), C.c_int(), C.c_double(), C.c_double()
        err = self._err()
        self._check(self.lib.momcref_load_pool_csv(str(path).encode(), C.byref(M), C.byref(n), C.byref(mc),
                                                   C.byref(ss), None, None, None, 0, err, 1024), err)
        wpc = (n.value + 63) // 64
        words = np.zeros((M.value, wpc), np.uint64)
        rec3 = np.zeros((M.value, 3), np.uint32)
        stamps = np.zeros(M.value, np.int64)
        self._check(self.lib.momcref_load_pool_csv(str(path).encode(), C.byref(M), C.byref(n), C.byref(mc),
                                                   C.byref(ss), _p(words, _u64p), _p(rec3, C.POINTER(C.c_uint32)),
                                                   _p(stamps, C.POINTER(C.c_longlong)), M.value, err, 1024), err)
        return {"n": n.value, "mc": mc.value, "ss": ss.value, "words": words, "rec3": rec3, "stamps": stamps}

    def save_archive_csv(self, path, vals, words, n, fs, r):
        vals = np.ascontiguousarray(vals, np.float64)
        F, k = vals.shape
        r = np.ascontiguousarray(r, np.float64)
        err = self._err()
        wp = _p(np.ascontiguousarray(words, np.uint64), _u64p) if words is not None else None
        self._check(self.lib.momcref_save_archive_csv(_p(vals, _dp), wp, F, k, n, fs, _p(r, _dp), r.shape[0],
                                                      str(path).encode(), err, 1024), err)

    def load_archive_csv(self, path):
        F, k, n, nr = C.c_size_t(), C.c_int(), C.c_int(), C.c_int()
        fs = C.c_double()
        r = np.zeros(16, np.float64)
        err = self._err()
        args = (str(path).encode(), C.byref(F), C.byref(k), C.byref(n), C.byref(fs), C.byref(nr), _p(r, _dp))
        self._check(self.lib.momcref_load_archive_csv(*args, None, None, None, 0, err, 1024), err)
        wpc = (n.value + 63) // 64
        vals = np.zeros((F.value, k.value), np.float64)
        words = np.zeros((F.value, max(wpc, 1)), np.uint64)
        has = np.zeros(F.value, np.uint8)
        self._check(self.lib.momcref_load_archive_csv(*args, _p(vals, _dp), _p(words, _u64p),
                                                      _p(has, C.POINTER(C.c_ubyte)), F.value, err, 1024), err)
        return {"values": vals, "words": words[:, :wpc], "has_cfg": has.astype(bool), "n": n.value,
                "fs": fs.value, "reference": r[: nr.value].tolist()}

    def convergence_trace(self, inst, words, stamps, r, checkpoints):
        words = np.ascontiguousarray(words, np.uint64)
        stamps = np.ascontiguousarray(stamps, np.int64)
        r = np.ascontiguousarray(r, np.float64)
        el = np.zeros(checkpoints, np.float64)
        hv = np.zeros(checkpoints, np.float64)
        sm = np.zeros(checkpoints, np.int64)
        err = self._err()
        self._check(self.lib.momcref_convergence_trace(inst.h, _p(words, _u64p), _p(stamps, C.POINTER(C.c_longlong)),
                                                       words.shape[0], _p(r, _dp), checkpoints, _p(el, _dp),
                                                       _p(hv, _dp), _p(sm, C.POINTER(C.c_longlong)), err, 1024), err)
        return el, hv, sm

    def bench(self, cfg: CfgC, instance_path="", n=10, density=0.5, k=3, instance_seed=1, weight_count=55,
              weight_resolution=0, runs=1, ref="exact", checkpoints=0) -> dict:
        rep = C.create_string_buffer(1 << 16)
        err = self._err()
        rc = self.lib.momcref_bench(instance_path.encode(), n, density, k, instance_seed, C.byref(cfg), weight_count,
                                    weight_resolution, runs, ref.encode(), checkpoints, rep, 1 << 16, err, 1024)
        self._check(rc, err)
        out = {}
        for line in rep.value.decode().splitlines():
            key, _, val = line.partition(" = ")
            out[key] = val
        return out


class RefInstance:
    def __init__(self, lib: RefLib, h):
        self.lib = lib
        self.h = h
        n, k, m = C.c_int(), C.c_int(), C.c_int()
        lib.lib.momcref_instance_dims(h, C.byref(n), C.byref(k), C.byref(m))
        self.n, self.k, self.m = n.value, k.value, m.value

    def edges(self):
        ei = np.zeros(self.m, np.int32)
        ej = np.zeros(self.m, np.int32)
        w = np.zeros((self.m, self.k), np.float64)
        self.lib.lib.momcref_instance_edges(self.h, _p(ei, _ip), _p(ej, _ip), _p(w, _dp))
        return ei, ej, w

    def save(self, path):
        err = RefLib._err()
        RefLib._check(self.lib.lib.momcref_instance_save(self.h, str(path).encode(), err, 1024), err)

    def __del__(self):
        try:
            self.lib.lib.momcref_instance_free(self.h)
        except Exception:
            pass


def pool_fold(words: np.ndarray) -> int:
    """SURVEY.md Appendix A pool fold: f = f*1099511628211 (mod 2^64) XOR v over canonical order."""
    f = 0
    mask = (1 << 64) - 1
    for v in np.asarray(words, np.uint64).reshape(-1).tolist():
        f = ((f * 1099511628211) & mask) ^ int(v)
    return f


ORACLE_SO = os.path.join(HERE, "_ref", "libmomc_oracle.so")


class OracleLib:
    """The C restatement (oracle/momc_oracle.c; cpu_baseline kind "port")."""

    def __init__(self, path: str = ORACLE_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing: run oracle/build_ref.sh")
        L = self.lib = C.CDLL(path)
        L.oracle_philox.argtypes = [C.c_uint64, _u32p, _u32p]
        L.oracle_derive_key.restype = C.c_uint64
        L.oracle_derive_key.argtypes = [C.c_uint64, C.c_uint64]
        L.oracle_run_key.restype = C.c_uint64
        L.oracle_run_key.argtypes = [C.c_uint64, C.c_uint32]
        L.oracle_tag_word.restype = C.c_uint32
        L.oracle_tag_word.argtypes = [C.c_uint32, C.c_uint32]
        L.oracle_ziggurat_tables.argtypes = [_u32p, _dp, _dp]
        L.oracle_stream_u32.argtypes = [C.c_uint64, C.c_uint32, C.c_uint32, C.c_uint32, C.c_int, _u32p]
        L.oracle_stream_normals.argtypes = [C.c_uint64, C.c_uint32, C.c_uint32, C.c_uint32, C.c_int, _dp]
        L.oracle_stream_below.argtypes = [C.c_uint64, C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint64, C.c_int, _u64p]
        L.oracle_resolution_for_interior_count.argtypes = [C.c_int, C.c_int]
        L.oracle_das_dennis.restype = C.c_longlong
        L.oracle_das_dennis.argtypes = [C.c_int, C.c_int, C.c_int, _ip, C.c_longlong]
        L.oracle_scalarize.argtypes = [C.c_int, C.c_int, C.c_int, _ip, _ip, _dp, _ip, C.c_int, _dp, _dp]
        L.oracle_integrate_one.argtypes = [_dp, C.c_int, C.c_double, C.POINTER(CfgC), C.c_uint64, C.c_uint32,
                                           C.c_uint32, _dp, _dp]
        L.oracle_run_sampler.argtypes = [C.c_int, C.c_int, C.c_int, _ip, _ip, _dp, _ip, C.c_int, C.c_int,
                                         C.POINTER(CfgC), C.c_int, C.c_int, _u64p, _ip]
        for nm in ("oracle_cut_values", "oracle_evaluate_cuts"):
            getattr(L, nm).argtypes = [C.c_int, C.c_int, C.c_int, _ip, _ip, _dp, _u64p, C.c_size_t, _dp]
        L.oracle_filter_values.restype = C.c_size_t
        L.oracle_filter_values.argtypes = [_dp, C.c_size_t, C.c_int]
        L.oracle_filter_pool.restype = C.c_size_t
        L.oracle_filter_pool.argtypes = [C.c_int, C.c_int, C.c_int, _ip, _ip, _dp, _u64p, C.c_size_t, _dp, _u64p]
        L.oracle_hypervolume.argtypes = [_dp, C.c_size_t, C.c_int, _dp, _dp, C.POINTER(C.c_longlong)]
        L.oracle_reference_point_sampled.argtypes = [C.c_int, C.c_int, C.c_int, _ip, _ip, _dp, C.c_int, C.c_uint64,
                                                     _dp]

    def philox(self, key, ctr):
        c = np.asarray(ctr, dtype=np.uint32)
        out = np.zeros(4, np.uint32)
        self.lib.oracle_philox(key, _p(c, _u32p), _p(out, _u32p))
        return out

    def derive_key(self, seed, ctx):
        return int(self.lib.oracle_derive_key(seed, ctx))

    def run_key(self, seed, run):
        return int(self.lib.oracle_run_key(seed, run))

    def tag_word(self, tag, step=0):
        return int(self.lib.oracle_tag_word(tag, step))

    def ziggurat_tables(self):
        kn = np.zeros(128, np.uint32)
        wn = np.zeros(128, np.float64)
        fn = np.zeros(128, np.float64)
        self.lib.oracle_ziggurat_tables(_p(kn, _u32p), _p(wn, _dp), _p(fn, _dp))
        return kn, wn, fn

    def stream_u32(self, key, hi, mid, lo, count):
        out = np.zeros(count, np.uint32)
        self.lib.oracle_stream_u32(key, hi, mid, lo, count, _p(out, _u32p))
        return out

    def stream_normals(self, key, hi, mid, lo, count):
        out = np.zeros(count, np.float64)
        self.lib.oracle_stream_normals(key, hi, mid, lo, count, _p(out, _dp))
        return out

    def stream_below(self, key, hi, mid, lo, bound, count):
        out = np.zeros(count, np.uint64)
        self.lib.oracle_stream_below(key, hi, mid, lo, bound, count, _p(out, _u64p))
        return out

    def resolution_for_interior_count(self, k, count):
        return int(self.lib.oracle_resolution_for_interior_count(k, count))

    def das_dennis(self, k, h, interior=True):
        n = self.lib.oracle_das_dennis(k, h, int(interior), None, 0)
        out = np.zeros((max(n, 0), k), np.int32)
        self.lib.oracle_das_dennis(k, h, int(interior), _p(out, _ip), n)
        return out

    @staticmethod
    def _inst(inst):
        n, k, ei, ej, w = inst
        return (n, k, len(ei), _p(np.ascontiguousarray(ei, np.int32), _ip),
                _p(np.ascontiguousarray(ej, np.int32), _ip), _p(np.ascontiguousarray(w, np.float64), _dp))

    def scalarize(self, inst, nums, H):
        n = inst[0]
        nums = np.ascontiguousarray(nums, np.int32)
        J = np.zeros((n, n), np.float64)
        c0 = C.c_double()
        keep = [np.ascontiguousarray(a) for a in inst[2:]]
        args = self._inst((inst[0], inst[1], keep[0], keep[1], keep[2]))
        rc = self.lib.oracle_scalarize(*args, _p(nums, _ip), H, _p(J, _dp), C.byref(c0))
        if rc:
            raise RefError(rc, "degenerate scalarized coupling: normalization undefined")
        return J, c0.value

    def integrate_one(self, J, c0, cfg, key, weight, traj):
        n = J.shape[0]
        J = np.ascontiguousarray(J, np.float64)
        x = np.zeros(n, np.float64)
        y = np.zeros(n, np.float64)
        bad = self.lib.oracle_integrate_one(_p(J, _dp), n, c0, C.byref(cfg), key, weight, traj, _p(x, _dp), _p(y, _dp))
        return x, y, bad

    def run_sampler(self, inst, nums, H, cfg, runs=1, threads=None):
        n, k, ei, ej, w = inst
        ei = np.ascontiguousarray(ei, np.int32)
        ej = np.ascontiguousarray(ej, np.int32)
        w = np.ascontiguousarray(w, np.float64)
        nums = np.ascontiguousarray(nums, np.int32)
        L = nums.shape[0]
        wpc = (n + 63) // 64
        words = np.zeros((runs * L * cfg.batch_size, wpc), np.uint64)
        info = np.zeros(3, np.int32)
        th = threads if threads is not None else (os.cpu_count() or 1)
        rc = self.lib.oracle_run_sampler(n, k, len(ei), _p(ei, _ip), _p(ej, _ip), _p(w, _dp), _p(nums, _ip), L, H,
                                         C.byref(cfg), runs, th, _p(words, _u64p), _p(info, _ip))
        if rc == 2:
            raise RefError(2, "degenerate scalarized coupling: normalization undefined")
        if rc == 1:
            raise RefError(1, f"numerical failure at step {info[0]} (run {info[1]}, weight {info[2]})")
        return words

    def _eval(self, fn, inst, words):
        n, k, ei, ej, w = inst
        ei = np.ascontiguousarray(ei, np.int32)
        ej = np.ascontiguousarray(ej, np.int32)
        w = np.ascontiguousarray(w, np.float64)
        words = np.ascontiguousarray(words, np.uint64)
        out = np.zeros((words.shape[0], k), np.float64)
        fn(n, k, len(ei), _p(ei, _ip), _p(ej, _ip), _p(w, _dp), _p(words, _u64p), words.shape[0], _p(out, _dp))
        return out

    def cut_values(self, inst, words):
        return self._eval(self.lib.oracle_cut_values, inst, words)

    def evaluate_cuts(self, inst, words):
        return self._eval(self.lib.oracle_evaluate_cuts, inst, words)

    def filter_values(self, vals):
        v = np.array(vals, dtype=np.float64, copy=True, order="C")
        f = self.lib.oracle_filter_values(_p(v, _dp), v.shape[0], v.shape[1])
        return v[:f].copy()

    def filter_pool(self, inst, words):
        n, k, ei, ej, w = inst
        ei = np.ascontiguousarray(ei, np.int32)
        ej = np.ascontiguousarray(ej, np.int32)
        w = np.ascontiguousarray(w, np.float64)
        words = np.ascontiguousarray(words, np.uint64)
        M = words.shape[0]
        wpc = (n + 63) // 64
        vals = np.zeros((M, k), np.float64)
        cfgs = np.zeros((M, wpc), np.uint64)
        f = self.lib.oracle_filter_pool(n, k, len(ei), _p(ei, _ip), _p(ej, _ip), _p(w, _dp), _p(words, _u64p), M,
                                        _p(vals, _dp), _p(cfgs, _u64p))
        return vals[:f].copy(), cfgs[:f].copy()

    def hypervolume(self, vals, r):
        vals = np.ascontiguousarray(vals, np.float64)
        r = np.ascontiguousarray(r, np.float64)
        out = C.c_double()
        bad = C.c_longlong()
        rc = self.lib.oracle_hypervolume(_p(vals, _dp), vals.shape[0], vals.shape[1], _p(r, _dp), C.byref(out),
                                         C.byref(bad))
        if rc:
            raise RefError(rc, "reference point not dominated by archive entry "
                               f"{bad.value // 64} (objective {bad.value % 64})")
        return out.value

    def reference_point_sampled(self, inst, count, seed):
        n, k, ei, ej, w = inst
        ei = np.ascontiguousarray(ei, np.int32)
        ej = np.ascontiguousarray(ej, np.int32)
        w = np.ascontiguousarray(w, np.float64)
        r = np.zeros(k, np.float64)
        self.lib.oracle_reference_point_sampled(n, k, len(ei), _p(ei, _ip), _p(ej, _ip), _p(w, _dp), count, seed,
                                                _p(r, _dp))
        return r
