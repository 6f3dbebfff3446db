"""In-tree build of libmomc_b200.so for sm_100a (nvcc cross-compiles without a GPU).

Each translation unit under csrc/ is compiled in parallel with
``-gencode arch=compute_100a,code=sm_100a -lineinfo`` and linked (static cudart) into
``paper_2604_26477_b200/libmomc_b200.so``. Objects are cached by content hash of the
sources + flags, so unchanged units are not recompiled.
"""
from __future__ import annotations

import concurrent.futures as cf
import hashlib
import os
import shutil
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
OBJ = os.path.join(PKG, "build_obj")
LIB = os.path.join(PKG, "libmomc_b200.so")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ARCH + ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xcompiler", "-O2",
                     "-I" + os.path.join(ROOT, "include")]


def _nvcc() -> str:
    for cand in (shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def _sources():
    return sorted(os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith(".cu"))


def _headers_digest() -> str:
    h = hashlib.sha256()
    for d in (CSRC, os.path.join(ROOT, "include")):
        for f in sorted(os.listdir(d)):
            p = os.path.join(d, f)
            if os.path.isfile(p) and f.endswith((".cuh", ".h", ".hpp")):
                h.update(f.encode())
                with open(p, "rb") as fh:
                    h.update(fh.read())
    return h.hexdigest()


def _compile(src: str, hdr: str, verbose: bool) -> str:
    with open(src, "rb") as fh:
        digest = hashlib.sha256(fh.read() + hdr.encode() + " ".join(NVCC_FLAGS).encode()).hexdigest()[:16]
    obj = os.path.join(OBJ, os.path.basename(src)[:-3] + "." + digest + ".o")
    if os.path.exists(obj):
        return obj
    cmd = [_nvcc()] + NVCC_FLAGS + ["-Xptxas", "-v", "-c", src, "-o", obj + ".tmp"]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src}:\n{res.stderr[-6000:]}")
    with open(os.path.join(OBJ, os.path.basename(src) + ".ptxas.log"), "w") as fh:
        fh.write(res.stderr)
    os.replace(obj + ".tmp", obj)
    if verbose:
        print(f"  compiled {os.path.basename(src)}", file=sys.stderr)
    return obj


def build(verbose: bool = False, jobs: int | None = None) -> str:
    os.makedirs(OBJ, exist_ok=True)
    hdr = _headers_digest()
    srcs = _sources()
    with cf.ThreadPoolExecutor(max_workers=jobs or os.cpu_count() or 4) as ex:
        objs = list(ex.map(lambda s: _compile(s, hdr, verbose), srcs))
    link_key = hashlib.sha256("".join(objs).encode()).hexdigest()[:16]
    stamp = LIB + ".stamp"
    if os.path.exists(LIB) and os.path.exists(stamp) and open(stamp).read() == link_key:
        return LIB
    cmd = [_nvcc()] + ARCH + ["-shared", "-o", LIB + ".tmp"] + objs + ["-lcudart_static", "-lrt", "-ldl", "-lpthread"]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"link failed:\n{res.stderr[-4000:]}")
    os.replace(LIB + ".tmp", LIB)
    with open(stamp, "w") as fh:
        fh.write(link_key)
    # drop stale objects of earlier source versions
    keep = set(objs)
    for f in os.listdir(OBJ):
        p = os.path.join(OBJ, f)
        if f.endswith(".o") and p not in keep:
            os.remove(p)
    return LIB


PROF_SRC = os.path.join(PKG, "prof", "cupti_traffic.cpp")
PROF_LIB = os.path.join(PKG, "libmomc_b200_prof.so")


def build_prof(verbose: bool = False) -> str | None:
    """libmomc_b200_prof.so: in-process DRAM traffic of kernels through the CUPTI range profiler
    (bench.py's roofline.traffic). Measurement tooling, separate from the product library; None
    when CUPTI is not installed."""
    cuda = os.path.dirname(os.path.dirname(_nvcc()))
    inc = os.path.join(cuda, "include")
    if not os.path.exists(os.path.join(inc, "cupti_range_profiler.h")):
        return None
    with open(PROF_SRC, "rb") as fh:
        key = hashlib.sha256(fh.read()).hexdigest()[:16]
    stamp = PROF_LIB + ".stamp"
    if os.path.exists(PROF_LIB) and os.path.exists(stamp) and open(stamp).read() == key:
        return PROF_LIB
    cmd = ["g++", "-O2", "-fPIC", "-shared", "-std=c++17", "-I" + inc, PROF_SRC, "-o", PROF_LIB + ".tmp",
           "-L" + os.path.join(cuda, "lib64"), "-Wl,-rpath," + os.path.join(cuda, "lib64"), "-lcupti", "-lcuda"]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        if verbose:
            print(f"  (prof library not built: {res.stderr[-500:]})", file=sys.stderr)
        return None
    os.replace(PROF_LIB + ".tmp", PROF_LIB)
    with open(stamp, "w") as fh:
        fh.write(key)
    return PROF_LIB


if __name__ == "__main__":
    print(build(verbose=True))
    print(build_prof(verbose=True))
