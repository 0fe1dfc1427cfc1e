"""Build the sm_100a C-ABI library in-tree (nvcc cross-compiles without a GPU)."""

import os
import subprocess

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIB = os.path.join(PKG, "libgee_b200.so")
SOURCES = ["gee_capi.cu", "gee_projection.cu", "gee_push.cu", "gee_prep.cu", "gee_hot.cu", "gee_gather.cu", "gee_tiles.cu", "gee_reduce.cu", "gee_wide.cu", "gee_compact.cu", "gee_pack.cu", "gee_synth.cu"]
HEADERS = ["gee_common.cuh"]
NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC", "-shared",
]


def _nvcc():
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if cand and (os.path.sep not in cand or os.path.exists(cand)):
            return cand
    return "nvcc"


def _stale(target, deps):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


IO_LIB = os.path.join(PKG, "libgee_io.so")
IO_SOURCES = ["gee_io.cpp"]
CXX_FLAGS = ["-O3", "-std=c++17", "-fPIC", "-shared", "-pthread", "-Wall", "-Wextra", "-static-libstdc++", "-static-libgcc"]


def build_io_library(force=False, verbose=False):
    """Compile the host IO library (text parsers, GEECSR1/GEEEMB1 readers and
    writers; pure C++, no CUDA) into paper_2402_04403_b200/libgee_io.so."""
    srcs = [os.path.join(CSRC, s) for s in IO_SOURCES]
    deps = srcs + [os.path.join(ROOT, "include", "gee_io.h")]
    if not force and not _stale(IO_LIB, deps):
        return IO_LIB
    tmp = IO_LIB + ".tmp"
    cmd = [os.environ.get("CXX", "g++"), *CXX_FLAGS, "-o", tmp, *srcs]
    if verbose:
        print(" ".join(cmd))
    subprocess.run(cmd, check=True, cwd=CSRC)
    os.replace(tmp, IO_LIB)
    return IO_LIB


CHECKED_LIB = os.path.join(PKG, "libgee_b200_checked.so")


def build_library(force=False, verbose=False, checked=False):
    """Compile every CUDA source into paper_2402_04403_b200/libgee_b200.so
    (one nvcc process per source, in parallel, then one link).  checked=True
    builds libgee_b200_checked.so instead, with -DGEE_CHECKED: device-side
    bounds checks (GEE_DCHECK) in the hot kernels; the GPU test suite runs
    against it by putting it in place of libgee_b200.so."""
    from concurrent.futures import ThreadPoolExecutor

    lib = CHECKED_LIB if checked else LIB
    srcs = [os.path.join(CSRC, s) for s in SOURCES]
    hdrs = [os.path.join(CSRC, h) for h in HEADERS] + [
        os.path.join(ROOT, "include", "gee_b200.h"), os.path.join(ROOT, "include", "gee_synth.h")]
    if not force and not _stale(lib, srcs + hdrs):
        return lib
    objdir = os.path.join(PKG, "build_checked" if checked else "build")
    os.makedirs(objdir, exist_ok=True)
    compile_flags = [f for f in NVCC_FLAGS if f != "-shared"] + (["-DGEE_CHECKED"] if checked else [])

    def obj(src):
        o = os.path.join(objdir, os.path.basename(src) + ".o")
        if force or _stale(o, [src] + hdrs):
            cmd = [_nvcc(), *compile_flags, "-c", "-o", o + ".tmp", src]
            if verbose:
                print(" ".join(cmd))
            subprocess.run(cmd, check=True, cwd=CSRC)
            os.replace(o + ".tmp", o)
        return o

    with ThreadPoolExecutor(max_workers=min(len(srcs), os.cpu_count() or 4)) as ex:
        objs = list(ex.map(obj, srcs))
    tmp = lib + ".tmp"
    cmd = [_nvcc(), "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", tmp, *objs]
    if verbose:
        print(" ".join(cmd))
    subprocess.run(cmd, check=True, cwd=CSRC)
    os.replace(tmp, lib)
    return lib
