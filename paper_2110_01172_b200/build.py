"""In-tree build of the native library (no JIT cache, no pip install).

Outputs (git-ignored, but they travel to the GPU box with the snapshot):
  paper_2110_01172_b200/lib/libsdct_b200.so   CUDA kernels + C ABI + C++ API
  paper_2110_01172_b200/_sdct<EXT_SUFFIX>     pybind11 module (reference-compatible)

All device code is compiled for sm_100a only:
  nvcc -gencode arch=compute_100a,code=sm_100a -lineinfo -O3
"""
from __future__ import annotations

import concurrent.futures as cf
import glob
import os
import subprocess
import sys
import sysconfig

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
INC = os.path.join(ROOT, "include")
OBJ = os.path.join(ROOT, "build", "obj")
LIB = os.path.join(PKG, "lib")
LIBSO = os.path.join(LIB, "libsdct_b200.so")
EXT = sysconfig.get_config_var("EXT_SUFFIX") or ".so"
PYMOD = os.path.join(PKG, "_sdct" + EXT)

NVCC = os.environ.get("NVCC", "nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVFLAGS = ["-std=c++17", "--expt-relaxed-constexpr", "-O3", "-lineinfo", "-Xcompiler", "-fPIC",
           "-Xcompiler", "-O3", "-I", INC, "-I", CSRC]
CXXFLAGS = ["-std=c++20", "-O2", "-fPIC", "-I", INC]


def _newest(paths):
    return max((os.path.getmtime(p) for p in paths if os.path.exists(p)), default=0.0)


def _headers():
    return (glob.glob(os.path.join(CSRC, "*.cuh")) + glob.glob(os.path.join(CSRC, "*.h"))
            + glob.glob(os.path.join(INC, "*.h")) + glob.glob(os.path.join(INC, "sdct", "*.hpp")))


def _run(cmd):
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(" ".join(cmd) + "\n" + r.stdout + r.stderr)
        raise RuntimeError(f"build step failed: {os.path.basename(cmd[-1])}")
    return r


def _compile(src, hdr_time, verbose=False):
    obj = os.path.join(OBJ, os.path.basename(src) + ".o")
    if os.path.exists(obj) and os.path.getmtime(obj) >= max(os.path.getmtime(src), hdr_time):
        return obj
    if src.endswith(".cu"):
        cmd = [NVCC] + ARCH + NVFLAGS + ["-c", src, "-o", obj]
        if verbose:
            cmd.insert(1, "-Xptxas=-v")
    else:
        cmd = ["g++"] + CXXFLAGS + ["-I", _cuda_inc(), "-c", src, "-o", obj]
    _run(cmd)
    return obj


def _cuda_inc():
    for base in (os.environ.get("CUDA_HOME", ""), "/usr/local/cuda"):
        if base and os.path.isdir(os.path.join(base, "include")):
            return os.path.join(base, "include")
    return "/usr/local/cuda/include"


def build(verbose: bool = False, jobs: int | None = None) -> str:
    os.makedirs(OBJ, exist_ok=True)
    os.makedirs(LIB, exist_ok=True)
    hdr_time = _newest(_headers())
    lib_srcs = sorted(glob.glob(os.path.join(CSRC, "*.cu"))) + [os.path.join(CSRC, "host_api.cpp")]
    jobs = jobs or min(8, os.cpu_count() or 4)
    with cf.ThreadPoolExecutor(jobs) as ex:
        objs = list(ex.map(lambda s: _compile(s, hdr_time, verbose), lib_srcs))
    if not os.path.exists(LIBSO) or os.path.getmtime(LIBSO) < _newest(objs):
        _run([NVCC] + ARCH + ["-shared", "-o", LIBSO] + objs + ["-Xlinker", "-soname=libsdct_b200.so"])
    # pybind11 module over the C++ API
    import pybind11

    pysrc = os.path.join(CSRC, "pymodule.cpp")
    if not os.path.exists(PYMOD) or os.path.getmtime(PYMOD) < max(
            os.path.getmtime(pysrc), os.path.getmtime(LIBSO), hdr_time):
        _run(["g++"] + CXXFLAGS + ["-shared", "-I", pybind11.get_include(),
                                   "-I", sysconfig.get_paths()["include"], pysrc, "-o", PYMOD,
                                   "-L", LIB, "-lsdct_b200", "-Wl,-rpath,$ORIGIN/lib"])
    # C++ drop-in check program (tests/cpp/api_smoke.cpp) against the C++ API
    src = os.path.join(ROOT, "tests", "cpp", "api_smoke.cpp")
    exe = os.path.join(LIB, "api_smoke")
    if os.path.exists(src) and (not os.path.exists(exe) or os.path.getmtime(exe) < max(
            os.path.getmtime(src), os.path.getmtime(LIBSO), hdr_time)):
        _run(["g++"] + CXXFLAGS + [src, "-o", exe, "-L", LIB, "-lsdct_b200", "-pthread", "-Wl,-rpath,$ORIGIN"])
    return LIBSO


if __name__ == "__main__":
    build(verbose="-v" in sys.argv)
    print(LIBSO)
    print(PYMOD)
