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
# SDCT_BUILD_TAG / SDCT_EXTRA_NVFLAGS: developer A/B builds of the library
# into build/obj_<tag> and paper_2110_01172_b200/lib_<tag> (selected at run
# time with LD_LIBRARY_PATH); the default build uses neither.
_TAG = os.environ.get("SDCT_BUILD_TAG", "")
OBJ = os.path.join(ROOT, "build", "obj" + ("_" + _TAG if _TAG else ""))
LIB = os.path.join(PKG, "lib" + ("_" + _TAG if _TAG else ""))
LIBSO = os.path.join(LIB, "libsdct_b200.so")
EXT = sysconfig.get_config_var("EXT_SUFFIX") or ".so"
PYMOD = os.path.join(PKG, "_sdct" + EXT)

NVCC = os.environ.get("NVCC", "nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVFLAGS = ["-std=c++17", "--expt-relaxed-constexpr", "-O3", "-lineinfo", "-Xcompiler", "-fPIC",
           "-Xcompiler", "-O3", "-I", INC, "-I", CSRC] + os.environ.get("SDCT_EXTRA_NVFLAGS", "").split()
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
    if _TAG:
        return LIBSO  # A/B library only: the module and programs link the default one
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
    build_acceptance()
    return LIBSO


REFERENCE = "/root/reference/proj"
ACC_BIN = os.path.join(ROOT, "tests", "cpp", "bin", "acceptance_dropin")
# headers of the hot path come from this repo (the drop-in); the reference's
# own headers serve everything off the path (PGM/DCTB I/O, compression app,
# quadratic oracles, bench helper, Amdahl model)
DROPIN_HEADERS = ["tensor", "exec", "errors", "dct1d", "dct2d", "transforms_ext", "rfft", "force", "plan_handle",
                  "device"]
REFERENCE_HEADERS = ["io", "compress", "oracle", "bench", "amdahl", "verify"]
REFERENCE_SUPPORT = ["oracle", "bench", "compress", "amdahl", "io"]


def build_acceptance() -> str | None:
    """The reference's own acceptance program (proj/tests/acceptance.cpp),
    compiled unmodified from where it lies in /root/reference against this
    repo's include/sdct and linked with libsdct_b200.so: the compatibility
    check of SURVEY.md §8(b). Its off-path helpers (oracle.cpp, bench.cpp,
    compress.cpp, amdahl.cpp, io.cpp) are compiled from the reference too and
    call the drop-in where they call the transforms. Output (git-ignored,
    travels to the GPU box): tests/cpp/bin/acceptance_dropin. Skipped when the
    reference tree is absent (the GPU box uses the prebuilt binary)."""
    if not os.path.isdir(REFERENCE):
        return None
    import shutil
    import tempfile

    srcs = [os.path.join(REFERENCE, "tests", "acceptance.cpp")] + [
        os.path.join(REFERENCE, "src", f + ".cpp") for f in REFERENCE_SUPPORT]
    hdrs = [os.path.join(INC, "sdct", h + ".hpp") for h in DROPIN_HEADERS] + [
        os.path.join(REFERENCE, "include", "sdct", h + ".hpp") for h in REFERENCE_HEADERS]
    if os.path.exists(ACC_BIN) and os.path.getmtime(ACC_BIN) >= _newest(srcs + hdrs + [LIBSO]):
        return ACC_BIN
    os.makedirs(os.path.dirname(ACC_BIN), exist_ok=True)
    tmp = tempfile.mkdtemp(prefix="sdct_acc_")
    try:
        inc = os.path.join(tmp, "inc", "sdct")
        os.makedirs(inc)
        for h in hdrs:
            os.symlink(h, os.path.join(inc, os.path.basename(h)))
        objs = []
        for src in srcs:
            obj = os.path.join(tmp, os.path.basename(src) + ".o")
            _run(["g++", "-std=c++20", "-O2", "-pthread", "-I", os.path.join(tmp, "inc"), "-I", INC, "-c", src,
                  "-o", obj])
            objs.append(obj)
        _run(["g++", "-o", ACC_BIN] + objs + ["-L", LIB, "-lsdct_b200", "-pthread",
                                             "-Wl,-rpath,$ORIGIN/../../../paper_2110_01172_b200/lib"])
    finally:
        shutil.rmtree(tmp, ignore_errors=True)
    return ACC_BIN


if __name__ == "__main__":
    build(verbose="-v" in sys.argv)
    print(LIBSO)
    print(PYMOD)
