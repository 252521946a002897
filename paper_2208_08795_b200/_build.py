"""In-tree build of the native pieces (no GPU needed; nvcc cross-compiles).

    python paper_2208_08795_b200/_build.py        # or __graft_entry__.build()

Outputs (git-ignored, shipped to the GPU box by gpurun's snapshot):
  paper_2208_08795_b200/lib/libpcs_gpu.so  -- sm_100a kernels + C-ABI
                                              (include/pcs_gpu.h) + the C++
                                              drop-in namespace pcs
  paper_2208_08795_b200/_core*.so          -- pybind11 module over the drop-in
"""
from __future__ import annotations

import os
import subprocess
import sys
import sysconfig

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
INC = os.path.join(ROOT, "include")
LIBDIR = os.path.join(PKG, "lib")
OBJDIR = os.path.join(PKG, "build")
LIB = os.path.join(LIBDIR, "libpcs_gpu.so")
CUDA = os.environ.get("CUDA_HOME", "/usr/local/cuda")
NVCC = os.path.join(CUDA, "bin", "nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
# A/B builds only (tools/ab_versions.py): extra nvcc flags, e.g. -DPCS_...
EXTRA_NVCC = os.environ.get("PCS_NVCC_EXTRA", "").split()

CU_SRCS = ["full_kernels.cu", "cluster_kernels.cu", "npdu_kernels.cu", "rows_kernels.cu", "morton_kernels.cu",
           "morton_tmem_kernels.cu", "stream_kernels.cu",
           "sample_dispatch.cu",
           "sort_kernels.cu", "metrics_kernels.cu"]
CXX_SRCS = ["capi.cpp", "pcs_api.cpp", "io.cpp"]
HEADERS = ["device_common.cuh", "sampler_common.cuh", "rows_common.cuh", "tmem.cuh", "internal.h"]


def core_path():
    return os.path.join(PKG, "_core" + sysconfig.get_config_var("EXT_SUFFIX"))


def _newer(target, deps):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def _run(cmd, verbose):
    if verbose:
        print(" ".join(cmd), flush=True)
    subprocess.run(cmd, check=True)


def _headers():
    hs = [os.path.join(CSRC, h) for h in HEADERS] + [os.path.join(INC, "pcs_gpu.h")]
    hs += [os.path.join(INC, "pcs", f) for f in os.listdir(os.path.join(INC, "pcs"))]
    return hs


def build(verbose=False):
    os.makedirs(LIBDIR, exist_ok=True)
    os.makedirs(OBJDIR, exist_ok=True)
    hdrs = _headers()
    objs, jobs = [], []
    for src in CU_SRCS:
        s = os.path.join(CSRC, src)
        o = os.path.join(OBJDIR, src + ".o")
        objs.append(o)
        if _newer(o, [s] + hdrs):
            jobs.append([NVCC, *ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC",
                         "-Xptxas", "-warn-spills", *EXTRA_NVCC, "-I", INC, "-c", s, "-o", o])
    for src in CXX_SRCS:
        s = os.path.join(CSRC, src)
        o = os.path.join(OBJDIR, src + ".o")
        objs.append(o)
        if _newer(o, [s] + hdrs):
            jobs.append(["g++", "-std=c++20", "-O2", "-fPIC", "-Wall", "-I", INC,
                         "-I", os.path.join(CUDA, "include"), "-c", s, "-o", o])
    # translation units compile in parallel (template-heavy kernels dominate)
    procs = []
    for cmd in jobs:
        if verbose:
            print(" ".join(cmd), flush=True)
        procs.append((cmd, subprocess.Popen(cmd)))
    failed = [cmd for cmd, pr in procs if pr.wait() != 0]
    if failed:
        for cmd in failed:
            out = cmd[cmd.index("-o") + 1]
            if os.path.exists(out):
                os.remove(out)
        raise subprocess.CalledProcessError(1, failed[0])
    if _newer(LIB, objs):
        _run([NVCC, *ARCH, "-shared", "-cudart", "static", "-o", LIB, *objs], verbose)
    core = core_path()
    mod_src = os.path.join(CSRC, "pybind_module.cpp")
    if _newer(core, [mod_src, LIB] + hdrs):
        import pybind11

        _run(["g++", "-std=c++20", "-O2", "-fPIC", "-shared", "-I", INC,
              "-I", pybind11.get_include(), "-I", sysconfig.get_paths()["include"],
              mod_src, "-o", core, "-L", LIBDIR, "-lpcs_gpu", "-Wl,-rpath,$ORIGIN/lib"],
             verbose)
    # the C++ drop-in API test (tests/cpp, run by the GPU suite)
    test_src = os.path.join(ROOT, "tests", "cpp", "test_pcs_api.cpp")
    test_bin = os.path.join(OBJDIR, "test_pcs_api")
    if os.path.exists(test_src) and _newer(test_bin, [test_src, LIB] + hdrs):
        _run(["g++", "-std=c++20", "-O2", "-Wall", "-I", INC, test_src, "-o", test_bin,
              "-L", LIBDIR, "-lpcs_gpu", "-Wl,-rpath,$ORIGIN/../lib"], verbose)
    return LIB, core


if __name__ == "__main__":
    build(verbose="-q" not in sys.argv)
