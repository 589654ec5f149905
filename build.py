#!/usr/bin/env python3
"""Build every native artefact in-tree (no JIT cache): the sm_100a CUDA library, the C++ API
library, the pybind11 module, and the test-infrastructure checkers under oracle/.

    python build.py            # incremental
    python build.py --force    # rebuild everything

Outputs (git-ignored, shipped to the GPU box by the gpurun snapshot):
    paper_1903_10722_b200/libffsga_cuda.so     kernels + C ABI (include/ffsga_cuda.h)
    paper_1903_10722_b200/libffsga.so          C++ API mirror of the reference (namespace ffsga)
    paper_1903_10722_b200/_core*.so            pybind11 module with the reference's Python API
    paper_1903_10722_b200/bin/ffsga            command-line front end (reference tools/main.cpp)
    oracle/liboracle.so, oracle/_ref/*.so      checkers (oracle/Makefile)
"""
from __future__ import annotations

import argparse
import concurrent.futures as cf
import os
import subprocess
import sys
import sysconfig

ROOT = os.path.dirname(os.path.abspath(__file__))
PKG = os.path.join(ROOT, "paper_1903_10722_b200")
CSRC = os.path.join(PKG, "csrc")
BUILD = os.path.join(ROOT, "build")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
CXX = os.environ.get("CXX", "g++")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVFLAGS = ["-O3", "-lineinfo", "-std=c++17", "--fmad=false", "-Xcompiler", "-fPIC",
           "-I" + os.path.join(ROOT, "include")]
CU_SOURCES = ["kernels.cu", "capi.cu"]
HOST_SOURCES = ["host/model.cpp", "host/islands.cpp", "host/solver.cpp", "host/io.cpp"]
NLOHMANN = "/opt/prime-rl/.venv/lib/python3.12/site-packages/include/cudnn_frontend/thirdparty/nlohmann"


def _newer(out, deps):
    if not os.path.exists(out):
        return True
    t = os.path.getmtime(out)
    return any(os.path.getmtime(d) > t for d in deps if os.path.exists(d))


def _run(cmd):
    print("+", " ".join(cmd), flush=True)
    subprocess.run(cmd, check=True)


def _headers(d, exts=(".h", ".cuh", ".hpp")):
    out = []
    for base, _, files in os.walk(d):
        out += [os.path.join(base, f) for f in files if f.endswith(exts)]
    return out


def build_cuda(force=False, checked=False):
    """checked: the same library with device-side bounds and invariant checks (-DFFSGA_CHECKED)
    into paper_1903_10722_b200/checked/ -- the stand-in for compute-sanitizer."""
    bdir = os.path.join(BUILD, "checked") if checked else BUILD
    os.makedirs(bdir, exist_ok=True)
    hdrs = _headers(CSRC) + [os.path.join(ROOT, "include", "ffsga_cuda.h")]
    objs, jobs = [], []
    extra = ["-DFFSGA_CHECKED"] if checked else []
    for src in CU_SOURCES:
        s = os.path.join(CSRC, src)
        o = os.path.join(bdir, src.replace(".cu", ".o"))
        objs.append(o)
        if force or _newer(o, [s] + hdrs):
            jobs.append([NVCC] + ARCH + NVFLAGS + extra + ["-c", s, "-o", o])
    with cf.ThreadPoolExecutor(max_workers=4) as ex:
        list(ex.map(_run, jobs))
    if checked:
        os.makedirs(os.path.join(PKG, "checked"), exist_ok=True)
    lib = os.path.join(PKG, "checked", "libffsga_cuda.so") if checked else os.path.join(PKG, "libffsga_cuda.so")
    if force or jobs or _newer(lib, objs):
        _run([NVCC] + ARCH + ["-shared", "-o", lib] + objs + ["-lcudart_static", "-lrt", "-ldl", "-lpthread"])
    return lib


def build_host(force=False):
    """C++ API (namespace ffsga) over the C ABI, then the pybind11 module."""
    hostdir = os.path.join(CSRC, "host")
    if not os.path.isdir(hostdir):
        return None
    inc = ["-I" + os.path.join(ROOT, "include"), "-I" + hostdir, "-I" + NLOHMANN]
    srcs = [os.path.join(CSRC, s) for s in HOST_SOURCES if os.path.exists(os.path.join(CSRC, s))]
    hdrs = _headers(hostdir) + [os.path.join(ROOT, "include", "ffsga_cuda.h")]
    lib = os.path.join(PKG, "libffsga.so")
    cuda_lib = os.path.join(PKG, "libffsga_cuda.so")
    if force or _newer(lib, srcs + hdrs + [cuda_lib]):
        _run([CXX, "-std=c++20", "-O2", "-ffp-contract=off", "-fPIC", "-shared", "-Wall", "-Wextra", "-Wno-dangling-reference"] + inc + srcs +
             ["-L" + PKG, "-lffsga_cuda", "-Wl,-rpath,$ORIGIN", "-o", lib])
    import pybind11
    mod_src = os.path.join(CSRC, "bindings", "module.cpp")
    if not os.path.exists(mod_src):
        return lib
    mod = os.path.join(PKG, "_core" + sysconfig.get_config_var("EXT_SUFFIX"))
    if force or _newer(mod, [mod_src, lib] + hdrs):
        _run([CXX, "-std=c++20", "-O2", "-ffp-contract=off", "-fPIC", "-shared"] + inc +
             ["-I" + pybind11.get_include(), "-I" + sysconfig.get_paths()["include"], mod_src,
              "-L" + PKG, "-lffsga", "-lffsga_cuda", "-Wl,-rpath,$ORIGIN", "-o", mod])
    return lib


def build_cli(force=False):
    """The command-line front end (reference proj/tools/main.cpp) -> paper_1903_10722_b200/bin/ffsga."""
    src = os.path.join(CSRC, "tools", "ffsga_cli.cpp")
    if not os.path.exists(src):
        return None
    hostdir = os.path.join(CSRC, "host")
    out = os.path.join(PKG, "bin", "ffsga")
    lib = os.path.join(PKG, "libffsga.so")
    if force or _newer(out, [src, lib] + _headers(hostdir)):
        os.makedirs(os.path.dirname(out), exist_ok=True)
        _run([CXX, "-std=c++20", "-O2", "-ffp-contract=off", "-Wall", "-Wextra", "-I" + os.path.join(ROOT, "include"),
              "-I" + hostdir, "-I" + NLOHMANN, src, "-L" + PKG, "-lffsga", "-lffsga_cuda",
              "-Wl,-rpath,$ORIGIN/..", "-o", out])
    return out


def build_oracle(force=False):
    args = ["make", "-s", "-f", os.path.join(ROOT, "oracle", "Makefile"), "all", "acceptance", "unit"]
    if force:
        args.append("-B")
    _run(args)


def main(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--force", action="store_true")
    ap.add_argument("--skip-oracle", action="store_true")
    ap.add_argument("--checked", action="store_true", help="also build the checked library (FFSGA_CHECKED)")
    a = ap.parse_args(argv)
    build_cuda(a.force)
    if a.checked:
        build_cuda(a.force, checked=True)
    build_host(a.force)
    build_cli(a.force)
    if not a.skip_oracle:
        build_oracle(a.force)


if __name__ == "__main__":
    sys.exit(main())
