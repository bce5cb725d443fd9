"""In-tree build of the B200 extension: csrc/*.cu + the C++ drop-in API into
paper_2506_02007_b200/lib/libeventscope_b200.so (sm_100a only).

The .so is git-ignored but travels to the GPU box with the gpurun snapshot;
nothing is JIT-compiled at import time on the box.
"""
from __future__ import annotations

import os
import shutil
import subprocess

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIBDIR = os.path.join(PKG, "lib")
LIB = os.path.join(LIBDIR, "libeventscope_b200.so")
INCLUDE = os.path.join(ROOT, "include")

GENCODE = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC", "--expt-relaxed-constexpr",
              "-I", INCLUDE] + GENCODE
CXX_FLAGS = ["-std=c++20", "-O2", "-fPIC", "-Wall", "-Wextra", "-I", INCLUDE, "-I", "/usr/local/cuda/include"]

CU_SOURCES = ["es_kernels.cu", "es_em_mma.cu", "es_em_diag.cu", "es_em_diag_tc.cu", "es_em_full.cu", "es_em_wide.cu", "es_score_mma.cu", "es_runtime.cu"]
CXX_SOURCES = ["eventscope_api.cpp"]
HEADERS = ["es_kernels.h", "es_chol.cuh", "es_layout.h", "es_tc.cuh", "es_mma.cuh"]


def _nvcc() -> str:
    for c in ("/usr/local/cuda/bin/nvcc", shutil.which("nvcc") or ""):
        if c and os.path.exists(c):
            return c
    raise RuntimeError("nvcc not found: the B200 extension cannot be built")


def _cxx() -> str:
    return "/usr/bin/g++" if os.path.exists("/usr/bin/g++") else (shutil.which("g++") or "g++")


def _inputs():
    files = [os.path.join(CSRC, f) for f in CU_SOURCES + CXX_SOURCES + HEADERS]
    for d, _, fs in os.walk(INCLUDE):
        files += [os.path.join(d, f) for f in fs]
    files.append(os.path.abspath(__file__))
    return files


def needs_build() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    return any(os.path.getmtime(f) > t for f in _inputs())


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not needs_build():
        return LIB
    os.makedirs(LIBDIR, exist_ok=True)
    objdir = os.path.join(LIBDIR, "obj")
    os.makedirs(objdir, exist_ok=True)
    nvcc = _nvcc()
    env = dict(os.environ)
    env.pop("CXX", None)
    env.pop("CC", None)
    objs = []
    procs = []
    for src in CU_SOURCES:
        obj = os.path.join(objdir, src + ".o")
        cmd = [nvcc, *NVCC_FLAGS, "-ccbin", _cxx(), "-c", os.path.join(CSRC, src), "-o", obj]
        procs.append((cmd, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT, env=env)))
        objs.append(obj)
    for src in CXX_SOURCES:
        obj = os.path.join(objdir, src + ".o")
        cmd = [_cxx(), *CXX_FLAGS, "-c", os.path.join(CSRC, src), "-o", obj]
        procs.append((cmd, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT, env=env)))
        objs.append(obj)
    for cmd, p in procs:
        out, _ = p.communicate()
        if p.returncode != 0:
            raise RuntimeError("build failed: " + " ".join(cmd) + "\n" + out.decode(errors="replace"))
        if verbose and out:
            print(out.decode(errors="replace"))
    tmp = LIB + ".tmp"
    link = [nvcc, "-shared", *GENCODE, "-ccbin", _cxx(), "-o", tmp, *objs, "-ldl"]
    r = subprocess.run(link, stdout=subprocess.PIPE, stderr=subprocess.STDOUT, env=env)
    if r.returncode != 0:
        raise RuntimeError("link failed: " + " ".join(link) + "\n" + r.stdout.decode(errors="replace"))
    os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    print(build(force=True, verbose=True))
