"""Build the native libraries in-tree (they travel to the GPU box with the repo).

libkrcuda.so  — CUDA kernels + the kr_* C ABI (include/kr_engine.h), sm_100a.
libkrhost.so  — C++ host side: instance loader, payoff assembly, sparsifier,
                bundle I/O (include/kr_host.h).
"""
from __future__ import annotations

import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PKG = os.path.join(ROOT, "paper_2112_03804_b200")
LIBDIR = os.path.join(PKG, "lib")
CUDA_SRC = [os.path.join(PKG, "csrc", "cuda", f) for f in ("kr_engine.cu", "kr_solver.cu", "kr_kron.cu", "kr_factors_dev.cu", "kr_devengine.cu", "kr_kfengine.cu", "kr_comm.cu", "kr_jit.cu")]
HOST_SRC = [os.path.join(PKG, "csrc", "host", f) for f in ("kr_host.cpp",)]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
# the system g++ links libstdc++ dynamically (a statically linked libstdc++
# inside a Python extension clashes with the process copy in iostreams)
CXX = "/usr/bin/g++" if os.path.exists("/usr/bin/g++") else "g++"

NVCC_FLAGS = [
    "-O3", "-std=c++17",
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-lineinfo",
    # bitwise parity with the reference's x86-64 build: never contract a*b+c
    "-fmad=false",
    "-ccbin", CXX,
    "-Xcompiler", "-fPIC", "-shared", "-cudart", "static",
    "-I", os.path.join(ROOT, "include"),
    "-I", os.path.join(PKG, "csrc", "cuda"),
]

CXX_FLAGS = ["-std=c++20", "-O3", "-ffp-contract=off", "-fPIC", "-shared", "-pthread", "-Wall", "-Wextra",
             "-I", os.path.join(ROOT, "include"), "-I", os.path.join(PKG, "csrc", "host")]


def _stale(target, sources):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    deps = list(sources)
    for d in (os.path.join(ROOT, "include"), os.path.join(PKG, "csrc", "cuda"), os.path.join(PKG, "csrc", "host")):
        if os.path.isdir(d):
            deps += [os.path.join(d, f) for f in os.listdir(d)]
    return any(os.path.getmtime(s) > t for s in deps if os.path.exists(s))


def build_cuda(force=False, verbose=False):
    """One object per .cu, compiled in parallel, then one shared-library link
    (no relocatable device code: kernels never cross translation units)."""
    from concurrent.futures import ThreadPoolExecutor
    os.makedirs(LIBDIR, exist_ok=True)
    out = os.path.join(LIBDIR, "libkrcuda.so")
    srcs = [s for s in CUDA_SRC if os.path.exists(s)]
    if not (force or _stale(out, srcs)):
        return out
    objdir = os.path.join(ROOT, "build", "cuda")
    os.makedirs(objdir, exist_ok=True)
    compile_flags = [f for f in NVCC_FLAGS if f not in ("-shared",)]
    objs = [os.path.join(objdir, os.path.basename(s) + ".o") for s in srcs]

    def one(so):
        s, o = so
        cmd = [NVCC, *compile_flags, "-c", "-o", o, s]
        if verbose:
            print(" ".join(cmd), file=sys.stderr)
        subprocess.run(cmd, check=True)

    with ThreadPoolExecutor(max_workers=max(1, min(len(srcs), os.cpu_count() or 1))) as ex:
        list(ex.map(one, zip(srcs, objs)))
    # NCCL is bound at run time (dlopen in kr_comm.cu), so a process shares
    # PyTorch's copy
    cmd = [NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-ccbin", CXX, "-shared", "-cudart", "static",
           "-o", out, *objs, "-ldl"]
    if verbose:
        print(" ".join(cmd), file=sys.stderr)
    subprocess.run(cmd, check=True)
    return out


def build_cuda_variant(name, defines=(), replace=None, verbose=False):
    """lib/libkrcuda_<name>.so: the same sources with extra -D flags and / or
    some translation units swapped for other files (`replace` maps a source
    basename to a path).  Loaded with KR_CUDA_LIB_VARIANT=<name>: A/B timing of
    a kernel change on one box, and the bounds-checked build (KR_CHECKED)."""
    from concurrent.futures import ThreadPoolExecutor
    replace = replace or {}
    out = os.path.join(LIBDIR, f"libkrcuda_{name}.so")
    if not replace and not _stale(out, CUDA_SRC):
        return out
    objdir = os.path.join(ROOT, "build", f"cuda_{name}")
    os.makedirs(objdir, exist_ok=True)
    srcs = [replace.get(os.path.basename(s), s) for s in CUDA_SRC]
    flags = [f for f in NVCC_FLAGS if f != "-shared"] + [f"-D{d}" for d in defines]
    objs = [os.path.join(objdir, os.path.basename(s) + ".o") for s in srcs]

    def one(so):
        cmd = [NVCC, *flags, "-c", "-o", so[1], so[0]]
        if verbose:
            print(" ".join(cmd), file=sys.stderr)
        subprocess.run(cmd, check=True)

    with ThreadPoolExecutor(max_workers=max(1, min(len(srcs), os.cpu_count() or 1))) as ex:
        list(ex.map(one, zip(srcs, objs)))
    subprocess.run([NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-ccbin", CXX, "-shared", "-cudart", "static",
                    "-o", out, *objs, "-ldl"], check=True)
    return out


def build_host(force=False, verbose=False):
    os.makedirs(LIBDIR, exist_ok=True)
    out = os.path.join(LIBDIR, "libkrhost.so")
    srcs = [s for s in HOST_SRC if os.path.exists(s)]
    if not srcs:
        return None
    if force or _stale(out, srcs):
        cmd = [CXX, *CXX_FLAGS, "-o", out, *srcs]
        if verbose:
            print(" ".join(cmd), file=sys.stderr)
        subprocess.run(cmd, check=True)
    return out


def build_cli(force=False, verbose=False):
    """krb200: the C++ CLI (tools/krb200_cli.cpp) over both C ABIs."""
    src = os.path.join(ROOT, "tools", "krb200_cli.cpp")
    out = os.path.join(LIBDIR, "krb200")
    deps = [src, os.path.join(LIBDIR, "libkrhost.so"), os.path.join(LIBDIR, "libkrcuda.so")]
    if force or _stale(out, deps):
        cmd = [CXX, "-std=c++20", "-O2", "-Wall", "-Wextra", "-I", os.path.join(ROOT, "include"), "-o", out, src,
               "-L", LIBDIR, "-lkrhost", "-lkrcuda", "-Wl,-rpath,$ORIGIN", "-ldl", "-lpthread", "-lrt"]
        if verbose:
            print(" ".join(cmd), file=sys.stderr)
        subprocess.run(cmd, check=True)
    return out


def build_all(force=False, verbose=False):
    out = build_host(force, verbose), build_cuda(force, verbose)
    build_cli(force, verbose)
    # the bounds-checked build (KR_CUDA_LIB_VARIANT=checked), kept current
    build_cuda_variant("checked", ["KR_CHECKED"], verbose=verbose)
    return out


if __name__ == "__main__":
    build_all(force="--force" in sys.argv, verbose=True)
