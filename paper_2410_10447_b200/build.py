"""Build the in-tree CUDA library libmdr_b200.so for sm_100a (nvcc, no JIT).

    python -m paper_2410_10447_b200.build          # incremental
    python -m paper_2410_10447_b200.build --force  # rebuild

Every translation unit is compiled with --fmad=false so double/float
expressions are evaluated exactly as written (the reference's
-ffp-contract=off, CMakeLists.txt:24); the fast paths request FMA explicitly.
"""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
INCLUDE = os.path.join(ROOT, "include")
LIB = os.path.join(HERE, "libmdr_b200.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
CU = ["reduce.cu", "dock.cu", "ls_multi.cu", "grid.cu", "cluster.cu", "bench_reduce.cu", "tc05_reduce.cu"]
CPP = ["capi.cpp", "dropin.cpp", "multi.cpp"]


def sources():
    return [os.path.join(CSRC, f) for f in CU + CPP if os.path.exists(os.path.join(CSRC, f))]


def _deps():
    files = sources()
    for d in (CSRC, INCLUDE):
        for f in os.listdir(d):
            if f.endswith((".h", ".cuh", ".hpp")):
                files.append(os.path.join(d, f))
    return files


def up_to_date(lib: str = LIB) -> bool:
    if not os.path.exists(lib):
        return False
    t = os.path.getmtime(lib)
    return all(os.path.getmtime(f) <= t for f in _deps())


def build(force: bool = False, verbose: bool = False, variant: str | None = None, defines=()) -> str:
    """Build the product library, or (variant = name, defines = ["-DX=1", ...])
    an experiment build into variants/<name>/libmdr_b200.so (A/B timing and
    instrumented runs; loaded with MDR_LIB_PATH, never by default)."""
    lib = LIB if variant is None else os.path.join(HERE, "variants", variant, "libmdr_b200.so")
    if not force and up_to_date(lib):
        return lib
    objdir = os.path.join(HERE, "build" if variant is None else os.path.join("variants", variant, "build"))
    os.makedirs(objdir, exist_ok=True)
    common = ["-O3", "-lineinfo", "-std=c++17", "--fmad=false", "-Xcompiler", "-fPIC,-ffp-contract=off",
              f"-I{INCLUDE}", f"-I{CSRC}"] + list(defines) + os.environ.get("MDR_NVCC_EXTRA", "").split()
    objs, procs = [], []
    headers = [f for f in _deps() if f not in sources()]
    flags_file = os.path.join(objdir, "flags.txt")
    flags = " ".join(common)
    same_flags = os.path.exists(flags_file) and open(flags_file).read() == flags
    for src in sources():
        obj = os.path.join(objdir, os.path.basename(src) + ".o")
        objs.append(obj)
        # incremental: an object newer than its source and every header, built
        # with the same flags, is reused (a header change rebuilds everything)
        if (not force and same_flags and os.path.exists(obj)
                and all(os.path.getmtime(f) <= os.path.getmtime(obj) for f in [src] + headers)):
            continue
        if src.endswith(".cu"):
            cmd = [NVCC, *ARCH, *common, "-c", src, "-o", obj] + (["-Xptxas", "-v"] if verbose else [])
        else:  # host-only C++ (C-ABI, drop-in C++ API): g++, C++20, no FP contraction
            cmd = [os.environ.get("CXX", "g++"), "-std=c++20", "-O2", "-fPIC", "-ffp-contract=off", "-Wall",
                   f"-I{INCLUDE}", f"-I{CSRC}", "-I/usr/local/cuda/include", *defines, "-c", src, "-o", obj]
        procs.append((src, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True)))
    for src, p in procs:
        out, _ = p.communicate()
        if p.returncode != 0:
            raise RuntimeError(f"nvcc failed for {src}:\n{out}")
        if verbose and out:
            print(out)
    with open(flags_file, "w") as f:
        f.write(flags)
    link = [NVCC, *ARCH, "-shared", "-cudart", "shared", "-Xcompiler", "-pthread", "-o", lib, *objs,
            "-Xlinker", "-rpath,/usr/local/cuda/lib64"]
    p = subprocess.run(link, capture_output=True, text=True)
    if p.returncode != 0:
        raise RuntimeError("link failed:\n" + p.stdout + p.stderr)
    return lib


if __name__ == "__main__":
    # python -m paper_2410_10447_b200.build [--force] [-v] [--variant NAME -DX=1 ...]
    argv = sys.argv[1:]
    var = argv[argv.index("--variant") + 1] if "--variant" in argv else None
    print(build(force="--force" in argv, verbose="-v" in argv, variant=var,
                defines=[a for a in argv if a.startswith("-D")]))
