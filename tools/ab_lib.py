#!/usr/bin/env python3
"""Build an A/B variant of libmdr_b200.so: recompile ONE source with extra
nvcc flags and link it with the in-tree objects of everything else.

  python tools/ab_lib.py grid.cu ab/lib_u4.so -DMDR_GRID_UNROLL=4
"""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "paper_2410_10447_b200"))
import build as b  # noqa: E402

src, out, extra = sys.argv[1], sys.argv[2], sys.argv[3:]
b.build()
objdir = os.path.join(b.HERE, "build")
os.makedirs(os.path.dirname(os.path.abspath(out)), exist_ok=True)
var = os.path.abspath(out) + ".o"
common = ["-O3", "-lineinfo", "-std=c++17", "--fmad=false", "-Xcompiler", "-fPIC,-ffp-contract=off",
          f"-I{b.INCLUDE}", f"-I{b.CSRC}"]
subprocess.run([b.NVCC, *b.ARCH, *common, *extra, "-c", os.path.join(b.CSRC, src), "-o", var], check=True)
objs = [var if os.path.basename(s) == src else os.path.join(objdir, os.path.basename(s) + ".o") for s in b.sources()]
subprocess.run([b.NVCC, *b.ARCH, "-shared", "-cudart", "shared", "-Xcompiler", "-pthread", "-o", out, *objs,
                "-Xlinker", "-rpath,/usr/local/cuda/lib64"], check=True)
os.remove(var)
print(out)
