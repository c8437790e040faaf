"""The drop-in C++ API (include/mdreduce_b200.hpp): it compiles against the
header, links libmdr_b200.so, and the reference's own test scenarios
(tests/cpp/test_dropin.cpp) pass on the GPU."""
import os
import subprocess

import pytest

from paper_2410_10447_b200._abi import Instance, serialize_instance

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIBDIR = os.path.join(ROOT, "paper_2410_10447_b200")


def _compile(tmp_path):
    exe = tmp_path / "test_dropin"
    cmd = ["g++", "-std=c++20", "-O1", f"-I{ROOT}/include", os.path.join(ROOT, "tests", "cpp", "test_dropin.cpp"),
           f"-L{LIBDIR}", "-lmdr_b200", f"-Wl,-rpath,{LIBDIR}", "-o", str(exe)]
    subprocess.run(cmd, check=True, capture_output=True, text=True)
    return exe


def test_dropin_header_compiles_and_links(tmp_path):
    from paper_2410_10447_b200 import build

    build.build()
    assert _compile(tmp_path).exists()


@pytest.mark.gpu
def test_dropin_reference_scenarios_on_gpu(tmp_path, instances, dev):
    exe = _compile(tmp_path)
    for name in ("s1", "s2", "s3"):
        inst: Instance = instances[name]
        (tmp_path / f"{name}.mdri").write_text(serialize_instance(inst))
    out = subprocess.run([str(exe), str(tmp_path)], capture_output=True, text=True, timeout=600)
    print(out.stdout)
    assert out.returncode == 0, out.stdout + out.stderr
