"""The C-ABI boundary (include/mdr.h): the built library loads without a GPU
and exports every function the header declares, and the Python binding
declares a prototype for each of them.  No compute calls (CPU suite)."""
import ctypes
import os
import re

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_functions():
    src = open(os.path.join(ROOT, "include", "mdr.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(mdr_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_header_function():
    from paper_2410_10447_b200 import build

    lib = ctypes.CDLL(build.build())
    names = header_functions()
    assert len(names) > 40
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing


def test_python_binding_covers_header():
    from paper_2410_10447_b200 import _lib

    declared = set(_lib.exported_symbols()) | set(_lib._OPTIONAL)
    missing = [n for n in header_functions() if n not in declared]
    assert not missing, missing
