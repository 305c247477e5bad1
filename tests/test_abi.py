"""CPU-side checks of the boundary: libv3db.so builds for sm_100a, loads without a GPU and
exports every function include/v3db.h declares (no compute calls here)."""
import ctypes
import os
import subprocess

import pytest

from paper_2603_03065_b200 import _lib, build as libbuild


@pytest.fixture(scope="module")
def lib_path():
    return libbuild.build()


def test_header_declares_the_north_star_entry_points():
    names = _lib.header_functions()
    for fn in ("v3db_build_snapshot", "v3db_query_batch", "v3db_free"):
        assert fn in names


def test_library_exports_every_header_symbol(lib_path):
    lib = ctypes.CDLL(lib_path)
    missing = [fn for fn in _lib.header_functions() if not hasattr(lib, fn)]
    assert missing == []
    # every declared symbol has a ctypes signature in the binding (and nothing extra)
    assert sorted(_lib._SIGS) == _lib.header_functions()


def test_library_is_sm100a_code(lib_path):
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", lib_path], capture_output=True, text=True)
    assert "sm_100a" in out.stdout


def test_error_path_without_gpu(lib_path):
    """Validation happens on the host before any CUDA call: a NULL snapshot is EINVAL."""
    lib = _lib.load(lib_path)
    rc = lib.v3db_query_batch(None, None, 0, 1, 1, None, None, None, None, None, None)
    assert rc == _lib.V3DB_EINVAL
    assert b"NULL snapshot" in lib.v3db_last_error()
    lib.v3db_free(None)  # NULL-safe


def test_no_cpu_fallback_in_product_path():
    """The product package never imports the oracle (oracle is test-only)."""
    pkg = os.path.dirname(_lib.__file__)
    for root, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh")):
                src = open(os.path.join(root, f)).read()
                assert "import oracle" not in src and "from oracle" not in src, f
