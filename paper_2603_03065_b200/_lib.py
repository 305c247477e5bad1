"""ctypes loader for libv3db.so (the C ABI of include/v3db.h).

Argument marshalling only.  The library is built in-tree by ``__graft_entry__.build()``
(or ``python -m paper_2603_03065_b200.build``); if it is missing, importing the ops
raises -- there is no CPU fallback.
"""
from __future__ import annotations

import ctypes
import os
import re

HERE = os.path.dirname(os.path.abspath(__file__))
# V3DB_LIB=debug loads the debug build (device-side invariant traps, identical results); a path to a
# .so loads that build (experiment variants under tools/)
_V = os.environ.get("V3DB_LIB", "")
LIB_PATH = (_V if _V.endswith(".so") else
            os.path.join(HERE, "libv3db_debug.so" if _V == "debug" else "libv3db.so"))
HEADER = os.path.join(os.path.dirname(HERE), "include", "v3db.h")

V3DB_OK, V3DB_EINVAL, V3DB_EINFEASIBLE, V3DB_ENOMEM, V3DB_ECUDA = range(5)
STATUS_NAMES = {0: "V3DB_OK", 1: "V3DB_EINVAL", 2: "V3DB_EINFEASIBLE", 3: "V3DB_ENOMEM", 4: "V3DB_ECUDA"}
SCAN_AUTO, SCAN_GENERIC, SCAN_ROTATED, SCAN_LIST_MAJOR = 0, 1, 2, 3
SHAPE_GREEDY, SHAPE_REBALANCE = 0, 1
FIELD_CENTROIDS, FIELD_CODEBOOKS, FIELD_IDS, FIELD_CODES, FIELD_COUNTS, FIELD_LIST_OF = range(6)
KIND_INT8, KIND_FX16 = 0, 1
(OPT_LUT_W32, OPT_COARSE_SIMT, OPT_SCHED, OPT_FX_NOROT, OPT_FX_W12, OPT_SCAN_SEG, OPT_SCAN_NS, OPT_SCAN_CAP,
 OPT_SCAN_FIRST, OPT_SCAN_DIRECT, OPT_LM_NT, OPT_AUTO_SCAN, OPT_COARSE_2PASS, OPT_SELECT_CTA, OPT_FX_COARSE, OPT_FX_SCAN, OPT_COARSE_KEYS,
 OPT_LM_STATIC) = range(18)

_c_i8p = ctypes.c_void_p
_c_i32p = ctypes.c_void_p

_SIGS = {
    "v3db_build_snapshot": (ctypes.c_int, [_c_i8p, ctypes.c_int64, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32,
                                           ctypes.c_int32, ctypes.c_int32, _c_i32p, _c_i32p, ctypes.c_void_p,
                                           ctypes.POINTER(ctypes.c_void_p)]),
    "v3db_build_snapshot_ex": (ctypes.c_int, [_c_i8p, ctypes.c_int64, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32,
                                              ctypes.c_int32, ctypes.c_int32, _c_i32p, _c_i32p, ctypes.c_int32,
                                              ctypes.c_void_p, ctypes.c_void_p, ctypes.POINTER(ctypes.c_void_p)]),
    "v3db_query_batch": (ctypes.c_int, [ctypes.c_void_p, _c_i8p, ctypes.c_int64, ctypes.c_int32, ctypes.c_int32,
                                        _c_i32p, _c_i32p, _c_i32p, _c_i32p, _c_i32p, ctypes.c_void_p]),
    "v3db_query_batch_ex": (ctypes.c_int, [ctypes.c_void_p, _c_i8p, ctypes.c_int64, ctypes.c_int32, ctypes.c_int32,
                                           _c_i32p, _c_i32p, _c_i32p, _c_i32p, _c_i32p, ctypes.c_int32,
                                           ctypes.c_void_p]),
    "v3db_query_batch_host": (ctypes.c_int, [ctypes.c_void_p, _c_i8p, ctypes.c_int64, ctypes.c_int32,
                                             ctypes.c_int32, _c_i32p, _c_i32p, _c_i32p, _c_i32p, _c_i32p,
                                             ctypes.c_void_p]),
    "v3db_witness_batch": (ctypes.c_int, [ctypes.c_void_p, _c_i8p, ctypes.c_int64, ctypes.c_int32, _c_i32p, _c_i32p,
                                          _c_i32p, _c_i32p, _c_i32p, ctypes.c_void_p]),
    "v3db_encode_fixed_point": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int64, ctypes.c_double, ctypes.c_void_p,
                                               ctypes.c_void_p]),
    "v3db_build_snapshot_fx": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32, ctypes.c_int32,
                                              ctypes.c_int32, ctypes.c_int32, ctypes.c_int32, _c_i32p, _c_i32p,
                                              ctypes.c_void_p, ctypes.POINTER(ctypes.c_void_p)]),
    "v3db_query_batch_fx": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32,
                                           ctypes.c_int32, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                           ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]),
    "v3db_query_batch_fx_host": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64, ctypes.c_double,
                                                ctypes.c_int32, ctypes.c_int32, ctypes.c_void_p, ctypes.c_void_p,
                                                ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]),
    "v3db_snapshot_kind": (ctypes.c_int, [ctypes.c_void_p]),
    "v3db_free": (None, [ctypes.c_void_p]),
    "v3db_snapshot_info": (ctypes.c_int, [ctypes.c_void_p, ctypes.POINTER(ctypes.c_int64)]),
    "v3db_snapshot_export": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int32, ctypes.c_void_p, ctypes.c_size_t]),
    "v3db_last_error": (ctypes.c_char_p, []),
    "v3db_profile_enable": (ctypes.c_int, [ctypes.c_int32]),
    "v3db_profile_read": (ctypes.c_int, [ctypes.POINTER(ctypes.c_float), ctypes.c_int32]),
    "v3db_kernel_launches": (ctypes.c_int64, []),
    "v3db_set_option": (ctypes.c_int, [ctypes.c_int32, ctypes.c_int64]),
    "v3db_get_option": (ctypes.c_int64, [ctypes.c_int32]),
}

_lib = None


class V3DBError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{STATUS_NAMES.get(status, status)}: {msg}")
        self.status = status


def header_functions(path: str = HEADER) -> list[str]:
    """Names of the functions include/v3db.h declares."""
    src = open(path).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(v3db_[a-z_0-9]+)\s*\(", src)))


def load(path: str = LIB_PATH) -> ctypes.CDLL:
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise ImportError(f"{path} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
                          "(there is no CPU fallback)")
    lib = ctypes.CDLL(path)
    for name, (res, args) in _SIGS.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def check(status: int) -> None:
    if status != V3DB_OK:
        raise V3DBError(status, load().v3db_last_error().decode(errors="replace"))
