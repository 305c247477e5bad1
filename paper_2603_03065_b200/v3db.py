"""Thin Python binding of the C ABI (include/v3db.h) -- same entry points, argument
marshalling only.  Every query step runs in libv3db.so's CUDA kernels; torch is used for
device memory and streams only.  Functions mirror the C names without the ``v3db_`` prefix:

  build_snapshot(db, nlist, list_cap, m, ks, centroid_rows, codeword_rows, stream=None) -> Snapshot
  query_batch(s, queries, nprobe, k, trace=True, algo=SCAN_AUTO, out=None, stream=None) -> dict
  query_batch_host(s, queries_host, nprobe, k, out) -> None          (end-to-end, host buffers)
  snapshot_info(s) -> dict;  snapshot_export(s, field) -> numpy array;  free(s)
  NEXT-1, 16-bit fixed point: encode_fixed_point(x, v_max) -> int32 tensor;
  build_snapshot_fx(db_int32, ...) -> Snapshot;  query_batch_fx(s, queries_int32, nprobe, k) -> dict
"""
from __future__ import annotations

import ctypes

import numpy as np
import torch

from . import _lib
from ._lib import (FIELD_CENTROIDS, FIELD_CODEBOOKS, FIELD_CODES, FIELD_COUNTS, FIELD_IDS,  # noqa: F401
                   FIELD_LIST_OF, KIND_FX16, KIND_INT8, SCAN_AUTO, SCAN_GENERIC, SCAN_ROTATED, SCAN_LIST_MAJOR, SHAPE_GREEDY, SHAPE_REBALANCE,
                   V3DBError, OPT_LUT_W32, OPT_COARSE_SIMT, OPT_SCHED, OPT_FX_NOROT, OPT_FX_W12,
                   OPT_SCAN_SEG, OPT_SCAN_NS, OPT_SCAN_CAP, OPT_SCAN_FIRST, OPT_SCAN_DIRECT, OPT_LM_NT, OPT_AUTO_SCAN, OPT_COARSE_2PASS,
                   OPT_SELECT_CTA, OPT_FX_COARSE, OPT_FX_SCAN, OPT_COARSE_KEYS, OPT_LM_STATIC)


def _stream_ptr(stream) -> ctypes.c_void_p:
    if stream is None:
        stream = torch.cuda.current_stream()
    return ctypes.c_void_p(stream.cuda_stream)


def _ptr(t) -> ctypes.c_void_p:
    return ctypes.c_void_p(t.data_ptr()) if t is not None else ctypes.c_void_p(0)


def _need(t: torch.Tensor, dtype, device_type: str, shape, name: str) -> None:
    if t.dtype != dtype or t.device.type != device_type or tuple(t.shape) != tuple(shape) or not t.is_contiguous():
        raise ValueError(f"{name}: expected contiguous {dtype} {device_type} tensor of shape {tuple(shape)}, got "
                         f"{t.dtype} {t.device} {tuple(t.shape)}")


class Snapshot:
    """Owner of a v3db_snapshot_t handle (library-owned device memory)."""

    def __init__(self, handle: ctypes.c_void_p):
        self._h = handle
        self.info = snapshot_info(self)
        self.kind = int(_lib.load().v3db_snapshot_kind(handle))

    @property
    def handle(self) -> ctypes.c_void_p:
        if not self._h:
            raise ValueError("snapshot has been freed")
        return self._h

    def __getattr__(self, name):
        info = self.__dict__.get("info")
        if info is not None and name in info:
            return info[name]
        raise AttributeError(name)

    def free(self) -> None:
        if self._h:
            _lib.load().v3db_free(self._h)
            self._h = None

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass


def build_snapshot(db: torch.Tensor, nlist: int, list_cap: int, m: int, ks: int, centroid_rows, codeword_rows,
                   stream=None, rule: int = 0, stats: dict | None = None) -> Snapshot:
    """v3db_build_snapshot(_ex): db is a CUDA int8 [n][dim] tensor; the row samples are host arrays.
    rule = SHAPE_GREEDY (BASELINE.json) or SHAPE_REBALANCE (the paper's Alg. 1); `stats`, if given,
    receives {"moved", "rounds"}."""
    lib = _lib.load()
    if db.dtype != torch.int8 or db.device.type != "cuda" or db.dim() != 2 or not db.is_contiguous():
        raise ValueError("db must be a contiguous CUDA int8 [n][dim] tensor")
    cent = np.ascontiguousarray(np.asarray(centroid_rows, dtype=np.int32).reshape(-1))
    code = np.ascontiguousarray(np.asarray(codeword_rows, dtype=np.int32).reshape(-1))
    if cent.size != nlist or code.size != m * ks:
        raise ValueError("centroid_rows must have nlist entries and codeword_rows m*ks entries")
    h = ctypes.c_void_p()
    st = (ctypes.c_int64 * 2)()
    _lib.check(lib.v3db_build_snapshot_ex(_ptr(db), db.shape[0], db.shape[1], nlist, list_cap, m, ks,
                                          cent.ctypes.data_as(ctypes.c_void_p), code.ctypes.data_as(ctypes.c_void_p),
                                          rule, ctypes.cast(st, ctypes.c_void_p), _stream_ptr(stream),
                                          ctypes.byref(h)))
    if stats is not None:
        stats.update(moved=int(st[0]), rounds=int(st[1]))
    return Snapshot(h)


def encode_fixed_point(x: torch.Tensor, v_max: float, stream=None) -> torch.Tensor:
    """v3db_encode_fixed_point: round((2^16 - 1) v / v_max) of a CUDA float32 tensor (PAPER.md:781-782,
    DESIGN.md R18) -> CUDA int32 tensor of the same shape."""
    lib = _lib.load()
    if x.dtype != torch.float32 or x.device.type != "cuda" or not x.is_contiguous():
        raise ValueError("x must be a contiguous CUDA float32 tensor")
    out = torch.empty(x.shape, dtype=torch.int32, device=x.device)
    _lib.check(lib.v3db_encode_fixed_point(_ptr(x), x.numel(), float(v_max), _ptr(out), _stream_ptr(stream)))
    return out


def build_snapshot_fx(db: torch.Tensor, nlist: int, list_cap: int, m: int, ks: int, centroid_rows, codeword_rows,
                      stream=None) -> Snapshot:
    """v3db_build_snapshot_fx: db is a CUDA int32 [n][dim] tensor of 16-bit fixed-point coordinates."""
    lib = _lib.load()
    if db.dtype != torch.int32 or db.device.type != "cuda" or db.dim() != 2 or not db.is_contiguous():
        raise ValueError("db must be a contiguous CUDA int32 [n][dim] tensor")
    cent = np.ascontiguousarray(np.asarray(centroid_rows, dtype=np.int32).reshape(-1))
    code = np.ascontiguousarray(np.asarray(codeword_rows, dtype=np.int32).reshape(-1))
    if cent.size != nlist or code.size != m * ks:
        raise ValueError("centroid_rows must have nlist entries and codeword_rows m*ks entries")
    h = ctypes.c_void_p()
    _lib.check(lib.v3db_build_snapshot_fx(_ptr(db), db.shape[0], db.shape[1], nlist, list_cap, m, ks,
                                          cent.ctypes.data_as(ctypes.c_void_p), code.ctypes.data_as(ctypes.c_void_p),
                                          _stream_ptr(stream), ctypes.byref(h)))
    return Snapshot(h)


def query_batch_fx(s: Snapshot, queries: torch.Tensor, nprobe: int, k: int, trace: bool = True,
                   out: dict | None = None, stream=None) -> dict:
    """v3db_query_batch_fx: Steps 1-5 on a fixed-point snapshot.  out_ids (int32) / out_dist (int64)
    [nq][k]; with trace, trace_lists (int32) / trace_list_dist (int64) [nq][nprobe] and
    trace_cand_dist (int64) [nq][nprobe][L]."""
    lib = _lib.load()
    nq = queries.shape[0]
    _need(queries, torch.int32, "cuda", (nq, s.dim), "queries")
    if out is None:
        out = alloc_outputs_fx(s, nq, nprobe, k, trace, device=queries.device)
    _need(out["out_ids"], torch.int32, "cuda", (nq, k), "out_ids")
    _need(out["out_dist"], torch.int64, "cuda", (nq, k), "out_dist")
    for key, dt, shape in (("trace_lists", torch.int32, (nq, nprobe)), ("trace_list_dist", torch.int64, (nq, nprobe)),
                           ("trace_cand_dist", torch.int64, (nq, nprobe, s.list_cap))):
        if out.get(key) is not None:
            _need(out[key], dt, "cuda", shape, key)
    _lib.check(lib.v3db_query_batch_fx(s.handle, _ptr(queries), nq, nprobe, k, _ptr(out["out_ids"]),
                                       _ptr(out["out_dist"]), _ptr(out.get("trace_lists")),
                                       _ptr(out.get("trace_list_dist")), _ptr(out.get("trace_cand_dist")),
                                       _stream_ptr(stream)))
    return out


def query_batch_fx_host(s: Snapshot, queries: torch.Tensor, v_max: float, nprobe: int, k: int, out: dict,
                        stream=None) -> dict:
    """v3db_query_batch_fx_host: HOST float32 queries and HOST output buffers (alloc_outputs_fx with
    device="cpu", pin=True); the call copies in, encodes, runs Steps 1-5, copies out, synchronizes."""
    lib = _lib.load()
    nq = queries.shape[0]
    _need(queries, torch.float32, "cpu", (nq, s.dim), "queries")
    _need(out["out_ids"], torch.int32, "cpu", (nq, k), "out_ids")
    _need(out["out_dist"], torch.int64, "cpu", (nq, k), "out_dist")
    tl, tld, tcd = out.get("trace_lists"), out.get("trace_list_dist"), out.get("trace_cand_dist")
    if tl is not None:
        _need(tl, torch.int32, "cpu", (nq, nprobe), "trace_lists")
    if tld is not None:
        _need(tld, torch.int64, "cpu", (nq, nprobe), "trace_list_dist")
    if tcd is not None:
        _need(tcd, torch.int64, "cpu", (nq, nprobe, s.list_cap), "trace_cand_dist")
    _lib.check(lib.v3db_query_batch_fx_host(s.handle, _ptr(queries), nq, float(v_max), nprobe, k, _ptr(out["out_ids"]),
                                            _ptr(out["out_dist"]), _ptr(tl), _ptr(tld), _ptr(tcd),
                                            _stream_ptr(stream)))
    return out


def alloc_outputs_fx(s: Snapshot, nq: int, nprobe: int, k: int, trace: bool = True, device="cuda",
                     pin=False) -> dict:
    """Output buffers of query_batch_fx (int32 ids / lists, int64 distances)."""
    def t(shape, dt):
        return torch.empty(shape, dtype=dt, device=device, pin_memory=(device == "cpu" and pin))
    out = {"out_ids": t((nq, k), torch.int32), "out_dist": t((nq, k), torch.int64)}
    if trace:
        out["trace_lists"] = t((nq, nprobe), torch.int32)
        out["trace_list_dist"] = t((nq, nprobe), torch.int64)
        out["trace_cand_dist"] = t((nq, nprobe, s.list_cap), torch.int64)
    return out


def alloc_outputs(s: Snapshot, nq: int, nprobe: int, k: int, trace: bool = True, device="cuda", pin=False) -> dict:
    kw = dict(dtype=torch.int32, device=device)
    if device == "cpu" and pin:
        kw["pin_memory"] = True
    out = {"out_ids": torch.empty((nq, k), **kw), "out_dist": torch.empty((nq, k), **kw)}
    if trace:
        out["trace_lists"] = torch.empty((nq, nprobe), **kw)
        out["trace_list_dist"] = torch.empty((nq, nprobe), **kw)
        out["trace_cand_dist"] = torch.empty((nq, nprobe, s.list_cap), **kw)
    return out


def query_batch(s: Snapshot, queries: torch.Tensor, nprobe: int, k: int, trace: bool = True,
                algo: int = SCAN_AUTO, out: dict | None = None, stream=None) -> dict:
    """v3db_query_batch(_ex): Steps 1-5 on the GPU.  Returns (or fills) a dict of CUDA int32
    tensors out_ids/out_dist [nq][k] and, with trace, trace_lists/trace_list_dist [nq][nprobe],
    trace_cand_dist [nq][nprobe][L]."""
    lib = _lib.load()
    nq = queries.shape[0]
    _need(queries, torch.int8, "cuda", (nq, s.dim), "queries")
    if out is None:
        out = alloc_outputs(s, nq, nprobe, k, trace, device=queries.device)
    _need(out["out_ids"], torch.int32, "cuda", (nq, k), "out_ids")
    _need(out["out_dist"], torch.int32, "cuda", (nq, k), "out_dist")
    tl, tld, tcd = out.get("trace_lists"), out.get("trace_list_dist"), out.get("trace_cand_dist")
    if tl is not None:
        _need(tl, torch.int32, "cuda", (nq, nprobe), "trace_lists")
    if tld is not None:
        _need(tld, torch.int32, "cuda", (nq, nprobe), "trace_list_dist")
    if tcd is not None:
        _need(tcd, torch.int32, "cuda", (nq, nprobe, s.list_cap), "trace_cand_dist")
    _lib.check(lib.v3db_query_batch_ex(s.handle, _ptr(queries), nq, nprobe, k, _ptr(out["out_ids"]),
                                       _ptr(out["out_dist"]), _ptr(tl), _ptr(tld), _ptr(tcd), algo,
                                       _stream_ptr(stream)))
    return out


def query_batch_host(s: Snapshot, queries: torch.Tensor, nprobe: int, k: int, out: dict, stream=None) -> dict:
    """v3db_query_batch_host: HOST buffers (pin them for asynchronous DMA); the call copies
    queries in, runs Steps 1-5 on the GPU, copies the outputs back and synchronizes."""
    lib = _lib.load()
    nq = queries.shape[0]
    _need(queries, torch.int8, "cpu", (nq, s.dim), "queries")
    for name in ("out_ids", "out_dist"):
        _need(out[name], torch.int32, "cpu", (nq, k), name)
    tl, tld, tcd = out.get("trace_lists"), out.get("trace_list_dist"), out.get("trace_cand_dist")
    if tl is not None:
        _need(tl, torch.int32, "cpu", (nq, nprobe), "trace_lists")
    if tld is not None:
        _need(tld, torch.int32, "cpu", (nq, nprobe), "trace_list_dist")
    if tcd is not None:
        _need(tcd, torch.int32, "cpu", (nq, nprobe, s.list_cap), "trace_cand_dist")
    _lib.check(lib.v3db_query_batch_host(s.handle, _ptr(queries), nq, nprobe, k, _ptr(out["out_ids"]),
                                         _ptr(out["out_dist"]), _ptr(tl), _ptr(tld), _ptr(tcd),
                                         _stream_ptr(stream)))
    return out


def witness_batch(s: Snapshot, queries: torch.Tensor, nprobe: int, lut_sel: bool = True, stream=None) -> dict:
    """v3db_witness_batch: the prover witness of each query (§4.7) as CUDA int32 tensors:
    list_order/list_dist [nq][nlist] (S^sorted_idx,dist), lut_sel [nq][nprobe][L][M] (selected LUT
    entries), cand_items/cand_dist [nq][nprobe*L] (S^sorted_item,dist)."""
    lib = _lib.load()
    nq = queries.shape[0]
    _need(queries, torch.int8, "cuda", (nq, s.dim), "queries")
    kw = dict(dtype=torch.int32, device=queries.device)
    nsel = nprobe * s.list_cap
    out = {"list_order": torch.empty((nq, s.nlist), **kw), "list_dist": torch.empty((nq, s.nlist), **kw),
           "cand_items": torch.empty((nq, nsel), **kw), "cand_dist": torch.empty((nq, nsel), **kw)}
    if lut_sel:
        out["lut_sel"] = torch.empty((nq, nprobe, s.list_cap, s.m), **kw)
    _lib.check(lib.v3db_witness_batch(s.handle, _ptr(queries), nq, nprobe, _ptr(out["list_order"]),
                                      _ptr(out["list_dist"]), _ptr(out.get("lut_sel")), _ptr(out["cand_items"]),
                                      _ptr(out["cand_dist"]), _stream_ptr(stream)))
    return out


_INFO_KEYS = ("n", "dim", "nlist", "list_cap", "m", "ks", "d", "total_valid")


def snapshot_info(s: Snapshot) -> dict:
    buf = (ctypes.c_int64 * 8)()
    _lib.check(_lib.load().v3db_snapshot_info(s.handle, buf))
    return dict(zip(_INFO_KEYS, list(buf)))


def snapshot_export(s: Snapshot, field: int) -> np.ndarray:
    """v3db_snapshot_export: canonical snapshot arrays as numpy (test-only introspection)."""
    i = s.info
    wide = np.int32 if s.kind == KIND_FX16 else np.int8
    shapes = {
        FIELD_CENTROIDS: ((i["nlist"], i["dim"]), wide),
        FIELD_CODEBOOKS: ((i["m"], i["ks"], i["d"]), wide),
        FIELD_IDS: ((i["nlist"], i["list_cap"]), np.int32),
        FIELD_CODES: ((i["nlist"], i["list_cap"], i["m"]), np.uint8),
        FIELD_COUNTS: ((i["nlist"],), np.int32),
        FIELD_LIST_OF: ((i["n"],), np.int32),
    }
    shape, dt = shapes[field]
    arr = np.empty(shape, dtype=dt)
    _lib.check(_lib.load().v3db_snapshot_export(s.handle, field, arr.ctypes.data_as(ctypes.c_void_p), arr.nbytes))
    return arr


def free(s: Snapshot) -> None:
    s.free()


def profile_enable(on: bool = True) -> None:
    """v3db_profile_enable: record CUDA events around each query kernel (bench.py)."""
    _lib.check(_lib.load().v3db_profile_enable(1 if on else 0))


def profile_read(detail: bool = False) -> tuple:
    """v3db_profile_read: (coarse ms, scan ms) of the most recent profiled query call; with
    detail=True (coarse, scan, scan main kernel, scan prologue, scan epilogue) in ms."""
    buf = (ctypes.c_float * 5)()
    _lib.check(_lib.load().v3db_profile_read(buf, 5))
    return tuple(float(x) for x in buf) if detail else (float(buf[0]), float(buf[1]))


def kernel_launches() -> int:
    """v3db_kernel_launches: kernels launched by libv3db since load."""
    return int(_lib.load().v3db_kernel_launches())


def set_option(key: int, value: int) -> int:
    """v3db_set_option (V3DB_OPT_* keys, 0 = default); returns the previous value."""
    lib = _lib.load()
    prev = int(lib.v3db_get_option(key))
    _lib.check(lib.v3db_set_option(key, int(value)))
    return prev


class option:
    """Context manager: `with v3db.option(v3db.OPT_LUT_W32, 1): ...` restores the old value."""

    def __init__(self, key: int, value: int):
        self.key, self.value, self.prev = key, value, None

    def __enter__(self):
        self.prev = set_option(self.key, self.value)
        return self

    def __exit__(self, *exc):
        set_option(self.key, self.prev)
        return False
