"""Loading of the in-tree native libraries (ctypes over the C-ABI of include/tdg.h).

The CUDA library is built in-tree (csrc/Makefile -> lib/libtdg.so) so the exact .so
travels with the repo to the GPU box. There is no fallback: if the library is missing or
no sm_100 device is present, the product API raises.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
import threading

PKG_DIR = os.path.dirname(os.path.abspath(__file__))
LIB_DIR = os.path.join(PKG_DIR, "lib")
CSRC_DIR = os.path.join(PKG_DIR, "csrc")
# TDG_SO in the environment selects another build of the same library (A/B variants built
# with scripts/variants.sh under lib_variants/; measurement only)
TDG_SO = os.environ.get("TDG_SO") or os.path.join(LIB_DIR, "libtdg.so")

TDG_OK, TDG_ERR_INVALID, TDG_ERR_CUDA, TDG_ERR_NOMEM, TDG_ERR_RANGE, TDG_ERR_IO = 0, -1, -2, -3, -4, -5

_lock = threading.Lock()
_TDG = None


def build(jobs: int = 8) -> None:
    """Compile every native library of the package for sm_100a (nvcc cross-compiles; no GPU needed)."""
    subprocess.run(["make", "-s", "-C", CSRC_DIR, f"-j{jobs}"], check=True)


def ensure_built() -> None:
    need = [TDG_SO, os.path.join(LIB_DIR, "libtdg_gen.so")]
    if not all(os.path.exists(p) for p in need):
        build()


class TdgError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"tdg status {status}: {msg}")
        self.status = status


class tdg_csr(C.Structure):
    _fields_ = [("n", C.c_int64), ("m", C.c_int64), ("offsets", C.c_void_p), ("neighbors", C.c_void_p)]


class tdg_times(C.Structure):
    _fields_ = [(k, C.c_double) for k in ("h2d_ms", "build_ms", "support_ms", "peel_ms", "scan_ms",
                                          "process_ms", "d2h_ms", "total_ms")] + \
               [(k, C.c_uint64) for k in ("triangles", "support_probes", "levels", "sublevels", "scans", "compactions", "probes", "hits",
                                          "dead_probes")] + \
               [("t_max", C.c_uint32), ("kernel_launches", C.c_uint32), ("compact_ms", C.c_double),
                ("rebuild_ms", C.c_double), ("table_rebuilds", C.c_uint64)]

    def as_dict(self) -> dict:
        return {k: getattr(self, k) for k, _ in self._fields_}


class tdg_graph_stats(C.Structure):
    _fields_ = [(k, C.c_uint64) for k in ("n", "m", "d_max", "sum_deg_sq", "sum_dplus_sq", "wedge_count",
                                          "deg_sum_dplus_sq", "deg_s1")]

    def as_dict(self) -> dict:
        return {k: getattr(self, k) for k, _ in self._fields_}


# (name, restype, argtypes) of every entry point include/tdg.h declares.
_vp, _u64, _u32, _i32 = C.c_void_p, C.c_uint64, C.c_uint32, C.c_int
_P = C.POINTER
SIGNATURES = [
    ("tdg_version", C.c_char_p, []),
    ("tdg_last_error", C.c_char_p, []),
    ("tdg_context_create", _i32, [C.c_int, _P(_vp)]),
    ("tdg_context_destroy", _i32, [_vp]),
    ("tdg_context_set_stream", _i32, [_vp, _vp]),
    ("tdg_context_stream", _vp, [_vp]),
    ("tdg_context_trim", _i32, [_vp]),
    ("tdg_truss", _i32, [_vp, _P(tdg_csr), _vp, _vp, _vp, _u64, _P(_u64), _P(tdg_times)]),
    ("tdg_truss_device", _i32, [_vp, _P(tdg_csr), _vp, _vp, _vp, _u64, _P(_u64), _P(tdg_times)]),
    ("tdg_counters", _i32, [_vp, _P(_u64), _u64]),
    ("tdg_filter_mode", _i32, [_vp, _P(C.c_int), _P(C.c_double)]),
    ("tdg_support", _i32, [_vp, _P(tdg_csr), _vp, _P(tdg_times)]),
    ("tdg_support_device", _i32, [_vp, _P(tdg_csr), _vp, _P(tdg_times)]),
    ("tdg_support_shard", _i32, [_vp, _P(tdg_csr), _u32, _u32, _vp, _P(tdg_times)]),
    ("tdg_support_shard_device", _i32, [_vp, _P(tdg_csr), _u32, _u32, _vp, _P(tdg_times)]),
    ("tdg_build_truss_graph", _i32, [_vp, _P(tdg_csr), _vp, _vp, _vp]),
    ("tdg_stats", _i32, [_vp, _P(tdg_csr), _P(tdg_graph_stats)]),
    ("tdg_triangle_count", _i32, [_vp, _P(tdg_csr), _P(_u64), _P(tdg_times)]),
    ("tdg_ktruss_components", _i32, [_vp, _P(tdg_csr), _vp, _u32, _vp, _P(_u64)]),
    ("tdg_kcore", _i32, [_vp, _P(tdg_csr), _vp, _P(_u32)]),
    ("tdg_coreness_order", _i32, [_vp, _u64, _vp, _vp]),
    ("tdg_reorder", _i32, [_vp, _P(tdg_csr), _vp, _vp, _vp]),
    ("tdg_read_edge_list", _i32, [_vp, C.c_char_p, _P(_P(_u64)), _P(_u64)]),
    ("tdg_free", None, [_vp]),
    ("tdg_canonicalize", _i32, [_vp, _vp, _u64, _vp, _vp, _vp, _P(C.c_int64), _P(C.c_int64)]),
    ("tdg_scan", _i32, [_vp, _vp, _u64, _u32, _vp, _vp, _vp, _P(_u64)]),
    ("tdg_process_sublevel", _i32, [_vp, _P(tdg_csr), _vp, _u32, _vp, _u64, _vp, _vp, _vp, _vp, _P(_u64)]),
]


def tdg():
    """The loaded libtdg.so with typed entry points (raises if it cannot be loaded)."""
    global _TDG
    with _lock:
        if _TDG is None:
            if not os.path.exists(TDG_SO):
                ensure_built()
            L = C.CDLL(TDG_SO)
            for name, res, args in SIGNATURES:
                f = getattr(L, name)
                f.restype = res
                f.argtypes = args
            _TDG = L
    return _TDG


def check(status: int) -> None:
    if status != TDG_OK:
        raise TdgError(status, tdg().tdg_last_error().decode(errors="replace"))
