"""Seeded config generator (ctypes over lib/libtdg_gen.so; rules in include/tdg_gen.h).

Benchmark/test infrastructure: produces the CSR that the GPU path and the CPU
reference consume byte-identically. Not on the decomposition path.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

from ._lib import LIB_DIR, ensure_built

_GEN = None

CONFIG_NAMES = {
    1: "C1 RMAT-16 ef16 (0.57,0.19,0.19,0.05) seed1, permuted",
    2: "C2 G(n=2^22, m=33554432) seed2",
    3: "C3 RMAT-22 ef16 seed3, permuted",
    4: "C4 planted clique: G(2^21, 5*2^21) + 2000 cliques U{8..256} seed4",
    5: "C5 RMAT-25 ef16 seed5, permuted",
}


def _gen():
    global _GEN
    if _GEN is None:
        ensure_built()
        L = C.CDLL(os.path.join(LIB_DIR, "libtdg_gen.so"))
        vp = C.POINTER(C.c_void_p)
        L.tdg_gen_rmat.argtypes = [C.c_uint32, C.c_uint32, C.c_uint64, C.c_double, C.c_double,
                                   C.c_double, C.c_double, C.c_int, vp]
        L.tdg_gen_gnm.argtypes = [C.c_int64, C.c_int64, C.c_uint64, vp]
        L.tdg_gen_planted.argtypes = [C.c_int64, C.c_int64, C.c_uint32, C.c_uint32, C.c_uint32,
                                      C.c_uint64, vp]
        L.tdg_gen_config.argtypes = [C.c_int, C.c_int, vp]
        L.tdg_gen_from_pairs.argtypes = [C.c_void_p, C.c_int64, C.c_int64, vp]
        L.tdg_gen_n.argtypes = [C.c_void_p]
        L.tdg_gen_n.restype = C.c_int64
        L.tdg_gen_m.argtypes = [C.c_void_p]
        L.tdg_gen_m.restype = C.c_int64
        L.tdg_gen_fill_csr.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p]
        L.tdg_gen_free.argtypes = [C.c_void_p]
        L.tdg_gen_last_error.restype = C.c_char_p
        _GEN = L
    return _GEN


def _finish(rc, h, alloc=None):
    L = _gen()
    if rc != 0:
        raise RuntimeError("graph generator: " + L.tdg_gen_last_error().decode())
    try:
        n, m = L.tdg_gen_n(h), L.tdg_gen_m(h)
        if alloc is None:
            off = np.empty(n + 1, np.int64)
            nb = np.empty(max(2 * m, 1), np.int32)
        else:
            off, nb = alloc(n, m)
        rc = L.tdg_gen_fill_csr(h, off.ctypes.data, nb.ctypes.data)
        if rc != 0:
            raise RuntimeError("graph generator: " + L.tdg_gen_last_error().decode())
        return n, m, off, nb[: 2 * m]
    finally:
        L.tdg_gen_free(h)


def config(cfg: int, scale_override: int = 0, alloc=None):
    """CSR (n, m, offsets int64[n+1], neighbors int32[2m]) of BASELINE config 1..5.

    ``alloc(n, m) -> (offsets, neighbors)`` lets the caller supply (e.g. pinned) buffers.
    """
    h = C.c_void_p()
    rc = _gen().tdg_gen_config(cfg, scale_override, C.byref(h))
    return _finish(rc, h, alloc)


def rmat(scale: int, ef: int = 16, seed: int = 1, a=0.57, b=0.19, c=0.19, d=0.05, permute=True):
    h = C.c_void_p()
    rc = _gen().tdg_gen_rmat(scale, ef, seed, a, b, c, d, int(permute), C.byref(h))
    return _finish(rc, h)


def gnm(n: int, m: int, seed: int):
    h = C.c_void_p()
    return _finish(_gen().tdg_gen_gnm(n, m, seed, C.byref(h)), h)


def planted(n: int, m_bg: int, cliques: int, smin: int, smax: int, seed: int):
    h = C.c_void_p()
    return _finish(_gen().tdg_gen_planted(n, m_bg, cliques, smin, smax, seed, C.byref(h)), h)


def from_pairs(pairs, n_hint: int = 0):
    arr = np.ascontiguousarray(np.asarray(pairs, dtype=np.int64).reshape(-1))
    h = C.c_void_p()
    rc = _gen().tdg_gen_from_pairs(arr.ctypes.data, len(arr) // 2, n_hint, C.byref(h))
    return _finish(rc, h)
