"""oracle — CPU checkers for the PKT truss path. TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline / --impl reference)
may import this package, and only as the checker or the timed CPU baseline. The
product (paper_1707_02000_b200) never imports it.

Two checkers:
  * ``Oracle``    — ctypes over build/liboracle.so, the plain-C restatement oracle.c
                    (each function cites the reference file:line it follows).
  * ``Reference`` — ctypes over _ref/libtrussdec_ref.so, the unmodified reference
                    sources (/root/reference/proj/src) compiled by oracle/Makefile.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "build", "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libtrussdec_ref.so")

_i64p = np.ctypeslib.ndpointer(dtype=np.int64, flags="C_CONTIGUOUS")
_i32p = np.ctypeslib.ndpointer(dtype=np.int32, flags="C_CONTIGUOUS")
_u32p = np.ctypeslib.ndpointer(dtype=np.uint32, flags="C_CONTIGUOUS")
_u64p = np.ctypeslib.ndpointer(dtype=np.uint64, flags="C_CONTIGUOUS")
_u8p = np.ctypeslib.ndpointer(dtype=np.uint8, flags="C_CONTIGUOUS")


def build() -> None:
    """Compile the checkers (oracle.c always; the reference only when its tree exists)."""
    subprocess.run(["make", "-s", "-C", HERE, "all"], check=True)


@dataclass
class Csr:
    """Undirected CSR as the C-ABI takes it: int64 offsets[n+1], int32 neighbors[2m]."""
    n: int
    m: int
    offsets: np.ndarray
    neighbors: np.ndarray
    labels: np.ndarray | None = None

    @staticmethod
    def from_arrays(offsets, neighbors, labels=None) -> "Csr":
        off = np.ascontiguousarray(offsets, dtype=np.int64)
        nb = np.ascontiguousarray(neighbors, dtype=np.int32)
        return Csr(len(off) - 1, len(nb) // 2, off, nb, labels)


@dataclass
class PktResult:
    truss: np.ndarray
    nsl: list = field(default_factory=list)
    barriers: int = 0
    support: np.ndarray | None = None
    times: dict = field(default_factory=dict)


class Oracle:
    """The C restatement (oracle.c)."""

    def __init__(self, path: str = ORACLE_SO):
        if not os.path.exists(path):
            build()
        L = self.lib = C.CDLL(path)
        L.or_mt64_seed.argtypes = [C.c_void_p, C.c_uint64]
        L.or_mt64_next.argtypes = [C.c_void_p]
        L.or_mt64_next.restype = C.c_uint64
        L.or_generate_er.argtypes = [C.c_uint32, C.c_double, C.c_uint64, _u64p, C.c_int64]
        L.or_generate_er.restype = C.c_int64
        L.or_generate_rmat.argtypes = [C.c_uint32, C.c_uint32, C.c_uint64, C.c_double, C.c_double,
                                       C.c_double, C.c_double, _u64p, C.c_int64]
        L.or_generate_rmat.restype = C.c_int64
        L.or_canonicalize.argtypes = [_u64p, C.c_int64, _i64p, _i32p, _u64p,
                                      C.POINTER(C.c_int64), C.POINTER(C.c_int64)]
        L.or_build_truss_graph.argtypes = [C.c_int64, C.c_int64, _i64p, _i32p, _u32p, _u32p, _u32p]
        L.or_support_am4.argtypes = [C.c_int64, C.c_int64, _i64p, _i32p, _u32p, _u32p, _u32p]
        L.or_triangle_oracle.argtypes = [C.c_int64, C.c_int64, _i64p, _i32p, _u32p]
        L.or_triangle_oracle.restype = C.c_int64
        L.or_scan.argtypes = [C.c_int64, _u32p, C.c_uint32, _u8p, _u8p, _u32p, C.POINTER(C.c_uint64)]
        L.or_process_sublevel.argtypes = [C.c_int64, _i64p, _i32p, _u32p, _u32p, _u32p, C.c_uint32,
                                          _u32p, C.c_uint64, _u8p, _u8p, _u8p, _u32p,
                                          C.POINTER(C.c_uint64), _u32p]
        L.or_truss_pkt.argtypes = [C.c_int64, C.c_int64, _i64p, _i32p, _u32p, _u32p, _u32p,
                                   C.c_uint64, C.POINTER(C.c_uint64), C.POINTER(C.c_uint64)]
        L.or_truss_wc.argtypes = [C.c_int64, C.c_int64, _i64p, _i32p, _u32p]

        class _Stats(C.Structure):
            _fields_ = [(k, C.c_uint64) for k in ("d_max", "sum_deg_sq", "sum_dplus_sq", "wedge_count",
                                                   "deg_order_sum_dplus_sq", "deg_order_s1")]
        self._Stats = _Stats
        L.or_stats_compute.argtypes = [C.c_int64, C.c_int64, _i64p, _i32p, C.POINTER(_Stats)]

    # -- mt19937_64 restatement
    def mt64(self, seed: int, count: int) -> list[int]:
        st = (C.c_uint64 * 313)()
        self.lib.or_mt64_seed(C.cast(st, C.c_void_p), seed)
        return [self.lib.or_mt64_next(C.cast(st, C.c_void_p)) for _ in range(count)]

    # -- generators + canonicalize (tests/helpers.hpp fixtures)
    def generate_er(self, n: int, p: float, seed: int) -> np.ndarray:
        cnt = self.lib.or_generate_er(n, p, seed, np.zeros(2, np.uint64), 0)
        out = np.zeros(max(2 * cnt, 2), np.uint64)
        self.lib.or_generate_er(n, p, seed, out, cnt)
        return out[: 2 * cnt].reshape(-1, 2)

    def generate_rmat(self, scale: int, ef: int, seed: int, a=0.57, b=0.19, c=0.19, d=0.05) -> np.ndarray:
        cnt = (1 << scale) * ef
        out = np.zeros(2 * cnt, np.uint64)
        self.lib.or_generate_rmat(scale, ef, seed, a, b, c, d, out, cnt)
        return out.reshape(-1, 2)

    def canonicalize(self, pairs) -> Csr:
        pairs = np.ascontiguousarray(np.asarray(pairs, dtype=np.uint64).reshape(-1, 2))
        k = len(pairs)
        off = np.zeros(2 * k + 2, np.int64)
        nb = np.zeros(max(2 * k, 1), np.int32)
        lab = np.zeros(2 * k + 1, np.uint64)
        n, m = C.c_int64(), C.c_int64()
        rc = self.lib.or_canonicalize(pairs.reshape(-1), k, off, nb, lab, C.byref(n), C.byref(m))
        if rc != 0:
            raise MemoryError("or_canonicalize failed")
        return Csr(n.value, m.value, off[: n.value + 1].copy(), nb[: 2 * m.value].copy(),
                   lab[: n.value].copy())

    def complete_graph(self, n):
        return self.canonicalize([(u, v) for u in range(n) for v in range(u + 1, n)])

    def cycle_graph(self, n):
        return self.canonicalize([(u, (u + 1) % n) for u in range(n)])

    def star_graph(self, leaves):
        return self.canonicalize([(0, v) for v in range(1, leaves + 1)])

    def er_graph(self, n, p, seed):
        return self.canonicalize(self.generate_er(n, p, seed))

    def rmat_graph(self, scale, ef, seed):
        return self.canonicalize(self.generate_rmat(scale, ef, seed))

    # -- path functions
    def build_truss_graph(self, g: Csr):
        eo = np.zeros(max(g.n, 1), np.uint32)
        eid = np.zeros(max(2 * g.m, 1), np.uint32)
        el = np.zeros(max(2 * g.m, 1), np.uint32)
        self.lib.or_build_truss_graph(g.n, g.m, g.offsets, g.neighbors, eo, eid, el)
        return eo[: g.n], eid[: 2 * g.m], el[: 2 * g.m].reshape(-1, 2)

    def stats(self, g: Csr) -> dict:
        st = self._Stats()
        self.lib.or_stats_compute(g.n, g.m, g.offsets, g.neighbors, C.byref(st))
        return {k: getattr(st, k) for k, _ in st._fields_}

    def support_am4(self, g: Csr) -> np.ndarray:
        eo, eid, _ = self.build_truss_graph(g)
        s = np.zeros(max(g.m, 1), np.uint32)
        self.lib.or_support_am4(g.n, g.m, g.offsets, g.neighbors, np.ascontiguousarray(eo) if g.n else
                                np.zeros(1, np.uint32), np.ascontiguousarray(eid) if g.m else
                                np.zeros(1, np.uint32), s)
        return s[: g.m]

    def triangle_oracle(self, g: Csr):
        s = np.zeros(max(g.m, 1), np.uint32)
        cnt = self.lib.or_triangle_oracle(g.n, g.m, g.offsets, g.neighbors, s)
        if cnt < 0:
            raise RuntimeError("triangle_oracle: refusing graph with n > 512")
        return cnt, s[: g.m]

    def truss_pkt(self, g: Csr) -> PktResult:
        truss = np.zeros(max(g.m, 1), np.uint32)
        sup = np.zeros(max(g.m, 1), np.uint32)
        cap = max(g.m, 1) + 2
        nsl = np.zeros(cap, np.uint32)
        nlen, bar = C.c_uint64(), C.c_uint64()
        rc = self.lib.or_truss_pkt(g.n, g.m, g.offsets, g.neighbors, truss, sup, nsl, cap,
                                   C.byref(nlen), C.byref(bar))
        if rc != 0:
            raise MemoryError("or_truss_pkt failed")
        return PktResult(truss[: g.m], [int(x) for x in nsl[: nlen.value]], bar.value, sup[: g.m])

    def truss_wc(self, g: Csr) -> np.ndarray:
        truss = np.zeros(max(g.m, 1), np.uint32)
        self.lib.or_truss_wc(g.n, g.m, g.offsets, g.neighbors, truss)
        return truss[: g.m]

    def scan(self, s, level, processed, in_curr, curr):
        cs = C.c_uint64()
        self.lib.or_scan(len(s), s, level, processed, in_curr, curr, C.byref(cs))
        return cs.value

    def process_sublevel(self, g: Csr, s, level, curr, curr_size, in_curr, in_next, processed, next_):
        _, eid, el = self.build_truss_graph(g)
        ns = C.c_uint64()
        mark = np.zeros(g.n + 1, np.uint32)
        self.lib.or_process_sublevel(g.n, g.offsets, g.neighbors, np.ascontiguousarray(eid),
                                     np.ascontiguousarray(el.reshape(-1)), s, level, curr, curr_size,
                                     in_curr, in_next, processed, next_, C.byref(ns), mark)
        return ns.value


class Reference:
    """The unmodified reference library (oracle/_ref/libtrussdec_ref.so)."""

    def __init__(self, path: str = REF_SO):
        if not os.path.exists(path):
            build()
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing (build it where /root/reference exists)")
        L = self.lib = C.CDLL(path)
        L.ref_last_error.restype = C.c_char_p
        L.ref_truss_parallel.argtypes = [C.c_int64, C.c_int64, _i64p, _i32p, C.c_int, _u32p, _u32p,
                                         C.c_uint64, C.POINTER(C.c_uint64), C.POINTER(C.c_uint64),
                                         C.POINTER(C.c_double)]
        L.ref_truss_parallel_kcore.argtypes = [C.c_int64, C.c_int64, _i64p, _i32p, C.c_int,
                                               C.POINTER(C.c_double)]
        L.ref_prepare.argtypes = [C.c_int64, C.c_int64, _i64p, _i32p, C.c_int, C.c_int, C.POINTER(C.c_double)]
        L.ref_prepare.restype = C.c_void_p
        L.ref_run.argtypes = [C.c_void_p, C.c_int, C.POINTER(C.c_double), C.POINTER(C.c_uint32)]
        L.ref_free.argtypes = [C.c_void_p]
        L.ref_read_edge_list.argtypes = [C.c_char_p, C.c_void_p, C.c_uint64, C.POINTER(C.c_uint64)]
        L.ref_support_am4.argtypes = [C.c_int64, C.c_int64, _i64p, _i32p, C.c_int, _u32p]
        L.ref_build_truss_graph.argtypes = [C.c_int64, C.c_int64, _i64p, _i32p, _u32p, _u32p, _u32p]
        L.ref_truss_wc.argtypes = [C.c_int64, C.c_int64, _i64p, _i32p, _u32p]
        L.ref_truss_oracle.argtypes = [C.c_int64, C.c_int64, _i64p, _i32p, _u32p]
        L.ref_ktruss_components.argtypes = [C.c_int64, C.c_int64, _i64p, _i32p, _u32p, C.c_uint32, _u32p,
                                            C.POINTER(C.c_uint64)]
        L.ref_kcore_order.argtypes = [C.c_int64, C.c_int64, _i64p, _i32p, C.c_int, _u32p, C.POINTER(C.c_uint32),
                                      _u32p]
        L.ref_reorder.argtypes = [C.c_int64, C.c_int64, _i64p, _i32p, _u32p, _i64p, _i32p]
        L.ref_triangle_count.argtypes = [C.c_int64, C.c_int64, _i64p, _i32p, C.c_int]
        L.ref_triangle_count.restype = C.c_int64
        L.ref_make_graph.argtypes = [C.c_int, C.c_int64, C.c_double, C.c_uint64, C.c_void_p, C.c_int64,
                                     C.c_int64, C.c_int64, _i64p, _i32p, C.POINTER(C.c_int64),
                                     C.POINTER(C.c_int64)]

    def _check(self, rc):
        if rc != 0:
            raise RuntimeError(self.lib.ref_last_error().decode())

    @staticmethod
    def max_threads() -> int:
        return os.cpu_count() or 1

    def truss_parallel(self, g: Csr, workers: int) -> PktResult:
        truss = np.zeros(max(g.m, 1), np.uint32)
        cap = max(g.m, 1) + 2
        nsl = np.zeros(cap, np.uint32)
        nlen, bar = C.c_uint64(), C.c_uint64()
        t = (C.c_double * 6)()
        self._check(self.lib.ref_truss_parallel(g.n, g.m, g.offsets, g.neighbors, workers, truss, nsl,
                                                cap, C.byref(nlen), C.byref(bar), t))
        times = dict(zip(("build", "support", "scan", "processing", "engine", "total"), list(t)))
        return PktResult(truss[: g.m], [int(x) for x in nsl[: nlen.value]], bar.value, None, times)

    def truss_parallel_kcore(self, g: Csr, workers: int) -> dict:
        t = (C.c_double * 7)()
        self._check(self.lib.ref_truss_parallel_kcore(g.n, g.m, g.offsets, g.neighbors, workers, t))
        return dict(zip(("kcore", "reorder", "build", "support", "scan", "processing", "engine"), list(t)))

    def prepare(self, g: Csr, workers: int, kcore: bool):
        """Preprocess once (kcore -> coreness_order -> reorder if kcore) + build_truss_graph.
        Returns (handle, {kcore, reorder, build} seconds); run with run(), release with free()."""
        t = (C.c_double * 3)()
        h = self.lib.ref_prepare(g.n, g.m, g.offsets, g.neighbors, workers, 1 if kcore else 0, t)
        if not h:
            raise RuntimeError(self.lib.ref_last_error().decode())
        return h, dict(zip(("kcore", "reorder", "build"), list(t)))

    def run(self, h, workers: int) -> dict:
        """truss_parallel on a prepared graph: {support, scan, processing, engine, t_max}."""
        t = (C.c_double * 4)()
        tm = C.c_uint32()
        self._check(self.lib.ref_run(h, workers, t, C.byref(tm)))
        d = dict(zip(("support", "scan", "processing", "engine"), list(t)))
        d["t_max"] = tm.value
        return d

    def free(self, h):
        self.lib.ref_free(h)

    def read_edge_list(self, path: str) -> np.ndarray:
        """graph.cpp:152-200: (k, 2) uint64 pairs; raises RuntimeError with the reference's message."""
        k = C.c_uint64()
        buf = np.zeros(2 * 1024, np.uint64)
        self._check(self.lib.ref_read_edge_list(os.fsencode(path), buf.ctypes.data, 1024, C.byref(k)))
        if k.value > 1024:
            buf = np.zeros(2 * k.value, np.uint64)
            self._check(self.lib.ref_read_edge_list(os.fsencode(path), buf.ctypes.data, k.value, C.byref(k)))
        return buf[: 2 * k.value].reshape(-1, 2)

    def support_am4(self, g: Csr, workers: int = 1) -> np.ndarray:
        s = np.zeros(max(g.m, 1), np.uint32)
        self._check(self.lib.ref_support_am4(g.n, g.m, g.offsets, g.neighbors, workers, s))
        return s[: g.m]

    def build_truss_graph(self, g: Csr):
        eo = np.zeros(max(g.n, 1), np.uint32)
        eid = np.zeros(max(2 * g.m, 1), np.uint32)
        el = np.zeros(max(2 * g.m, 1), np.uint32)
        self._check(self.lib.ref_build_truss_graph(g.n, g.m, g.offsets, g.neighbors, eo, eid, el))
        return eo[: g.n], eid[: 2 * g.m], el[: 2 * g.m].reshape(-1, 2)

    def truss_wc(self, g: Csr) -> np.ndarray:
        t = np.zeros(max(g.m, 1), np.uint32)
        self._check(self.lib.ref_truss_wc(g.n, g.m, g.offsets, g.neighbors, t))
        return t[: g.m]

    def truss_oracle(self, g: Csr) -> np.ndarray:
        t = np.zeros(max(g.m, 1), np.uint32)
        self._check(self.lib.ref_truss_oracle(g.n, g.m, g.offsets, g.neighbors, t))
        return t[: g.m]

    def ktruss_subgraphs(self, g: Csr, truss, k: int) -> list[list[int]]:
        """truss_serial.cpp:176-210 on the reference library; raises on invalid k."""
        comp = np.zeros(max(g.m, 1), np.uint32)
        nc = C.c_uint64()
        tr = np.ascontiguousarray(truss, np.uint32) if g.m else np.zeros(1, np.uint32)
        self._check(self.lib.ref_ktruss_components(g.n, g.m, g.offsets, g.neighbors, tr, k, comp, C.byref(nc)))
        out = [[] for _ in range(nc.value)]
        for e, c in enumerate(comp[: g.m].tolist()):
            if c != 0xFFFFFFFF:
                out[c].append(e)
        return out

    def kcore_order(self, g: Csr, workers: int = 1):
        """kcore_parallel + coreness_order: (core[n], c_max, perm[n])."""
        core = np.zeros(max(g.n, 1), np.uint32)
        perm = np.zeros(max(g.n, 1), np.uint32)
        cm = C.c_uint32()
        self._check(self.lib.ref_kcore_order(g.n, g.m, g.offsets, g.neighbors, workers, core, C.byref(cm), perm))
        return core[: g.n], cm.value, perm[: g.n]

    def reorder(self, g: Csr, perm) -> Csr:
        off = np.zeros(g.n + 1, np.int64)
        nb = np.zeros(max(2 * g.m, 1), np.int32)
        self._check(self.lib.ref_reorder(g.n, g.m, g.offsets, g.neighbors, np.ascontiguousarray(perm, np.uint32),
                                         off, nb))
        return Csr(g.n, g.m, off, nb[: 2 * g.m])

    def triangle_count(self, g: Csr, workers: int = 1) -> int:
        return int(self.lib.ref_triangle_count(g.n, g.m, g.offsets, g.neighbors, workers))

    def make_graph(self, kind: int, a: int, b: float, seed: int, pairs=None) -> Csr:
        cap_n, cap_nb = 1 << 20, 1 << 24
        if pairs is not None:
            cap_n = max(cap_n, 2 * len(pairs) + 1)
            cap_nb = max(cap_nb, 2 * len(pairs))
        off = np.zeros(cap_n + 1, np.int64)
        nb = np.zeros(cap_nb, np.int32)
        n, m = C.c_int64(), C.c_int64()
        pp = None
        if pairs is not None:
            arr = np.ascontiguousarray(np.asarray(pairs, dtype=np.int64).reshape(-1))
            pp, npairs = arr.ctypes.data_as(C.c_void_p), len(arr) // 2
        else:
            npairs = 0
        self._check(self.lib.ref_make_graph(kind, a, b, seed, pp, npairs, cap_n, cap_nb, off, nb,
                                            C.byref(n), C.byref(m)))
        return Csr(n.value, m.value, off[: n.value + 1].copy(), nb[: 2 * m.value].copy())
