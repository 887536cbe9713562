"""Python host mirror of the reference's truss-decomposition interface, over the C-ABI.

Names, argument meaning and error behaviour follow the reference (paths relative to
/root/reference/proj):

  build_truss_graph(CsrGraph) -> TrussGraph              include/trussdec/graph.hpp:69
  stats(CsrGraph) -> GraphStats                          graph.hpp:74
  support_am4(TrussGraph, workers) -> SupportArray       include/trussdec/triangle.hpp:16
  triangle_count(TrussGraph, workers) -> int             triangle.hpp:19 (triangle.cpp:90-116)
  truss_parallel(TrussGraph, workers) -> ParallelDecomposition
                                                         include/trussdec/truss_parallel.hpp:72
  scan(s, level, LevelFrontier, workers)                 truss_parallel.hpp:62
  process_sublevel(LevelFrontier, TrussGraph, s, level, MarkScratchPool, workers)
                                                         truss_parallel.hpp:67-68

Everything computes on the B200 through lib/libtdg.so; there is no CPU path. Errors map
like the C++ shim: TDG_ERR_INVALID -> ValueError (std::invalid_argument),
TDG_ERR_NOMEM -> MemoryError (std::bad_alloc), others -> RuntimeError.
Arrays are numpy (uint32 per-edge, int64 offsets, int32 neighbours).
"""
from __future__ import annotations

import ctypes as C
import os
import threading
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from ._lib import tdg_csr, tdg_graph_stats, tdg_times


def _raise(status: int):
    msg = _lib.tdg().tdg_last_error().decode(errors="replace")
    if status == _lib.TDG_ERR_INVALID:
        raise ValueError(msg)
    if status == _lib.TDG_ERR_NOMEM:
        raise MemoryError(msg)
    raise RuntimeError(f"tdg status {status}: {msg}")


def _ck(status: int):
    if status != _lib.TDG_OK:
        _raise(status)


def _ptr(a) -> int | None:
    if a is None:
        return None
    if hasattr(a, "data_ptr"):  # torch tensor
        return a.data_ptr()
    return a.ctypes.data


@dataclass
class CsrGraph:
    """graph.hpp:21-31 (offsets widened to int64 at the C-ABI; ids int32)."""
    n: int
    m: int
    offsets: np.ndarray
    neighbors: np.ndarray
    labels: np.ndarray | None = None

    @staticmethod
    def from_arrays(offsets, neighbors, labels=None) -> "CsrGraph":
        off = np.ascontiguousarray(offsets, dtype=np.int64)
        nb = np.ascontiguousarray(neighbors, dtype=np.int32)
        if len(off) == 0:
            off = np.zeros(1, np.int64)
        return CsrGraph(len(off) - 1, len(nb) // 2, off, nb, labels)

    def degree(self, u: int) -> int:
        return int(self.offsets[u + 1] - self.offsets[u])

    def label_of(self, u: int) -> int:
        return u if self.labels is None else int(self.labels[u])

    def _view(self) -> tdg_csr:
        nb = self.neighbors if len(self.neighbors) else np.zeros(1, np.int32)
        self._keep = nb
        return tdg_csr(self.n, self.m, self.offsets.ctypes.data, nb.ctypes.data)


@dataclass
class TrussGraph:
    """graph.hpp:35-49: CSR + eid[2m] + el[m] (u<v) + eo[n]."""
    csr: CsrGraph
    eid: np.ndarray
    el: np.ndarray
    eo: np.ndarray

    def n(self) -> int:
        return self.csr.n

    def m(self) -> int:
        return self.csr.m

    @staticmethod
    def core_array_bytes(n: int, m: int) -> int:
        return 28 * m + 8 * n


@dataclass
class TrussnessResult:
    """truss_serial.hpp:12-18."""
    truss: np.ndarray
    t_max: int = 0
    kclass_sizes: dict = field(default_factory=dict)

    def finalize(self):  # truss_serial.cpp:10-17
        if len(self.truss):
            vals, cnt = np.unique(self.truss, return_counts=True)
            self.kclass_sizes = {int(v): int(c) for v, c in zip(vals, cnt)}
            self.t_max = int(vals[-1])
        else:
            self.kclass_sizes, self.t_max = {}, 0


@dataclass
class SubLevelTrace:
    """truss_parallel.hpp:27-40."""
    nsl: list = field(default_factory=list)
    barriers: int = 0

    def sublevel_total(self) -> int:
        return int(sum(self.nsl))

    def expected_barriers(self, t_max: int) -> int:
        return t_max + 2 * self.sublevel_total()


@dataclass
class PhaseTimes:
    """truss_parallel.hpp:42-46 (seconds)."""
    support: float = 0.0
    scan: float = 0.0
    processing: float = 0.0


@dataclass
class ParallelDecomposition:
    """truss_parallel.hpp:48-52, plus the GPU's own timing/trace record (`gpu`)."""
    result: TrussnessResult
    trace: SubLevelTrace
    times: PhaseTimes
    gpu: dict = field(default_factory=dict)


class LevelFrontier:
    """truss_parallel.hpp:15-24."""

    def __init__(self, m: int):
        self.curr = np.zeros(max(m, 1), np.uint32)
        self.next = np.zeros(max(m, 1), np.uint32)
        self.curr_size = 0
        self.next_size = 0
        self.in_curr = np.zeros(max(m, 1), np.uint8)
        self.in_next = np.zeros(max(m, 1), np.uint8)
        self.processed = np.zeros(max(m, 1), np.uint8)
        self.todo = m
        self.level = 0


class MarkScratchPool:
    """truss_parallel.hpp:55-59. The GPU keeps no dense per-worker mark arrays; kept for
    signature compatibility."""

    def __init__(self, workers: int, n: int):
        self.workers, self.n = workers, n


@dataclass
class GraphStats:
    n: int
    m: int
    d_max: int
    wedge_count: int
    sum_deg_sq: int
    sum_dplus_sq: int
    deg_sum_dplus_sq: int = 0
    deg_s1: int = 0


class Context:
    """A tdg_context: one CUDA stream + cached device buffers on one device."""

    def __init__(self, device: int = -1):
        self._h = C.c_void_p()
        _ck(_lib.tdg().tdg_context_create(device, C.byref(self._h)))

    @property
    def handle(self):
        return self._h

    def set_stream(self, stream_ptr: int | None):
        _ck(_lib.tdg().tdg_context_set_stream(self._h, stream_ptr))

    def trim(self):
        _ck(_lib.tdg().tdg_context_trim(self._h))

    def close(self):
        if self._h:
            _lib.tdg().tdg_context_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    COUNTER_NAMES = ("filter", "pbits", "walk", "slots", "hits", "dead", "dec", "repair", "next", "cross",
                     "comp_in", "comp_kept", "comp_long", "scan_in", "scan_out", "tasks", "sorted", "marks",
                     "rebuild_edges", "rebuild_buckets",
                     "sup_tab_elems", "sup_segments", "sup_search", "sup_hub")

    def counters(self) -> dict:
        """tdg_counters: access tallies of this context's last truss/support call (per-probe
        peel tallies only if TDG_COUNT=1 was in the environment during that call)."""
        out = (C.c_uint64 * len(self.COUNTER_NAMES))()
        _ck(_lib.tdg().tdg_counters(self._h, out, len(out)))
        return dict(zip(self.COUNTER_NAMES, list(out)))

    # -- host-pointer entry points
    def filter_mode(self) -> tuple[bool, float]:
        """tdg_filter_mode: (hash mode chosen?, false-positive estimate of the rank-mode filters)
        of the graph this context last decomposed."""
        h, e = C.c_int(), C.c_double()
        _ck(_lib.tdg().tdg_filter_mode(self._h, C.byref(h), C.byref(e)))
        return bool(h.value), e.value

    def truss(self, g: CsrGraph, want_support: bool = False):
        """tdg_truss: returns (truss u32[m], nsl list, support or None, times dict)."""
        truss = np.zeros(max(g.m, 1), np.uint32)
        sup = np.zeros(max(g.m, 1), np.uint32) if want_support else None
        cap = g.n + 2
        nsl = np.zeros(cap, np.uint32)
        nlen = C.c_uint64()
        t = tdg_times()
        v = g._view()
        _ck(_lib.tdg().tdg_truss(self._h, C.byref(v), truss.ctypes.data, _ptr(sup), nsl.ctypes.data, cap,
                                 C.byref(nlen), C.byref(t)))
        return truss[: g.m], [int(x) for x in nsl[: nlen.value]], (sup[: g.m] if sup is not None else None), t.as_dict()

    def truss_host_ptrs(self, n: int, m: int, off_ptr: int, nb_ptr: int, truss_ptr: int, nsl: np.ndarray):
        """tdg_truss on raw (e.g. pinned) host buffers; returns (nsl_len, times dict)."""
        nlen = C.c_uint64()
        t = tdg_times()
        v = tdg_csr(n, m, off_ptr, nb_ptr)
        _ck(_lib.tdg().tdg_truss(self._h, C.byref(v), truss_ptr, None, nsl.ctypes.data, len(nsl),
                                 C.byref(nlen), C.byref(t)))
        return nlen.value, t.as_dict()

    def truss_device(self, n: int, m: int, off_ptr: int, nb_ptr: int, truss_ptr: int, nsl: np.ndarray,
                     support_ptr: int | None = None):
        """tdg_truss_device on device buffers; returns (nsl_len, times dict)."""
        nlen = C.c_uint64()
        t = tdg_times()
        v = tdg_csr(n, m, off_ptr, nb_ptr)
        _ck(_lib.tdg().tdg_truss_device(self._h, C.byref(v), truss_ptr, support_ptr, nsl.ctypes.data, len(nsl),
                                        C.byref(nlen), C.byref(t)))
        return nlen.value, t.as_dict()

    def support(self, g: CsrGraph):
        s = np.zeros(max(g.m, 1), np.uint32)
        t = tdg_times()
        v = g._view()
        _ck(_lib.tdg().tdg_support(self._h, C.byref(v), s.ctypes.data, C.byref(t)))
        return s[: g.m], t.as_dict()

    def support_shard(self, g: CsrGraph, shard: int, nshards: int):
        """Partial supports of one shard (tdg_support_shard): the shards' arrays sum to support()."""
        s = np.zeros(max(g.m, 1), np.uint32)
        t = tdg_times()
        v = g._view()
        _ck(_lib.tdg().tdg_support_shard(self._h, C.byref(v), shard, nshards, s.ctypes.data, C.byref(t)))
        return s[: g.m], t.as_dict()

    def support_shard_device(self, n: int, m: int, off_ptr: int, nb_ptr: int, shard: int, nshards: int,
                             support_ptr: int) -> dict:
        """tdg_support_shard_device on device buffers (partial supports stay in HBM for the all-reduce)."""
        t = tdg_times()
        v = tdg_csr(n, m, off_ptr, nb_ptr)
        _ck(_lib.tdg().tdg_support_shard_device(self._h, C.byref(v), shard, nshards, support_ptr, C.byref(t)))
        return t.as_dict()

    def build_truss_graph(self, g: CsrGraph) -> TrussGraph:
        eo = np.zeros(max(g.n, 1), np.uint32)
        eid = np.zeros(max(2 * g.m, 1), np.uint32)
        el = np.zeros(max(2 * g.m, 1), np.uint32)
        v = g._view()
        _ck(_lib.tdg().tdg_build_truss_graph(self._h, C.byref(v), eo.ctypes.data, eid.ctypes.data, el.ctypes.data))
        return TrussGraph(g, eid[: 2 * g.m], el[: 2 * g.m].reshape(-1, 2), eo[: g.n])

    def triangle_count(self, g: CsrGraph) -> int:
        cnt = C.c_uint64()
        v = g._view()
        _ck(_lib.tdg().tdg_triangle_count(self._h, C.byref(v), C.byref(cnt), None))
        return cnt.value

    def stats(self, g: CsrGraph) -> GraphStats:
        st = tdg_graph_stats()
        v = g._view()
        _ck(_lib.tdg().tdg_stats(self._h, C.byref(v), C.byref(st)))
        d = st.as_dict()
        return GraphStats(d["n"], d["m"], d["d_max"], d["wedge_count"], d["sum_deg_sq"], d["sum_dplus_sq"],
                          d["deg_sum_dplus_sq"], d["deg_s1"])


_tls = threading.local()


def default_context() -> Context:
    """Per-thread default context: ctypes releases the GIL during the C calls, so threads
    sharing one context would race on its device buffers and pinned control block."""
    ctx = getattr(_tls, "ctx", None)
    if ctx is None:
        ctx = _tls.ctx = Context(-1)
    return ctx


# ---------------------------------------------------------------- reference-named API
def build_truss_graph(g: CsrGraph) -> TrussGraph:
    return default_context().build_truss_graph(g)


def stats(g: CsrGraph) -> GraphStats:
    return default_context().stats(g)


def triangle_count(tg: TrussGraph | CsrGraph, workers: int = 1) -> int:
    """triangle.cpp:90-116."""
    g = tg.csr if isinstance(tg, TrussGraph) else tg
    return default_context().triangle_count(g)


def support_am4(tg: TrussGraph | CsrGraph, workers: int = 1) -> np.ndarray:
    g = tg.csr if isinstance(tg, TrussGraph) else tg
    return default_context().support(g)[0]


def allreduce_partial_supports(partial, group=None):
    """Sum the shards' partial supports over the process group, in place (the one exchange of
    the sharded support pass). `partial` is a torch tensor of m 32-bit words (on
    the GPU under NCCL, on the host under gloo) or a numpy uint32 array (gloo). Sums are taken
    on the int32 view: two's-complement addition is the same bits as uint32 addition."""
    import torch
    import torch.distributed as dist

    if isinstance(partial, np.ndarray):
        t = torch.from_numpy(partial.view(np.int32))
        dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
        return partial
    t = partial.view(torch.int32) if partial.dtype != torch.int32 else partial
    dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
    return partial


def support_am4_sharded(tg: TrussGraph | CsrGraph, group=None, ctx: Context | None = None) -> np.ndarray:
    """support_am4 (triangle.cpp:26-61) over the ranks of a torch.distributed group: every
    rank holds the graph, counts the triangles of its equal-work shard on its own GPU and the
    partial supports are summed with ONE all-reduce of m u32 (NCCL: device buffers; gloo: host).
    Every rank returns the full support array."""
    import torch
    import torch.distributed as dist

    g = tg.csr if isinstance(tg, TrussGraph) else tg
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    ctx = ctx or default_context()
    if dist.get_backend(group) == "nccl":
        dev = torch.device("cuda", torch.cuda.current_device())
        off = torch.from_numpy(np.ascontiguousarray(g.offsets, np.int64)).to(dev)
        nb = torch.from_numpy(np.ascontiguousarray(g.neighbors, np.int32)).to(dev)
        part = torch.zeros(max(g.m, 1), dtype=torch.int32, device=dev)
        ctx.set_stream(torch.cuda.current_stream().cuda_stream)
        try:
            ctx.support_shard_device(g.n, g.m, off.data_ptr(), nb.data_ptr(), rank, world, part.data_ptr())
        finally:
            ctx.set_stream(None)
        allreduce_partial_supports(part, group)
        return part[: g.m].cpu().numpy().view(np.uint32)
    part = ctx.support_shard(g, rank, world)[0]
    return allreduce_partial_supports(np.ascontiguousarray(part), group)


def truss_parallel(tg: TrussGraph | CsrGraph, workers: int = 1) -> ParallelDecomposition:
    g = tg.csr if isinstance(tg, TrussGraph) else tg
    truss, nsl, _, t = default_context().truss(g)
    res = TrussnessResult(truss)
    res.finalize()
    # reference tally (truss_parallel.cpp:113,122,132,140)
    barriers = (res.t_max if g.m else 1) + 2 * int(sum(nsl))
    times = PhaseTimes(t["support_ms"] * 1e-3, t["scan_ms"] * 1e-3, (t["peel_ms"] - t["scan_ms"]) * 1e-3)
    return ParallelDecomposition(res, SubLevelTrace(nsl, barriers), times, t)


def scan(s: np.ndarray, level: int, frontier: LevelFrontier, workers: int = 1) -> None:
    s = np.ascontiguousarray(s, dtype=np.uint32)
    cs = C.c_uint64()
    _ck(_lib.tdg().tdg_scan(default_context().handle, s.ctypes.data, len(s), level, frontier.processed.ctypes.data,
                            frontier.in_curr.ctypes.data, frontier.curr.ctypes.data, C.byref(cs)))
    frontier.curr_size = cs.value


def process_sublevel(frontier: LevelFrontier, tg: TrussGraph | CsrGraph, s: np.ndarray, level: int,
                     scratch: MarkScratchPool | None = None, workers: int = 1) -> None:
    g = tg.csr if isinstance(tg, TrussGraph) else tg
    if s.dtype != np.uint32 or not s.flags.c_contiguous:
        raise ValueError("s must be a contiguous uint32 array (modified in place)")
    out = np.zeros(max(g.m, 1), np.uint32)
    ns = C.c_uint64()
    v = g._view()
    _ck(_lib.tdg().tdg_process_sublevel(default_context().handle, C.byref(v), s.ctypes.data, level,
                                        frontier.curr.ctypes.data, frontier.curr_size, frontier.in_curr.ctypes.data,
                                        frontier.in_next.ctypes.data, frontier.processed.ctypes.data,
                                        out.ctypes.data, C.byref(ns)))
    base = frontier.next_size
    frontier.next[base: base + ns.value] = out[: ns.value]
    frontier.next_size = base + ns.value


def ktruss_subgraphs(tg: TrussGraph | CsrGraph, res: TrussnessResult | np.ndarray, k: int) -> list[list[int]]:
    """truss_serial.cpp:176-210: the maximal k-trusses (connected components of the edges
    with truss >= k) as lists of edge ids, in the reference's order (components by first
    edge id, edges ascending). Computed on the GPU (tdg_ktruss_components)."""
    g = tg.csr if isinstance(tg, TrussGraph) else tg
    truss = np.ascontiguousarray(res.truss if isinstance(res, TrussnessResult) else res, dtype=np.uint32)
    comp = np.zeros(max(g.m, 1), np.uint32)
    nc = C.c_uint64()
    v = g._view()
    tr = truss if len(truss) else np.zeros(1, np.uint32)
    _ck(_lib.tdg().tdg_ktruss_components(default_context().handle, C.byref(v), tr.ctypes.data, k,
                                         comp.ctypes.data, C.byref(nc)))
    comp = comp[: g.m]
    sel = np.nonzero(comp != 0xFFFFFFFF)[0]
    order = np.argsort(comp[sel], kind="stable")
    groups = np.split(sel[order], np.cumsum(np.bincount(comp[sel], minlength=nc.value))[:-1]) if nc.value else []
    return [grp.astype(np.int64).tolist() for grp in groups]


@dataclass
class CorenessResult:
    """kcore.hpp:9-12."""
    core: np.ndarray
    c_max: int = 0


def kcore_parallel(g: CsrGraph, workers: int = 1) -> CorenessResult:
    """kcore.cpp:68-127 on the GPU (tdg_kcore)."""
    core = np.zeros(max(g.n, 1), np.uint32)
    cmax = C.c_uint32()
    v = g._view()
    _ck(_lib.tdg().tdg_kcore(default_context().handle, C.byref(v), core.ctypes.data, C.byref(cmax)))
    return CorenessResult(core[: g.n], cmax.value)


def coreness_order(res: CorenessResult) -> np.ndarray:
    """kcore.cpp:129-138: perm[v] = new id (stable by (coreness, id)), on the GPU."""
    core = np.ascontiguousarray(res.core, np.uint32)
    n = len(core)
    perm = np.zeros(max(n, 1), np.uint32)
    _ck(_lib.tdg().tdg_coreness_order(default_context().handle, n, core.ctypes.data if n else None,
                                      perm.ctypes.data))
    return perm[:n]


def reorder(g: CsrGraph, perm) -> CsrGraph:
    """graph.cpp:103-133: relabel vertex v as perm[v] and re-sort every adjacency list."""
    p = np.ascontiguousarray(perm, np.uint32)
    if len(p) != g.n:
        raise ValueError("reorder: permutation size does not match vertex count")
    off = np.zeros(g.n + 1, np.int64)
    nb = np.zeros(max(2 * g.m, 1), np.int32)
    v = g._view()
    pp = p if len(p) else np.zeros(1, np.uint32)
    _ck(_lib.tdg().tdg_reorder(default_context().handle, C.byref(v), pp.ctypes.data, off.ctypes.data, nb.ctypes.data))
    labels = None
    if g.labels is not None:
        labels = np.empty_like(g.labels)
        labels[p] = g.labels
    return CsrGraph(g.n, g.m, off, nb[: 2 * g.m], labels)


def read_edge_list(path: str) -> np.ndarray:
    """graph.cpp:152-200 (tdg_read_edge_list): the text edge list at `path` (plain or gzip;
    '#' / '%' comment lines, blank lines, any whitespace) as raw label pairs, shape (k, 2)
    uint64, in file order. Parsed on the GPU; raises RuntimeError with the reference's
    message ("<path>:<line>: <why>") on malformed input."""
    pairs = C.POINTER(C.c_uint64)()
    k = C.c_uint64()
    L = _lib.tdg()
    _ck(L.tdg_read_edge_list(default_context().handle, os.fsencode(path), C.byref(pairs), C.byref(k)))
    try:
        out = np.ctypeslib.as_array(pairs, shape=(2 * k.value,)).copy() if k.value else np.zeros(0, np.uint64)
    finally:
        if pairs:
            L.tdg_free(pairs)
    return out.reshape(-1, 2)


def canonicalize(pairs) -> CsrGraph:
    """graph.cpp:19-71 on the GPU (tdg_canonicalize): raw label pairs -> CsrGraph with dense
    ids in first-appearance order, loops dropped, duplicates merged, labels kept."""
    raw = np.ascontiguousarray(np.asarray(pairs, dtype=np.uint64).reshape(-1))
    k = len(raw) // 2
    off = np.zeros(2 * k + 2, np.int64)
    nb = np.zeros(max(2 * k, 1), np.int32)
    lab = np.zeros(max(2 * k, 1), np.uint64)
    n, m = C.c_int64(), C.c_int64()
    rp = raw if len(raw) else np.zeros(2, np.uint64)
    _ck(_lib.tdg().tdg_canonicalize(default_context().handle, rp.ctypes.data, k, off.ctypes.data, nb.ctypes.data,
                                    lab.ctypes.data, C.byref(n), C.byref(m)))
    return CsrGraph(n.value, m.value, off[: n.value + 1].copy(), nb[: 2 * m.value].copy(), lab[: n.value].copy())
