// trussdec_gpu.hpp — C++ host shim over the C-ABI (include/tdg.h) that keeps the
// reference's entry points, argument meaning and error behaviour (paths relative to
// /root/reference/proj):
//
//   ParallelDecomposition truss_parallel(const TrussGraph&, int workers)  truss_parallel.hpp:72
//   SupportArray          support_am4(const TrussGraph&, int workers)     triangle.hpp:16
//   TrussGraph            build_truss_graph(const CsrGraph&)              graph.hpp:69
//   GraphStats            stats(const CsrGraph&)                          graph.hpp:74
//   void scan(const SupportArray&, uint32_t, LevelFrontier&, int)         truss_parallel.hpp:62
//   void process_sublevel(LevelFrontier&, const TrussGraph&, SupportArray&,
//                         uint32_t, MarkScratchPool&, int)                truss_parallel.hpp:67-68
//
// The types below mirror the reference's field-for-field (graph.hpp:21-49,
// truss_serial.hpp:12-18, truss_parallel.hpp:15-59), so the call sites read the same.
// Two ways to drop in:
//   * use trussdec_gpu::{CsrGraph, TrussGraph, ...} directly; or
//   * keep the reference's own types and call the templated adapters
//     trussdec_gpu::truss_parallel_as<trussdec::ParallelDecomposition>(tg, workers) /
//     support_am4_as<trussdec::SupportArray>(tg, workers), which only touch the members
//     the reference declares (csr.n, csr.m, csr.offsets, csr.neighbors, result.truss,
//     result.finalize(), trace.nsl, trace.barriers, times.*).
//
// `workers` is accepted for signature compatibility and ignored (the GPU decides its own
// parallelism), as `workers < 1` is clamped by the reference (truss_parallel.cpp:107).
// Errors: TDG_ERR_INVALID -> std::invalid_argument, TDG_ERR_NOMEM -> std::bad_alloc,
// anything else -> std::runtime_error(tdg_last_error()). No CPU fallback exists.
#pragma once

#include <atomic>
#include <cstdint>
#include <map>
#include <new>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "tdg.h"

namespace trussdec_gpu {

using VertexId = std::uint32_t;
using EdgeId = std::uint32_t;
using SupportArray = std::vector<std::uint32_t>;

struct CsrGraph {
    std::uint32_t n = 0;
    std::uint32_t m = 0;
    std::vector<std::uint32_t> offsets;
    std::vector<VertexId> neighbors;
    std::vector<std::uint64_t> labels;
    std::uint32_t degree(VertexId u) const { return offsets[u + 1] - offsets[u]; }
    std::uint64_t label_of(VertexId u) const { return labels.empty() ? u : labels[u]; }
};

struct RawEdgeList {  // graph.hpp:13-15
    std::vector<std::pair<std::uint64_t, std::uint64_t>> edges;
};

struct TrussGraph {
    CsrGraph csr;
    std::vector<EdgeId> eid;
    std::vector<std::pair<VertexId, VertexId>> el;
    std::vector<std::uint32_t> eo;
    std::uint32_t n() const { return csr.n; }
    std::uint32_t m() const { return csr.m; }
    static std::uint64_t core_array_bytes(std::uint64_t n, std::uint64_t m) { return 28 * m + 8 * n; }
};

struct GraphStats {
    std::uint32_t n = 0, m = 0, d_max = 0;
    std::uint64_t wedge_count = 0, sum_deg_sq = 0, sum_dplus_sq = 0;
    std::int64_t triangle_count = -1, c_max = -1, t_max = -1;
};

struct TrussnessResult {
    std::vector<std::uint32_t> truss;
    std::uint32_t t_max = 0;
    std::map<std::uint32_t, std::uint64_t> kclass_sizes;
    void finalize() {  // truss_serial.cpp:10-17
        t_max = 0;
        kclass_sizes.clear();
        for (std::uint32_t t : truss) {
            t_max = t > t_max ? t : t_max;
            kclass_sizes[t]++;
        }
    }
};

struct LevelFrontier {
    std::vector<EdgeId> curr, next;
    std::atomic<std::size_t> curr_size{0}, next_size{0};
    std::vector<std::uint8_t> in_curr, in_next, processed;
    std::size_t todo = 0;
    std::uint32_t level = 0;
    explicit LevelFrontier(std::uint32_t m)
        : curr(m), next(m), in_curr(m, 0), in_next(m, 0), processed(m, 0), todo(m) {}
};

struct SubLevelTrace {
    std::vector<std::uint32_t> nsl;
    std::uint64_t barriers = 0;
    std::uint64_t sublevel_total() const {
        std::uint64_t s = 0;
        for (std::uint32_t c : nsl) s += c;
        return s;
    }
    std::uint64_t expected_barriers(std::uint32_t t_max) const { return t_max + 2 * sublevel_total(); }
};

struct PhaseTimes {
    double support = 0, scan = 0, processing = 0;
};

struct ParallelDecomposition {
    TrussnessResult result;
    SubLevelTrace trace;
    PhaseTimes times;
};

/// The GPU keeps no per-worker mark arrays (truss_parallel.hpp:55-59); this stub exists
/// so process_sublevel keeps the reference signature.
struct MarkScratchPool {
    MarkScratchPool(int, std::uint32_t) {}
};

/// Context used by the shim's free functions (one per thread, on the current device).
tdg_context* default_context();

[[noreturn]] void raise_status(int status);
inline void check(int status) {
    if (status != TDG_OK) raise_status(status);
}

template <class Csr>
tdg_csr view(const Csr& g, std::vector<std::int64_t>& off64) {
    off64.assign(g.offsets.begin(), g.offsets.end());
    if (off64.empty()) off64.push_back(0);
    return tdg_csr{static_cast<std::int64_t>(g.n), static_cast<std::int64_t>(g.m), off64.data(),
                   reinterpret_cast<const std::int32_t*>(g.neighbors.data())};
}

// ---- templated adapters: work on the reference's own types as well as ours ----

template <class PD, class TG>
PD truss_parallel_as(const TG& tg, int /*workers*/) {
    std::vector<std::int64_t> off64;
    const tdg_csr g = view(tg.csr, off64);
    PD out;
    out.result.truss.resize(tg.csr.m);
    std::vector<std::uint32_t> nsl(static_cast<std::size_t>(tg.csr.n) + 2);
    std::uint64_t len = 0;
    tdg_times t{};
    check(tdg_truss(default_context(), &g, out.result.truss.data(), nullptr, nsl.data(), nsl.size(), &len, &t));
    nsl.resize(len);
    out.trace.nsl.assign(nsl.begin(), nsl.end());
    out.result.finalize();
    // Reference tally (truss_parallel.cpp:113,122,132,140): 1 after support, one per
    // visited level (t_max - 1 of them), two per sub-level.
    std::uint64_t sum = 0;
    for (std::uint32_t c : nsl) sum += c;
    out.trace.barriers = (tg.csr.m ? out.result.t_max : 1) + 2 * sum;
    out.times.support = t.support_ms * 1e-3;
    out.times.scan = t.scan_ms * 1e-3;
    out.times.processing = (t.peel_ms - t.scan_ms) * 1e-3;
    return out;
}

template <class SA, class TG>
SA support_am4_as(const TG& tg, int /*workers*/) {
    std::vector<std::int64_t> off64;
    const tdg_csr g = view(tg.csr, off64);
    SA s(tg.csr.m, 0);
    check(tdg_support(default_context(), &g, s.data(), nullptr));
    return s;
}

struct CorenessResult {  // kcore.hpp:9-12
    std::vector<std::uint32_t> core;
    std::uint32_t c_max = 0;
};

// ---- reference-named entry points on the mirrored types ----
CorenessResult kcore_parallel(const CsrGraph& g, int workers);                    // kcore.hpp:19
std::vector<VertexId> coreness_order(const CorenessResult& res);                   // kcore.hpp:23
CsrGraph reorder(const CsrGraph& g, const std::vector<VertexId>& perm);            // graph.hpp:72
std::uint64_t triangle_count(const TrussGraph& tg, int workers);  // triangle.hpp:19
std::vector<std::vector<EdgeId>> ktruss_subgraphs(const TrussGraph& tg, const TrussnessResult& res,
                                                  std::uint32_t k);  // truss_serial.hpp:43-45
RawEdgeList read_edge_list(const std::string& path);  // graph.hpp:78 (GPU-parsed)
CsrGraph canonicalize(const RawEdgeList& raw);         // graph.hpp:69 (GPU)
TrussGraph build_truss_graph(const CsrGraph& g);
GraphStats stats(const CsrGraph& g);
SupportArray support_am4(const TrussGraph& tg, int workers);
ParallelDecomposition truss_parallel(const TrussGraph& tg, int workers);
void scan(const SupportArray& s, std::uint32_t level, LevelFrontier& frontier, int workers);
void process_sublevel(LevelFrontier& frontier, const TrussGraph& tg, SupportArray& s,
                      std::uint32_t level, MarkScratchPool& scratch, int workers);

}  // namespace trussdec_gpu
