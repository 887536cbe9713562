// ref_capi.cpp — a C wrapper around the UNMODIFIED reference library, compiled together
// with the reference sources (/root/reference/proj/src/*.cpp) by oracle/Makefile into
// oracle/_ref/libtrussdec_ref.so. TEST / BASELINE INFRASTRUCTURE ONLY: used to pin the
// C restatement (oracle.c), to generate tests/golden fixtures, and as bench.py's
// `--impl reference` / cpu_baseline arm. Not part of the product.
//
// The CSR handed in is the generator's (int64 offsets, int32 sorted neighbours); it is
// turned into a trussdec::CsrGraph directly (no canonicalize, so edge ids line up),
// narrowing offsets to the reference's uint32 (graph.hpp:21-31).

#include <omp.h>

#include <chrono>
#include <cstdint>
#include <cstring>
#include <exception>
#include <string>
#include <vector>

#include "trussdec/generate.hpp"
#include "trussdec/graph.hpp"
#include "trussdec/kcore.hpp"
#include "trussdec/triangle.hpp"
#include "trussdec/truss_parallel.hpp"
#include "trussdec/truss_serial.hpp"

using namespace trussdec;

namespace {

thread_local std::string g_err;

double now() {
    return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

CsrGraph to_csr(int64_t n, int64_t m, const int64_t* off, const int32_t* nb) {
    CsrGraph g;
    g.n = static_cast<uint32_t>(n);
    g.m = static_cast<uint32_t>(m);
    g.offsets.resize(static_cast<size_t>(n) + 1);
    for (int64_t i = 0; i <= n; i++) g.offsets[i] = static_cast<uint32_t>(off[i]);
    g.neighbors.resize(static_cast<size_t>(2 * m));
    std::memcpy(g.neighbors.data(), nb, static_cast<size_t>(2 * m) * sizeof(uint32_t));
    return g;
}

int from_csr(const CsrGraph& g, int64_t cap_n, int64_t cap_nb, int64_t* off, int32_t* nb,
             int64_t* n_out, int64_t* m_out) {
    *n_out = g.n;
    *m_out = g.m;
    if (static_cast<int64_t>(g.n) > cap_n || static_cast<int64_t>(g.neighbors.size()) > cap_nb) return -4;
    for (uint32_t i = 0; i <= g.n; i++) off[i] = g.n ? g.offsets[i] : 0;
    if (g.n == 0) off[0] = 0;
    std::memcpy(nb, g.neighbors.data(), g.neighbors.size() * sizeof(uint32_t));
    return 0;
}

template <typename F>
int guarded(F&& f) {
    try {
        return f();
    } catch (const std::exception& e) {
        g_err = e.what();
        return -1;
    }
}

}  // namespace

extern "C" {

const char* ref_last_error(void) { return g_err.c_str(); }
int ref_max_threads(void) { return omp_get_max_threads(); }

// times[0..5] = build_truss_graph, support, scan, processing, engine wall, total (s)
int ref_truss_parallel(int64_t n, int64_t m, const int64_t* off, const int32_t* nb, int workers,
                       uint32_t* truss_out, uint32_t* nsl_out, uint64_t nsl_cap, uint64_t* nsl_len,
                       uint64_t* barriers, double* times) {
    return guarded([&] {
        double t0 = now();
        CsrGraph g = to_csr(n, m, off, nb);
        double t1 = now();
        TrussGraph tg = build_truss_graph(g);
        double t2 = now();
        ParallelDecomposition dec = truss_parallel(tg, workers);
        double t3 = now();
        if (truss_out) std::memcpy(truss_out, dec.result.truss.data(), static_cast<size_t>(m) * 4);
        *nsl_len = dec.trace.nsl.size();
        for (size_t i = 0; i < dec.trace.nsl.size() && i < nsl_cap; i++) nsl_out[i] = dec.trace.nsl[i];
        if (barriers) *barriers = dec.trace.barriers;
        if (times) {
            times[0] = t2 - t1;
            times[1] = dec.times.support;
            times[2] = dec.times.scan;
            times[3] = dec.times.processing;
            times[4] = t3 - t2;
            times[5] = t3 - t0;
        }
        return 0;
    });
}

// Reference preprocessing pipeline of trussdec.cpp:92-97 (kcore -> coreness_order ->
// reorder) followed by build + truss_parallel. times: kcore, reorder, build, support,
// scan, processing, engine wall.
int ref_truss_parallel_kcore(int64_t n, int64_t m, const int64_t* off, const int32_t* nb,
                             int workers, double* times) {
    return guarded([&] {
        CsrGraph g = to_csr(n, m, off, nb);
        double t0 = now();
        CorenessResult cores = kcore_parallel(g, workers);
        double t1 = now();
        CsrGraph r = reorder(g, coreness_order(cores));
        double t2 = now();
        TrussGraph tg = build_truss_graph(r);
        double t3 = now();
        ParallelDecomposition dec = truss_parallel(tg, workers);
        double t4 = now();
        times[0] = t1 - t0;
        times[1] = t2 - t1;
        times[2] = t3 - t2;
        times[3] = dec.times.support;
        times[4] = dec.times.scan;
        times[5] = dec.times.processing;
        times[6] = t4 - t3;
        return 0;
    });
}

// Prepared graph for repeated engine runs (bench.py --impl reference / cpu_baseline): the
// reference's preprocessing runs once — with kcore != 0 its own pipeline kcore_parallel ->
// coreness_order -> reorder (trussdec.cpp:92-97) — then build_truss_graph; ref_run times
// truss_parallel alone, as the CLI's bench command does (trussdec.cpp:319-323).
// prep_times: kcore, reorder, build (s). run times: support, scan, processing, engine (s).
void* ref_prepare(int64_t n, int64_t m, const int64_t* off, const int32_t* nb, int workers, int kcore,
                  double* prep_times) {
    TrussGraph* out = nullptr;
    guarded([&] {
        CsrGraph g = to_csr(n, m, off, nb);
        double t0 = now(), t1 = t0, t2 = t0;
        if (kcore) {
            CorenessResult cores = kcore_parallel(g, workers);
            t1 = now();
            g = reorder(g, coreness_order(cores));
            t2 = now();
        }
        out = new TrussGraph(build_truss_graph(g));
        const double t3 = now();
        if (prep_times) {
            prep_times[0] = t1 - t0;
            prep_times[1] = t2 - t1;
            prep_times[2] = t3 - t2;
        }
        return 0;
    });
    return out;
}

int ref_run(void* h, int workers, double* times, uint32_t* t_max) {
    return guarded([&] {
        const TrussGraph& tg = *static_cast<const TrussGraph*>(h);
        const double t0 = now();
        ParallelDecomposition dec = truss_parallel(tg, workers);
        const double t1 = now();
        times[0] = dec.times.support;
        times[1] = dec.times.scan;
        times[2] = dec.times.processing;
        times[3] = t1 - t0;
        if (t_max) *t_max = dec.result.t_max;
        return 0;
    });
}

void ref_free(void* h) { delete static_cast<TrussGraph*>(h); }

int ref_support_am4(int64_t n, int64_t m, const int64_t* off, const int32_t* nb, int workers,
                    uint32_t* s_out) {
    return guarded([&] {
        TrussGraph tg = build_truss_graph(to_csr(n, m, off, nb));
        SupportArray s = support_am4(tg, workers);
        std::memcpy(s_out, s.data(), static_cast<size_t>(m) * 4);
        return 0;
    });
}

int ref_build_truss_graph(int64_t n, int64_t m, const int64_t* off, const int32_t* nb,
                          uint32_t* eo, uint32_t* eid, uint32_t* el) {
    return guarded([&] {
        TrussGraph tg = build_truss_graph(to_csr(n, m, off, nb));
        std::memcpy(eo, tg.eo.data(), static_cast<size_t>(n) * 4);
        std::memcpy(eid, tg.eid.data(), static_cast<size_t>(2 * m) * 4);
        for (int64_t e = 0; e < m; e++) {
            el[2 * e] = tg.el[e].first;
            el[2 * e + 1] = tg.el[e].second;
        }
        return 0;
    });
}

int ref_truss_wc(int64_t n, int64_t m, const int64_t* off, const int32_t* nb, uint32_t* truss_out) {
    return guarded([&] {
        TrussGraph tg = build_truss_graph(to_csr(n, m, off, nb));
        TrussnessResult r = truss_wc(tg, support_am4(tg, 1));
        std::memcpy(truss_out, r.truss.data(), static_cast<size_t>(m) * 4);
        return 0;
    });
}

int ref_truss_oracle(int64_t n, int64_t m, const int64_t* off, const int32_t* nb, uint32_t* truss_out) {
    return guarded([&] {
        TrussnessResult r = truss_oracle(to_csr(n, m, off, nb));
        std::memcpy(truss_out, r.truss.data(), static_cast<size_t>(m) * 4);
        return 0;
    });
}

int64_t ref_triangle_count(int64_t n, int64_t m, const int64_t* off, const int32_t* nb, int workers) {
    int64_t out = -1;
    guarded([&] {
        out = static_cast<int64_t>(triangle_count(build_truss_graph(to_csr(n, m, off, nb)), workers));
        return 0;
    });
    return out;
}

// ktruss_subgraphs (truss_serial.cpp:176-210) flattened to comp_out[e] = component index or
// 0xFFFFFFFF; returns -1 with the reference's exception message on invalid k.
int ref_ktruss_components(int64_t n, int64_t m, const int64_t* off, const int32_t* nb, const uint32_t* truss,
                          uint32_t k, uint32_t* comp_out, uint64_t* ncomp) {
    return guarded([&] {
        TrussGraph tg = build_truss_graph(to_csr(n, m, off, nb));
        TrussnessResult res;
        res.truss.assign(truss, truss + m);
        res.finalize();
        auto comps = ktruss_subgraphs(tg, res, k);
        for (int64_t e = 0; e < m; e++) comp_out[e] = 0xffffffffu;
        for (size_t c = 0; c < comps.size(); c++)
            for (EdgeId e : comps[c]) comp_out[e] = static_cast<uint32_t>(c);
        *ncomp = comps.size();
        return 0;
    });
}

// kcore_parallel + coreness_order (kcore.cpp:68-138) and reorder (graph.cpp:103-133).
int ref_kcore_order(int64_t n, int64_t m, const int64_t* off, const int32_t* nb, int workers, uint32_t* core_out,
                    uint32_t* c_max, uint32_t* perm_out) {
    return guarded([&] {
        CorenessResult r = kcore_parallel(to_csr(n, m, off, nb), workers);
        std::memcpy(core_out, r.core.data(), static_cast<size_t>(n) * 4);
        *c_max = r.c_max;
        std::vector<VertexId> p = coreness_order(r);
        std::memcpy(perm_out, p.data(), static_cast<size_t>(n) * 4);
        return 0;
    });
}

int ref_reorder(int64_t n, int64_t m, const int64_t* off, const int32_t* nb, const uint32_t* perm,
                int64_t* off_out, int32_t* nb_out) {
    return guarded([&] {
        CsrGraph r = reorder(to_csr(n, m, off, nb), std::vector<VertexId>(perm, perm + n));
        for (int64_t i = 0; i <= n; i++) off_out[i] = r.offsets[i];
        std::memcpy(nb_out, r.neighbors.data(), static_cast<size_t>(2 * m) * 4);
        return 0;
    });
}

// read_edge_list (graph.cpp:152-200): pairs into a caller buffer of cap pairs; *npairs is
// the file's pair count (also when it exceeds cap: call again with a bigger buffer).
int ref_read_edge_list(const char* path, uint64_t* pairs, uint64_t cap, uint64_t* npairs) {
    return guarded([&] {
        RawEdgeList raw = read_edge_list(path);
        *npairs = raw.edges.size();
        for (uint64_t i = 0; i < raw.edges.size() && i < cap; i++) {
            pairs[2 * i] = raw.edges[i].first;
            pairs[2 * i + 1] = raw.edges[i].second;
        }
        return 0;
    });
}

// Fixture graphs exactly as the reference tests build them (tests/helpers.hpp:12-43):
// kind 0 = er_graph(n, p, seed), kind 1 = rmat_graph(scale=n, ef=(int)p, seed),
// kind 2 = canonicalize(pairs). CSR written into caller buffers (capacities given).
int ref_make_graph(int kind, int64_t a, double b, uint64_t seed, const int64_t* pairs,
                   int64_t npairs, int64_t cap_n, int64_t cap_nb, int64_t* off, int32_t* nb,
                   int64_t* n_out, int64_t* m_out) {
    return guarded([&] {
        RawEdgeList raw;
        if (kind == 0) raw = generate_er(static_cast<uint32_t>(a), b, seed);
        else if (kind == 1) raw = generate_rmat(static_cast<uint32_t>(a), static_cast<uint32_t>(b), seed);
        else
            for (int64_t i = 0; i < npairs; i++)
                raw.edges.emplace_back(static_cast<uint64_t>(pairs[2 * i]), static_cast<uint64_t>(pairs[2 * i + 1]));
        return from_csr(canonicalize(raw), cap_n, cap_nb, off, nb, n_out, m_out);
    });
}

}  // extern "C"
