// C++ drop-in test: the reference's own unit cases (tests/test_truss_parallel.cpp,
// tests/test_triangle.cpp under /root/reference/proj) written against the shim's
// reference-named API (trussdec_gpu::*), running on the GPU through libtdg.so.
#include <algorithm>
#include <cstdio>
#include <map>
#include <vector>

#include "trussdec_gpu.hpp"

using namespace trussdec_gpu;

static int failures = 0;
#define CHECK(c)                                                          \
    do {                                                                  \
        if (!(c)) {                                                       \
            std::printf("CHECK failed %s:%d: %s\n", __FILE__, __LINE__, #c); \
            failures++;                                                   \
        }                                                                 \
    } while (0)

static CsrGraph make_graph(std::vector<std::pair<uint32_t, uint32_t>> edges, uint32_t n) {
    for (auto& e : edges) if (e.first > e.second) std::swap(e.first, e.second);
    std::sort(edges.begin(), edges.end());
    CsrGraph g;
    g.n = n;
    g.m = static_cast<uint32_t>(edges.size());
    g.offsets.assign(n + 1, 0);
    for (auto& e : edges) { g.offsets[e.first + 1]++; g.offsets[e.second + 1]++; }
    for (uint32_t i = 0; i < n; i++) g.offsets[i + 1] += g.offsets[i];
    g.neighbors.resize(2ull * g.m);
    std::vector<uint32_t> cur(g.offsets.begin(), g.offsets.end() - 1);
    for (auto& e : edges) { g.neighbors[cur[e.first]++] = e.second; g.neighbors[cur[e.second]++] = e.first; }
    return g;
}

static CsrGraph complete_graph(uint32_t n) {
    std::vector<std::pair<uint32_t, uint32_t>> e;
    for (uint32_t u = 0; u < n; u++)
        for (uint32_t v = u + 1; v < n; v++) e.emplace_back(u, v);
    return make_graph(e, n);
}

int main() {
    {   // support on a triangle, K4 and a path (test_triangle.cpp:13-22)
        CHECK(support_am4(build_truss_graph(complete_graph(3)), 1) == (SupportArray{1, 1, 1}));
        SupportArray k4 = support_am4(build_truss_graph(complete_graph(4)), 2);
        CHECK(k4 == SupportArray(6, 2));
        CHECK(support_am4(build_truss_graph(make_graph({{0, 1}, {1, 2}}, 3)), 1) == (SupportArray{0, 0}));
    }
    {   // build_truss_graph layout (graph.cpp:73-101) on K4
        TrussGraph tg = build_truss_graph(complete_graph(4));
        CHECK(tg.el.size() == 6 && tg.el[0] == std::make_pair(0u, 1u) && tg.el[5] == std::make_pair(2u, 3u));
        CHECK(tg.eo[0] == 0 && tg.eo[3] == 12);
    }
    {   // scan collects exactly the edges at the level (test_truss_parallel.cpp:25-36)
        TrussGraph tg = build_truss_graph(complete_graph(4));
        SupportArray s = support_am4(tg, 1);
        LevelFrontier f(tg.m());
        scan(s, 0, f, 2);
        CHECK(f.curr_size.load() == 0);
        scan(s, 2, f, 2);
        std::vector<EdgeId> c(f.curr.begin(), f.curr.begin() + f.curr_size.load());
        std::sort(c.begin(), c.end());
        CHECK(c == (std::vector<EdgeId>{0, 1, 2, 3, 4, 5}));
    }
    {   // ownership rule decrements the third edge once (:72-88)
        TrussGraph tg = build_truss_graph(complete_graph(3));
        SupportArray s{0, 0, 1};
        LevelFrontier f(3);
        MarkScratchPool scratch(2, tg.n());
        f.curr[0] = 0; f.curr[1] = 1; f.curr_size.store(2); f.in_curr[0] = f.in_curr[1] = 1;
        process_sublevel(f, tg, s, 0, scratch, 2);
        CHECK(s[2] == 0);
        CHECK(f.next_size.load() == 1 && f.next[0] == 2);
        CHECK(f.processed[0] == 1 && f.processed[1] == 1 && f.in_curr[0] == 0);
    }
    {   // K4 decomposition trace (:107-116)
        ParallelDecomposition par = truss_parallel(build_truss_graph(complete_graph(4)), 4);
        for (uint32_t t : par.result.truss) CHECK(t == 4);
        CHECK(par.trace.nsl == (std::vector<uint32_t>{0, 0, 1}));
        CHECK(par.trace.barriers == par.trace.expected_barriers(par.result.t_max));
    }
    {   // triangle plus pendant (:118-126)
        ParallelDecomposition d = truss_parallel(build_truss_graph(make_graph({{0, 1}, {0, 2}, {1, 2}, {0, 3}}, 4)), 2);
        CHECK(d.result.kclass_sizes.at(2) == 1 && d.result.kclass_sizes.at(3) == 3);
    }
    {   // closed forms (acceptance.cpp:109-124)
        for (uint32_t n = 3; n <= 8; n++)
            for (uint32_t t : truss_parallel(build_truss_graph(complete_graph(n)), 4).result.truss) CHECK(t == n);
    }
    {   // error behaviour: invalid CSR -> std::invalid_argument
        CsrGraph bad = complete_graph(3);
        bad.m = 5;
        bool threw = false;
        try { truss_parallel(build_truss_graph(bad), 1); } catch (const std::invalid_argument&) { threw = true; } catch (...) {}
        CHECK(threw);
    }
    std::printf(failures ? "FAILED (%d)\n" : "all shim checks passed\n", failures);
    return failures ? 1 : 0;
}
