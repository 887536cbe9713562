// Drop-in check on the reference's OWN types: a caller that already
// holds trussdec::TrussGraph (built by the reference library itself) switches
// trussdec::truss_parallel / support_am4 to the GPU with
//   trussdec_gpu::truss_parallel_as<trussdec::ParallelDecomposition>(tg, w)
//   trussdec_gpu::support_am4_as<trussdec::SupportArray>(tg, w)
// and gets identical results, traces and invariants. Compiled against the reference headers
// (/root/reference/proj/include) and linked with oracle/_ref/libtrussdec_ref.so (the
// unmodified reference sources) + libtdg.so; test infrastructure only.
#include <cstdio>
#include <vector>

#include "trussdec/generate.hpp"
#include "trussdec/graph.hpp"
#include "trussdec/triangle.hpp"
#include "trussdec/truss_parallel.hpp"
#include "trussdec/truss_serial.hpp"
#include "trussdec_gpu.hpp"

static int failures = 0;
#define CHECK(c)                                                          \
    do {                                                                  \
        if (!(c)) {                                                       \
            std::printf("CHECK failed %s:%d: %s\n", __FILE__, __LINE__, #c); \
            failures++;                                                   \
        }                                                                 \
    } while (0)

static void check_graph(const trussdec::CsrGraph& g, const char* what) {
    const trussdec::TrussGraph tg = trussdec::build_truss_graph(g);
    // the reference itself
    const trussdec::ParallelDecomposition ref = trussdec::truss_parallel(tg, 4);
    const trussdec::SupportArray sref = trussdec::support_am4(tg, 4);
    // the GPU, called with the reference's types
    const auto gpu = trussdec_gpu::truss_parallel_as<trussdec::ParallelDecomposition>(tg, 4);
    const auto sgpu = trussdec_gpu::support_am4_as<trussdec::SupportArray>(tg, 4);
    CHECK(gpu.result.truss == ref.result.truss);
    CHECK(gpu.result.t_max == ref.result.t_max);
    CHECK(gpu.result.kclass_sizes == ref.result.kclass_sizes);
    CHECK(gpu.trace.nsl == ref.trace.nsl);
    CHECK(gpu.trace.barriers == ref.trace.barriers);
    CHECK(gpu.trace.barriers == gpu.trace.expected_barriers(gpu.result.t_max) || tg.m() == 0);
    CHECK(sgpu == sref);
    std::printf("%s: n=%u m=%u t_max=%u sublevels=%llu ok=%d\n", what, tg.n(), tg.m(), gpu.result.t_max,
                static_cast<unsigned long long>(gpu.trace.sublevel_total()), failures == 0);
}

int main() {
    check_graph(trussdec::canonicalize(trussdec::generate_er(200, 0.1, 3)), "er(200,0.1,3)");
    check_graph(trussdec::canonicalize(trussdec::generate_rmat(10, 16, 5)), "rmat(10,16,5)");
    check_graph(trussdec::canonicalize(trussdec::generate_rmat(12, 8, 9)), "rmat(12,8,9)");
    {   // triangle + pendant (test_truss_parallel.cpp:118-126)
        trussdec::RawEdgeList raw;
        raw.edges = {{0, 1}, {1, 2}, {0, 2}, {2, 3}};
        check_graph(trussdec::canonicalize(raw), "triangle+pendant");
    }
    {   // empty graph
        trussdec::RawEdgeList raw;
        raw.edges = {{5, 5}};
        check_graph(trussdec::canonicalize(raw), "loop-only");
    }
    if (failures) {
        std::printf("%d reference-type shim checks FAILED\n", failures);
        return 1;
    }
    std::printf("all reference-type shim checks passed\n");
    return 0;
}
