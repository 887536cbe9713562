// trussdec_gpu.cpp — non-template parts of the C++ shim (see trussdec_gpu.hpp).
#include "trussdec_gpu.hpp"

namespace trussdec_gpu {

namespace {
struct CtxHolder {
    tdg_context* ctx = nullptr;
    ~CtxHolder() {
        if (ctx) tdg_context_destroy(ctx);
    }
};
thread_local CtxHolder t_ctx;
}  // namespace

tdg_context* default_context() {
    if (!t_ctx.ctx) check(tdg_context_create(-1, &t_ctx.ctx));  // -1: current device
    return t_ctx.ctx;
}

void raise_status(int status) {
    const std::string msg = tdg_last_error();
    if (status == TDG_ERR_INVALID) throw std::invalid_argument(msg);
    if (status == TDG_ERR_NOMEM) throw std::bad_alloc();
    throw std::runtime_error(msg);
}

RawEdgeList read_edge_list(const std::string& path) {
    std::uint64_t* pairs = nullptr;
    std::uint64_t k = 0;
    check(tdg_read_edge_list(default_context(), path.c_str(), &pairs, &k));
    RawEdgeList raw;
    raw.edges.resize(k);
    for (std::uint64_t i = 0; i < k; i++) raw.edges[i] = {pairs[2 * i], pairs[2 * i + 1]};
    tdg_free(pairs);
    return raw;
}

CsrGraph canonicalize(const RawEdgeList& raw) {
    const std::uint64_t k = raw.edges.size();
    std::vector<std::uint64_t> flat(2 * k + 2);
    for (std::uint64_t i = 0; i < k; i++) {
        flat[2 * i] = raw.edges[i].first;
        flat[2 * i + 1] = raw.edges[i].second;
    }
    std::vector<std::int64_t> off(2 * k + 2);
    std::vector<std::int32_t> nb(2 * k + 1);
    std::vector<std::uint64_t> lab(2 * k + 1);
    std::int64_t n = 0, m = 0;
    check(tdg_canonicalize(default_context(), flat.data(), k, off.data(), nb.data(), lab.data(), &n, &m));
    CsrGraph g;
    g.n = static_cast<std::uint32_t>(n);
    g.m = static_cast<std::uint32_t>(m);
    g.offsets.assign(off.begin(), off.begin() + n + 1);
    g.neighbors.assign(nb.begin(), nb.begin() + 2 * m);
    g.labels.assign(lab.begin(), lab.begin() + n);
    return g;
}

TrussGraph build_truss_graph(const CsrGraph& g) {
    TrussGraph tg;
    tg.csr = g;
    tg.eid.assign(2ull * g.m, 0);
    tg.el.resize(g.m);
    tg.eo.resize(g.n);
    std::vector<std::int64_t> off64;
    const tdg_csr v = view(g, off64);
    std::vector<std::uint32_t> el2(2ull * g.m + 1);
    std::vector<std::uint32_t> eo(g.n + 1ull), eid(2ull * g.m + 1);
    check(tdg_build_truss_graph(default_context(), &v, eo.data(), eid.data(), el2.data()));
    for (std::uint32_t u = 0; u < g.n; u++) tg.eo[u] = eo[u];
    for (std::uint64_t j = 0; j < 2ull * g.m; j++) tg.eid[j] = eid[j];
    for (std::uint32_t e = 0; e < g.m; e++) tg.el[e] = {el2[2ull * e], el2[2ull * e + 1]};
    return tg;
}

GraphStats stats(const CsrGraph& g) {
    std::vector<std::int64_t> off64;
    const tdg_csr v = view(g, off64);
    tdg_graph_stats st{};
    check(tdg_stats(default_context(), &v, &st));
    GraphStats out;
    out.n = static_cast<std::uint32_t>(st.n);
    out.m = static_cast<std::uint32_t>(st.m);
    out.d_max = static_cast<std::uint32_t>(st.d_max);
    out.wedge_count = st.wedge_count;
    out.sum_deg_sq = st.sum_deg_sq;
    out.sum_dplus_sq = st.sum_dplus_sq;
    return out;
}

SupportArray support_am4(const TrussGraph& tg, int workers) { return support_am4_as<SupportArray>(tg, workers); }

CorenessResult kcore_parallel(const CsrGraph& g, int /*workers*/) {
    std::vector<std::int64_t> off64;
    const tdg_csr v = view(g, off64);
    CorenessResult r;
    r.core.assign(g.n, 0);
    check(tdg_kcore(default_context(), &v, r.core.data(), &r.c_max));
    return r;
}

std::vector<VertexId> coreness_order(const CorenessResult& res) {
    std::vector<VertexId> perm(res.core.size());
    check(tdg_coreness_order(default_context(), res.core.size(), res.core.data(), perm.data()));
    return perm;
}

CsrGraph reorder(const CsrGraph& g, const std::vector<VertexId>& perm) {
    if (perm.size() != g.n) throw std::invalid_argument("reorder: permutation size does not match vertex count");
    std::vector<std::int64_t> off64;
    const tdg_csr v = view(g, off64);
    std::vector<std::int64_t> noff(g.n + 1ull);
    CsrGraph out;
    out.n = g.n;
    out.m = g.m;
    out.neighbors.resize(2ull * g.m);
    check(tdg_reorder(default_context(), &v, perm.data(), noff.data(),
                      reinterpret_cast<std::int32_t*>(out.neighbors.data())));
    out.offsets.assign(noff.begin(), noff.end());
    if (!g.labels.empty()) {
        out.labels.resize(g.n);
        for (VertexId u = 0; u < g.n; u++) out.labels[perm[u]] = g.labels[u];
    }
    return out;
}

std::uint64_t triangle_count(const TrussGraph& tg, int /*workers*/) {
    std::vector<std::int64_t> off64;
    const tdg_csr v = view(tg.csr, off64);
    std::uint64_t c = 0;
    check(tdg_triangle_count(default_context(), &v, &c, nullptr));
    return c;
}

std::vector<std::vector<EdgeId>> ktruss_subgraphs(const TrussGraph& tg, const TrussnessResult& res, std::uint32_t k) {
    std::vector<std::int64_t> off64;
    const tdg_csr v = view(tg.csr, off64);
    std::vector<std::uint32_t> comp(tg.csr.m + 1ull);
    std::uint64_t nc = 0;
    check(tdg_ktruss_components(default_context(), &v, res.truss.data(), k, comp.data(), &nc));
    std::vector<std::vector<EdgeId>> out(nc);
    for (std::uint32_t e = 0; e < tg.csr.m; e++)
        if (comp[e] != 0xffffffffu) out[comp[e]].push_back(e);  // ascending edge ids per component
    return out;
}

ParallelDecomposition truss_parallel(const TrussGraph& tg, int workers) {
    return truss_parallel_as<ParallelDecomposition>(tg, workers);
}

void scan(const SupportArray& s, std::uint32_t level, LevelFrontier& f, int /*workers*/) {
    std::uint64_t cs = 0;
    check(tdg_scan(default_context(), s.data(), s.size(), level, f.processed.data(), f.in_curr.data(),
                   f.curr.data(), &cs));
    f.curr_size.store(cs);
}

void process_sublevel(LevelFrontier& f, const TrussGraph& tg, SupportArray& s, std::uint32_t level,
                      MarkScratchPool&, int /*workers*/) {
    std::vector<std::int64_t> off64;
    const tdg_csr v = view(tg.csr, off64);
    std::uint64_t ns = 0;
    // The reference appends to next after next_size entries already present (it is reset
    // by the driver between sub-levels, truss_parallel.cpp:139); keep that contract.
    const std::size_t base = f.next_size.load();
    std::vector<std::uint32_t> out(tg.csr.m + 1ull);
    check(tdg_process_sublevel(default_context(), &v, s.data(), level, f.curr.data(), f.curr_size.load(),
                               f.in_curr.data(), f.in_next.data(), f.processed.data(), out.data(), &ns));
    for (std::uint64_t i = 0; i < ns; i++) f.next[base + i] = out[i];
    f.next_size.store(base + ns);
}

}  // namespace trussdec_gpu
