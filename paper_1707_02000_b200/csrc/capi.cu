// capi.cu — the extern "C" boundary (include/tdg.h): contexts, device buffers, H2D/D2H,
// phase timing with CUDA events, error mapping. All compute is in build.cu / support.cu /
// peel.cu; there is no host compute path.

#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <cstdint>
#include <new>
#include <string>
#include <vector>
#include <algorithm>

#include <zlib.h>

#include "tdg.h"
#include "tdg_kernels.h"

using namespace tdg;
namespace tdg { extern const char* g_ingest_step; }

#ifndef TDG_SUP_TAB
#define TDG_SUP_TAB_DEFAULT 4096
#else
#define TDG_SUP_TAB_DEFAULT TDG_SUP_TAB
#endif
namespace {

thread_local std::string g_err;

struct Fail {
    int code;
    std::string msg;
};

void ck(cudaError_t e, const char* what) {
    if (e != cudaSuccess) {
        cudaGetLastError();
        throw Fail{e == cudaErrorMemoryAllocation ? TDG_ERR_NOMEM : TDG_ERR_CUDA,
                    std::string(what) + ": " + cudaGetErrorString(e)};
    }
}

// Device->host copy ordered on the context's (non-blocking) stream, then waited for. A
// plain cudaMemcpy runs on the legacy stream and would not wait for work queued on it.
void d2h(cudaStream_t st, void* dst, const void* src, size_t bytes, const char* what) {
    ck(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, st), what);
    ck(cudaStreamSynchronize(st), what);
}

struct DevBuf {
    void* p = nullptr;
    size_t cap = 0;
    void ensure(size_t bytes, const char* name) {
        if (bytes < 256) bytes = 256;
        if (bytes <= cap) return;
        release();
        bytes = (bytes + (2u << 20) - 1) & ~size_t((2u << 20) - 1);
        cudaError_t e = cudaMalloc(&p, bytes);
        if (e != cudaSuccess) {
            p = nullptr;
            cudaGetLastError();
            throw Fail{TDG_ERR_NOMEM, std::string("device allocation of ") + name + " (" +
                                          std::to_string(bytes >> 20) + " MiB) failed: " + cudaGetErrorString(e)};
        }
        cap = bytes;
    }
    void release() {
        if (p) cudaFree(p);
        p = nullptr;
        cap = 0;
    }
    template <class T> T* as() const { return static_cast<T*>(p); }
};

struct HostCtl {
    PeelCtl peel;
    SupportCtl sup;
    StatsAcc stats;
    uint32_t word;  // small D2H scalar (component count, c_max, reorder check)
};

}  // namespace

namespace {
bool peel_filter();
}  // namespace

struct tdg_context {
    int device = 0;
    int sms = 148;
    cudaStream_t own = nullptr;
    cudaStream_t stream = nullptr;
    // persistent per-graph arrays (live through the peel)
    DevBuf off64, off, adj, eo, up, P, eid, el, opos, oeid, sbeg, dl, pbits, hbo, htab, filt;
    // one arena for the m-sized scratch: the build + support arrays and the peel lists share
    // it (they are never live at the same time; layout in ensure_arena)
    DevBuf arena;
    DevBuf fctl;  // FilterCtl of the resident graph
    DevBuf cchunk, nsl, ctl, sctl, sacc, cub, truss, sup, f0, f1, f2, bsum, bhist, bcur, trace;
    DevBuf kdeg, kcore, kL0, kL1, kA0, kA1, kwpre, kctl, ktmp, knoff, knadj, kperm, kbad, ing, ptext, pscr, ppairs;
    // arena views (recomputed by ensure_arena)
    uint32_t *src = nullptr, *flag = nullptr, *pos = nullptr, *oadj = nullptr, *osrc = nullptr, *stask = nullptr,
             *sx = nullptr, *s = nullptr, *L0 = nullptr, *L1 = nullptr, *A0 = nullptr, *A1 = nullptr, *F0 = nullptr,
             *F1 = nullptr, *cscr = nullptr;
    unsigned long long *ss = nullptr, *wpre = nullptr;
    size_t word = 0;
    HostCtl* hctl = nullptr;
    cudaEvent_t ev[8] = {};
    uint32_t launches = 0;

    void use() { ck(cudaSetDevice(device), "cudaSetDevice"); }

    // Arena of 14 "words" of 4(m+1) bytes (256-aligned). Build + support use words
    //   2-3 src (-> support work prefix wpre), 4-5 flag (-> internal-id scratch), 6-7 pos,
    //   8 oadj, 9 osrc, 10 stask, 11 sx, 12 s,
    // the peel uses 0-1 ss (packed state), 2-3 wpre, 4-7 cscr (task descriptors + a sorted
    // curr list / compaction scratch), 8 L0, 9 L1, 10 A0, 11 A1, 12 F0, 13 F1.
    // s (12) is read by k_peel_init while it writes ss (0-1); F0 (12) is first written by the
    // peel's first scan, after that.
    static constexpr int kArenaWords = 14;
    static size_t arena_word(uint64_t m) { return (4 * (m + 1) + 255) & ~size_t(255); }
    void ensure_arena(uint64_t m) {
        word = arena_word(m);
        arena.ensure(kArenaWords * word, "arena (build / support / peel scratch)");
        char* b = arena.as<char>();
        auto w32 = [&](int i) { return reinterpret_cast<uint32_t*>(b + i * word); };
        ss = reinterpret_cast<unsigned long long*>(b);
        wpre = reinterpret_cast<unsigned long long*>(b + 2 * word);
        src = w32(2);
        cscr = flag = w32(4);
        pos = w32(6);
        L0 = oadj = w32(8);
        L1 = osrc = w32(9);
        A0 = stask = w32(10);
        A1 = sx = w32(11);
        F0 = s = w32(12);
        F1 = w32(13);
    }

    void ensure_graph(uint64_t n, uint64_t m) {
        const uint64_t slots = 2 * m;
        off64.ensure((n + 1) * 8, "offsets64");
        off.ensure((n + 1) * 4, "offsets");
        adj.ensure(slots * 4, "adj");
        eo.ensure(n * 4, "eo");
        up.ensure((n + 1) * 4, "up");
        P.ensure((n + 1) * 4, "P");
        eid.ensure(slots * 4, "eid");
        el.ensure(m * 8, "el");
        opos.ensure((n + 1) * 4, "opos");
        oeid.ensure(m * 4, "oeid");
        sbeg.ensure((n + 1) * 4, "sbeg");
        dl.ensure(n * 4, "dl");
        ensure_arena(m);
        ctl.ensure(sizeof(PeelCtl), "ctl");
        sctl.ensure(sizeof(SupportCtl), "sctl");
        sacc.ensure(sizeof(StatsAcc), "stats");
        cub.ensure(build_cub_bytes(static_cast<uint32_t>(n), static_cast<uint32_t>(m)), "cub");
        bsum.ensure(sizeof(unsigned long long) * kMaxChunks, "bsum");
    }
    void ensure_peel(uint64_t n, uint64_t m) {
        ensure_arena(m);
        if (bhist.cap == 0) {
            bhist.ensure(kBuckets * 4, "bhist");
            ck(cudaMemsetAsync(bhist.p, 0, kBuckets * 4, stream), "memset");
        }
        bcur.ensure(kBuckets * 4, "bcur");
        nsl.ensure((n + 2) * 4, "nsl");
        cchunk.ensure(chunk_cap(m) * 12, "compaction chunks");
        pbits.ensure((m + 31) / 32 * 4, "processed bitmap");
    }
    static uint64_t chunk_cap(uint64_t m) { return (2 * m) / 512 + (2 * m) / 2048 + 2; }

    BuildBufs build_bufs(const int64_t* off64_dev) const {
        BuildBufs b;
        b.off64 = off64_dev;
        b.off = off.as<uint32_t>();
        b.adj = adj.as<uint32_t>();
        b.src = src;
        b.eo = eo.as<uint32_t>();
        b.up = up.as<uint32_t>();
        b.P = P.as<uint32_t>();
        b.eid = eid.as<uint32_t>();
        b.el = el.as<uint2>();
        b.flag = flag;
        b.pos = pos;
        b.opos = opos.as<uint32_t>();
        b.oadj = oadj;
        b.oeid = oeid.as<uint32_t>();
        b.osrc = osrc;
        b.stask = stask;
        b.sx = sx;
        b.sbeg = sbeg.as<uint32_t>();
        b.cub_tmp = cub.p;
        b.cub_bytes = cub.cap;
        return b;
    }
    DevGraph dev_graph(uint32_t n, uint32_t m) const {
        DevGraph g;
        g.n = n;
        g.m = m;
        g.off = off.as<uint32_t>();
        g.adj = adj.as<uint32_t>();
        g.eid = eid.as<uint32_t>();
        g.el = el.as<uint2>();
        g.dl = dl.as<uint32_t>();
        g.opos = opos.as<uint32_t>();
        g.oadj = oadj;
        g.oeid = oeid.as<uint32_t>();
        g.osrc = osrc;
        g.stask = stask;
        g.sx = sx;
        g.sbeg = sbeg.as<uint32_t>();
        g.htab = htab.as<uint32_t>();
        g.hbo = hbo.as<uint32_t>();
        g.nbuckets = htab.cap / 32;
        g.filt = peel_filter() ? filt.as<unsigned long long>() : nullptr;
        g.fctl = fctl.as<FilterCtl>();
        return g;
    }
    PeelBufs peel_bufs(uint32_t n) const {
        PeelBufs p;
        p.s = s;
        p.ss = ss;
        p.L[0] = L0;
        p.L[1] = L1;
        p.A[0] = A0;
        p.A[1] = A1;
        p.F[0] = F0;
        p.F[1] = F1;
        p.wpre = wpre;
        p.bsum = bsum.as<unsigned long long>();
        p.ctl = ctl.as<PeelCtl>();
        p.nsl = nsl.as<uint32_t>();
        p.nsl_cap = n + 1;
        const char* ch = std::getenv("TDG_COUNT");
        p.count = (ch && ch[0] == '1') ? 1u : 0u;
        p.bhist = bhist.as<uint32_t>();
        p.bcur = bcur.as<uint32_t>();
        uint32_t bits = 0;
        while ((1ull << bits) < n) bits++;
        p.bshift = bits > kBucketBits ? bits - kBucketBits : 0;
        p.trace = nullptr;
        p.trace_cap = 0;
        if (std::getenv("TDG_TRACE")) {
            p.trace = trace.as<unsigned long long>();
            p.trace_cap = static_cast<uint32_t>(trace.cap / 32);
        }
        const uint64_t cc = cchunk.cap / 12;
        p.chunk_cap = static_cast<uint32_t>(cc);
        p.chunks = cchunk.as<uint2>();
        p.ckept = reinterpret_cast<uint32_t*>(p.chunks + cc);
        // compaction scratch: 2 x 2m u32 in words 4-7; the sub-level task descriptors (16 B per
        // curr edge) share it — compaction runs only between a scan and the first sub-level
        p.sadj = cscr;
        p.seid = cscr + word / 2;  // 2 words later (word is in bytes: 2 * word / 4 u32)
        p.desc = reinterpret_cast<uint4*>(cscr);
        p.pbits = pbits.as<uint32_t>();
        p.hbo_w = hbo.as<uint32_t>();
        p.htab_w = htab.as<uint32_t>();
        p.filt_w = peel_filter() ? filt.as<unsigned long long>() : nullptr;
        p.rebuild_num = kPeelRebuildNum;
        p.rebuild_den = kPeelRebuildDen;
        p.nseg = kPeelRebuildMax + 1;
        if (const char* rb = std::getenv("TDG_REBUILD")) {  // diagnostic: "num/den[/max]", "0/0" = never
            unsigned a = 0, b = 0, mx = kPeelRebuildMax;
            if (std::sscanf(rb, "%u/%u/%u", &a, &b, &mx) >= 2) {
                p.rebuild_num = a;
                p.rebuild_den = b;
                p.nseg = (mx < 16 ? mx : 16) + 1;
            }
        }
        return p;
    }
    void trim() {
        DevBuf* all[] = {&fctl, &off64, &off, &adj, &eo, &up, &P, &eid, &el, &opos, &oeid, &sbeg, &dl, &pbits, &hbo, &htab, &filt,
                         &arena, &cchunk, &nsl, &ctl, &sctl, &sacc, &cub, &truss, &sup, &f0, &f1, &f2, &bsum, &bhist,
                         &bcur, &trace, &kdeg, &kcore, &kL0, &kL1, &kA0, &kA1, &kwpre, &kctl, &ktmp, &knoff, &knadj,
                         &kperm, &kbad, &ing, &ptext, &pscr, &ppairs};
        for (DevBuf* b : all) b->release();
        word = 0;
    }
    KcoreBufs kcore_bufs(uint64_t n, uint64_t m) {
        kdeg.ensure((n + 2) * 4, "kdeg");
        kcore.ensure((n + 2) * 4, "kcore");
        kL0.ensure(n * 4, "kL0");
        kL1.ensure(n * 4, "kL1");
        kA0.ensure(n * 4, "kA0");
        kA1.ensure(n * 4, "kA1");
        kwpre.ensure(n * 8, "kwpre");
        kctl.ensure(kKcoreCtlBytes, "kctl");
        ktmp.ensure(2 * m * 4, "ktmp");
        bsum.ensure(sizeof(unsigned long long) * kMaxChunks, "bsum");
        cub.ensure(kcore_cub_bytes(static_cast<uint32_t>(n), static_cast<uint32_t>(m)), "cub");
        KcoreBufs b;
        b.deg = kdeg.as<uint32_t>();
        b.core = kcore.as<uint32_t>();
        b.L0 = kL0.as<uint32_t>();
        b.L1 = kL1.as<uint32_t>();
        b.A0 = kA0.as<uint32_t>();
        b.A1 = kA1.as<uint32_t>();
        b.tmp_adj = ktmp.as<uint32_t>();
        b.wpre = kwpre.as<unsigned long long>();
        b.bsum = bsum.as<unsigned long long>();
        b.ctl = kctl.p;
        b.cub_tmp = cub.p;
        b.cub_bytes = cub.cap;
        return b;
    }
    float ms(int a, int b) const {
        float t = 0;
        cudaEventElapsedTime(&t, ev[a], ev[b]);
        return t;
    }
};

namespace {

void destroy_ctx(tdg_context* ctx);

// ctx == NULL: one default context per calling thread (created lazily on the thread's
// current device, destroyed when the thread exits), so threads that pass NULL never share
// device buffers or the pinned control block.
struct DefaultCtx {
    tdg_context* c = nullptr;
    ~DefaultCtx() {
        if (c) destroy_ctx(c);
    }
};
thread_local DefaultCtx g_default;

template <class F>
int guarded(F&& f) {
    try {
        f();
        return TDG_OK;
    } catch (const Fail& e) {
        g_err = e.msg;
        return e.code;
    } catch (const std::bad_alloc&) {
        g_err = "host allocation failed";
        return TDG_ERR_NOMEM;
    } catch (const std::exception& e) {
        g_err = e.what();
        return TDG_ERR_INVALID;
    }
}

void create_ctx(int device, tdg_context** out) {
    int count = 0;
    cudaError_t e = cudaGetDeviceCount(&count);
    if (e != cudaSuccess || count == 0) {
        cudaGetLastError();
        throw Fail{TDG_ERR_CUDA, "no CUDA device available (this library has no CPU path)"};
    }
    if (device == -1) ck(cudaGetDevice(&device), "cudaGetDevice");
    if (device < 0 || device >= count) throw Fail{TDG_ERR_INVALID, "device index out of range"};
    cudaDeviceProp prop;
    ck(cudaGetDeviceProperties(&prop, device), "cudaGetDeviceProperties");
    if (prop.major != 10 || prop.minor != 0)
        throw Fail{TDG_ERR_CUDA, std::string("device ") + prop.name + " is not sm_100 (B200); kernels are built for sm_100a only"};
    if (!prop.cooperativeLaunch) throw Fail{TDG_ERR_CUDA, "device lacks cooperative launch"};
    auto* c = new tdg_context;
    c->device = device;
    c->sms = prop.multiProcessorCount;
    ck(cudaSetDevice(device), "cudaSetDevice");
    ck(cudaStreamCreateWithFlags(&c->own, cudaStreamNonBlocking), "cudaStreamCreate");
    c->stream = c->own;
    for (auto& ev : c->ev) ck(cudaEventCreate(&ev), "cudaEventCreate");
    ck(cudaMallocHost(reinterpret_cast<void**>(&c->hctl), sizeof(HostCtl)), "cudaMallocHost");
    std::memset(c->hctl, 0, sizeof(HostCtl));
    *out = c;
}

void destroy_ctx(tdg_context* ctx) {
    cudaSetDevice(ctx->device);
    cudaStreamSynchronize(ctx->stream);
    ctx->trim();
    for (auto& ev : ctx->ev) if (ev) cudaEventDestroy(ev);
    if (ctx->own) cudaStreamDestroy(ctx->own);
    if (ctx->hctl) cudaFreeHost(ctx->hctl);
    if (g_default.c == ctx) g_default.c = nullptr;
    delete ctx;
    cudaGetLastError();  // (at process exit the runtime may already be unloading)
}

tdg_context* resolve(tdg_context* ctx) {
    if (ctx) return ctx;
    if (!g_default.c) {
        int dev = 0;
        cudaGetDevice(&dev);
        create_ctx(dev, &g_default.c);
    }
    return g_default.c;
}

struct Dims {
    uint32_t n, m;
};

Dims check_graph(const tdg_csr* g, bool host_ptrs) {
    if (!g) throw Fail{TDG_ERR_INVALID, "graph is NULL"};
    if (g->n < 0 || g->m < 0) throw Fail{TDG_ERR_INVALID, "negative n or m"};
    if (static_cast<uint64_t>(g->n) >= 0xffffffffull)
        throw Fail{TDG_ERR_RANGE, "graph exceeds 32-bit vertex id width"};
    if (2 * static_cast<uint64_t>(g->m) > 0xffffffffull)
        throw Fail{TDG_ERR_RANGE, "graph exceeds 32-bit edge width (2m too large)"};  // graph.cpp:48-49
    if (!g->offsets || (g->m > 0 && !g->neighbors)) throw Fail{TDG_ERR_INVALID, "NULL CSR array"};
    if (host_ptrs && (g->offsets[0] != 0 || g->offsets[g->n] != 2 * g->m))
        throw Fail{TDG_ERR_INVALID, "offsets must start at 0 and end at 2m"};
    return Dims{static_cast<uint32_t>(g->n), static_cast<uint32_t>(g->m)};
}

// Upload / alias the CSR and build eo/eid/el (+ orientation). Records ev[0], ev[1], ev[2].
// Peel membership filters (tdg_common.cuh); TDG_PEEL_FILTER=0 disables them (A/B).
bool peel_filter() {
    static const bool on = [] {
        const char* e = std::getenv("TDG_PEEL_FILTER");
        return !(e && e[0] == '0');
    }();
    return on;
}

// internal=true (truss / support): edge ids become oriented slots before the hash tables are
// filled (build.cu launch_internal_ids); results go back to reference ids via oeid.
void stage_and_build(tdg_context* c, const tdg_csr* g, Dims d, bool host_ptrs, bool orient, bool tables,
                     bool internal = false) {
    c->ensure_graph(d.n, d.m);
    const int64_t* off64 = g->offsets;
    ck(cudaEventRecord(c->ev[0], c->stream), "event");
    if (host_ptrs) {
        ck(cudaMemcpyAsync(c->off64.p, g->offsets, (size_t(d.n) + 1) * 8, cudaMemcpyHostToDevice, c->stream), "H2D offsets");
        if (d.m)
            ck(cudaMemcpyAsync(c->adj.p, g->neighbors, size_t(d.m) * 8, cudaMemcpyHostToDevice, c->stream), "H2D neighbors");
        off64 = c->off64.as<int64_t>();
    } else if (d.m) {
        ck(cudaMemcpyAsync(c->adj.p, g->neighbors, size_t(d.m) * 8, cudaMemcpyDeviceToDevice, c->stream), "D2D neighbors");
    }
    ck(cudaEventRecord(c->ev[1], c->stream), "event");
    ck(launch_build(c->build_bufs(off64), d.n, d.m, orient, c->stream, &c->launches), "build kernels");
    if (internal)  // flag (2m+1 u32) is free once the build is done
        ck(launch_internal_ids(c->build_bufs(off64), d.m, c->flag, c->stream, &c->launches),
           "internal edge ids");
    if (tables) {  // neighbour -> edge-id hash tables (+ filters): sizes depend on n and m only
        c->hbo.ensure((size_t(d.n) + 1) * 4, "table offsets");
        c->htab.ensure(htab_buckets(d.n, d.m) * 32, "hash tables");
        ck(launch_htab_fill(c->off.as<uint32_t>(), c->adj.as<uint32_t>(), c->src, c->eid.as<uint32_t>(), d.n, d.m,
                            c->up.as<uint32_t>(), c->hbo.as<uint32_t>(), c->htab.as<uint32_t>(), c->cub.p, c->cub.cap,
                            c->stream, &c->launches), "hash fill");
        if (peel_filter()) {
            c->filt.ensure(filter_words(d.n, d.m) * 8, "filters");
            c->fctl.ensure(sizeof(FilterCtl), "filter control");
            ck(launch_filter_fill(c->hbo.as<uint32_t>(), c->adj.as<uint32_t>(), c->src, d.n, d.m,
                                  c->filt.as<unsigned long long>(), c->fctl.as<FilterCtl>(), c->stream, &c->launches),
               "filter fill");
        }
    }
    ck(cudaEventRecord(c->ev[2], c->stream), "event");
}

void check_peel_ctl(const PeelCtl& pc) {
    if (pc.nsl_overflow) throw Fail{TDG_ERR_RANGE, "sub-level trace overflow: a level index reached n+1"};
    if (pc.chunk_overflow) throw Fail{TDG_ERR_RANGE, "internal error: compaction chunk table too small"};
}

void fill_times(tdg_times* t, tdg_context* c, bool host, bool peel) {
    if (!t) return;
    std::memset(t, 0, sizeof(*t));
    t->h2d_ms = host ? c->ms(0, 1) : 0.0;
    t->build_ms = c->ms(1, 2);
    t->support_ms = c->ms(2, 3);
    if (peel) {
        t->peel_ms = c->ms(3, 6);
        t->d2h_ms = host ? c->ms(4, 5) : 0.0;
        t->total_ms = c->ms(0, 5);
    } else {
        t->d2h_ms = host ? c->ms(3, 5) : 0.0;
        t->total_ms = c->ms(0, 5);
    }
    t->triangles = c->hctl->sup.tri3 / 3;
    t->support_probes = c->hctl->sup.probes;
    t->kernel_launches = c->launches;
}

int truss_impl(tdg_context* ctx, const tdg_csr* g, uint32_t* truss_out, uint32_t* support_out,
               uint32_t* nsl_out, uint64_t nsl_cap, uint64_t* nsl_len, tdg_times* times, bool host) {
    return guarded([&] {
        tdg_context* c = resolve(ctx);
        c->use();
        const Dims d = check_graph(g, host);
        if (!truss_out && d.m) throw Fail{TDG_ERR_INVALID, "truss_out is NULL"};
        c->launches = 0;
        stage_and_build(c, g, d, host, true, true, true);
        c->ensure_peel(d.n, d.m);
        if (std::getenv("TDG_TRACE")) c->trace.ensure(size_t(32) << 20, "trace");
        const DevGraph dg = c->dev_graph(d.n, d.m);
        ck(launch_support(dg, c->s, c->wpre, c->bsum.as<unsigned long long>(),
                          c->sctl.as<SupportCtl>(), c->sms, c->stream, &c->launches), "support kernels");
        uint32_t* sup_dev = nullptr;
        if (support_out && d.m) {
            if (host) { c->sup.ensure(size_t(d.m) * 4, "support copy"); sup_dev = c->sup.as<uint32_t>(); }
            else sup_dev = support_out;
            ck(launch_to_ref(dg.oeid, c->s, d.m, 0, sup_dev, c->stream, &c->launches), "support copy");
        }
        ck(cudaEventRecord(c->ev[3], c->stream), "event");
        const PeelBufs pb = c->peel_bufs(d.n);
        ck(launch_peel(dg, pb, c->sms, c->stream, &c->launches), "peel kernel");
        ck(cudaEventRecord(c->ev[6], c->stream), "event");
        uint32_t* tdev = truss_out;
        if (host) { c->truss.ensure(size_t(d.m) * 4, "truss"); tdev = c->truss.as<uint32_t>(); }
        ck(launch_finalize(pb.ss, dg.oeid, d.m, tdev, pb.ctl, c->stream, &c->launches), "finalize kernel");
        ck(cudaEventRecord(c->ev[4], c->stream), "event");
        if (host && d.m) {
            ck(cudaMemcpyAsync(truss_out, tdev, size_t(d.m) * 4, cudaMemcpyDeviceToHost, c->stream), "D2H truss");
            if (sup_dev) ck(cudaMemcpyAsync(support_out, sup_dev, size_t(d.m) * 4, cudaMemcpyDeviceToHost, c->stream), "D2H support");
        }
        ck(cudaEventRecord(c->ev[5], c->stream), "event");
        ck(cudaMemcpyAsync(&c->hctl->peel, pb.ctl, sizeof(PeelCtl), cudaMemcpyDeviceToHost, c->stream), "D2H ctl");
        ck(cudaMemcpyAsync(&c->hctl->sup, c->sctl.p, sizeof(SupportCtl), cudaMemcpyDeviceToHost, c->stream), "D2H sctl");
        ck(cudaStreamSynchronize(c->stream), "decomposition");
        const PeelCtl& pc = c->hctl->peel;
        check_peel_ctl(pc);
        const uint64_t len = d.m ? pc.levels_len : 0;
        if (const char* tp = std::getenv("TDG_TRACE")) {  // diagnostic dump: level, cs, W, ns, K
            const size_t k = std::min<size_t>(pc.sublevels, c->trace.cap / 32);
            std::vector<unsigned long long> h(4 * k);
            if (k) d2h(c->stream, h.data(), c->trace.p, 32 * k, "D2H trace");
            if (FILE* f = std::fopen(tp, "w")) {
                for (size_t i = 0; i < k; i++)
                    std::fprintf(f, "%llu %llu %llu %llu %llu\n", h[4 * i] >> 32, h[4 * i] & 0xffffffffull, h[4 * i + 1],
                                 h[4 * i + 2], h[4 * i + 3]);
                std::fclose(f);
            }
        }
        if (std::getenv("TDG_SUP_DEBUG"))  // diagnostic: block geometry of the support pass
            std::fprintf(stderr, "tdg support: %s geometry, %.1f %% of the work has an owner list above %u keys\n",
                         c->hctl->sup.big_geometry ? "big" : "small",
                         c->hctl->sup.work_items ? 100.0 * double(c->hctl->sup.big_work) / double(c->hctl->sup.work_items) : 0.0,
                         unsigned(TDG_SUP_TAB_DEFAULT / 4));
        if (std::getenv("TDG_FILTER_DEBUG") && c->fctl.p && peel_filter() && d.m) {  // diagnostic: filter mode of this graph
            FilterCtl fc;
            d2h(c->stream, &fc, c->fctl.p, sizeof(fc), "D2H filter control");
            std::fprintf(stderr, "tdg filter: %s mode, fp estimate %.4f (keys %llu)\n", fc.hashed ? "hash" : "rank",
                         fc.keys ? double(fc.fp) / 262144.0 / double(fc.keys) : 0.0, fc.keys);
        }
        if (nsl_len) *nsl_len = len;
        if (nsl_out && len) {
            const uint64_t k = len < nsl_cap ? len : nsl_cap;
            if (k) d2h(c->stream, nsl_out, pb.nsl, k * 4, "D2H nsl");
        }
        if (times) {
            fill_times(times, c, host, true);
            times->levels = len;
            times->sublevels = pc.sublevels;
            times->scans = pc.scans;
            times->compactions = pc.compactions;
            times->scan_ms = pc.scan_ns * 1e-6;
            times->process_ms = pc.proc_ns * 1e-6;
            times->compact_ms = pc.compact_ns * 1e-6;
            times->rebuild_ms = pc.rebuild_ns * 1e-6;
            times->table_rebuilds = pc.table_rebuilds;
            times->probes = pc.probes;
            times->hits = pc.cnt[kCntHits];
            times->dead_probes = pc.cnt[kCntDead];
            times->t_max = d.m ? pc.t_max : 0;
        }
    });
}

int support_impl(tdg_context* ctx, const tdg_csr* g, uint32_t* support_out, tdg_times* times, bool host,
                 uint32_t shard = 0, uint32_t nshards = 1) {
    return guarded([&] {
        tdg_context* c = resolve(ctx);
        c->use();
        if (nshards == 0 || shard >= nshards) throw Fail{TDG_ERR_INVALID, "shard must be < nshards"};
        const Dims d = check_graph(g, host);
        if (!support_out && d.m) throw Fail{TDG_ERR_INVALID, "support_out is NULL"};
        c->launches = 0;
        stage_and_build(c, g, d, host, true, false, true);
        const DevGraph dg = c->dev_graph(d.n, d.m);
        uint32_t* sdev = support_out;
        if (host) { c->sup.ensure(size_t(d.m) * 4 + 4, "support copy"); sdev = c->sup.as<uint32_t>(); }
        ck(launch_support(dg, c->s, c->wpre, c->bsum.as<unsigned long long>(),
                          c->sctl.as<SupportCtl>(), c->sms, c->stream, &c->launches, shard, nshards), "support kernels");
        ck(launch_to_ref(dg.oeid, c->s, d.m, 0, sdev, c->stream, &c->launches), "support to ref ids");
        ck(cudaEventRecord(c->ev[3], c->stream), "event");
        if (host && d.m)
            ck(cudaMemcpyAsync(support_out, sdev, size_t(d.m) * 4, cudaMemcpyDeviceToHost, c->stream), "D2H support");
        ck(cudaEventRecord(c->ev[5], c->stream), "event");
        ck(cudaMemcpyAsync(&c->hctl->sup, c->sctl.p, sizeof(SupportCtl), cudaMemcpyDeviceToHost, c->stream), "D2H sctl");
        ck(cudaStreamSynchronize(c->stream), "support");
        fill_times(times, c, host, false);
    });
}

}  // namespace

extern "C" {

const char* tdg_version(void) { return "tdg 0.1 (sm_100a)"; }
const char* tdg_last_error(void) { return g_err.c_str(); }

int tdg_context_create(int device, tdg_context** out) {
    return guarded([&] {
        if (!out) throw Fail{TDG_ERR_INVALID, "out is NULL"};
        create_ctx(device, out);
    });
}

int tdg_context_destroy(tdg_context* ctx) {
    return guarded([&] {
        if (ctx) destroy_ctx(ctx);
    });
}

int tdg_context_set_stream(tdg_context* ctx, void* stream) {
    return guarded([&] {
        tdg_context* c = resolve(ctx);
        c->stream = stream ? static_cast<cudaStream_t>(stream) : c->own;
    });
}

void* tdg_context_stream(tdg_context* ctx) {
    tdg_context* c = nullptr;
    if (guarded([&] { c = resolve(ctx); }) != TDG_OK) return nullptr;
    return c->stream;
}

int tdg_context_trim(tdg_context* ctx) {
    return guarded([&] {
        tdg_context* c = resolve(ctx);
        c->use();
        ck(cudaStreamSynchronize(c->stream), "sync");
        c->trim();
    });
}

int tdg_truss(tdg_context* ctx, const tdg_csr* g, uint32_t* truss_out, uint32_t* support_out,
              uint32_t* nsl_out, uint64_t nsl_cap, uint64_t* nsl_len, tdg_times* times) {
    return truss_impl(ctx, g, truss_out, support_out, nsl_out, nsl_cap, nsl_len, times, true);
}

int tdg_truss_device(tdg_context* ctx, const tdg_csr* g, uint32_t* truss_out, uint32_t* support_out,
                     uint32_t* nsl_out, uint64_t nsl_cap, uint64_t* nsl_len, tdg_times* times) {
    return truss_impl(ctx, g, truss_out, support_out, nsl_out, nsl_cap, nsl_len, times, false);
}

int tdg_support(tdg_context* ctx, const tdg_csr* g, uint32_t* support_out, tdg_times* times) {
    return support_impl(ctx, g, support_out, times, true);
}

int tdg_support_device(tdg_context* ctx, const tdg_csr* g, uint32_t* support_out, tdg_times* times) {
    return support_impl(ctx, g, support_out, times, false);
}

int tdg_support_shard(tdg_context* ctx, const tdg_csr* g, uint32_t shard, uint32_t nshards, uint32_t* support_out,
                      tdg_times* times) {
    return support_impl(ctx, g, support_out, times, true, shard, nshards);
}

int tdg_support_shard_device(tdg_context* ctx, const tdg_csr* g, uint32_t shard, uint32_t nshards,
                             uint32_t* support_out, tdg_times* times) {
    return support_impl(ctx, g, support_out, times, false, shard, nshards);
}

int tdg_build_truss_graph(tdg_context* ctx, const tdg_csr* g, uint32_t* eo, uint32_t* eid, uint32_t* el) {
    return guarded([&] {
        if (!eo || !eid || !el) throw Fail{TDG_ERR_INVALID, "NULL output array"};
        tdg_context* c = resolve(ctx);
        c->use();
        const Dims d = check_graph(g, true);
        c->launches = 0;
        stage_and_build(c, g, d, true, false, false);
        if (d.n) ck(cudaMemcpyAsync(eo, c->eo.p, size_t(d.n) * 4, cudaMemcpyDeviceToHost, c->stream), "D2H eo");
        if (d.m) {
            ck(cudaMemcpyAsync(eid, c->eid.p, size_t(d.m) * 8, cudaMemcpyDeviceToHost, c->stream), "D2H eid");
            ck(cudaMemcpyAsync(el, c->el.p, size_t(d.m) * 8, cudaMemcpyDeviceToHost, c->stream), "D2H el");
        }
        ck(cudaStreamSynchronize(c->stream), "build");
    });
}

int tdg_triangle_count(tdg_context* ctx, const tdg_csr* g, uint64_t* count, tdg_times* times) {
    return guarded([&] {
        if (!count) throw Fail{TDG_ERR_INVALID, "count is NULL"};
        tdg_context* c = resolve(ctx);
        c->use();
        const Dims d = check_graph(g, true);
        c->launches = 0;
        stage_and_build(c, g, d, true, true, false);
        ck(launch_triangle_count(c->dev_graph(d.n, d.m), c->wpre,
                                 c->bsum.as<unsigned long long>(), c->sctl.as<SupportCtl>(), c->sms, c->stream,
                                 &c->launches), "triangle count");
        ck(cudaEventRecord(c->ev[3], c->stream), "event");
        ck(cudaEventRecord(c->ev[5], c->stream), "event");
        ck(cudaMemcpyAsync(&c->hctl->sup, c->sctl.p, sizeof(SupportCtl), cudaMemcpyDeviceToHost, c->stream), "D2H sctl");
        ck(cudaStreamSynchronize(c->stream), "triangle count");
        *count = c->hctl->sup.tri3;
        fill_times(times, c, true, false);
        if (times) times->triangles = *count;
    });
}

int tdg_ktruss_components(tdg_context* ctx, const tdg_csr* g, const uint32_t* truss, uint32_t k,
                          uint32_t* comp_of_edge, uint64_t* ncomp) {
    return guarded([&] {
        if (!ncomp || (g && g->m && (!truss || !comp_of_edge))) throw Fail{TDG_ERR_INVALID, "NULL argument"};
        tdg_context* c = resolve(ctx);
        c->use();
        const Dims d = check_graph(g, true);
        uint32_t t_max = 0;
        for (uint32_t e = 0; e < d.m; e++) t_max = truss[e] > t_max ? truss[e] : t_max;
        if (k < 2 || (t_max > 0 && k > t_max))  // truss_serial.cpp:179-180
            throw Fail{TDG_ERR_INVALID, "ktruss_subgraphs: k out of range [2, t_max]"};
        *ncomp = 0;
        c->launches = 0;
        stage_and_build(c, g, d, true, false, false);
        if (d.m == 0) { ck(cudaStreamSynchronize(c->stream), "sync"); return; }
        // scratch: s <- truss, stamp-buffer halves / lists for the rest
        c->ensure_peel(d.n, d.m);
        c->truss.ensure(size_t(d.m) * 4, "truss");
        c->f0.ensure((size_t(d.m) + 1) * 4, "flag");
        c->f1.ensure((size_t(d.m) + 1) * 4, "rank");
        c->cub.ensure(ktruss_cub_bytes(d.m), "cub");
        ck(cudaMemcpyAsync(c->truss.p, truss, size_t(d.m) * 4, cudaMemcpyHostToDevice, c->stream), "H2D truss");
        KtrussBufs kb;
        kb.parent = c->dl.as<uint32_t>();
        kb.first = c->up.as<uint32_t>();
        kb.root_of_edge = c->L0;
        kb.flag = c->f0.as<uint32_t>();
        kb.rank = c->f1.as<uint32_t>();
        kb.comp = c->L1;
        kb.cub_tmp = c->cub.p;
        kb.cub_bytes = c->cub.cap;
        ck(launch_ktruss(c->el.as<uint2>(), c->truss.as<uint32_t>(), d.n, d.m, k, kb, c->stream, &c->launches),
           "ktruss kernels");
        ck(cudaMemcpyAsync(comp_of_edge, kb.comp, size_t(d.m) * 4, cudaMemcpyDeviceToHost, c->stream), "D2H comp");
        ck(cudaMemcpyAsync(&c->hctl->word, kb.rank + d.m, 4, cudaMemcpyDeviceToHost, c->stream), "D2H ncomp");
        ck(cudaStreamSynchronize(c->stream), "ktruss");
        *ncomp = c->hctl->word;
    });
}

int tdg_kcore(tdg_context* ctx, const tdg_csr* g, uint32_t* core_out, uint32_t* c_max) {
    return guarded([&] {
        if (!c_max || (g && g->n && !core_out)) throw Fail{TDG_ERR_INVALID, "NULL argument"};
        tdg_context* c = resolve(ctx);
        c->use();
        const Dims d = check_graph(g, true);
        c->launches = 0;
        *c_max = 0;
        stage_and_build(c, g, d, true, false, false);
        const KcoreBufs kb = c->kcore_bufs(d.n, d.m);
        ck(launch_kcore(c->off.as<uint32_t>(), c->adj.as<uint32_t>(), d.n, kb, c->sms, c->stream, &c->launches,
                        kb.deg + d.n), "kcore kernel");
        if (d.n) {
            ck(cudaMemcpyAsync(core_out, kb.core, size_t(d.n) * 4, cudaMemcpyDeviceToHost, c->stream), "D2H core");
            ck(cudaMemcpyAsync(&c->hctl->word, kb.deg + d.n, 4, cudaMemcpyDeviceToHost, c->stream), "D2H c_max");
        }
        ck(cudaStreamSynchronize(c->stream), "kcore");
        *c_max = d.n ? c->hctl->word : 0;
    });
}

int tdg_coreness_order(tdg_context* ctx, uint64_t n, const uint32_t* core, uint32_t* perm_out) {
    return guarded([&] {
        if (n && (!core || !perm_out)) throw Fail{TDG_ERR_INVALID, "NULL argument"};
        if (n >= 0xffffffffull) throw Fail{TDG_ERR_RANGE, "too many vertices"};
        tdg_context* c = resolve(ctx);
        c->use();
        if (n == 0) return;
        c->launches = 0;
        const KcoreBufs kb = c->kcore_bufs(n, 0);
        c->kperm.ensure(n * 4, "perm");
        ck(cudaMemcpyAsync(kb.A0, core, n * 4, cudaMemcpyHostToDevice, c->stream), "H2D core");
        // sort keys come from a copy so the caller's order array stays untouched
        ck(cudaMemcpyAsync(kb.core, kb.A0, n * 4, cudaMemcpyDeviceToDevice, c->stream), "D2D core");
        ck(launch_coreness_order(kb.core, static_cast<uint32_t>(n), kb, c->kperm.as<uint32_t>(), c->stream,
                                 &c->launches), "coreness order");
        ck(cudaMemcpyAsync(perm_out, c->kperm.p, n * 4, cudaMemcpyDeviceToHost, c->stream), "D2H perm");
        ck(cudaStreamSynchronize(c->stream), "coreness order");
    });
}

int tdg_reorder(tdg_context* ctx, const tdg_csr* g, const uint32_t* perm, int64_t* out_offsets,
                int32_t* out_neighbors) {
    return guarded([&] {
        tdg_context* c = resolve(ctx);
        c->use();
        const Dims d = check_graph(g, true);
        if (!out_offsets || (d.n && !perm) || (d.m && !out_neighbors)) throw Fail{TDG_ERR_INVALID, "NULL argument"};
        c->launches = 0;
        stage_and_build(c, g, d, true, false, false);
        const KcoreBufs kb = c->kcore_bufs(d.n, d.m);
        c->kperm.ensure((size_t(d.n) + 1) * 4, "perm");
        c->knoff.ensure((size_t(d.n) + 1) * 4, "noff");
        c->knadj.ensure(size_t(d.m) * 8, "nadj");
        c->kbad.ensure(4, "bad");
        if (d.n) ck(cudaMemcpyAsync(c->kperm.p, perm, size_t(d.n) * 4, cudaMemcpyHostToDevice, c->stream), "H2D perm");
        ck(launch_reorder(c->off.as<uint32_t>(), c->adj.as<uint32_t>(), c->kperm.as<uint32_t>(), d.n, d.m, kb,
                          c->knoff.as<uint32_t>(), c->knadj.as<uint32_t>(), c->kbad.as<uint32_t>(), c->stream,
                          &c->launches), "reorder");
        ck(cudaMemcpyAsync(&c->hctl->word, c->kbad.p, 4, cudaMemcpyDeviceToHost, c->stream), "D2H check");
        ck(cudaStreamSynchronize(c->stream), "reorder");
        if (c->hctl->word)  // graph.cpp:106-113
            throw Fail{TDG_ERR_INVALID, "reorder: permutation is not a bijection on 0..n-1"};
        std::vector<uint32_t> noff(size_t(d.n) + 1);
        d2h(c->stream, noff.data(), c->knoff.p, noff.size() * 4, "D2H offsets");
        for (size_t i = 0; i < noff.size(); i++) out_offsets[i] = noff[i];
        if (d.m) d2h(c->stream, out_neighbors, c->knadj.p, size_t(d.m) * 8, "D2H neighbors");
    });
}

int tdg_canonicalize(tdg_context* ctx, const uint64_t* pairs, uint64_t npairs, int64_t* offsets, int32_t* neighbors,
                     uint64_t* labels, int64_t* n_out, int64_t* m_out) {
    return guarded([&] {
        if (!n_out || !m_out || !offsets || (npairs && (!pairs || !neighbors || !labels)))
            throw Fail{TDG_ERR_INVALID, "NULL argument"};
        if (2 * npairs >= 0xffffffffull)  // graph.cpp:30-31, 48-49 (32-bit ids and slots)
            throw Fail{TDG_ERR_RANGE, "graph exceeds 32-bit edge width (2m too large)"};
        tdg_context* c = resolve(ctx);
        c->use();
        *n_out = 0;
        *m_out = 0;
        offsets[0] = 0;
        if (npairs == 0) return;
        const uint64_t N = 2 * npairs;
        // carve one allocation (8-byte arrays first)
        const size_t cubb = ingest_cub_bytes(npairs);
        const size_t bytes = 8 * (N * 4 + 2 * npairs + 1) + 4 * (N * 15 + 8) + cubb + 256;
        c->ing.ensure(bytes, "ingest");
        char* p = static_cast<char*>(c->ing.p);
        auto take8 = [&](uint64_t cnt) { auto* r = reinterpret_cast<unsigned long long*>(p); p += 8 * cnt; return r; };
        auto take4 = [&](uint64_t cnt) { auto* r = reinterpret_cast<uint32_t*>(p); p += 4 * cnt; return r; };
        IngestBufs B;
        B.labels_in = take8(N);
        B.key_sorted = take8(N);
        B.glabel = take8(N);
        B.labels_out = take8(N);
        B.keys = take8(npairs);
        B.keys_sorted = take8(npairs);
        B.nuniq = take8(1);
        B.pos_in = take4(N);
        B.pos_sorted = take4(N);
        B.head = take4(N + 1);
        B.gidx = take4(N + 1);
        B.first_pos = take4(N);
        B.gseq = take4(N);
        B.first_sorted = take4(N);
        B.gsorted = take4(N);
        B.rank_of = take4(N);
        B.vid = take4(N);
        B.deg = take4(N + 1);
        B.off = take4(N + 1);
        B.cursor = take4(N + 1);
        B.nb_tmp = take4(N);
        B.nb = take4(N);
        p = reinterpret_cast<char*>((reinterpret_cast<uintptr_t>(p) + 255) & ~uintptr_t(255));
        B.cub_tmp = p;
        B.cub_bytes = cubb;
        c->launches = 0;
        ck(cudaMemcpyAsync(B.labels_in, pairs, N * 8, cudaMemcpyHostToDevice, c->stream), "H2D pairs");
        uint64_t n = 0, m = 0;
        {
            const cudaError_t e = launch_ingest(B, npairs, c->stream, &n, &m, &c->launches);
            ck(e, (std::string("ingest kernels after step '") + g_ingest_step + "'").c_str());
        }
        std::vector<uint32_t> off(n + 1);
        d2h(c->stream, off.data(), B.off, (n + 1) * 4, "D2H offsets");
        for (uint64_t i = 0; i <= n; i++) offsets[i] = off[i];
        if (m) d2h(c->stream, neighbors, B.nb, 2 * m * 4, "D2H neighbors");
        d2h(c->stream, labels, B.labels_out, n * 8, "D2H labels");
        *n_out = static_cast<int64_t>(n);
        *m_out = static_cast<int64_t>(m);
    });
}

int tdg_read_edge_list(tdg_context* ctx, const char* path, uint64_t** pairs_out, uint64_t* npairs) {
    return guarded([&] {
        if (!path || !pairs_out || !npairs) throw Fail{TDG_ERR_INVALID, "NULL argument"};
        *pairs_out = nullptr;
        *npairs = 0;
        const std::string p(path);
        // host: read / inflate (gzopen reads plain text too, as the reference)
        gzFile f = gzopen(path, "rb");
        if (!f) throw Fail{TDG_ERR_IO, "cannot open input file: " + p};
        std::vector<unsigned char> text;
        for (;;) {
            const size_t at = text.size(), blk = size_t(64) << 20;
            text.resize(at + blk);
            const int r = gzread(f, text.data() + at, static_cast<unsigned>(blk));
            if (r < 0) {
                gzclose(f);
                throw Fail{TDG_ERR_IO, "read error: " + p};
            }
            text.resize(at + static_cast<size_t>(r));
            if (static_cast<size_t>(r) < blk) break;
        }
        gzclose(f);
        tdg_context* c = resolve(ctx);
        c->use();
        c->launches = 0;
        // GPU: parse chunks of <= 1 GiB cut after a '\n' (segment counts stay 32-bit)
        std::vector<uint64_t> out;
        const size_t N = text.size(), kChunk = size_t(1) << 30;
        for (size_t c0 = 0; c0 < N;) {
            size_t c1 = std::min(N, c0 + kChunk);
            if (c1 < N) {
                while (c1 > c0 && text[c1 - 1] != '\n') c1--;
                if (c1 == c0) throw Fail{TDG_ERR_IO, p + ": line longer than 1 GiB"};
            }
            const uint64_t nb = c1 - c0, nseg = (nb + 255) / 256;
            c->ptext.ensure(nb, "edge-list text");
            const size_t sb = parse_scratch_bytes(nb);
            c->pscr.ensure(sb + 8, "parse scratch");
            auto* err = reinterpret_cast<unsigned long long*>(c->pscr.as<char>() + (c->pscr.cap - 8));
            ck(cudaMemcpyAsync(c->ptext.p, text.data() + c0, nb, cudaMemcpyHostToDevice, c->stream), "H2D text");
            ck(launch_parse_count(c->ptext.as<unsigned char>(), nb, c->pscr.p, c->pscr.cap - 8, err, c->stream,
                                  &c->launches), "parse kernels");
            unsigned long long e = 0;
            uint32_t total = 0;
            d2h(c->stream, &e, err, 8, "D2H parse status");
            if (e != ~0ull) {
                const size_t pos = c0 + static_cast<size_t>(e >> 2);
                const uint64_t lineno = 1 + static_cast<uint64_t>(std::count(text.begin(), text.begin() + pos, '\n'));
                std::string why;
                switch (static_cast<uint32_t>(e & 3)) {
                    case kParseNegative: why = "negative vertex label"; break;
                    case kParseTrailing: why = "trailing characters after edge"; break;
                    default: {
                        size_t q = pos;
                        while (q < N && text[q] != '\n') q++;
                        why = "expected two nonnegative integers, got '" +
                              std::string(reinterpret_cast<const char*>(text.data() + pos), q - pos) + "'";
                    }
                }
                throw Fail{TDG_ERR_IO, p + ":" + std::to_string(lineno) + ": " + why};
            }
            d2h(c->stream, &total, c->pscr.as<uint32_t>() + 2 * nseg + 1, 4, "D2H edge count");
            if (total) {
                c->ppairs.ensure(size_t(total) * 16, "edge pairs");
                ck(launch_parse_write(c->ptext.as<unsigned char>(), nb, c->pscr.p, c->ppairs.as<unsigned long long>(),
                                      c->stream, &c->launches), "parse kernels");
                const size_t at = out.size();
                out.resize(at + 2 * size_t(total));
                d2h(c->stream, out.data() + at, c->ppairs.p, size_t(total) * 16, "D2H edge pairs");
            }
            c0 = c1;
        }
        if (!out.empty()) {
            auto* h = static_cast<uint64_t*>(std::malloc(out.size() * 8));
            if (!h) throw std::bad_alloc();
            std::memcpy(h, out.data(), out.size() * 8);
            *pairs_out = h;
        }
        *npairs = out.size() / 2;
    });
}

void tdg_free(void* p) { std::free(p); }

int tdg_stats(tdg_context* ctx, const tdg_csr* g, tdg_graph_stats* out) {
    return guarded([&] {
        if (!out) throw Fail{TDG_ERR_INVALID, "out is NULL"};
        tdg_context* c = resolve(ctx);
        c->use();
        const Dims d = check_graph(g, true);
        c->launches = 0;
        stage_and_build(c, g, d, true, true, false);
        std::memset(out, 0, sizeof(*out));
        out->n = d.n;
        out->m = d.m;
        if (d.m == 0) return;
        ck(launch_stats(c->off.as<uint32_t>(), c->eo.as<uint32_t>(), c->opos.as<uint32_t>(), d.n,
                        c->sacc.as<StatsAcc>(), c->stream, &c->launches), "stats kernel");
        ck(cudaMemcpyAsync(&c->hctl->stats, c->sacc.p, sizeof(StatsAcc), cudaMemcpyDeviceToHost, c->stream), "D2H stats");
        ck(cudaStreamSynchronize(c->stream), "stats");
        const StatsAcc& a = c->hctl->stats;
        out->d_max = a.d_max;
        out->sum_deg_sq = a.sum_deg_sq;
        out->sum_dplus_sq = a.sum_dplus_sq;
        out->wedge_count = (a.sum_deg_sq - 2ull * d.m) / 2;
        out->deg_sum_dplus_sq = a.deg_sum_dplus_sq;
        out->deg_s1 = a.deg_s1;
    });
}

int tdg_scan(tdg_context* ctx, const uint32_t* s, uint64_t m, uint32_t level, const uint8_t* processed,
             uint8_t* in_curr, uint32_t* curr, uint64_t* curr_size) {
    return guarded([&] {
        if (!curr_size || (m && (!s || !processed || !in_curr || !curr))) throw Fail{TDG_ERR_INVALID, "NULL argument"};
        if (m > 0x7fffffffull) throw Fail{TDG_ERR_RANGE, "m too large"};
        tdg_context* c = resolve(ctx);
        c->use();
        *curr_size = 0;
        if (m == 0) return;
        const uint32_t mm = static_cast<uint32_t>(m);
        c->ensure_peel(0, m);
        c->ctl.ensure(sizeof(PeelCtl), "ctl");
        c->bsum.ensure(sizeof(unsigned long long) * kMaxChunks, "bsum");
        c->f0.ensure(m, "processed");
        c->f1.ensure(m, "in_curr");
        ck(cudaMemcpyAsync(c->s, s, m * 4, cudaMemcpyHostToDevice, c->stream), "H2D s");
        ck(cudaMemcpyAsync(c->f0.p, processed, m, cudaMemcpyHostToDevice, c->stream), "H2D processed");
        ck(cudaMemcpyAsync(c->f1.p, in_curr, m, cudaMemcpyHostToDevice, c->stream), "H2D in_curr");
        ck(cudaMemsetAsync(c->ctl.p, 0, sizeof(PeelCtl), c->stream), "memset");
        DevGraph dg;
        dg.m = mm;
        PeelBufs pb = c->peel_bufs(0);
        ck(launch_step_scan(dg, pb, level, c->f0.as<uint8_t>(), c->f1.as<uint8_t>(), c->sms, c->stream), "scan");
        ck(cudaMemcpyAsync(&c->hctl->peel, pb.ctl, sizeof(PeelCtl), cudaMemcpyDeviceToHost, c->stream), "D2H ctl");
        ck(cudaMemcpyAsync(in_curr, c->f1.p, m, cudaMemcpyDeviceToHost, c->stream), "D2H in_curr");
        ck(cudaStreamSynchronize(c->stream), "scan");
        const uint32_t cs = c->hctl->peel.ph[0].out_size;
        if (cs) d2h(c->stream, curr, pb.L[0], size_t(cs) * 4, "D2H curr");
        *curr_size = cs;
    });
}

int tdg_process_sublevel(tdg_context* ctx, const tdg_csr* g, uint32_t* s, uint32_t level, const uint32_t* curr,
                         uint64_t curr_size, uint8_t* in_curr, uint8_t* in_next, uint8_t* processed,
                         uint32_t* next, uint64_t* next_size) {
    return guarded([&] {
        tdg_context* c = resolve(ctx);
        c->use();
        const Dims d = check_graph(g, true);
        if (!next_size || (d.m && (!s || !in_curr || !in_next || !processed || !next)) || (curr_size && !curr))
            throw Fail{TDG_ERR_INVALID, "NULL argument"};
        if (curr_size > d.m) throw Fail{TDG_ERR_INVALID, "curr_size exceeds m"};
        *next_size = 0;
        c->launches = 0;
        stage_and_build(c, g, d, true, false, true);
        if (d.m == 0) { ck(cudaStreamSynchronize(c->stream), "sync"); return; }
        c->ensure_peel(d.n, d.m);
        c->f0.ensure(d.m, "processed");
        c->f1.ensure(d.m, "in_curr");
        c->f2.ensure(d.m, "in_next");
        const size_t m = d.m;
        ck(cudaMemcpyAsync(c->s, s, m * 4, cudaMemcpyHostToDevice, c->stream), "H2D s");
        ck(cudaMemcpyAsync(c->f0.p, processed, m, cudaMemcpyHostToDevice, c->stream), "H2D processed");
        ck(cudaMemcpyAsync(c->f1.p, in_curr, m, cudaMemcpyHostToDevice, c->stream), "H2D in_curr");
        ck(cudaMemcpyAsync(c->f2.p, in_next, m, cudaMemcpyHostToDevice, c->stream), "H2D in_next");
        if (curr_size) ck(cudaMemcpyAsync(c->L0, curr, curr_size * 4, cudaMemcpyHostToDevice, c->stream), "H2D curr");
        ck(cudaMemsetAsync(c->ctl.p, 0, sizeof(PeelCtl), c->stream), "memset");
        const DevGraph dg = c->dev_graph(d.n, d.m);
        const PeelBufs pb = c->peel_bufs(d.n);
        ck(launch_step_process(dg, pb, level, static_cast<uint32_t>(curr_size), c->f1.as<uint8_t>(),
                               c->f2.as<uint8_t>(), c->f0.as<uint8_t>(), c->sms, c->stream), "process_sublevel");
        ck(cudaMemcpyAsync(s, c->s, m * 4, cudaMemcpyDeviceToHost, c->stream), "D2H s");
        ck(cudaMemcpyAsync(processed, c->f0.p, m, cudaMemcpyDeviceToHost, c->stream), "D2H processed");
        ck(cudaMemcpyAsync(in_curr, c->f1.p, m, cudaMemcpyDeviceToHost, c->stream), "D2H in_curr");
        ck(cudaMemcpyAsync(in_next, c->f2.p, m, cudaMemcpyDeviceToHost, c->stream), "D2H in_next");
        ck(cudaMemcpyAsync(&c->hctl->peel, pb.ctl, sizeof(PeelCtl), cudaMemcpyDeviceToHost, c->stream), "D2H ctl");
        ck(cudaStreamSynchronize(c->stream), "process_sublevel");
        check_peel_ctl(c->hctl->peel);
        const uint32_t ns = c->hctl->peel.ph[1].out_size;
        if (ns) d2h(c->stream, next, pb.L[1], size_t(ns) * 4, "D2H next");
        *next_size = ns;
    });
}

static_assert(int(TDG_CNT_SCAN_IN) == int(kCntScanIn) && int(TDG_CNT_MARKS) == int(kCntMarks) &&
                  int(TDG_CNT_REBUILD_BUCKETS) == int(kCntRebuildBuckets) &&
                  int(TDG_CNT_COMP_LONG) == int(kCntCompLong) && int(TDG_CNT_SUP_TAB_ELEMS) == int(kPeelCnt),
              "tdg.h counter order must follow PeelCnt");

int tdg_counters(tdg_context* ctx, uint64_t* out, uint64_t cap) {
    return guarded([&] {
        if (!out && cap) throw Fail{TDG_ERR_INVALID, "out is NULL"};
        tdg_context* c = resolve(ctx);
        uint64_t v[TDG_NCOUNTERS];
        for (int i = 0; i < kPeelCnt; i++) v[i] = c->hctl->peel.cnt[i];
        v[TDG_CNT_SUP_TAB_ELEMS] = c->hctl->sup.tab_elems;
        v[TDG_CNT_SUP_SEGMENTS] = c->hctl->sup.tab_segments;
        v[TDG_CNT_SUP_SEARCH] = c->hctl->sup.search_items;
        v[TDG_CNT_SUP_HUB] = c->hctl->sup.hub_items;
        for (uint64_t i = 0; i < cap && i < TDG_NCOUNTERS; i++) out[i] = v[i];
    });
}

int tdg_filter_mode(tdg_context* ctx, int* hashed, double* fp_estimate) {
    return guarded([&] {
        tdg_context* c = resolve(ctx);
        c->use();
        if (!c->fctl.p) throw Fail{TDG_ERR_INVALID, "no filtered graph is resident in this context"};
        FilterCtl fc;
        d2h(c->stream, &fc, c->fctl.p, sizeof(fc), "D2H filter control");
        if (hashed) *hashed = fc.hashed ? 1 : 0;
        if (fp_estimate) *fp_estimate = fc.keys ? double(fc.fp) / 262144.0 / double(fc.keys) : 0.0;
    });
}

}  // extern "C"
