/*
 * tdg.h — C-ABI of the B200 (sm_100a) PKT truss-decomposition path.
 *
 * This is the drop-in boundary: plain pointers and sizes, no C++/torch types. Each entry
 * point replaces a reference function (paths relative to /root/reference/):
 *
 *   tdg_truss            <- trussdec::truss_parallel(const TrussGraph&, int)
 *                           proj/include/trussdec/truss_parallel.hpp:72, impl
 *                           proj/src/truss_parallel.cpp:106-150 (support pass + level-
 *                           synchronous peel; truss[e] = final support + 2).
 *   tdg_support          <- trussdec::support_am4(const TrussGraph&, int)
 *                           proj/include/trussdec/triangle.hpp:16, proj/src/triangle.cpp:26-61
 *   tdg_build_truss_graph<- trussdec::build_truss_graph(const CsrGraph&)
 *                           proj/include/trussdec/graph.hpp:69, proj/src/graph.cpp:73-101
 *   tdg_stats            <- trussdec::stats(const CsrGraph&)  proj/src/graph.cpp:135-150
 *   tdg_triangle_count   <- trussdec::triangle_count(const TrussGraph&, int)  triangle.cpp:90-116
 *   tdg_ktruss_components<- trussdec::ktruss_subgraphs(tg, res, k)  truss_serial.cpp:176-210
 *   tdg_canonicalize     <- trussdec::canonicalize(const RawEdgeList&)  graph.cpp:19-71
 *   tdg_read_edge_list   <- trussdec::read_edge_list(const std::string&) graph.cpp:152-200
 *   tdg_kcore / tdg_coreness_order / tdg_reorder
 *                        <- kcore_parallel / coreness_order (kcore.cpp:68-138), reorder (graph.cpp:103-133)
 *   tdg_scan             <- trussdec::scan(...)              truss_parallel.hpp:62, .cpp:21-37
 *   tdg_process_sublevel <- trussdec::process_sublevel(...)  truss_parallel.hpp:67-68, .cpp:39-104
 *
 * Graph input (tdg_csr): undirected simple graph, adjacency lists sorted ascending,
 * symmetric, no loops/duplicates (the reference's unchecked precondition,
 * graph.hpp:19-20). n vertices, m undirected edges, offsets[n+1] (int64),
 * neighbors[2m] (int32). Like the reference (graph.cpp:48-49) 2m must fit in uint32.
 *
 * Edge ids: the reference's — rank of (u,v), u<v, in ascending lexicographic order of the
 * INPUT numbering (graph.cpp:86-99). Every per-edge output is indexed by it. The GPU
 * orders work internally by degree but always scatters back to these ids.
 *
 * Pointers: the plain entry points take HOST pointers and copy in/out (timed as h2d/d2h);
 * the *_device variants take DEVICE pointers (inputs already resident in HBM).
 *
 * Status: 0 = ok, < 0 = error; tdg_last_error() returns a thread-local message.
 * Threading: a context owns one CUDA stream and its device buffers; calls on one
 * context are serialised by the caller; distinct contexts are independent (reentrant).
 * ctx == NULL selects the calling thread's default context (created lazily on the thread's
 * current device, destroyed at thread exit), so threads passing NULL never share buffers.
 * There is no CPU fallback: without a usable sm_100 device every compute call fails.
 */
#ifndef TDG_H
#define TDG_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TDG_OK 0
#define TDG_ERR_INVALID (-1)   /* bad argument / contract violation (std::invalid_argument) */
#define TDG_ERR_CUDA (-2)      /* CUDA runtime error or no usable device                  */
#define TDG_ERR_NOMEM (-3)     /* device or pinned allocation failed (std::bad_alloc)    */
#define TDG_ERR_RANGE (-4)     /* graph exceeds 32-bit edge width (graph.cpp:48-49)      */
#define TDG_ERR_IO (-5)        /* file cannot be opened / read, or malformed edge-list text
                                  (the reference's std::runtime_error, graph.cpp:153-186)   */

typedef struct tdg_context tdg_context;

typedef struct tdg_csr {
    int64_t n;
    int64_t m;
    const int64_t* offsets;   /* n+1 */
    const int32_t* neighbors; /* 2m, each list sorted ascending */
} tdg_csr;

/* Phase timings (CUDA events on the context stream, milliseconds) and trace counters.
 * support_ms/peel_ms mirror PhaseTimes{support, scan+processing}
 * (truss_parallel.hpp:42-46). */
typedef struct tdg_times {
    double h2d_ms;      /* host -> device copy of the CSR (host-pointer entry points) */
    double build_ms;    /* edge-id map + degree orientation (graph.cpp:73-101 equivalent) */
    double support_ms;  /* support pass (triangle.cpp:26-61 equivalent)                  */
    double peel_ms;     /* level loop: scans + sub-levels (truss_parallel.cpp:119-144)    */
    double scan_ms;     /*   of which scan phases   (device clock, PhaseTimes::scan)       */
    double process_ms;  /*   of which sub-levels    (device clock, PhaseTimes::processing) */
    double d2h_ms;      /* device -> host copy of the per-edge result                     */
    double total_ms;    /* whole call, device-side                                        */
    uint64_t triangles; /* sum(support) / 3                                               */
    uint64_t support_probes; /* support-pass probe items (binary searches)                */
    uint64_t levels;    /* trace length = last non-empty level + 1                       */
    uint64_t sublevels; /* sum(nsl)                                                       */
    uint64_t scans;     /* scan passes actually executed (levels are skipped on device)   */
    uint64_t compactions; /* adjacency compactions executed inside the peel               */
    uint64_t probes;    /* peel probe items (hash lookups) over all sub-levels            */
    uint64_t hits;      /* peel triangle visits (0 unless TDG_COUNT=1 in the env)         */
    uint64_t dead_probes; /* probes of already-processed slots (same diagnostic switch)   */
    uint32_t t_max;     /* max trussness (0 when m == 0)                                  */
    uint32_t kernel_launches; /* kernels this call launched                               */
    double compact_ms;  /*   of process_ms: adjacency compactions (device clock)          */
    double rebuild_ms;  /*   of process_ms: hash-table rebuilds on the live graph         */
    uint64_t table_rebuilds; /* hash-table rebuilds executed inside the peel              */
} tdg_times;

typedef struct tdg_graph_stats {
    uint64_t n, m, d_max;
    uint64_t sum_deg_sq;      /* sum_v d(v)^2                 (graph.cpp:144)           */
    uint64_t sum_dplus_sq;    /* sum_v d+(v)^2, natural order (graph.cpp:145-147)       */
    uint64_t wedge_count;     /* (sum_deg_sq - 2m) / 2        (graph.cpp:148)           */
    uint64_t deg_sum_dplus_sq;/* sum_u d+(u)^2 under the (degree, id) orientation       */
    uint64_t deg_s1;          /* S1 = sum_{u->v} (d+(u) + d+(v)) under that orientation */
} tdg_graph_stats;

const char* tdg_version(void);
const char* tdg_last_error(void);

/* Context: one CUDA stream + grow-only device buffers on `device` (-1 = current device). */
int tdg_context_create(int device, tdg_context** out);
int tdg_context_destroy(tdg_context* ctx);
/* Use an external CUDA stream (cudaStream_t as void*; NULL = the context's own). */
int tdg_context_set_stream(tdg_context* ctx, void* stream);
void* tdg_context_stream(tdg_context* ctx);
/* Release cached device buffers (they are re-grown on the next call). */
int tdg_context_trim(tdg_context* ctx);

/* truss_parallel: truss_out[m] (host), nsl_out[min(nsl_cap, len)] (host) with
 * *nsl_len = trace length; support_out[m] optional (initial supports, may be NULL);
 * times optional. */
int tdg_truss(tdg_context* ctx, const tdg_csr* g, uint32_t* truss_out, uint32_t* support_out,
              uint32_t* nsl_out, uint64_t nsl_cap, uint64_t* nsl_len, tdg_times* times);
/* Same with g->offsets / g->neighbors / truss_out / support_out in DEVICE memory
 * (nsl_out stays a host array). Synchronises the stream before returning. */
int tdg_truss_device(tdg_context* ctx, const tdg_csr* g, uint32_t* truss_out,
                     uint32_t* support_out, uint32_t* nsl_out, uint64_t nsl_cap,
                     uint64_t* nsl_len, tdg_times* times);

/* support_am4: support_out[m] (host / device). */
int tdg_support(tdg_context* ctx, const tdg_csr* g, uint32_t* support_out, tdg_times* times);
int tdg_support_device(tdg_context* ctx, const tdg_csr* g, uint32_t* support_out,
                       tdg_times* times);
/* Sharded support pass (the reference has no distributed code — this is the
 * multi-GPU form of support_am4, proj/src/triangle.cpp:26-61). Every rank holds the whole
 * graph; shard `shard` of `nshards` counts only the triangles found in its equal-work stretch
 * of the probe axis and writes PARTIAL supports (support_out[m], host / device, reference
 * edge ids). The element-wise sum over all shards (one all-reduce of m u32) is exactly
 * support_am4's result; there is no other exchange. */
int tdg_support_shard(tdg_context* ctx, const tdg_csr* g, uint32_t shard, uint32_t nshards,
                      uint32_t* support_out, tdg_times* times);
int tdg_support_shard_device(tdg_context* ctx, const tdg_csr* g, uint32_t shard,
                             uint32_t nshards, uint32_t* support_out, tdg_times* times);

/* build_truss_graph: eo[n], eid[2m], el[2m] (el[2e], el[2e+1] = u < v). Host pointers. */
int tdg_build_truss_graph(tdg_context* ctx, const tdg_csr* g, uint32_t* eo, uint32_t* eid,
                          uint32_t* el);

/* triangle_count (proj/src/triangle.cpp:90-116): number of triangles.
 * Host-pointer graph. */
int tdg_triangle_count(tdg_context* ctx, const tdg_csr* g, uint64_t* count, tdg_times* times);

/* ktruss_subgraphs (proj/src/truss_serial.cpp:176-210): the maximal
 * k-trusses = connected components of the edges with truss >= k. truss[m] and
 * comp_of_edge[m] are host arrays: comp_of_edge[e] = component index (components numbered
 * in the order of their first edge id, as the reference returns them) or 0xFFFFFFFF for
 * truss[e] < k; *ncomp = number of components. k < 2 or k > t_max (when t_max > 0) is
 * TDG_ERR_INVALID (the reference's std::invalid_argument). */
int tdg_ktruss_components(tdg_context* ctx, const tdg_csr* g, const uint32_t* truss, uint32_t k,
                          uint32_t* comp_of_edge, uint64_t* ncomp);

/* Vertex ordering before the path (the CLI's --reorder kcore pipeline,
 * tools/trussdec.cpp:92-97):
 *   tdg_kcore          <- kcore_parallel (proj/src/kcore.cpp:68-127): core_out[n], *c_max.
 *   tdg_coreness_order <- coreness_order (kcore.cpp:129-138): perm_out[v] = new id, vertices
 *                         stably sorted by (coreness, id).
 *   tdg_reorder        <- reorder (proj/src/graph.cpp:103-133): relabel by perm and re-sort
 *                         every list; out_offsets[n+1], out_neighbors[2m]. A perm that is not
 *                         a bijection on 0..n-1 is TDG_ERR_INVALID (std::invalid_argument).
 * All host pointers. */
int tdg_kcore(tdg_context* ctx, const tdg_csr* g, uint32_t* core_out, uint32_t* c_max);
int tdg_coreness_order(tdg_context* ctx, uint64_t n, const uint32_t* core, uint32_t* perm_out);
int tdg_reorder(tdg_context* ctx, const tdg_csr* g, const uint32_t* perm, int64_t* out_offsets,
                int32_t* out_neighbors);

/* Ingest <- canonicalize (proj/src/graph.cpp:19-71): pairs[2*npairs] raw
 * labels (duplicates, both orientations, self loops allowed). Labels get dense ids in
 * first-appearance order (a then b per pair), loops are dropped, pairs deduplicated; the
 * CSR is written to offsets[n+1], neighbors[2m], labels[n] (original label of every id).
 * Capacities: offsets 2*npairs+1, neighbors 2*npairs, labels 2*npairs. Host pointers. */
int tdg_canonicalize(tdg_context* ctx, const uint64_t* pairs, uint64_t npairs, int64_t* offsets,
                     int32_t* neighbors, uint64_t* labels, int64_t* n_out, int64_t* m_out);

/* read_edge_list (graph.cpp:152-200): the text edge list at `path` (plain or gzip, read and
 * inflated with zlib on the host, parsed on the GPU) as raw label pairs in file order:
 * *pairs_out = malloc'd host array of 2 * *npairs uint64 (u0, v0, u1, v1, ...; release with
 * tdg_free). Errors are TDG_ERR_IO with the reference's message ("cannot open input file:
 * <path>" or "<path>:<line>: <why>" for the first malformed line). */
int tdg_read_edge_list(tdg_context* ctx, const char* path, uint64_t** pairs_out, uint64_t* npairs);
void tdg_free(void* p);

/* stats (host-pointer graph). */
int tdg_stats(tdg_context* ctx, const tdg_csr* g, tdg_graph_stats* out);

/* Step functions on caller-held frontier state (host arrays of length m, flags 0/1),
 * for unit tests on hand-built states (tests/test_truss_parallel.cpp:25-105). They run
 * the same device code as tdg_truss. scan: curr[*curr_size] = unprocessed edges with
 * s == level, in_curr set. process_sublevel: drains curr (ownership rule, clamped
 * decrements with repair), appends to next[*next_size] (in_next set), then marks curr
 * processed and clears in_curr. The order inside curr/next is unspecified (as in the
 * reference); compare as sets. */
int tdg_scan(tdg_context* ctx, const uint32_t* s, uint64_t m, uint32_t level,
             const uint8_t* processed, uint8_t* in_curr, uint32_t* curr, uint64_t* curr_size);
int tdg_process_sublevel(tdg_context* ctx, const tdg_csr* g, uint32_t* s, uint32_t level,
                         const uint32_t* curr, uint64_t curr_size, uint8_t* in_curr,
                         uint8_t* in_next, uint8_t* processed, uint32_t* next,
                         uint64_t* next_size);

/* Access tallies of the context's last tdg_truss* / tdg_support* call, for byte models of
 * the kernels (bench.py roofline). out[i] for i < min(cap, TDG_NCOUNTERS), in this order.
 * The per-probe peel tallies (TDG_CNT_FILTER .. TDG_CNT_COMP_LONG) are counted only when
 * the environment holds TDG_COUNT=1 at the call (a slower diagnostic instantiation of the
 * peel kernel; the timed path never counts); the others are always counted. */
enum {
    TDG_CNT_FILTER = 0,     /* peel: membership-filter words read                          */
    TDG_CNT_PBITS,          /* peel: processed-bitmap words read by probes                 */
    TDG_CNT_WALK,           /* peel: hash-table walks (probes past filter + processed bit) */
    TDG_CNT_SLOTS,          /* peel: hash-table slots read (first + collisions)            */
    TDG_CNT_HITS,           /* peel: triangle visits (two edge-state words read)           */
    TDG_CNT_DEAD,           /* peel: probes whose own slot was already processed           */
    TDG_CNT_DEC,            /* peel: atomic decrements (truss_parallel.cpp:54)             */
    TDG_CNT_REPAIR,         /* peel: repairs (truss_parallel.cpp:58-62)                    */
    TDG_CNT_NEXT,           /* peel: next-frontier appends (truss_parallel.cpp:55-57)      */
    TDG_CNT_CROSS,          /* peel: near/far crosser appends                              */
    TDG_CNT_COMP_IN,        /* peel: adjacency-compaction entries read                     */
    TDG_CNT_COMP_KEPT,      /* peel: compaction entries written back (short lists)         */
    TDG_CNT_COMP_LONG,      /* peel: compaction entries kept in long lists (two copies)    */
    TDG_CNT_SCAN_IN,        /* peel: scan entries read (live-list entry + edge state)      */
    TDG_CNT_SCAN_OUT,       /* peel: scan entries written (curr / near / far lists)        */
    TDG_CNT_TASKS,          /* peel: sub-level tasks (curr edges at levels > 0)            */
    TDG_CNT_SORTED,         /* peel: tasks bucket-sorted by searched vertex                */
    TDG_CNT_MARKS,          /* peel: processed-bitmap marks                                */
    TDG_CNT_REBUILD_EDGES,  /* peel: live edges re-inserted by table rebuilds (2 inserts each) */
    TDG_CNT_REBUILD_BUCKETS,/* peel: table buckets cleared by rebuilds                     */
    TDG_CNT_SUP_TAB_ELEMS,  /* support: N+(owner) elements loaded into shared-memory tables */
    TDG_CNT_SUP_SEGMENTS,   /* support: owner segments served from a shared-memory table   */
    TDG_CNT_SUP_SEARCH,     /* support: 16-byte list quads binary-searched in global memory */
    TDG_CNT_SUP_HUB,        /* support: quads x passes of owners whose N+ exceeds one table */
    TDG_NCOUNTERS
};
int tdg_counters(tdg_context* ctx, uint64_t* out, uint64_t cap);
/* Diagnostic (no reference counterpart): how the membership filters of the graph resident
 * in ctx (the last truss / step call) choose a key's word — *hashed = 0: by the key's rank in
 * the id space (sorted probe lists share filter sectors), 1: by a multiplicative hash (chosen
 * on the device when rank-mode filters would pass too many probes: clustered vertex ids);
 * *fp_estimate = the probe-weighted false-positive estimate of the rank-mode fill. Results
 * never depend on the mode. Synchronises the stream. */
int tdg_filter_mode(tdg_context* ctx, int* hashed, double* fp_estimate);

#ifdef __cplusplus
}
#endif

#endif /* TDG_H */
