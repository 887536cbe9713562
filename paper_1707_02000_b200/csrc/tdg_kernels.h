// tdg_kernels.h — host-side launchers for the sm_100a kernels (internal, C++).
#pragma once

#include <cstddef>
#include <cstdint>
#include <cuda_runtime.h>

#include "tdg_common.cuh"

namespace tdg {

// ---- build (graph.cpp:73-101 equivalent + degree orientation) ----
struct BuildBufs {
    const int64_t* off64;  // device, n+1
    uint32_t* off;         // n+1
    uint32_t* adj;         // 2m
    uint32_t* src;         // 2m scratch (row of each slot)
    uint32_t* eo;          // n
    uint32_t* up;          // n+1 scratch
    uint32_t* P;           // n+1 edge-id base per vertex
    uint32_t* eid;         // 2m
    uint2* el;             // m
    uint32_t* flag;        // 2m+1 scratch
    uint32_t* pos;         // 2m+1 scratch
    uint32_t* opos;        // n+1
    uint32_t* oadj;        // m
    uint32_t* oeid;        // m
    uint32_t* osrc;        // m
    uint32_t* stask;       // m  support tasks: slot index, grouped by searched-list owner
    uint32_t* sx;          // m  owner of that slot
    uint32_t* sbeg;        // n+1 first support task of each owner (tasks are grouped by owner)
    void* cub_tmp;
    size_t cub_bytes;
};
size_t build_cub_bytes(uint32_t n, uint32_t m);
// with_orientation=false stops after eo/eid/el (tdg_build_truss_graph, step functions).
cudaError_t launch_build(const BuildBufs& b, uint32_t n, uint32_t m, bool with_orientation,
                         cudaStream_t st, uint32_t* launches);

// Internal edge ids (truss / support): after launch_build with orientation, rewrite eid[2m]
// and el[m] so edge {x,y} is identified by its oriented slot (position in oadj); r2i: m u32
// scratch. launch_to_ref scatters an internal-id array back: out[oeid[t]] = in[t] + add.
cudaError_t launch_internal_ids(const BuildBufs& b, uint32_t m, uint32_t* r2i, cudaStream_t st, uint32_t* launches);
cudaError_t launch_to_ref(const uint32_t* oeid, const uint32_t* in, uint32_t m, uint32_t add, uint32_t* out,
                          cudaStream_t st, uint32_t* launches);

// Per-vertex neighbour -> edge-id hash tables (tdg_common.cuh): bucket offsets hbo[n+1]
// (hq: n+1 scratch) and at most htab_buckets(n, m) buckets of 32 bytes; the membership filters
// of the big tables: filter_words(n, m) 64-bit words. All sizes follow from n and m.
inline uint64_t htab_buckets(uint64_t n, uint64_t m) { return (uint64_t(kHF) * 2 * m) / 4 + n + 1; }
inline uint64_t filter_words(uint64_t n, uint64_t m) { return (htab_buckets(n, m) >> kFShift) + 1; }
cudaError_t launch_htab_fill(const uint32_t* off, const uint32_t* adj, const uint32_t* src, const uint32_t* eid,
                             uint32_t n, uint32_t m, uint32_t* hq, uint32_t* hbo, uint32_t* htab, void* cub_tmp,
                             size_t cub_bytes, cudaStream_t st, uint32_t* launches);
// fctl: the graph's FilterCtl (word multiplier: rank mode, or hash mode when rank-mode filters
// would pass too much; decided on the device).
cudaError_t launch_filter_fill(const uint32_t* hbo, const uint32_t* adj, const uint32_t* src, uint32_t n, uint32_t m,
                               unsigned long long* filt, FilterCtl* fctl, cudaStream_t st, uint32_t* launches);

struct StatsAcc {
    unsigned long long d_max, sum_deg_sq, sum_dplus_sq, deg_sum_dplus_sq, deg_s1;
};
cudaError_t launch_stats(const uint32_t* off, const uint32_t* eo, const uint32_t* opos, uint32_t n,
                         StatsAcc* acc, cudaStream_t st, uint32_t* launches);

// ---- support (triangle.cpp:26-61 equivalent) ----
struct SupportCtl {
    unsigned long long tri3; // sum of supports
    uint32_t piece_head, pad0, smax, pad;
    unsigned long long probes;        // probe items of the support pass
    unsigned long long tab_elems;     // N+(owner) elements loaded into shared-memory tables
    unsigned long long tab_segments;  // owner segments served from a shared-memory table
    unsigned long long search_items;  // work items (16-byte list quads) binary-searched in global memory instead
    unsigned long long hub_items;     // quads x passes of owners whose N+ exceeds one table (d+ > 3/4 of its slots)
    unsigned long long big_work;      // work items whose owner list exceeds TDG_SUP_TAB / 4 keys (block geometry choice)
    unsigned long long work_items;    // all work items (16-byte list quads) of the pass
    unsigned long long big_geometry;  // 1: the 512-thread / 8192-slot geometry ran
};
constexpr uint32_t kMaxChunks = 1024;  // max blocks of a prep grid (one work chunk each)
// Requires internal edge ids (launch_internal_ids): s[m] is indexed by oriented slot.
// wpre: >= m u64 scratch; bsum: kMaxChunks u64. shard / nshards: only the triangles found in
// shard's stretch of the probe axis are counted (the shards' results sum to the supports).
cudaError_t launch_support(const DevGraph& g, uint32_t* s, unsigned long long* wpre,
                           unsigned long long* bsum, SupportCtl* ctl, int sm_count, cudaStream_t st,
                           uint32_t* launches, uint32_t shard = 0, uint32_t nshards = 1);

// triangle_count (triangle.cpp:90-116): count lands in ctl->tri3 (= T, not 3T).
cudaError_t launch_triangle_count(const DevGraph& g, unsigned long long* wpre, unsigned long long* bsum,
                                  SupportCtl* ctl, int sm_count, cudaStream_t st, uint32_t* launches);

// ---- k-truss components (truss_serial.cpp:176-210) ----
struct KtrussBufs {
    uint32_t* parent;        // n
    uint32_t* first;         // n: min qualifying edge id per root
    uint32_t* root_of_edge;  // m
    uint32_t* flag;          // m+1
    uint32_t* rank;          // m+1 (rank[m] = number of components)
    uint32_t* comp;          // m output
    void* cub_tmp;
    size_t cub_bytes;
};
size_t ktruss_cub_bytes(uint32_t m);
cudaError_t launch_ktruss(const uint2* el, const uint32_t* truss, uint32_t n, uint32_t m, uint32_t k,
                          const KtrussBufs& b, cudaStream_t st, uint32_t* launches);

// ---- vertex ordering (kcore.cpp:68-138, graph.cpp:103-133) ----
struct KcoreBufs {
    uint32_t* deg;            // n+1
    uint32_t* core;           // n+1
    uint32_t *L0, *L1, *A0, *A1;  // n each
    uint32_t* tmp_adj;        // 2m (reorder)
    unsigned long long* wpre;  // n
    unsigned long long* bsum;  // kMaxChunks
    void* ctl;                // device control block (kKcoreCtlBytes)
    void* cub_tmp;
    size_t cub_bytes;
};
constexpr size_t kKcoreCtlBytes = 256;
size_t kcore_cub_bytes(uint32_t n, uint32_t m);
cudaError_t launch_kcore(const uint32_t* off, const uint32_t* adj, uint32_t n, const KcoreBufs& b, int sm_count,
                         cudaStream_t st, uint32_t* launches, uint32_t* c_max_dev);
cudaError_t launch_coreness_order(const uint32_t* core, uint32_t n, const KcoreBufs& b, uint32_t* perm,
                                  cudaStream_t st, uint32_t* launches);
cudaError_t launch_reorder(const uint32_t* off, const uint32_t* adj, const uint32_t* perm, uint32_t n, uint32_t m,
                           const KcoreBufs& b, uint32_t* noff, uint32_t* nadj, uint32_t* bad, cudaStream_t st,
                           uint32_t* launches);

// ---- ingest (graph.cpp:19-71 canonicalize) ----
struct IngestBufs {
    unsigned long long *labels_in, *key_sorted, *glabel, *labels_out, *keys, *keys_sorted, *nuniq;
    uint32_t *pos_in, *pos_sorted, *head, *gidx, *first_pos, *gseq, *first_sorted, *gsorted, *rank_of, *vid;
    uint32_t *deg, *off, *cursor, *nb_tmp, *nb;
    void* cub_tmp;
    size_t cub_bytes;
};
size_t ingest_cub_bytes(uint64_t npairs);
// Synchronises the stream (sizes are read back). *n_out distinct labels, *m_out edges.
cudaError_t launch_ingest(const IngestBufs& B, uint64_t npairs, cudaStream_t st, uint64_t* n_out, uint64_t* m_out,
                          uint32_t* launches);

// ---- text edge-list parsing (graph.cpp:152-200 read_edge_list), edgelist.cu ----
enum ParseError : uint32_t { kParseNegative = 0, kParseExpected = 1, kParseTrailing = 2 };
size_t parse_scratch_bytes(uint64_t nbytes);
// Pass 1 over nbytes of text (< 2^31): per-segment edge counts + their exclusive scan in
// scratch (total edges at u32 index 2 * nseg + 1, nseg = ceil(nbytes / 256)); *err = min over
// failing lines of (line start << 2 | ParseError), or ~0.
cudaError_t launch_parse_count(const unsigned char* text, uint64_t nbytes, void* scratch, size_t scratch_bytes,
                               unsigned long long* err, cudaStream_t st, uint32_t* launches);
// Pass 2: the (u, v) pairs in file order (2 x u64 each).
cudaError_t launch_parse_write(const unsigned char* text, uint64_t nbytes, void* scratch, unsigned long long* pairs,
                               cudaStream_t st, uint32_t* launches);

// ---- peel (truss_parallel.cpp:21-150 equivalent) ----
struct PhaseCtr {
    unsigned long long work; // sub-level: total probe items (informational)
    uint32_t out_size;       // list appends (curr for a scan, next for a sub-level)
    uint32_t alive_size;     // scan: surviving alive edges
    uint32_t min_s;          // scan: min support over survivors (level skipping)
    uint32_t piece_head;     // sub-level: dynamic piece cursor
    uint32_t batch_head;     // sub-level / scan: dynamic batch cursor
    uint32_t far_size;       // scan: far-list appends (peel.cu near/far scan)
};
// Access tallies of one decomposition (bench.py's byte model of the peel). Entries below
// kCntProbe are counted per probe and only by the diagnostic count-mode instantiation of
// k_peel (PeelBufs::count); the rest are phase-level and always counted (leader thread).
enum PeelCnt : int {
    kCntFilter = 0,  // membership-filter words read
    kCntPbits,       // processed-bitmap words read by probes
    kCntWalk,        // table walks (probes that passed filter and processed bit)
    kCntSlots,       // table slots read (first slot + collisions)
    kCntHits,        // triangle visits (element found in the table; 2 state words read)
    kCntDead,        // probes whose own slot was already processed
    kCntDec,         // atomicSub decrements issued
    kCntRepair,      // repairs (+1 after a decrement at or below the level)
    kCntNext,        // next-frontier appends (+ stamp stores)
    kCntCross,       // crosser appends
    kCntProbe,       // ---- below: per-entry compaction tallies (count mode)
    kCntCompIn = kCntProbe,  // compaction: list entries read (adj + eid + processed bit)
    kCntCompKept,    // compaction: entries written back
    kCntCompLong,    // compaction: entries kept in long lists (staged through scratch: +1 copy)
    kCntScanIn,      // ---- below: phase-level, always counted. Scan: entries read (list + state)
    kCntScanOut,     // scan: entries written (curr + near + far lists)
    kCntTasks,       // sub-level tasks prepped (level > 0)
    kCntSorted,      // tasks bucket-sorted by searched vertex
    kCntMarks,       // processed-bitmap marks (one per curr edge)
    kCntRebuildEdges,    // live edges re-inserted by table rebuilds (two inserts each)
    kCntRebuildBuckets,  // table buckets cleared by rebuilds
    kPeelCnt
};
constexpr int kCntFirstPhase = kCntScanIn;

// Level-loop state carried from one k_peel segment to the next (a segment ends where the
// tables are rebuilt on the live graph, peel.cu).
struct PeelResume {
    uint32_t j, level, K, nA, ai, li, live_at_compact, live_at_rebuild, B, fi, nF, xp, cs, bar_target;
    unsigned long long t_exit;  // device clock when the segment ended
};
struct PeelCtl {
    PhaseCtr ph[3];
    uint32_t levels_len;   // last non-empty level + 1
    uint32_t sublevels;
    uint32_t scans;
    uint32_t compactions;
    uint32_t nsl_overflow;    // a level index reached the nsl capacity (n+1)
    uint32_t chunk_overflow;  // the compaction chunk table was too small
    uint32_t final_stamp;
    uint32_t t_max;
    uint32_t nchunks;  // long-list compaction chunks (built by k_peel_init)
    unsigned long long scan_ns;  // device-clock time in scan phases (leader thread)
    unsigned long long proc_ns;  // device-clock time in sub-level phases
    unsigned long long probes;   // probe items over all sub-levels (sum of W)
    unsigned long long compact_ns;  // device-clock time in adjacency compactions
    unsigned long long cnt[kPeelCnt];  // access tallies (PeelCnt); probe-level ones only in count mode
    uint32_t xcnt[2];  // crosser-list append counters (peel.cu near/far scan)
    uint32_t rebuilds;  // scans that re-split the far list
    uint32_t bar;       // grid-barrier arrival counter (TDG_FAST_BARRIER)
    uint32_t table_rebuilds;        // hash-table rebuilds on the live graph
    uint32_t done;                  // the level loop has finished (later segments are no-ops)
    unsigned long long rebuild_ns;  // device-clock time in table rebuilds
    PeelResume rs;
};
struct PeelBufs {
    uint32_t* s;               // support (u32): input of the peel / step-function I/O
    unsigned long long* ss;    // packed per-edge state: (stamp << 32) | support
    uint32_t* L[2];
    uint32_t* A[2];
    unsigned long long* wpre;  // per curr position: exclusive work prefix inside its chunk
    unsigned long long* bsum;  // per chunk (= block of the prep phase): total work
    PeelCtl* ctl;
    uint32_t* nsl;
    uint32_t nsl_cap;
    uint32_t count;       // diagnostic count mode: the k_peel<true> instantiation tallies every access
    uint32_t* bhist;      // kBuckets counters (zero between uses)
    uint32_t* bcur;       // kBuckets cursors
    uint32_t bshift;      // bucket = vertex >> bshift
    unsigned long long* trace;  // diagnostic (TDG_TRACE): 4 words per sub-level, or null
    uint32_t trace_cap;
    // compaction of long lists (degree > kBigList): fixed 512-slot chunks {vertex, index},
    // per-chunk kept counts, and a slot-aligned scratch copy of the kept entries
    uint2* chunks;
    uint32_t* ckept;
    uint32_t chunk_cap;
    uint32_t* sadj;
    uint32_t* seid;
    uint32_t* pbits;  // (m+31)/32 words: bit e set once edge e's sub-level has run
    uint32_t* F[2];   // m each: far live edges (support >= the near bound when split)
    // (far edges whose support crossed below the near bound are appended right after the
    // current near list A[ai], which the next scan reads as one list)
    // writable views of the graph's tables for the in-peel rebuild on the live graph (the
    // DevGraph pointers are the same arrays, read-only for the probes)
    uint32_t* hbo_w;
    uint32_t* htab_w;
    unsigned long long* filt_w;
    uint32_t rebuild_num, rebuild_den;  // rebuild once live <= num/den of the last (re)build (den 0: never)
    uint32_t seg, nseg;                 // this k_peel launch is segment seg of at most nseg
    uint4* desc;      // m: per-sub-level task descriptors (aliases the compaction scratch; a
                      // bucket-sorted curr list follows the descriptors)
};
// In-peel table rebuild (peel.cu): once live edges <= NUM/DEN of those at the last (re)build.
#ifndef TDG_REBUILD_NUM
#define TDG_REBUILD_NUM 1
#endif
#ifndef TDG_REBUILD_DEN
#define TDG_REBUILD_DEN 2  // 0 = never (compiled out)
#endif
#ifndef TDG_REBUILD_MAX
#define TDG_REBUILD_MAX 6  // at most this many rebuilds per decomposition (k_peel segments - 1)
#endif
constexpr uint32_t kPeelRebuildNum = TDG_REBUILD_NUM, kPeelRebuildDen = TDG_REBUILD_DEN, kPeelRebuildMax = TDG_REBUILD_MAX;
#ifndef TDG_BUCKET_BITS
#define TDG_BUCKET_BITS 16
#endif
constexpr uint32_t kBucketBits = TDG_BUCKET_BITS;
constexpr uint32_t kBuckets = 1u << kBucketBits;
// Whole level loop in one persistent cooperative launch.
cudaError_t launch_peel(const DevGraph& g, const PeelBufs& p, int sm_count, cudaStream_t st,
                        uint32_t* launches);
// truss[e] = s[e] + 2 and t_max.
cudaError_t launch_finalize(const unsigned long long* ss, const uint32_t* oeid, uint32_t m, uint32_t* truss, PeelCtl* ctl,
                            cudaStream_t st, uint32_t* launches);

// Step functions (tdg_scan / tdg_process_sublevel) on reference-style flags.
cudaError_t launch_step_scan(const DevGraph& g, const PeelBufs& p, uint32_t level,
                             const uint8_t* processed, uint8_t* in_curr, int sm_count,
                             cudaStream_t st);
cudaError_t launch_step_process(const DevGraph& g, const PeelBufs& p, uint32_t level,
                                uint32_t curr_size, uint8_t* in_curr, uint8_t* in_next,
                                uint8_t* processed, int sm_count, cudaStream_t st);

}  // namespace tdg
