// peel.cu — the level-synchronous PKT peel as ONE persistent cooperative kernel.
//
// Reference (paths relative to /root/reference/proj):
//   scan              src/truss_parallel.cpp:21-37
//   process_sublevel  src/truss_parallel.cpp:39-104 (try_decrement :49-63)
//   truss_parallel    src/truss_parallel.cpp:106-150 (level / sub-level driver)
//   BufferedAppender  include/trussdec/appender.hpp:12-40
//
// Semantics kept exactly: level = support value; curr(l) =
// {unprocessed e : s[e]==l}; each e1=(u,v) in curr visits every w in N(u)∩N(v),
// skips triangles with a processed peer, and for each peer target decrements only if
// s[target] > l and (other peer not in curr or e1 < other); the thread whose atomicSub
// returns l+1 appends target to next; a return <= l is repaired with +1; trussness =
// final support + 2. Sub-level sets (hence nsl) and results are therefore identical to
// the reference for any schedule.
//
// B200 design:
//  * Device-resident loop: every level and sub-level runs inside one cooperative launch;
//    a sub-level is two grid-barrier phases (prep, process); a level adds one scan phase.
//  * Flags -> stamps: stamp[e] = index of the sub-level in which e is (or was) curr, packed
//    with s[e] in one 64-bit word so a probe reads both with one random access.
//    processed(e) <=> 0 < stamp < K, in_curr(e) <=> stamp == K, next <=> stamp == K+1.
//    Entering next is the single stamp store by the appending thread, so the
//    reference's epilogue pass over curr (:97-102) and the flag swaps vanish.
//  * No dense X[n] mark array (MarkScratchPool, truss_parallel.hpp:55-59): N(u)∩N(v) is
//    computed by walking the shorter live list and looking each element up in the other
//    endpoint's neighbour -> edge-id hash table (built once per graph, build.cu).
//  * Item-balanced sub-levels: prep computes each curr edge's probe count and a chunked
//    prefix sum; process splits the sub-level's total probe count W into ~4 pieces per
//    warp, pulled dynamically, so a sub-level's critical path is ~W/(#warps) probes no
//    matter how skewed its edges are (hub-hub edges spread over many warps, tiny late
//    sub-levels use as many warps as they have probes).
//  * Level 0 needs no intersections: s[e1] >= #live triangles of e1, so s==0 edges have
//    none (the reference still marks/scans their lists).
//  * Levels with no edges are skipped: the scan that finds curr empty also returns the
//    minimum live support, which is the next non-empty level. Each scan compacts the
//    live-edge list, so later levels stream only survivors.

#include <cooperative_groups.h>

#include "intersect.cuh"
#include "tdg_kernels.h"

namespace cg = cooperative_groups;

namespace tdg {

namespace {

#ifndef TDG_PEEL_THREADS
#define TDG_PEEL_THREADS 256
#endif
constexpr int kPeelThreads = TDG_PEEL_THREADS;
#ifndef TDG_PEEL_MINB
#define TDG_PEEL_MINB 4  // min resident blocks/SM: 64 registers, 32 warps per SM
#endif
#ifndef TDG_PEEL_U
#define TDG_PEEL_U 3  // probe items per lane per window step (independent chains in flight)
#endif
constexpr int kScanItems = 8;
constexpr int kWarps = kPeelThreads / 32;

// Task of e1 = (u,v): probe the shorter live list a against the other endpoint b's
// neighbour -> edge-id hash table (ob = hbo[b], lb = its bucket count, tdg_common.cuh).
#ifndef TDG_HTAB_NC
#define TDG_HTAB_NC 0  // table slots through the read-only (non-coherent) path: tables never change in the peel
#endif
#ifndef TDG_FILT_NC
#define TDG_FILT_NC 0  // filter words through the read-only path
#endif
// Cold phases (rebuild, compaction, bucket sort) can be kept out of line so that they do not
// take part in the register allocation of the probe loop.
#ifndef TDG_NOINLINE_RB
#define TDG_NOINLINE_RB 0
#endif
#ifndef TDG_NOINLINE_COLD
#define TDG_NOINLINE_COLD 0
#endif
#if TDG_NOINLINE_RB
#define TDG_COLD_RB __device__ __noinline__
#else
#define TDG_COLD_RB __device__
#endif
#if TDG_NOINLINE_COLD
#define TDG_COLD __device__ __noinline__
#else
#define TDG_COLD __device__
#endif
// The process phase out of line: the probe loop gets a register allocation of its own; the
// level loop's state is saved around the call (once per sub-level) instead of being spilled
// and refilled inside the loop.
#ifndef TDG_NOINLINE_HOT
#define TDG_NOINLINE_HOT 0
#endif
#if TDG_NOINLINE_HOT
#define TDG_HOT __device__ __noinline__
#else
#define TDG_HOT __device__
#endif
#ifndef TDG_PEEL_FAST
#define TDG_PEEL_FAST 0  // engine fast path (intersect.cuh) for the peel's probe loop
#endif
#ifndef TDG_DIAG_RATIO
#define TDG_DIAG_RATIO 0  // diagnostic build: probe-weighted task-shape histograms, printed by the kernel
#endif
#if TDG_DIAG_RATIO
__device__ unsigned long long d_diag[16];
#endif
// la = the probe count (live length of the shorter list).
__device__ __forceinline__ ITask ptask(const DevGraph& g, uint32_t e1, uint32_t& la) {
    const uint2 p = g.el[e1];
    const uint32_t du = g.dl[p.x], dv = g.dl[p.y];
    const bool pu = du <= dv;
    const uint32_t a = pu ? p.x : p.y, b = pu ? p.y : p.x;
    ITask k;
    k.id = e1;
    k.oa = g.off[a];
    la = pu ? du : dv;
#if TDG_DIAG_RATIO
    {   // probe-weighted histograms of (searched live length / probe length) and of the searched length
        const uint32_t lbv = pu ? dv : du, r = la ? lbv / la : 0;
        const int rc = r < 2 ? 0 : r < 4 ? 1 : r < 8 ? 2 : r < 16 ? 3 : r < 64 ? 4 : 5;
        const int sc = lbv < 512 ? 0 : lbv < 2048 ? 1 : lbv < 8192 ? 2 : lbv < 32768 ? 3 : lbv < 131072 ? 4 : lbv < 524288 ? 5 : 6;
        atomicAdd(&d_diag[rc], static_cast<unsigned long long>(la));
        atomicAdd(&d_diag[6 + sc], static_cast<unsigned long long>(la));
        if (r < 8) atomicAdd(&d_diag[13 + (sc < 3 ? 0 : sc < 5 ? 1 : 2)], static_cast<unsigned long long>(la));
    }
#endif
    k.ob = g.hbo[b];
    k.lb = g.hbo[b + 1] - k.ob;
    return k;
}

__device__ __forceinline__ void reset_ctr(PhaseCtr* c) {
    c->work = 0;
    c->out_size = 0;
    c->alive_size = 0;
    c->min_s = 0xffffffffu;
    c->piece_head = 0;
    c->batch_head = 0;
    c->far_size = 0;
}

// Per-edge state packed in one 64-bit word: low half = support s[e], high half = the
// sub-level stamp. A probe reads both with ONE random access; atomics act on the low half.
__device__ __forceinline__ uint32_t* s_ptr(unsigned long long* ss, uint32_t e) {
    return reinterpret_cast<uint32_t*>(ss + e);
}
__device__ __forceinline__ uint32_t* stamp_ptr(unsigned long long* ss, uint32_t e) {
    return reinterpret_cast<uint32_t*>(ss + e) + 1;
}
__device__ __forceinline__ unsigned long long ld_state(const unsigned long long* ss, uint32_t e) {
    unsigned long long v;
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(ss + e));
    return v;
}
__device__ __forceinline__ uint32_t st_s(unsigned long long w) { return static_cast<uint32_t>(w); }
__device__ __forceinline__ uint32_t st_stamp(unsigned long long w) { return static_cast<uint32_t>(w >> 32); }

// Append every lane's valid targets (o[j] != kNone) to next with one atomic per warp.
template <int N>
__device__ __forceinline__ void emit_many(const uint32_t (&o)[N], uint32_t* ctr, uint32_t* next) {
    uint32_t c = 0;
#pragma unroll
    for (int j = 0; j < N; j++) c += o[j] != kNone ? 1u : 0u;
    if (!__any_sync(kFull, c != 0)) return;
    const uint32_t lane = lane_id();
    uint32_t incl = c;
#pragma unroll
    for (uint32_t d = 1; d < 32; d <<= 1) {
        const uint32_t t = __shfl_up_sync(kFull, incl, d);
        if (lane >= d) incl += t;
    }
    uint32_t base = 0;
    if (lane == 31) base = atomicAdd(ctr, incl);
    base = __shfl_sync(kFull, base, 31) + incl - c;
    TDG_CHECK(base + c >= base);
#pragma unroll
    for (int j = 0; j < N; j++)
        if (o[j] != kNone) next[base++] = o[j];
}

// Two-stage probes (TDG_PEEL_QUEUE): stage A (list element + edge id, processed bit, filter
// word — one level of independent random loads) pushes the ~1/3 of probes that survive into
// a per-warp shared-memory queue; stage B drains it in full batches of kQBatch candidates
// (table bucket -> value -> both peers' states -> atomics), so the long dependent chain runs
// with every lane busy instead of once per step for the few lanes whose probe survived.
#ifndef TDG_PEEL_QUEUE
#define TDG_PEEL_QUEUE 1
#endif
constexpr int kQB = TDG_PEEL_U > 3 ? TDG_PEEL_U : 3;  // candidates per lane per drain
constexpr uint32_t kQBatch = 32u * kQB;      // drain size
constexpr uint32_t kQCap = 2u * kQBatch;     // < kQBatch left + <= 32 * TDG_PEEL_U new (<= kQBatch)
static_assert(32 * TDG_PEEL_U <= int(kQBatch), "one engine step must fit behind a partial batch");

// process_sublevel's inner loop (truss_parallel.cpp:80-88) as a probe-engine policy: a hit
// is w in N(u) ∩ N(v): slot ja of the probe list (its eid is one peer) found in the other
// endpoint's hash table (whose value is the other peer's id). kCount = the diagnostic
// instantiation that also tallies every access class of the probe (PeelCnt, for the byte
// model of bench.py); the timed path is the kCount = false instantiation.
template <bool kCount, uint32_t kShift = kFShift>
struct PeelPolicy {
    const DevGraph& g;
    unsigned long long* ss;
    uint32_t level, K;
    const uint32_t* curr;
    PhaseCtr* ph;
    uint32_t* next;
    const uint32_t* elems;
    unsigned long long* cnt;      // PeelCnt counters (kCount only)
    uint32_t B;                   // near bound (phase_scan): decrements from B append to X
    uint32_t* X;
    uint32_t* xcnt;
    const uint32_t* pbits;        // edges processed in earlier sub-levels (or null)
    const uint4* desc;            // task descriptors written by phase_prep
    uint32_t* qbuf;               // this warp's candidate queue (TDG_PEEL_QUEUE): 5 x kQCap u32, SoA
    uint32_t nq = 0;              // queued candidates (warp-uniform)
    static constexpr bool kFast = TDG_PEEL_FAST;
    static constexpr int kUnroll = TDG_PEEL_U;
    static_assert(kUnroll > 1, "the peel's probe loop is the U-chain form (run)");

    __device__ ITask load(uint32_t t) const {
        const uint4 d = desc[t];
        return ITask{d.x, d.y, d.z, d.w};
    }
    // Triangle visits {e1 = ids[q], ea[q], eb[q]} (eb[q] == kNone: no visit), all lanes together:
    // both peers' state words -> skip on a processed peer (:85) -> ownership + clamp
    // (try_decrement, truss_parallel.cpp:49-63) with all atomics issued before any result is
    // used -> one warp append for all next / crosser targets.
    template <int U>
    __device__ __forceinline__ void apply(const uint32_t (&ea)[U], const uint32_t (&eb)[U], const uint32_t (&ids)[U],
                                          uint32_t (&cn)[kCntProbe]) const {
        unsigned long long wa[U], wb[U];
#pragma unroll
        for (int q = 0; q < U; q++) {
            wa[q] = 0;
            wb[q] = 0;
            if (eb[q] != kNone) {
                wa[q] = ld_state(ss, ea[q]);
                wb[q] = ld_state(ss, eb[q]);
                if constexpr (kCount) cn[kCntHits]++;
            }
        }
        // try_dec (truss_parallel.cpp:49-63) split so all atomics issue before any result is used
        uint32_t tg[2 * U], pv[2 * U];
#pragma unroll
        for (int q = 0; q < U; q++) {
            tg[2 * q] = kNone;
            tg[2 * q + 1] = kNone;
            if (eb[q] != kNone) {
                const uint32_t sa = st_stamp(wa[q]), sb = st_stamp(wb[q]);
                if (!((sa != 0 && sa < K) || (sb != 0 && sb < K))) {  // :85 processed peer
                    const uint32_t id = ids[q];
                    if (st_s(wa[q]) > level && !(sb == K && id >= eb[q])) tg[2 * q] = ea[q];      // :86, :52-53
                    if (st_s(wb[q]) > level && !(sa == K && id >= ea[q])) tg[2 * q + 1] = eb[q];  // :87
                }
            }
        }
#pragma unroll
        for (int j = 0; j < 2 * U; j++)
            if (tg[j] != kNone) pv[j] = atomicSub(s_ptr(ss, tg[j]), 1u);  // :54
        uint32_t o[2 * U], c[2 * U];
#pragma unroll
        for (int j = 0; j < 2 * U; j++) {
            o[j] = kNone;
            c[j] = kNone;
            if (tg[j] != kNone) {
                if constexpr (kCount) cn[kCntDec]++;
                if (pv[j] == level + 1) {  // :55-57
                    st_relaxed(stamp_ptr(ss, tg[j]), K + 1);
                    o[j] = tg[j];
                    if constexpr (kCount) cn[kCntNext]++;
                } else if (pv[j] <= level) {
                    atomicAdd(s_ptr(ss, tg[j]), 1u);  // :58-62 repair
                    if constexpr (kCount) cn[kCntRepair]++;
                } else if (pv[j] == B) {
                    c[j] = tg[j];  // crossed below the near bound
                    if constexpr (kCount) cn[kCntCross]++;
                }
            }
        }
        emit_many(o, &ph->out_size, next);
        emit_many(c, xcnt, X);
    }
    // U hash-form probes per lane, stage by stage so the U chains' loads overlap:
    // list element + its edge id (coalesced) -> first table slot -> (collisions) ->
    // both peers' state words -> both decrements -> one warp append for all targets.
    template <int U>
    __device__ void run(const bool (&act)[U], const ITask (&ko)[U], const uint32_t (&ja)[U]) {
        if constexpr (TDG_PEEL_QUEUE) run_queued<U>(act, ko, ja);
        else run_fused<U>(act, ko, ja);
    }
    // Table lookup of key x in the table [ob, ob + lb) (hash h = hmix(x)): the partner edge id
    // or kNone. One 16-byte key vector per bucket; the value (same sector) only on a hit.
    __device__ __forceinline__ uint32_t table_find(uint32_t x, uint32_t h, uint32_t ob, uint32_t lb,
                                                   uint32_t (&cn)[kCntProbe]) const {
        uint32_t bi = hbucket(h, lb);
        TDG_CHECK(lb > 0 && uint64_t(ob) + lb <= g.nbuckets);
        uint4 kv = TDG_HTAB_NC ? __ldg(reinterpret_cast<const uint4*>(g.htab + 8ull * (ob + bi)))
                               : *reinterpret_cast<const uint4*>(g.htab + 8ull * (ob + bi));
        if constexpr (kCount) { cn[kCntWalk]++; cn[kCntSlots]++; }
        uint32_t sl = bucket_find(kv, x);
        while (sl == 4u && kv.w != kHEmpty) {  // home bucket full: the key may sit further on
            bi = hnext(bi, lb);
            kv = TDG_HTAB_NC ? __ldg(reinterpret_cast<const uint4*>(g.htab + 8ull * (ob + bi)))
                             : *reinterpret_cast<const uint4*>(g.htab + 8ull * (ob + bi));
            sl = bucket_find(kv, x);
            if constexpr (kCount) cn[kCntSlots]++;
        }
        const uint32_t eb = sl < 4u ? (g.htab[8ull * (ob + bi) + 4u + sl] & ~kHUp) : kNone;
        TDG_CHECK(eb == kNone || eb < g.m);
        return eb;
    }
    __device__ __forceinline__ void flush_counts(uint32_t (&cn)[kCntProbe]) const {
        if constexpr (kCount) {
#pragma unroll
            for (int k = 0; k < kCntProbe; k++) {
                const uint32_t t = __reduce_add_sync(kFull, cn[k]);
                if (lane_id() == 0 && t) atomicAdd(cnt + k, static_cast<unsigned long long>(t));
            }
        }
    }
    // Stage B: the first k (<= kQBatch) queued candidates -> table -> visit; the rest moves up.
    __device__ void drain(uint32_t k) {
        uint32_t* qx = qbuf;
        uint32_t* qea = qbuf + kQCap;
        uint32_t* qid = qbuf + 2 * kQCap;
        uint32_t* qob = qbuf + 3 * kQCap;
        uint32_t* qlb = qbuf + 4 * kQCap;
        const uint32_t lane = lane_id();
        uint32_t cn[kCntProbe] = {};
        __syncwarp();
        uint32_t x[kQB], ea[kQB], eb[kQB], ids[kQB], ob[kQB], lb[kQB];
#pragma unroll
        for (int r = 0; r < kQB; r++) {
            const uint32_t i = lane + 32u * r;
            eb[r] = kNone;
            ea[r] = kNone;
            ids[r] = kNone;
            if (i < k) {
                x[r] = qx[i];
                ea[r] = qea[i];
                ids[r] = qid[i];
                ob[r] = qob[i];
                lb[r] = qlb[i];
            }
        }
#pragma unroll
        for (int r = 0; r < kQB; r++)
            if (lane + 32u * r < k) eb[r] = table_find(x[r], hmix(x[r]), ob[r], lb[r], cn);
        apply<kQB>(ea, eb, ids, cn);
        flush_counts(cn);
        // move the leftover [k, nq) (< kQBatch entries, disjoint from [0, k)) to the front
        const uint32_t left = nq - k;
        __syncwarp();
        for (uint32_t i = lane; i < left; i += 32) {
            qx[i] = qx[k + i];
            qea[i] = qea[k + i];
            qid[i] = qid[k + i];
            qob[i] = qob[k + i];
            qlb[i] = qlb[k + i];
        }
        __syncwarp();
        nq = left;
    }
    __device__ void flush() {
        if constexpr (TDG_PEEL_QUEUE)
            if (nq) drain(nq);
    }
    // Stage A of U probes per lane: survivors of the processed bit and the filter are queued.
    template <int U>
    __device__ void run_queued(const bool (&act)[U], const ITask (&ko)[U], const uint32_t (&ja)[U]) {
        uint32_t x[U], ea[U], h[U];
        uint32_t cn[kCntProbe] = {};
#pragma unroll
        for (int q = 0; q < U; q++) {
            x[q] = kHEmpty;
            ea[q] = kNone;
            if (act[q]) {
                TDG_CHECK(uint64_t(ko[q].oa) + ja[q] < 2ull * g.m);
                x[q] = elems[ko[q].oa + ja[q]];
                ea[q] = g.eid[ko[q].oa + ja[q]];
                TDG_CHECK(ea[q] < g.m && x[q] < g.n);
            }
        }
        bool look[U];
        uint32_t pw[U];
        unsigned long long fw[U];
        const uint32_t fscale = g.filt ? __ldg(&g.fctl->fscale) : 0u;  // (uniform; FilterCtl, tdg_common.cuh)
#pragma unroll
        for (int q = 0; q < U; q++) {
            look[q] = act[q];
            h[q] = look[q] ? hmix(x[q]) : 0u;
            pw[q] = (pbits && look[q]) ? pbits[ea[q] >> 5] : 0u;
            if constexpr (kCount) cn[kCntPbits] += (pbits && look[q]) ? 1u : 0u;
            fw[q] = ~0ull;
            if (g.filt && look[q] && ko[q].lb >= kFMin) {
                fw[q] = TDG_FILT_NC ? __ldg(g.filt + fword_index(ko[q].ob, ko[q].lb, x[q], kShift, fscale)) : g.filt[fword_index(ko[q].ob, ko[q].lb, x[q], kShift, fscale)];
                if constexpr (kCount) cn[kCntFilter]++;
            }
        }
        uint32_t* qx = qbuf;
        uint32_t* qea = qbuf + kQCap;
        uint32_t* qid = qbuf + 2 * kQCap;
        uint32_t* qob = qbuf + 3 * kQCap;
        uint32_t* qlb = qbuf + 4 * kQCap;
#pragma unroll
        for (int q = 0; q < U; q++) {
            const unsigned long long fb = fbits(h[q]);
            if ((fw[q] & fb) != fb) look[q] = false;
            if ((pw[q] >> (ea[q] & 31u)) & 1u) look[q] = false;
            const uint32_t bal = __ballot_sync(kFull, look[q]);
            if (look[q]) {
                const uint32_t pos = nq + __popc(bal & lanemask_lt());
                qx[pos] = x[q];
                qea[pos] = ea[q];
                qid[pos] = ko[q].id;
                qob[pos] = ko[q].ob;
                qlb[pos] = ko[q].lb;
            }
            nq += __popc(bal);
        }
        if constexpr (kCount) {
#pragma unroll
            for (int q = 0; q < U; q++) {
                if (act[q]) {
                    const uint32_t sa = st_stamp(ld_state(ss, ea[q]));
                    cn[kCntDead] += (sa != 0 && sa < K) ? 1u : 0u;
                }
            }
        }
        flush_counts(cn);
        if (nq >= kQBatch) drain(kQBatch);
    }
    // Fused form (TDG_PEEL_QUEUE = 0): each lane's U probes run the whole chain in one step.
    template <int U>
    __device__ void run_fused(const bool (&act)[U], const ITask (&ko)[U], const uint32_t (&ja)[U]) const {
        uint32_t x[U], ea[U], eb[U], h[U];
        uint32_t cn[kCntProbe] = {};  // per-lane access tallies (kCount only; folded away otherwise)
#pragma unroll
        for (int q = 0; q < U; q++) {
            x[q] = kHEmpty;
            ea[q] = kNone;
            if (act[q]) {
                TDG_CHECK(uint64_t(ko[q].oa) + ja[q] < 2ull * g.m);
                x[q] = elems[ko[q].oa + ja[q]];
                ea[q] = g.eid[ko[q].oa + ja[q]];
                TDG_CHECK(ea[q] < g.m && x[q] < g.n);
            }
        }
        // membership filter of a big table: a certain miss skips the table (tdg_common.cuh)
        bool look[U];
#pragma unroll
        for (int q = 0; q < U; q++) {
            look[q] = act[q];  // (b itself is in N(a) but never in its own table: a plain miss)
            h[q] = look[q] ? hmix(x[q]) : 0u;
        }
        // ... and so does an own slot already processed in an earlier sub-level (:85): its
        // bit (L2-resident bitmap, consecutive lanes share words) is read beside the filter
        uint32_t pw[U];
#pragma unroll
        for (int q = 0; q < U; q++) {
            pw[q] = (pbits && look[q]) ? pbits[ea[q] >> 5] : 0u;
            if constexpr (kCount) cn[kCntPbits] += (pbits && look[q]) ? 1u : 0u;
        }
        if (g.filt) {
            unsigned long long fw[U];
            const uint32_t fscale = __ldg(&g.fctl->fscale);
#pragma unroll
            for (int q = 0; q < U; q++) {
                fw[q] = ~0ull;
                if (look[q] && ko[q].lb >= kFMin) {
                    fw[q] = TDG_FILT_NC ? __ldg(g.filt + fword_index(ko[q].ob, ko[q].lb, x[q], kShift, fscale)) : g.filt[fword_index(ko[q].ob, ko[q].lb, x[q], kShift, fscale)];
                    if constexpr (kCount) cn[kCntFilter]++;
                }
            }
#pragma unroll
            for (int q = 0; q < U; q++) {
                const unsigned long long fb = fbits(h[q]);
                if ((fw[q] & fb) != fb) look[q] = false;
            }
        }
#pragma unroll
        for (int q = 0; q < U; q++)
            if ((pw[q] >> (ea[q] & 31u)) & 1u) look[q] = false;
        // b's table: buckets [ob, ob + lb) of 8 words (4 keys, then their 4 values); one
        // 16-byte key-vector load per bucket, the value (same sector) only on a hit
        uint4 kv[U];
        uint32_t bi[U];
#pragma unroll
        for (int q = 0; q < U; q++) {
            kv[q] = make_uint4(kHEmpty, kHEmpty, kHEmpty, kHEmpty);
            bi[q] = 0;
            if (look[q]) {
                bi[q] = hbucket(h[q], ko[q].lb);
                TDG_CHECK(ko[q].lb > 0 && uint64_t(ko[q].ob) + ko[q].lb <= g.nbuckets);
                const uint4* kp = reinterpret_cast<const uint4*>(g.htab + 8ull * (ko[q].ob + bi[q]));
                kv[q] = TDG_HTAB_NC ? __ldg(kp) : *kp;
                if constexpr (kCount) { cn[kCntWalk]++; cn[kCntSlots]++; }
            }
        }
        uint32_t sl[U];
#pragma unroll
        for (int q = 0; q < U; q++) {
            sl[q] = bucket_find(kv[q], x[q]);
            while (sl[q] == 4u && kv[q].w != kHEmpty) {  // home bucket full: the key may sit further on
                bi[q] = hnext(bi[q], ko[q].lb);
                const uint4* kp = reinterpret_cast<const uint4*>(g.htab + 8ull * (ko[q].ob + bi[q]));
                kv[q] = TDG_HTAB_NC ? __ldg(kp) : *kp;
                sl[q] = bucket_find(kv[q], x[q]);
                if constexpr (kCount) cn[kCntSlots]++;
            }
        }
#pragma unroll
        for (int q = 0; q < U; q++) {
            eb[q] = (look[q] && sl[q] < 4u) ? (g.htab[8ull * (ko[q].ob + bi[q]) + 4u + sl[q]] & ~kHUp) : kNone;
            TDG_CHECK(eb[q] == kNone || eb[q] < g.m);
        }
        uint32_t ids[U];
#pragma unroll
        for (int q = 0; q < U; q++) ids[q] = ko[q].id;
        apply<U>(ea, eb, ids, cn);
        if constexpr (kCount) {
#pragma unroll
            for (int q = 0; q < U; q++) {
                if (act[q]) {
                    const uint32_t sa = st_stamp(ld_state(ss, ea[q]));
                    cn[kCntDead] += (sa != 0 && sa < K) ? 1u : 0u;
                }
            }
#pragma unroll
            for (int k = 0; k < kCntProbe; k++) {
                const uint32_t t = __reduce_add_sync(kFull, cn[k]);
                if (lane_id() == 0 && t) atomicAdd(cnt + k, static_cast<unsigned long long>(t));
            }
        }
    }
};

// scan (truss_parallel.cpp:21-37), near/far form. The live edges are split at a bound B:
// the NEAR list holds those with support < B, the FAR list the rest (at split time).
// Supports only fall, so a scan at level < B needs only the near list plus the far edges
// whose support has since crossed below B (the process phase appends them, once, to a
// crosser list when its atomicSub returns exactly B). When the level reaches B the far
// list is re-split with a new bound. Each scan reads three input segments — near A, crossers
// X, and (on a re-split) far F — and writes: s == level -> curr (stamp K); s < B -> near
// out; else -> far out. Far entries whose support is already below the old bound are
// dropped (they crossed and sit in A/X). Block-aggregated appends: 3 atomics per 2048 edges.
struct ScanIn {
    const uint32_t* A;  // near list (or implicit 0..nA-1 when implicit)
    uint32_t nA;
    bool implicit;
    const uint32_t* X;  // crossers
    uint32_t nX;
    const uint32_t* F;  // far list (re-split scans only)
    uint32_t nF;
    uint32_t Bold;      // bound the far list was split at
    uint32_t B;         // bound of the outputs
};

__device__ void phase_scan(unsigned long long* ss, uint32_t level, uint32_t K, const ScanIn in, uint32_t* Aout,
                           uint32_t* Fout, uint32_t* curr, PhaseCtr* ph) {
    __shared__ uint32_t sh_c[kWarps], sh_a[kWarps], sh_f[kWarps];
    __shared__ uint32_t sh_bc, sh_ba, sh_bf;
    const uint32_t tid = threadIdx.x, lane = lane_id(), wid = tid >> 5;
    const uint64_t tile = uint64_t(kPeelThreads) * kScanItems;
    const uint64_t nAX = uint64_t(in.nA) + in.nX, ntot = nAX + in.nF;
    uint32_t local_min = 0xffffffffu;
    for (uint64_t t0 = uint64_t(blockIdx.x) * tile; t0 < ntot; t0 += uint64_t(gridDim.x) * tile) {
        uint32_t es[kScanItems];
        uint32_t kind = 0;  // 2 bits per item: 1 = curr, 2 = near, 3 = far
        uint32_t cc = 0, ca = 0, cf = 0;
#pragma unroll
        for (int k = 0; k < kScanItems; k++) {
            const uint64_t i = t0 + uint64_t(k) * kPeelThreads + tid;
            es[k] = 0;
            if (i < ntot) {
                const bool far_in = i >= nAX;
                const uint32_t e = i < in.nA ? (in.implicit ? static_cast<uint32_t>(i) : in.A[i])
                                             : (far_in ? in.F[i - nAX] : in.X[i - in.nA]);
                es[k] = e;
                TDG_CHECK(e != kNone);
                const unsigned long long w = ld_state(ss, e);
                const uint32_t sv = st_s(w);
                if (st_stamp(w) == 0 && !(far_in && sv < in.Bold)) {
                    if (sv == level) {
                        st_relaxed(stamp_ptr(ss, e), K);
                        kind |= 1u << (2 * k);
                        cc++;
                    } else if (sv < in.B) {
                        kind |= 2u << (2 * k);
                        ca++;
                        local_min = sv < local_min ? sv : local_min;
                    } else {
                        kind |= 3u << (2 * k);
                        cf++;
                    }
                }
            }
        }
        const uint32_t ic = warp_incl_scan(cc), ia = warp_incl_scan(ca), iff = warp_incl_scan(cf);
        if (lane == 31) { sh_c[wid] = ic; sh_a[wid] = ia; sh_f[wid] = iff; }
        __syncthreads();
        if (tid == 0) {
            uint32_t rc = 0, ra = 0, rf = 0;
            for (int w = 0; w < kWarps; w++) {
                const uint32_t c = sh_c[w], a = sh_a[w], f = sh_f[w];
                sh_c[w] = rc; sh_a[w] = ra; sh_f[w] = rf;
                rc += c; ra += a; rf += f;
            }
            sh_bc = rc ? atomicAdd(&ph->out_size, rc) : 0;
            sh_ba = ra ? atomicAdd(&ph->alive_size, ra) : 0;
            sh_bf = rf ? atomicAdd(&ph->far_size, rf) : 0;
        }
        __syncthreads();
        uint32_t pc = sh_bc + sh_c[wid] + ic - cc, pa = sh_ba + sh_a[wid] + ia - ca, pf = sh_bf + sh_f[wid] + iff - cf;
#pragma unroll
        for (int k = 0; k < kScanItems; k++) {
            const uint32_t f = (kind >> (2 * k)) & 3u;
            if (f == 1u) curr[pc++] = es[k];
            else if (f == 2u) Aout[pa++] = es[k];
            else if (f == 3u) Fout[pf++] = es[k];
        }
        __syncthreads();
    }
    for (int o = 16; o > 0; o >>= 1) local_min = min(local_min, __shfl_xor_sync(kFull, local_min, o));
    if (lane == 0 && local_min != 0xffffffffu) atomicMin(&ph->min_s, local_min);
}

// Near bound after a (re-)split at `level`: the window grows with the level so the number
// of far re-splits stays logarithmic in t_max.
#ifndef TDG_NEAR_ADD
#define TDG_NEAR_ADD 8
#define TDG_NEAR_DIV 4
#endif
__device__ __forceinline__ uint32_t near_bound(uint32_t level) {
    const unsigned long long b = static_cast<unsigned long long>(level) + TDG_NEAR_ADD + level / TDG_NEAR_DIV;
    return b > 0xfffffff0ull ? 0xfffffff0u : static_cast<uint32_t>(b);
}

// Sub-level prep: block b owns curr chunk b; probe count of e1 = min live degree.
// ---- locality: order a big sub-level's curr edges by the vertex whose hash table they
// probe (bucketed counting sort, 2^16 buckets of 2^bshift vertices), so concurrently
// running warps share hot tables in L2 instead of hitting DRAM for every lookup.
#ifndef TDG_SORT_MIN
#define TDG_SORT_MIN (1u << 20)
#endif
constexpr uint32_t kSortMin = TDG_SORT_MIN;

__device__ __forceinline__ uint32_t searched_vertex(const DevGraph& g, uint32_t e1) {
    const uint2 p = g.el[e1];
    return g.dl[p.x] <= g.dl[p.y] ? p.y : p.x;  // same choice as ptask
}

// Warp-aggregated bucket counter increment; returns this lane's rank among the lanes of
// its warp with the same bucket plus the counter's old value (all lanes must call).
__device__ __forceinline__ uint32_t bucket_add(uint32_t* ctr, uint32_t bucket, bool valid) {
    const uint32_t vm = __ballot_sync(kFull, valid);
    uint32_t pos = 0;
    if (valid) {
        const uint32_t grp = __match_any_sync(vm, bucket);
        const uint32_t leader = __ffs(grp) - 1;
        uint32_t base = 0;
        if (lane_id() == leader) base = atomicAdd(&ctr[bucket], static_cast<uint32_t>(__popc(grp)));
        base = __shfl_sync(grp, base, leader);
        pos = base + __popc(grp & lanemask_lt());
    }
    return pos;
}

TDG_COLD void phase_bucket_hist(const DevGraph& g, const uint32_t* curr, uint32_t cs, uint32_t* hist, uint32_t shift) {
    for (uint64_t i0 = uint64_t(blockIdx.x) * kPeelThreads + (threadIdx.x & ~31u); i0 < cs;
         i0 += uint64_t(gridDim.x) * kPeelThreads) {
        const uint64_t i = i0 + lane_id();
        const bool valid = i < cs;
        const uint32_t bk = valid ? (searched_vertex(g, curr[i]) >> shift) : 0;
        bucket_add(hist, bk, valid);
    }
}

// One block: cursor = exclusive scan of hist; hist is cleared for the next use.
TDG_COLD void phase_bucket_scan(uint32_t* hist, uint32_t* cursor) {
    constexpr uint32_t per = kBuckets / kPeelThreads;
    const uint32_t c0 = threadIdx.x * per;
    unsigned long long loc = 0;
    for (uint32_t c = 0; c < per; c++) loc += hist[c0 + c];
    unsigned long long tot;
    unsigned long long run = block_excl_scan64<kPeelThreads>(loc, tot);
    for (uint32_t c = 0; c < per; c++) {
        const uint32_t h = hist[c0 + c];
        cursor[c0 + c] = static_cast<uint32_t>(run);
        hist[c0 + c] = 0;
        run += h;
    }
}

TDG_COLD void phase_bucket_scatter(const DevGraph& g, const uint32_t* curr, uint32_t cs, uint32_t* cursor,
                                     uint32_t shift, uint32_t* out) {
    for (uint64_t i0 = uint64_t(blockIdx.x) * kPeelThreads + (threadIdx.x & ~31u); i0 < cs;
         i0 += uint64_t(gridDim.x) * kPeelThreads) {
        const uint64_t i = i0 + lane_id();
        const bool valid = i < cs;
        const uint32_t e = valid ? curr[i] : 0;
        const uint32_t bk = valid ? (searched_vertex(g, e) >> shift) : 0;
        const uint32_t pos = bucket_add(cursor, bk, valid);
        if (valid) out[pos] = e;
    }
}

// Task descriptors: prep resolves each task's three levels of dependent random loads
// (el -> dl -> off / table offset) once and stores {oa, la, ob, lb} in task order, so the
// process phase's window refills are one coalesced 16-byte load per lane (the descriptor
// loads were ~8 % of the peel's stall samples).

__device__ void phase_prep(const DevGraph& g, const uint32_t* curr, uint32_t cs, unsigned long long* wpre,
                           unsigned long long* bsum, uint4* desc) {
    prep_items<kPeelThreads>(cs, [&](uint32_t t) {
        uint32_t la;
        const ITask k = ptask(g, curr[t], la);
        desc[t] = make_uint4(k.id, k.oa, k.ob, k.lb);
        return la;
    }, wpre, bsum);
}

// Processed-edge bitmap (m bits: 65 MB at m = 523M, L2-resident) for the compaction, so
// that filtering a list costs an L2 lookup per entry instead of a DRAM sector.
__device__ void mark_processed(uint32_t* pbits, const uint32_t* curr, uint32_t cs) {
    for (uint32_t t = blockIdx.x * kPeelThreads + threadIdx.x; t < cs; t += gridDim.x * kPeelThreads) {
        const uint32_t e = curr[t];
        atomicOr(&pbits[e >> 5], 1u << (e & 31));
    }
}
__device__ __forceinline__ bool processed_bit(const uint32_t* pbits, uint32_t e) {
    return (ld_relaxed(pbits + (e >> 5)) >> (e & 31)) & 1u;
}

// Shared memory of the sub-level phases (one instance per block): the chunk offsets of the
// work prefix (or, in a fused small sub-level, its whole prefix and task descriptors) and the
// warps' candidate queues.
struct PeelShared {
    unsigned long long sboff[kMaxChunks + 1];
    uint32_t squeue[TDG_PEEL_QUEUE ? kWarps * 5 * kQCap : 1];
};
__device__ __forceinline__ PeelShared& peel_shared() {
    __shared__ __align__(16) PeelShared sh;
    return sh;
}

// process_sublevel (truss_parallel.cpp:39-104) for curr[0..cs) on the intersection engine.
template <bool kCount, uint32_t kShift = kFShift>
TDG_HOT unsigned long long phase_process(const DevGraph& g, unsigned long long* ss, uint32_t level,
                                            uint32_t K, const uint32_t* curr, uint32_t cs,
                                            const unsigned long long* wpre, const unsigned long long* bsum,
                                            uint32_t nchunks, PhaseCtr* ph, uint32_t* next,
                                            unsigned long long* cnt, uint32_t B, uint32_t* X, uint32_t* xcnt,
                                            const uint32_t* pbits, const uint4* desc) {
    PeelShared& sh = peel_shared();
    PeelPolicy<kCount, kShift> P{g, ss, level, K, curr, ph, next, g.adj, cnt, B, X, xcnt, pbits, desc,
                         sh.squeue + (TDG_PEEL_QUEUE ? (threadIdx.x >> 5) * 5 * kQCap : 0)};
    return process_items<kPeelThreads>(P, cs, wpre, bsum, nchunks, &ph->piece_head, sh.sboff);
}

// Small sub-levels (cs <= kFuseMax tasks: most of the thousands of late sub-levels) run prep
// and process as ONE phase: every block resolves all task descriptors itself (one task per
// thread) into shared memory and scans their probe counts there, then runs the usual
// process phase on that one-chunk prefix — no work-prefix round trip through global memory,
// one grid barrier per sub-level instead of two. Same probes, same sets.
#ifndef TDG_FUSE_MAX
#define TDG_FUSE_MAX 256
#endif
constexpr uint32_t kFuseMax = TDG_FUSE_MAX;
static_assert(kFuseMax <= uint32_t(kPeelThreads), "fused prep: one task per thread");
// layout inside PeelShared::sboff (u64 words): [0,1] chunk offsets of the one chunk, [2] its
// total (the "bsum"), [8, 8 + kFuseMax) the prefix, then the descriptors (16-byte aligned)
constexpr uint32_t kFusePre = 8, kFuseDesc = 8 + kFuseMax + (kFuseMax & 1);
static_assert((kFuseDesc * 8) % 16 == 0 && kFuseDesc * 8 + kFuseMax * 16 <= (kMaxChunks + 1) * 8,
              "fused prefix + descriptors alias the chunk-offset array");

__device__ void phase_fused_prep(const DevGraph& g, const uint32_t* curr, uint32_t cs) {
    PeelShared& sh = peel_shared();
    uint4* sdesc = reinterpret_cast<uint4*>(sh.sboff + kFuseDesc);
    const uint32_t t = threadIdx.x;
    uint32_t la = 0;
    if (t < cs) {
        const ITask k = ptask(g, curr[t], la);
        sdesc[t] = make_uint4(k.id, k.oa, k.ob, k.lb);
    }
    unsigned long long W;
    const unsigned long long ex = block_excl_scan64<kPeelThreads>(la, W);
    if (t < cs) sh.sboff[kFusePre + t] = ex;
    if (t == 0) sh.sboff[2] = W;
    __syncthreads();
}

// Adjacency compaction (between levels): drop processed edges (0 < stamp < K) from every
// live list, in place and order-preserving, and shrink dl. Lists of original degree above
// kBigList go through fixed chunks (below), the rest through flat warp tiles. Processed
// edges are skipped by every probe anyway (:85), so this only removes work; triangle sets
// seen by the peel are unchanged.
constexpr uint32_t kBigList = 2048;
#ifndef TDG_COMPACT_NUM
#define TDG_COMPACT_NUM 9  // compact once live edges <= NUM/DEN of those at the last compaction
#define TDG_COMPACT_DEN 10
#endif
constexpr unsigned long long kCompactNum = TDG_COMPACT_NUM, kCompactDen = TDG_COMPACT_DEN;


// Long lists (original degree > kBigList) are cut into fixed kChunk-slot chunks
// {vertex, index} (table built once by k_peel_init), so a hub's list is compacted by many
// warps at once. Pass A: each warp filters one chunk into the slot-aligned scratch and
// records its kept count. Pass B (after a grid barrier): each chunk copies its kept
// entries back to its list at the kept count of the list's earlier chunks; the list's
// last chunk stores the new live length.
constexpr uint32_t kChunk = 512;
constexpr int kCompactU = 4;  // entries per lane per compaction round

__device__ __forceinline__ bool long_list(const DevGraph& g, uint32_t u) { return g.off[u + 1] - g.off[u] > kBigList; }

template <bool kCount>
TDG_COLD void phase_compact_long(const DevGraph& g, const PeelBufs& pb, uint32_t nchunks) {
    const uint32_t lane = lane_id();
    const uint32_t gw = (blockIdx.x * kPeelThreads + threadIdx.x) >> 5, nw = (gridDim.x * kPeelThreads) >> 5;
    for (uint32_t c = gw; c < nchunks; c += nw) {
        const uint2 ck = pb.chunks[c];
        const uint32_t lo = ck.y * kChunk, dlu = g.dl[ck.x];
        uint32_t kept = 0;
        if (lo < dlu) {
            const uint32_t hi = min(dlu, lo + kChunk), o = g.off[ck.x];
            TDG_CHECK(ck.x < g.n && hi <= g.off[ck.x + 1] - o);
            for (uint32_t r0 = lo; r0 < hi; r0 += 32u * kCompactU) {
                uint32_t a[kCompactU], e[kCompactU], st[kCompactU];
#pragma unroll
                for (int q = 0; q < kCompactU; q++) {
                    const uint32_t i = r0 + 32u * q + lane;
                    a[q] = 0;
                    e[q] = 0;
                    if (i < hi) {
                        a[q] = g.adj[o + i];
                        e[q] = g.eid[o + i];
                    }
                }
#pragma unroll
                for (int q = 0; q < kCompactU; q++)
                    st[q] = (r0 + 32u * q + lane < hi) ? processed_bit(pb.pbits, e[q]) : 0u;
#pragma unroll
                for (int q = 0; q < kCompactU; q++) {
                    const bool keep = r0 + 32u * q + lane < hi && !st[q];
                    const uint32_t bal = __ballot_sync(kFull, keep);
                    if (keep) {
                        const uint32_t at = o + lo + kept + __popc(bal & lanemask_lt());
                        pb.sadj[at] = a[q];
                        pb.seid[at] = e[q];
                    }
                    kept += __popc(bal);
                }
            }
        }
        if (lane == 0) {
            pb.ckept[c] = kept;
            if constexpr (kCount) {
                if (lo < dlu) atomicAdd(&pb.ctl->cnt[kCntCompIn], static_cast<unsigned long long>(min(dlu, lo + kChunk) - lo));
                atomicAdd(&pb.ctl->cnt[kCntCompLong], static_cast<unsigned long long>(kept));
            }
        }
    }
}

TDG_COLD void phase_compact_copy(const DevGraph& g, const PeelBufs& pb, uint32_t nchunks) {
    const uint32_t lane = lane_id();
    const uint32_t gw = (blockIdx.x * kPeelThreads + threadIdx.x) >> 5, nw = (gridDim.x * kPeelThreads) >> 5;
    for (uint32_t c = gw; c < nchunks; c += nw) {
        const uint2 ck = pb.chunks[c];
        const uint32_t kept = pb.ckept[c];
        const uint32_t deg = g.off[ck.x + 1] - g.off[ck.x];
        const bool last = (ck.y + 1) * kChunk >= deg;
        if (kept == 0 && !last) continue;
        uint32_t before = 0;  // kept entries of the list's chunks 0 .. ck.y-1 (at c-ck.y ..)
        for (uint32_t k = lane; k < ck.y; k += 32) before += pb.ckept[c - ck.y + k];
#pragma unroll
        for (int d = 16; d > 0; d >>= 1) before += __shfl_xor_sync(kFull, before, d);
        const uint32_t o = g.off[ck.x], src = o + ck.y * kChunk;
        for (uint32_t i = lane; i < kept; i += 32) {
            g.adj[o + before + i] = pb.sadj[src + i];
            g.eid[o + before + i] = pb.seid[src + i];
        }
        if (last && lane == 0) g.dl[ck.x] = before + kept;
    }
}

// Pass 2 (short lists): a warp takes a tile of 32 consecutive vertices and walks their
// live entries as one flat item range (32*kCompactU items per round, lane -> vertex by a
// shuffle search over the tile's prefix), so short lists fill the lanes and every lane
// keeps kCompactU state loads in flight. Writes stay in list order: an entry's new slot is
// its list's kept count before this round (per-vertex counter in shared memory) plus the
// kept entries before it in the round.
template <bool kCount>
TDG_COLD void phase_compact_short(const DevGraph& g, const uint32_t* pbits, unsigned long long* cnt) {
    __shared__ uint32_t sh_kept[kWarps][32];
    const uint32_t lane = lane_id(), wid = threadIdx.x >> 5;
    const uint32_t gw = (blockIdx.x * kPeelThreads + threadIdx.x) >> 5, nw = (gridDim.x * kPeelThreads) >> 5;
    for (uint64_t v0 = uint64_t(gw) * 32; v0 < g.n; v0 += uint64_t(nw) * 32) {
        const uint64_t u = v0 + lane;
        uint32_t len = 0, o = 0;
        if (u < g.n && !long_list(g, static_cast<uint32_t>(u))) len = g.dl[u];
        const uint32_t incl = warp_incl_scan(len), excl = incl - len;
        const uint32_t total = __shfl_sync(kFull, incl, 31);
        if (total == 0) continue;
        if (len) o = g.off[u];
        sh_kept[wid][lane] = 0;
        __syncwarp();
        for (uint32_t r0 = 0; r0 < total; r0 += 32u * kCompactU) {
            uint32_t a[kCompactU], e[kCompactU], st[kCompactU], own[kCompactU], slot[kCompactU];
#pragma unroll
            for (int q = 0; q < kCompactU; q++) {
                const uint32_t item = r0 + 32u * q + lane;
                own[q] = warp_search_le(excl, item);
                const uint32_t ob = __shfl_sync(kFull, o, own[q]);
                const uint32_t ex = __shfl_sync(kFull, excl, own[q]);
                slot[q] = ob + (item - ex);
                a[q] = 0;
                e[q] = 0;
                if (item < total) {
                    TDG_CHECK(slot[q] < 2ull * g.m);
                    a[q] = g.adj[slot[q]];
                    e[q] = g.eid[slot[q]];
                }
            }
#pragma unroll
            for (int q = 0; q < kCompactU; q++)
                st[q] = (r0 + 32u * q + lane < total) ? processed_bit(pbits, e[q]) : 0u;
            __syncwarp();  // every read of this round precedes every write
#pragma unroll
            for (int q = 0; q < kCompactU; q++) {
                const bool act = r0 + 32u * q + lane < total;
                const bool keep = act && !st[q];
                const uint32_t bal = __ballot_sync(kFull, keep);
                const uint32_t prev_own = __shfl_up_sync(kFull, own[q], 1);
                const uint32_t heads = __ballot_sync(kFull, lane == 0 || own[q] != prev_own);
                const uint32_t le = lanemask_lt() | (1u << lane);
                const uint32_t seg_lo = 31u - __clz(heads & le);
                const uint32_t segmask = ~((1u << seg_lo) - 1u);
                const uint32_t before = __popc(bal & lanemask_lt() & segmask);
                const uint32_t kept0 = sh_kept[wid][own[q]];
                const uint32_t ob = __shfl_sync(kFull, o, own[q]);
                if (keep) {
                    g.adj[ob + kept0 + before] = a[q];
                    g.eid[ob + kept0 + before] = e[q];
                }
                const uint32_t next_own = __shfl_down_sync(kFull, own[q], 1);
                const bool tail = act && (lane == 31 || next_own != own[q] ||
                                          r0 + 32u * q + lane + 1 >= total);
                __syncwarp();
                if (tail) sh_kept[wid][own[q]] = kept0 + before + (keep ? 1u : 0u);
                __syncwarp();
            }
        }
        if (len) g.dl[u] = sh_kept[wid][lane];
        if constexpr (kCount) {
            const uint32_t kept = __reduce_add_sync(kFull, len ? sh_kept[wid][lane] : 0u);
            if (lane == 0) {
                atomicAdd(cnt + kCntCompIn, static_cast<unsigned long long>(total));
                atomicAdd(cnt + kCntCompKept, static_cast<unsigned long long>(kept));
            }
        }
        __syncwarp();
    }
}

__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

__device__ __forceinline__ uint32_t vload(const uint32_t* p) { return *reinterpret_cast<const volatile uint32_t*>(p); }

// Grid-wide barrier of the persistent kernel. TDG_FAST_BARRIER: one fire-and-forget
// red.release per block on a monotone arrival counter and an ld.acquire spin of thread 0
// (no returned atomic on the critical path); else cooperative_groups' grid.sync().
#ifndef TDG_FAST_BARRIER
#define TDG_FAST_BARRIER 1
#endif
struct GridBar {
    cg::grid_group grid;
    uint32_t* ctr;
    uint32_t target;
    __device__ __forceinline__ void sync() {
        if (TDG_FAST_BARRIER) {
            __syncthreads();
            if (threadIdx.x == 0) {
                target += gridDim.x;
                __threadfence();
                asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(ctr) : "memory");
                uint32_t v;
                do {
                    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(ctr) : "memory");
                } while (static_cast<int>(v - target) < 0);
            }
            __syncthreads();
        } else {
            grid.sync();
        }
    }
};

// The whole truss_parallel level loop (truss_parallel.cpp:119-144) in one launch.
// kShift: filter density of the tables this segment probes (the input graph's, or the rebuilt).
template <bool kCount, uint32_t kShift>
__global__ void __launch_bounds__(kPeelThreads, TDG_PEEL_MINB) k_peel(DevGraph g, PeelBufs pb) {
    GridBar grid{cg::this_grid(), &pb.ctl->bar, 0u};
    PeelCtl* ctl = pb.ctl;
    const bool leader = blockIdx.x == 0 && threadIdx.x == 0;
    // The level loop's state is volatile ON PURPOSE: it then lives in the thread's stack frame
    // (L1-resident local memory, a few accesses per phase) and never competes with the probe
    // loop for registers. Left to the register allocator, small changes to this loop moved
    // spills into the probe loop and cost up to 15 % of the peel (64 registers per thread).
    volatile uint32_t j = 0, level = 0, K = 1, nA = g.m, ai = 0, li = 0, live_at_compact = g.m, live_at_rebuild = g.m;
    volatile uint32_t B = 0, fi = 1, nF = 0, xp = 0;  // near bound, far list parity/size, crosser parity
    const uint32_t* volatile pend = nullptr;          // last sub-level's curr, not yet in pbits
    volatile uint32_t pend_n = 0;
    volatile bool implicit = true;
    volatile unsigned long long t_prev = leader ? gtimer() : 0;
    volatile unsigned long long sub_w = 0;
    const uint32_t nchunks = vload(&ctl->nchunks);
    volatile bool resumed = pb.seg > 0;
    volatile uint32_t cs = 0;
    if (resumed) {  // a later segment of the same decomposition: continue where the last one left
        if (vload(&ctl->done)) return;
        const PeelResume& rs = ctl->rs;
        j = rs.j; level = rs.level; K = rs.K; nA = rs.nA; ai = rs.ai; li = rs.li;
        live_at_compact = rs.live_at_compact; live_at_rebuild = rs.live_at_rebuild;
        B = rs.B; fi = rs.fi; nF = rs.nF; xp = rs.xp; cs = rs.cs;
        grid.target = rs.bar_target;
        implicit = false;
        if (leader) ctl->rebuild_ns += t_prev - rs.t_exit;
    }
    while (true) {
        if (!resumed) {
        // ---- scan at `level` (one grid barrier); re-split the far list once level >= B
        const bool resplit = implicit || level >= B;
        // (crossers sit right after the near list, in the same buffer: A[ai][nA .. nA + nX))
        ScanIn in{pb.A[ai], nA, implicit, pb.A[ai] + nA, vload(&ctl->xcnt[xp]), pb.F[fi], resplit ? nF : 0u, B, B};
        if (resplit) in.B = near_bound(level);
        if (leader) {
            reset_ctr(&ctl->ph[(j + 1) % 3]);
            ctl->scans++;
            ctl->cnt[kCntScanIn] += static_cast<unsigned long long>(in.nA) + in.nX + in.nF;
            ctl->cnt[kCntMarks] += pend_n;
            ctl->xcnt[xp ^ 1] = 0;  // crossers after this scan (read by the previous scan)
            if (resplit) ctl->rebuilds++;
        }
        // (every counter read after a barrier lives in the rotating phase slots, which are
        // reset two phases after they are written, so no block can observe a reset early)
        if (pend_n) mark_processed(pb.pbits, pend, pend_n);  // before the compaction that may follow
        pend_n = 0;
        phase_scan(pb.ss, level, K, in, pb.A[ai ^ 1], pb.F[fi ^ 1], pb.L[li], &ctl->ph[j % 3]);
        grid.sync();
        if (leader) { const unsigned long long t = gtimer(); ctl->scan_ns += t - t_prev; t_prev = t; }
        j++;
        const PhaseCtr* r = &ctl->ph[(j - 1) % 3];
        cs = vload(&r->out_size);
        nA = vload(&r->alive_size);
        const uint32_t mins = vload(&r->min_s);
        ai ^= 1;
        xp ^= 1;
        implicit = false;
        B = in.B;
        if (resplit) {
            fi ^= 1;
            nF = vload(&r->far_size);
        }
        if (leader) ctl->cnt[kCntScanOut] += static_cast<unsigned long long>(cs) + nA + (resplit ? nF : 0u);
        if (cs == 0) {
            if (nA == 0) {
                if (nF == 0) break;
                level = B;  // only far edges are left, all with support >= B
            } else {
                level = mins;  // skip empty levels
            }
            continue;
        }
        // ---- compaction once the live edge count fell below kCompactFrac of the last one
        const unsigned long long live = static_cast<unsigned long long>(cs) + nA + nF;
        if (level > 0 && live * kCompactDen < static_cast<unsigned long long>(live_at_compact) * kCompactNum) {
            if (leader) { reset_ctr(&ctl->ph[(j + 1) % 3]); ctl->compactions++; }
            phase_compact_long<kCount>(g, pb, nchunks);
            phase_compact_short<kCount>(g, pb.pbits, ctl->cnt);
            grid.sync();
            phase_compact_copy(g, pb, nchunks);
            grid.sync();
            unsigned long long t_c = 0;
            if (leader) { t_c = gtimer(); ctl->compact_ns += t_c - t_prev; }
            j++;
            live_at_compact = static_cast<uint32_t>(live);
            // ---- table rebuild on the live graph (kernels below): leave the launch here; the
            // host has queued the rebuild kernels and the next segment, which resumes at the
            // sub-levels of this level
            // (the denser rebuilt filters must fit the words allocated for the input graph's:
            // the live tables have at most kHF * live / 2 + min(n, 2 live) buckets)
            const unsigned long long nb_max = kHF * live / 2 + (2 * live < g.n ? 2 * live : g.n);
            if (kPeelRebuildDen && pb.seg + 1 < pb.nseg && pb.rebuild_den &&
                live * pb.rebuild_den <= static_cast<unsigned long long>(live_at_rebuild) * pb.rebuild_num &&
                (nb_max >> kFShiftRebuild) + 1 <= (g.nbuckets >> kFShift)) {
                if (leader) {
                    PeelResume& rs = ctl->rs;
                    rs.j = j; rs.level = level; rs.K = K; rs.nA = nA; rs.ai = ai; rs.li = li;
                    rs.live_at_compact = live_at_compact; rs.live_at_rebuild = static_cast<uint32_t>(live);
                    rs.B = B; rs.fi = fi; rs.nF = nF; rs.xp = xp; rs.cs = cs;
                    rs.bar_target = grid.target;
                    rs.t_exit = t_c;
                    ctl->table_rebuilds++;
                    ctl->cnt[kCntRebuildEdges] += live;
                }
                return;
            }
        }
        }  // !resumed
        resumed = false;
        // ---- sub-levels: prep + process (two grid barriers each; level 0 one)
        while (true) {
            if (leader) {
                if (level < pb.nsl_cap) pb.nsl[level]++; else ctl->nsl_overflow = 1;
                ctl->sublevels++;
                ctl->cnt[kCntMarks] += pend_n;
                if (level > 0) {
                    ctl->cnt[kCntTasks] += cs;
                    if (kSortMin && cs >= kSortMin && 5ull * cs <= 4ull * g.m) ctl->cnt[kCntSorted] += cs;
                }
                ctl->levels_len = level + 1;
                reset_ctr(&ctl->ph[(j + 1) % 3]);
            }
            // the previous sub-level's curr is processed now: mark it (read by this sub-level's
            // probes and by compaction; this sub-level's own curr is marked by the next phase)
            if (pend_n) mark_processed(pb.pbits, pend, pend_n);
            if (level > 0) {  // level 0: s[e1] == 0 bounds its live triangles to none
                const uint32_t* tasks = pb.L[li];
                const unsigned long long* wp = pb.wpre;
                const unsigned long long* bs = pb.bsum;
                const uint4* dsc = pb.desc;
                uint32_t nch = gridDim.x;
                if (kFuseMax && cs <= kFuseMax) {
                    phase_fused_prep(g, tasks, cs);
                    PeelShared& sh = peel_shared();
                    wp = sh.sboff + kFusePre;
                    bs = sh.sboff + 2;
                    dsc = reinterpret_cast<const uint4*>(sh.sboff + kFuseDesc);
                    nch = 1;
                } else {
                    // group big sub-levels by searched vertex; the sorted list sits after the task
                    // descriptors in the compaction scratch (16 + 4 bytes per task <= its 16m + 16)
                    if (kSortMin && cs >= kSortMin && 5ull * cs <= 4ull * g.m) {
                        phase_bucket_hist(g, tasks, cs, pb.bhist, pb.bshift);
                        grid.sync();
                        if (blockIdx.x == 0) phase_bucket_scan(pb.bhist, pb.bcur);
                        grid.sync();
                        uint32_t* Ls = reinterpret_cast<uint32_t*>(pb.desc + cs);
                        phase_bucket_scatter(g, tasks, cs, pb.bcur, pb.bshift, Ls);
                        grid.sync();
                        tasks = Ls;
                    }
                    phase_prep(g, tasks, cs, pb.wpre, pb.bsum, pb.desc);
                    grid.sync();
                }
                const unsigned long long W =
                    phase_process<kCount, kShift>(g, pb.ss, level, K, tasks, cs, wp, bs, nch, &ctl->ph[j % 3], pb.L[li ^ 1],
                                          ctl->cnt, B, pb.A[ai] + nA, &ctl->xcnt[xp], pb.pbits, dsc);
                if (leader) {
                    ctl->probes += W;
                    sub_w = W;
                }
            }
            grid.sync();
            if (leader) {
                const unsigned long long t = gtimer();
                if (pb.trace && ctl->sublevels <= pb.trace_cap) {  // diagnostic per-sub-level record
                    unsigned long long* r4 = pb.trace + 4ull * (ctl->sublevels - 1);
                    r4[0] = (static_cast<unsigned long long>(level) << 32) | cs;
                    r4[1] = sub_w;
                    r4[2] = t - t_prev;
                    r4[3] = K;
                }
                ctl->proc_ns += t - t_prev;
                t_prev = t;
                sub_w = 0;
            }
            j++;
            K++;
            const PhaseCtr* r = &ctl->ph[(j - 1) % 3];
            pend = pb.L[li];
            pend_n = cs;
            cs = vload(&r->out_size);
            li ^= 1;
            if (cs == 0) break;
        }
        level++;
    }
    if (leader) { ctl->final_stamp = K; ctl->done = 1; }
#if TDG_DIAG_RATIO
    if (leader) {
        printf("DIAG ratio lb/la (<2,<4,<8,<16,<64,>=64):");
        for (int i = 0; i < 6; i++) printf(" %llu", d_diag[i]);
        printf("\nDIAG lb (<512,<2K,<8K,<32K,<128K,<512K,>=512K):");
        for (int i = 6; i < 13; i++) printf(" %llu", d_diag[i]);
        printf("\nDIAG ratio<8 by lb (<8K,<128K,>=128K): %llu %llu %llu\n", d_diag[13], d_diag[14], d_diag[15]);
        for (int i = 0; i < 16; i++) d_diag[i] = 0;
    }
#endif
}

// ---- table rebuild on the live graph. The tables and filters are built for the input
// graph, but most of the peel's probes run when only a fraction of the edges is left (C5: 2/3
// of the probes with < 1/4 of the edges live), and their random accesses keep spreading over
// the full-size tables (16.7 GB + 0.75 GB of filters at C5). Right after a compaction (dl =
// live degree of every vertex, pbits = the processed edges) k_peel ends its segment; these
// kernels re-size the tables to the live degrees and refill them with the live edges only,
// in place, and the next segment resumes: the working set shrinks with the graph (filters
// become L2-resident), dead peers vanish from the tables. Same layout and lookup as the build
// (tdg_common.cuh); values carry no orientation bit (the peel ignores it). The kernels are
// queued with the segments and do nothing once the level loop has finished. (Run inside the
// cooperative kernel instead, the same phases cost the probe loop ~10 % through its register
// allocation.)
constexpr unsigned kRbBlocks = 592;
static_assert(kRbBlocks <= kMaxChunks, "one vertex chunk per block");

// Pass 1: block b owns vertex chunk b: hbo[x] = chunk-local exclusive prefix of nb(x) =
// hbuckets(dl[x]); bsum[b] = the chunk's bucket count.
__global__ void __launch_bounds__(kPeelThreads) k_rb_sizes(DevGraph g, PeelBufs pb) {
    if (pb.ctl->done) return;
    const uint32_t CH = chunk_len(g.n, gridDim.x);
    const uint64_t lo = uint64_t(blockIdx.x) * CH;
    const uint64_t hi = lo + CH < g.n ? lo + CH : g.n;
    unsigned long long run = 0;
    for (uint64_t x0 = lo; x0 < hi; x0 += kPeelThreads) {
        const uint64_t x = x0 + threadIdx.x;
        const unsigned long long nb = x < hi ? hbuckets(g.dl[x]) : 0u;
        unsigned long long tot;
        const unsigned long long ex = block_excl_scan64<kPeelThreads>(nb, tot);
        if (x < hi) pb.hbo_w[x] = static_cast<uint32_t>(run + ex);
        run += tot;
    }
    if (threadIdx.x == 0) pb.bsum[blockIdx.x] = run;
}

// Pass 2: chunk offsets added to the chunk-local prefixes; the new tables' buckets and filter
// words cleared.
__global__ void __launch_bounds__(kPeelThreads) k_rb_clear(DevGraph g, PeelBufs pb) {
    if (pb.ctl->done) return;
    __shared__ unsigned long long sboff[kMaxChunks + 1];
    const unsigned long long total = chunk_offsets<kPeelThreads>(pb.bsum, gridDim.x, sboff);
    const uint32_t CH = chunk_len(g.n, gridDim.x);
    const uint64_t lo = uint64_t(blockIdx.x) * CH;
    const uint64_t hi = lo + CH < g.n ? lo + CH : g.n;
    const uint32_t add = static_cast<uint32_t>(sboff[blockIdx.x]);
    for (uint64_t x = lo + threadIdx.x; x < hi; x += kPeelThreads) pb.hbo_w[x] += add;
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        pb.hbo_w[g.n] = static_cast<uint32_t>(total);
        pb.ctl->cnt[kCntRebuildBuckets] += total;
    }
    TDG_CHECK(total <= g.nbuckets);
    uint4* t4 = reinterpret_cast<uint4*>(pb.htab_w);
    const uint4 e4 = make_uint4(kHEmpty, kHEmpty, kHEmpty, kHEmpty);
    const uint64_t stride = uint64_t(gridDim.x) * kPeelThreads, tid = uint64_t(blockIdx.x) * kPeelThreads + threadIdx.x;
    for (uint64_t i = tid; i < 2 * total; i += stride) t4[i] = e4;
    if (pb.filt_w) {
        const uint64_t fw = (total >> kFShiftRebuild) + 1;
        for (uint64_t i = tid; i < fw; i += stride) pb.filt_w[i] = 0ull;
    }
}

// Pass 3a: tables of at most kHMid buckets, from the live lists (adj / eid [off[x], +dl[x])),
// in shared memory — one warp per table up to kHSmall buckets, the block for the rest — and
// written out with coalesced stores (as k_hbuild_small, build.cu).
__global__ void __launch_bounds__(256) k_rb_small(DevGraph g, PeelBufs pb) {
    if (pb.ctl->done) return;
    extern __shared__ uint32_t rb_smem[];  // 8 warps x kHSmall buckets x 8 words
    const uint32_t lane = threadIdx.x & 31u, w = threadIdx.x >> 5;
    uint32_t* t = rb_smem + w * kHSmall * 8u;
    const uint32_t nw = (gridDim.x * blockDim.x) >> 5;
    // a warp scans 32 vertices at a time and builds the non-empty small tables among them
    for (uint64_t x0 = uint64_t((blockIdx.x * blockDim.x + threadIdx.x) >> 5) * 32; x0 < g.n; x0 += uint64_t(nw) * 32) {
        const uint64_t xl = x0 + lane;
        uint32_t nbl = 0;
        if (xl < g.n) nbl = pb.hbo_w[xl + 1] - pb.hbo_w[xl];
        uint32_t todo = __ballot_sync(kFull, nbl != 0 && nbl <= kHSmall);
        while (todo) {
            const uint32_t src = __ffs(todo) - 1;
            todo &= todo - 1;
            const uint32_t x = static_cast<uint32_t>(x0) + src;
            const uint32_t nb = __shfl_sync(kFull, nbl, src);
            const uint32_t b0 = pb.hbo_w[x];
            for (uint32_t i = lane; i < 8u * nb; i += 32) t[i] = kHEmpty;
            __syncwarp();
            const uint32_t o = g.off[x], d = g.dl[x];
            for (uint32_t i = lane; i < d; i += 32) bucket_insert(t, nb, g.adj[o + i], g.eid[o + i]);
            __syncwarp();
            uint32_t* gt = pb.htab_w + 8ull * b0;
            for (uint32_t i = lane; i < 8u * nb; i += 32) gt[i] = t[i];
            __syncwarp();
        }
    }
    __syncthreads();
    __shared__ uint32_t q[256];
    __shared__ uint32_t qn;
    for (uint64_t c0 = uint64_t(blockIdx.x) * 256; c0 < g.n; c0 += uint64_t(gridDim.x) * 256) {
        if (threadIdx.x == 0) qn = 0;
        __syncthreads();
        const uint64_t x = c0 + threadIdx.x;
        if (x < g.n) {
            const uint32_t nb = pb.hbo_w[x + 1] - pb.hbo_w[x];
            if (nb > kHSmall && nb <= kHMid) q[atomicAdd(&qn, 1u)] = static_cast<uint32_t>(x);
        }
        __syncthreads();
        const uint32_t cnt = qn;
        for (uint32_t k = 0; k < cnt; k++) {
            const uint32_t v = q[k], b0 = pb.hbo_w[v], nb = pb.hbo_w[v + 1] - b0, o = g.off[v], d = g.dl[v];
            for (uint32_t i = threadIdx.x; i < 8u * nb; i += blockDim.x) rb_smem[i] = kHEmpty;
            __syncthreads();
            for (uint32_t i = threadIdx.x; i < d; i += blockDim.x) bucket_insert(rb_smem, nb, g.adj[o + i], g.eid[o + i]);
            __syncthreads();
            uint32_t* gt = pb.htab_w + 8ull * b0;
            for (uint32_t i = threadIdx.x; i < 8u * nb; i += blockDim.x) gt[i] = rb_smem[i];
            __syncthreads();
        }
    }
}

// Pass 3b: every live edge e = {u, v} (processed bit clear) enters the tables of more than
// kHMid buckets among its endpoints' (global CAS) and the filters of those with a filter.
// Internal edge ids follow the oriented lists, so consecutive edges share u.
__global__ void __launch_bounds__(256) k_rb_big(DevGraph g, PeelBufs pb) {
    if (pb.ctl->done) return;
    const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
    const uint32_t fscale = pb.filt_w ? g.fctl->fscale : 0u;
    for (uint64_t e0 = (uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) & ~31ull; e0 < g.m; e0 += stride) {
        const uint32_t w = pb.pbits[e0 >> 5];
        const uint64_t e = e0 + lane_id();
        if (e >= g.m || ((w >> lane_id()) & 1u)) continue;
        const uint2 p = g.el[e];
#pragma unroll
        for (int side = 0; side < 2; side++) {
            const uint32_t x = side ? p.y : p.x, y = side ? p.x : p.y;
            const uint32_t b0 = pb.hbo_w[x], nb = pb.hbo_w[x + 1] - b0;
            TDG_CHECK(nb > 0 && uint64_t(b0) + nb <= g.nbuckets);
            if (nb > kHMid) bucket_insert(pb.htab_w + 8ull * b0, nb, y, static_cast<uint32_t>(e));
            if (pb.filt_w && nb >= kFMin) atomicOr(&pb.filt_w[fword_index(b0, nb, y, kFShiftRebuild, fscale)], fbits(hmix(y)));
        }
    }
}

__global__ void k_peel_init(const uint32_t* __restrict__ off, uint32_t n, uint32_t* __restrict__ dl,
                            const uint32_t* __restrict__ s, uint32_t m, unsigned long long* __restrict__ ss,
                            PeelCtl* ctl, uint2* chunks, uint32_t chunk_cap) {
    for (uint32_t u = blockIdx.x * blockDim.x + threadIdx.x; u < n; u += gridDim.x * blockDim.x) {
        const uint32_t deg = off[u + 1] - off[u];
        dl[u] = deg;
        if (chunks && deg > kBigList) {  // compaction chunk table (order irrelevant)
            const uint32_t nc = (deg + kChunk - 1) / kChunk;
            const uint32_t base = atomicAdd(&ctl->nchunks, nc);
            if (base + nc <= chunk_cap)
                for (uint32_t k = 0; k < nc; k++) chunks[base + k] = make_uint2(u, k);
            else
                ctl->chunk_overflow = 1;
        }
    }
    if (ss)  // pack the support pass result with stamp 0
        for (uint32_t e = blockIdx.x * blockDim.x + threadIdx.x; e < m; e += gridDim.x * blockDim.x) ss[e] = s[e];
    if (blockIdx.x == 0 && threadIdx.x < 3) reset_ctr(&ctl->ph[threadIdx.x]);
}

// truss[ref id] = s + 2; ss is indexed by internal id, oeid maps it to the reference edge id.
__global__ void k_finalize(const unsigned long long* __restrict__ ss, const uint32_t* __restrict__ oeid, uint32_t m,
                           uint32_t* __restrict__ truss, PeelCtl* ctl) {
    uint32_t mx = 0;
    for (uint32_t e = blockIdx.x * blockDim.x + threadIdx.x; e < m; e += gridDim.x * blockDim.x) {
        const uint32_t t = static_cast<uint32_t>(ss[e]) + 2;  // truss_parallel.cpp:146-148
        truss[oeid[e]] = t;
        mx = t > mx ? t : mx;
    }
    for (int o = 16; o > 0; o >>= 1) mx = max(mx, __shfl_xor_sync(kFull, mx, o));
    if (lane_id() == 0 && mx) atomicMax(&ctl->t_max, mx);
}

// ---- step functions on reference-style flag arrays (tests/test_truss_parallel.cpp) ----
__global__ void k_step_stamps(const uint8_t* __restrict__ processed, const uint8_t* __restrict__ in_curr,
                              const uint32_t* __restrict__ s, uint32_t m, unsigned long long* __restrict__ ss,
                              PeelCtl* ctl) {
    for (uint32_t e = blockIdx.x * blockDim.x + threadIdx.x; e < m; e += gridDim.x * blockDim.x) {
        const unsigned long long st = processed[e] ? 1u : ((in_curr && in_curr[e]) ? 2u : 0u);
        ss[e] = (st << 32) | s[e];
    }
    if (blockIdx.x == 0 && threadIdx.x < 3) reset_ctr(&ctl->ph[threadIdx.x]);
}

__global__ void __launch_bounds__(kPeelThreads) k_step_scan(PeelBufs pb, uint32_t m, uint32_t level) {
    const ScanIn in{pb.A[0], m, true, nullptr, 0u, nullptr, 0u, 0u, 0xffffffffu};  // one near list, no far
    phase_scan(pb.ss, level, 2, in, pb.A[1], pb.A[1], pb.L[0], &pb.ctl->ph[0]);
}

__global__ void k_step_scan_flags(const uint32_t* __restrict__ curr, PeelCtl* ctl, uint8_t* in_curr) {
    const uint32_t cs = ctl->ph[0].out_size;
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < cs; i += gridDim.x * blockDim.x)
        in_curr[curr[i]] = 1;
}

__global__ void __launch_bounds__(kPeelThreads) k_step_prep(DevGraph g, PeelBufs pb, uint32_t cs) {
    phase_prep(g, pb.L[0], cs, pb.wpre, pb.bsum, pb.desc);
}

// Hand-built states may break the level-0 invariant, so the step form always probes.
__global__ void __launch_bounds__(kPeelThreads) k_step_process(DevGraph g, PeelBufs pb, uint32_t cs, uint32_t level,
                                                               uint32_t nchunks) {
    phase_process<false>(g, pb.ss, level, 2, pb.L[0], cs, pb.wpre, pb.bsum, nchunks, &pb.ctl->ph[1], pb.L[1],
                         nullptr, 0xffffffffu, nullptr, &pb.ctl->xcnt[0], nullptr, pb.desc);
}

// Epilogue (truss_parallel.cpp:97-102) + in_next flags for the appended edges; unpacks s.
__global__ void k_step_process_flags(const uint32_t* __restrict__ curr, uint32_t cs,
                                     const uint32_t* __restrict__ next, PeelCtl* ctl, uint8_t* in_curr,
                                     uint8_t* in_next, uint8_t* processed, const unsigned long long* __restrict__ ss,
                                     uint32_t* __restrict__ s, uint32_t m) {
    const uint32_t ns = ctl->ph[1].out_size;
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < cs || i < ns; i += gridDim.x * blockDim.x) {
        if (i < cs) { processed[curr[i]] = 1; in_curr[curr[i]] = 0; }
        if (i < ns) in_next[next[i]] = 1;
    }
    for (uint32_t e = blockIdx.x * blockDim.x + threadIdx.x; e < m; e += gridDim.x * blockDim.x)
        s[e] = static_cast<uint32_t>(ss[e]);
}

}  // namespace

cudaError_t launch_peel(const DevGraph& g, const PeelBufs& p, int sm_count, cudaStream_t st,
                        uint32_t* launches) {
    cudaError_t err = cudaMemsetAsync(p.ctl, 0, sizeof(PeelCtl), st);
    if (err != cudaSuccess) return err;
    if ((err = cudaMemsetAsync(p.nsl, 0, size_t(p.nsl_cap) * sizeof(uint32_t), st)) != cudaSuccess) return err;
    if (g.m == 0) return cudaSuccess;
    if (p.pbits && (err = cudaMemsetAsync(p.pbits, 0, size_t((g.m + 31) / 32) * 4, st)) != cudaSuccess) return err;
    k_peel_init<<<148 * 4, 256, 0, st>>>(g.off, g.n, g.dl, p.s, g.m, p.ss, p.ctl, p.chunks, p.chunk_cap);
    // count mode (diagnostic, PeelBufs::count): the instantiation that tallies every access;
    // segments after a rebuild probe the denser rebuilt filters (a second instantiation: a
    // run-time shift in the probe loop cost 15 % through its register allocation)
    const void* kern = p.count ? reinterpret_cast<const void*>(k_peel<true, kFShift>)
                               : reinterpret_cast<const void*>(k_peel<false, kFShift>);
    const void* kern_rb = p.count ? reinterpret_cast<const void*>(k_peel<true, kFShiftRebuild>)
                                  : reinterpret_cast<const void*>(k_peel<false, kFShiftRebuild>);
    int per_sm = 0;
    err = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kPeelThreads, 0);
    if (err != cudaSuccess) return err;
    if (per_sm < 1) return cudaErrorLaunchOutOfResources;
    unsigned blocks = static_cast<unsigned>(sm_count * per_sm);
    if (blocks > kMaxChunks) blocks = kMaxChunks;
    DevGraph gg = g;
    PeelBufs pp = p;
    void* args[] = {&gg, &pp};
    // one cooperative launch (an L2 persisting window on the processed bitmap was measured
    // here: the device-wide set-aside it needs shrank the normal L2 for every kernel, C5 peel
    // 2.52 -> 3.77 s and build 145 -> 252 ms; removed)
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(blocks);
    cfg.blockDim = dim3(kPeelThreads);
    cfg.dynamicSmemBytes = 0;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeCooperative;
    at[0].val.cooperative = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    // Segments: the level loop leaves its launch where the tables are to be rebuilt on the
    // live graph (at most kPeelRebuildMax times); the rebuild kernels and the next segment are
    // queued up front and do nothing once the loop has finished — no host round trip.
    const bool rebuild = kPeelRebuildDen != 0 && p.rebuild_den != 0 && p.hbo_w && p.htab_w;
    pp.nseg = rebuild && p.nseg > 1 ? p.nseg : 1;
    const size_t rb_smem = 8u * kHSmall * 8u * sizeof(uint32_t);
    if (rebuild) {
        err = cudaFuncSetAttribute(k_rb_small, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(rb_smem));
        if (err != cudaSuccess) return err;
    }
    (*launches)++;  // k_peel_init
    for (uint32_t seg = 0; seg < pp.nseg; seg++) {
        pp.seg = seg;
        if ((err = cudaLaunchKernelExC(&cfg, seg ? kern_rb : kern, args)) != cudaSuccess) return err;
        (*launches)++;
        if (seg + 1 < pp.nseg) {
            k_rb_sizes<<<kRbBlocks, kPeelThreads, 0, st>>>(gg, pp);
            k_rb_clear<<<kRbBlocks, kPeelThreads, 0, st>>>(gg, pp);
            k_rb_small<<<148u * 3u, 256, rb_smem, st>>>(gg, pp);
            k_rb_big<<<148u * 16u, 256, 0, st>>>(gg, pp);
            (*launches) += 4;
        }
    }
    return cudaGetLastError();
}

cudaError_t launch_finalize(const unsigned long long* ss, const uint32_t* oeid, uint32_t m, uint32_t* truss, PeelCtl* ctl,
                            cudaStream_t st, uint32_t* launches) {
    if (m == 0) return cudaSuccess;
    k_finalize<<<148 * 4, 256, 0, st>>>(ss, oeid, m, truss, ctl);
    (*launches)++;
    return cudaGetLastError();
}

cudaError_t launch_step_scan(const DevGraph& g, const PeelBufs& p, uint32_t level, const uint8_t* processed,
                             uint8_t* in_curr, int sm_count, cudaStream_t st) {
    k_step_stamps<<<sm_count * 2, 256, 0, st>>>(processed, nullptr, p.s, g.m, p.ss, p.ctl);
    k_step_scan<<<sm_count, kPeelThreads, 0, st>>>(p, g.m, level);
    k_step_scan_flags<<<sm_count, 256, 0, st>>>(p.L[0], p.ctl, in_curr);
    return cudaGetLastError();
}

cudaError_t launch_step_process(const DevGraph& g, const PeelBufs& p, uint32_t level, uint32_t curr_size,
                                uint8_t* in_curr, uint8_t* in_next, uint8_t* processed, int sm_count,
                                cudaStream_t st) {
    const uint32_t nchunks = static_cast<uint32_t>(sm_count);
    k_peel_init<<<sm_count, 256, 0, st>>>(g.off, g.n, g.dl, nullptr, 0, nullptr, p.ctl, nullptr, 0);
    k_step_stamps<<<sm_count * 2, 256, 0, st>>>(processed, in_curr, p.s, g.m, p.ss, p.ctl);
    k_step_prep<<<nchunks, kPeelThreads, 0, st>>>(g, p, curr_size);
    k_step_process<<<sm_count * 2, kPeelThreads, 0, st>>>(g, p, curr_size, level, nchunks);
    k_step_process_flags<<<sm_count, 256, 0, st>>>(p.L[0], curr_size, p.L[1], p.ctl, in_curr, in_next, processed,
                                                   p.ss, p.s, g.m);
    return cudaGetLastError();
}

}  // namespace tdg
