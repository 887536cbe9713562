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
//  * Flags -> stamps: stamp[e] = index of the sub-level in which e is (or was) curr.
//    processed(e) <=> 0 < stamp < K, in_curr(e) <=> stamp == K, next <=> stamp == K+1.
//    Entering next is the single stamp store by the appending thread, so the
//    reference's epilogue pass over curr (:97-102) and the flag swaps vanish.
//  * No dense X[n] mark array (MarkScratchPool, truss_parallel.hpp:55-59): N(u)∩N(v) is
//    computed by walking the shorter live list and binary-searching the longer one.
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

#include "tdg_kernels.h"

namespace cg = cooperative_groups;

namespace tdg {

namespace {

constexpr int kPeelThreads = 256;
constexpr int kScanItems = 8;
constexpr int kWarps = kPeelThreads / 32;

struct PTask {
    uint32_t e1;
    uint32_t oa, la;  // probe list (shorter live list)
    uint32_t ob, lb;  // searched list
    uint32_t b;       // vertex owning the searched list
};

__device__ __forceinline__ PTask ptask(const DevGraph& g, uint32_t e1) {
    const uint2 p = g.el[e1];
    const uint32_t du = g.dl[p.x], dv = g.dl[p.y];
    PTask k;
    k.e1 = e1;
    if (du <= dv) { k.oa = g.off[p.x]; k.la = du; k.ob = g.off[p.y]; k.lb = dv; k.b = p.y; }
    else          { k.oa = g.off[p.y]; k.la = dv; k.ob = g.off[p.x]; k.lb = du; k.b = p.x; }
    return k;
}

__device__ __forceinline__ void reset_ctr(PhaseCtr* c) {
    c->work = 0;
    c->out_size = 0;
    c->alive_size = 0;
    c->min_s = 0xffffffffu;
    c->piece_head = 0;
    c->batch_head = 0;
}

// try_decrement, truss_parallel.cpp:49-63. Returns target if this thread moved it to the
// level (it then owns the append), else kNone.
__device__ __forceinline__ uint32_t try_dec(uint32_t* s, uint32_t* stamp, uint32_t level, uint32_t K,
                                            uint32_t e1, uint32_t target, uint32_t other,
                                            bool other_in_curr) {
    if (ld_relaxed(&s[target]) <= level) return kNone;   // :52
    if (other_in_curr && e1 >= other) return kNone;      // :53 ownership
    const uint32_t prev = atomicSub(&s[target], 1u);     // :54
    if (prev == level + 1) {                             // :55-57
        st_relaxed(&stamp[target], K + 1);
        return target;
    }
    if (prev <= level) atomicAdd(&s[target], 1u);        // :58-62 repair
    return kNone;
}

// One triangle probe of e1 (truss_parallel.cpp:80-88): x = item j of the probe list.
__device__ __forceinline__ void peel_probe(const DevGraph& g, uint32_t* s, uint32_t* stamp,
                                           uint32_t level, uint32_t K, uint32_t e1, uint32_t oa,
                                           uint32_t ob, uint32_t lb, uint32_t b, uint32_t j,
                                           uint32_t& out0, uint32_t& out1) {
    const uint32_t x = g.adj[oa + j];
    if (x == b) return;
    // (Searching b in N(x) when x's list is shorter was measured slower: the extra random
    // dl[x]/off[x] loads miss L2, while the top of N(b)'s search tree stays cached.)
    const uint32_t p = lower_bound_u32(g.adj + ob, lb, x);
    if (p >= lb || g.adj[ob + p] != x) return;
    const uint32_t ea = g.eid[oa + j], eb = g.eid[ob + p];
    const uint32_t sa = ld_relaxed(&stamp[ea]), sb = ld_relaxed(&stamp[eb]);
    if ((sa != 0 && sa < K) || (sb != 0 && sb < K)) return;  // :85 processed peer
    out0 = try_dec(s, stamp, level, K, e1, ea, eb, sb == K);  // :86
    out1 = try_dec(s, stamp, level, K, e1, eb, ea, sa == K);  // :87
}

// Append up to two targets per lane to next, one atomic per warp (appender.hpp:12-40).
__device__ __forceinline__ void emit(uint32_t o0, uint32_t o1, PhaseCtr* out, uint32_t* next) {
    const uint32_t p0 = warp_append(o0 != kNone, &out->out_size);
    if (o0 != kNone) next[p0] = o0;
    const uint32_t p1 = warp_append(o1 != kNone, &out->out_size);
    if (o1 != kNone) next[p1] = o1;
}

__device__ __forceinline__ unsigned long long shfl64(unsigned long long v, uint32_t src) {
    const uint32_t lo = __shfl_sync(kFull, static_cast<uint32_t>(v), src);
    const uint32_t hi = __shfl_sync(kFull, static_cast<uint32_t>(v >> 32), src);
    return (static_cast<unsigned long long>(hi) << 32) | lo;
}

// Block-wide exclusive scan of a u64 per thread; returns the exclusive prefix and sets
// `total`. All threads of the block must call.
__device__ __forceinline__ unsigned long long block_excl_scan64(unsigned long long v, unsigned long long& total) {
    __shared__ unsigned long long sh[kWarps];
    const uint32_t lane = lane_id(), wid = threadIdx.x >> 5;
    unsigned long long x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const unsigned long long t = shfl64(x, lane >= static_cast<uint32_t>(o) ? lane - o : lane);
        if (lane >= static_cast<uint32_t>(o)) x += t;
    }
    if (lane == 31) sh[wid] = x;
    __syncthreads();
    unsigned long long woff = 0, tot = 0;
#pragma unroll
    for (int w = 0; w < kWarps; w++) {
        const unsigned long long t = sh[w];
        if (w < static_cast<int>(wid)) woff += t;
        tot += t;
    }
    __syncthreads();
    total = tot;
    return woff + x - v;
}

// scan (truss_parallel.cpp:21-37) over the live-edge list A: survivors with s==level
// become curr (stamp K), the others are compacted into Aout and their minimum support is
// reduced for level skipping. Block-aggregated appends: 2 atomics per 2048 edges.
__device__ void phase_scan(uint32_t* s, uint32_t* stamp, uint32_t level, uint32_t K, const uint32_t* Ain,
                           uint32_t nA, bool implicit, uint32_t* Aout, uint32_t* curr, PhaseCtr* ph) {
    __shared__ uint32_t sh_c[kWarps], sh_a[kWarps];
    __shared__ uint32_t sh_bc, sh_ba;
    const uint32_t tid = threadIdx.x, lane = lane_id(), wid = tid >> 5;
    const uint64_t tile = uint64_t(kPeelThreads) * kScanItems;
    uint32_t local_min = 0xffffffffu;
    for (uint64_t t0 = uint64_t(blockIdx.x) * tile; t0 < nA; t0 += uint64_t(gridDim.x) * tile) {
        uint32_t es[kScanItems];
        uint32_t kind = 0;  // 2 bits per item: 1 = curr, 2 = alive
        uint32_t cc = 0, ca = 0;
#pragma unroll
        for (int k = 0; k < kScanItems; k++) {
            const uint64_t i = t0 + uint64_t(k) * kPeelThreads + tid;
            es[k] = 0;
            if (i < nA) {
                const uint32_t e = implicit ? static_cast<uint32_t>(i) : Ain[i];
                es[k] = e;
                if (ld_relaxed(&stamp[e]) == 0) {
                    const uint32_t sv = ld_relaxed(&s[e]);
                    if (sv == level) {
                        st_relaxed(&stamp[e], K);
                        kind |= 1u << (2 * k);
                        cc++;
                    } else {
                        kind |= 2u << (2 * k);
                        ca++;
                        local_min = sv < local_min ? sv : local_min;
                    }
                }
            }
        }
        const uint32_t ic = warp_incl_scan(cc), ia = warp_incl_scan(ca);
        if (lane == 31) { sh_c[wid] = ic; sh_a[wid] = ia; }
        __syncthreads();
        if (tid == 0) {
            uint32_t rc = 0, ra = 0;
            for (int w = 0; w < kWarps; w++) {
                uint32_t c = sh_c[w], a = sh_a[w];
                sh_c[w] = rc; sh_a[w] = ra;
                rc += c; ra += a;
            }
            sh_bc = rc ? atomicAdd(&ph->out_size, rc) : 0;
            sh_ba = ra ? atomicAdd(&ph->alive_size, ra) : 0;
        }
        __syncthreads();
        uint32_t pc = sh_bc + sh_c[wid] + ic - cc, pa = sh_ba + sh_a[wid] + ia - ca;
#pragma unroll
        for (int k = 0; k < kScanItems; k++) {
            const uint32_t f = (kind >> (2 * k)) & 3u;
            if (f == 1u) curr[pc++] = es[k];
            else if (f == 2u) Aout[pa++] = es[k];
        }
        __syncthreads();
    }
    for (int o = 16; o > 0; o >>= 1) local_min = min(local_min, __shfl_xor_sync(kFull, local_min, o));
    if (lane == 0 && local_min != 0xffffffffu) atomicMin(&ph->min_s, local_min);
}

__device__ __forceinline__ uint32_t chunk_len(uint32_t cs, uint32_t nchunks) {
    return (cs + nchunks - 1) / nchunks;
}

// Sub-level prep: block b owns curr chunk b; writes the chunk-local exclusive prefix of
// probe counts (min live degree of the two endpoints) and the chunk total.
__device__ void phase_prep(const DevGraph& g, const uint32_t* curr, uint32_t cs, unsigned long long* wpre,
                           unsigned long long* bsum) {
    const uint32_t CH = chunk_len(cs, gridDim.x);
    const uint64_t lo = uint64_t(blockIdx.x) * CH;
    const uint64_t hi = lo + CH < cs ? lo + CH : cs;
    unsigned long long run = 0;
    for (uint64_t t0 = lo; t0 < hi; t0 += kPeelThreads) {
        const uint64_t i = t0 + threadIdx.x;
        unsigned long long w = 0;
        if (i < hi) w = ptask(g, curr[i]).la;
        unsigned long long tot;
        const unsigned long long ex = block_excl_scan64(w, tot);
        if (i < hi) wpre[i] = run + ex;
        run += tot;
    }
    if (threadIdx.x == 0) bsum[blockIdx.x] = run;
}

// process_sublevel (truss_parallel.cpp:39-104) for curr[0..cs): the W probe items are cut
// into pieces of P items (P ~ W / (4 * #warps), >= 32), pulled by warps dynamically. A
// warp walks its piece 32 items per step; lane k holds task i+k (the curr edges whose
// items can fall in the 32-item window), and each lane finds its item's owner with a
// 5-step shuffle search over the tasks' start offsets.
__device__ void phase_process(const DevGraph& g, uint32_t* s, uint32_t* stamp, uint32_t level, uint32_t K,
                              const uint32_t* curr, uint32_t cs, const unsigned long long* wpre,
                              const unsigned long long* bsum, uint32_t nchunks, PhaseCtr* ph,
                              uint32_t* next) {
    __shared__ unsigned long long sboff[kMaxChunks + 1];
    // chunk offsets (exclusive scan of bsum), redundantly per block
    {
        const uint32_t per = (nchunks + kPeelThreads - 1) / kPeelThreads;
        const uint32_t c0 = threadIdx.x * per;
        unsigned long long loc = 0;
        for (uint32_t c = c0; c < c0 + per && c < nchunks; c++) loc += bsum[c];
        unsigned long long tot;
        unsigned long long run = block_excl_scan64(loc, tot);
        for (uint32_t c = c0; c < c0 + per && c < nchunks; c++) {
            sboff[c] = run;
            run += bsum[c];
        }
        if (threadIdx.x == 0) sboff[nchunks] = tot;
        __syncthreads();
    }
    const unsigned long long W = sboff[nchunks];
    if (W == 0) return;
    const uint32_t CH = chunk_len(cs, nchunks);
    const uint32_t nwarps = (gridDim.x * kPeelThreads) >> 5;
    unsigned long long P = (W + 4ull * nwarps - 1) / (4ull * nwarps);
    P = (P + 31) & ~31ull;
    if (P < 32) P = 32;
    const unsigned long long npieces = (W + P - 1) / P;
    const uint32_t lane = lane_id();

    while (true) {
        uint32_t p = 0;
        if (lane == 0) p = atomicAdd(&ph->piece_head, 1u);
        p = __shfl_sync(kFull, p, 0);
        if (p >= npieces) break;
        const unsigned long long x0 = p * P;
        const unsigned long long x1 = x0 + P < W ? x0 + P : W;
        // task containing x0: largest chunk c with sboff[c] <= x0, then largest i in chunk
        uint32_t clo = 0, chi = nchunks;  // sboff[clo] <= x0 < sboff[chi]
        while (chi - clo > 1) {
            const uint32_t mid = (clo + chi) >> 1;
            if (sboff[mid] <= x0) clo = mid; else chi = mid;
        }
        uint32_t ilo = clo * CH, ihi = min(cs, (clo + 1) * CH);
        const unsigned long long rel = x0 - sboff[clo];
        while (ihi - ilo > 1) {
            const uint32_t mid = (ilo + ihi) >> 1;
            if (wpre[mid] <= rel) ilo = mid; else ihi = mid;
        }
        uint32_t i = ilo;
        // Lanes hold tasks i..i+31 (starts st); `end_held` = start of task i+32. A step
        // covers the items of held tasks only, so any mix of task sizes is handled.
        uint32_t held = kNone;
        PTask k{0, 0, 0, 0, 0, 0};
        unsigned long long st = ~0ull, end_held = ~0ull;
        for (unsigned long long base = x0; base < x1;) {
            if (held != i) {
                const uint32_t t = i + lane;
                if (t < cs) { k = ptask(g, curr[t]); st = sboff[t / CH] + wpre[t]; }
                else { st = ~0ull; }
                unsigned long long s32 = ~0ull;
                if (lane == 31 && t + 1 < cs) s32 = sboff[(t + 1) / CH] + wpre[t + 1];
                end_held = shfl64(s32, 31);
                held = i;
            }
            const unsigned long long limit = x1 < end_held ? x1 : end_held;
            const uint32_t relk = st <= base ? 0u : (st - base > 0xffffffffull ? 0xffffffffu : static_cast<uint32_t>(st - base));
            const uint32_t own = warp_owner(relk, lane);
            const unsigned long long so = shfl64(st, own);
            const uint32_t e1 = __shfl_sync(kFull, k.e1, own);
            const uint32_t oa = __shfl_sync(kFull, k.oa, own);
            const uint32_t ob = __shfl_sync(kFull, k.ob, own);
            const uint32_t lb = __shfl_sync(kFull, k.lb, own);
            const uint32_t bv = __shfl_sync(kFull, k.b, own);
            const unsigned long long x = base + lane;
            uint32_t o0 = kNone, o1 = kNone;
            if (x < limit) peel_probe(g, s, stamp, level, K, e1, oa, ob, lb, bv, static_cast<uint32_t>(x - so), o0, o1);
            emit(o0, o1, ph, next);
            const unsigned long long nb = base + 32 < limit ? base + 32 : limit;
            i = (nb >= end_held) ? i + 32 : i + warp_owner(relk, static_cast<uint32_t>(nb - base));
            base = nb;
        }
    }
}

// Adjacency compaction (between levels): drop processed edges (0 < stamp < K) from every
// live list, in place and order-preserving, and shrink dl. Lists longer than kBigList are
// compacted by a whole block (block scan per 1024-entry chunk), the rest by one warp
// (ballot per 32 entries). Processed edges are skipped by every probe anyway (:85), so
// this only removes work; triangle sets seen by the peel are unchanged.
constexpr uint32_t kBigList = 2048;
constexpr unsigned long long kCompactNum = 4, kCompactDen = 5;  // compact at <= 80% live

__device__ __forceinline__ bool processed_stamp(uint32_t st, uint32_t K) { return st != 0 && st < K; }

// Pass 1 (long lists). Must be separated from pass 2 by a grid barrier: pass 1 shrinks dl,
// which would otherwise let pass 2 see a list being compacted as "short".
__device__ void phase_compact_long(const DevGraph& g, const uint32_t* stamp, uint32_t K) {
    __shared__ uint32_t sh_big[kPeelThreads], sh_nbig;
    // 1) long lists: one block each (found per 256-vertex tile)
    for (uint64_t u0 = uint64_t(blockIdx.x) * kPeelThreads; u0 < g.n; u0 += uint64_t(gridDim.x) * kPeelThreads) {
        if (threadIdx.x == 0) sh_nbig = 0;
        __syncthreads();
        const uint64_t uu = u0 + threadIdx.x;
        if (uu < g.n && g.dl[uu] > kBigList) sh_big[atomicAdd(&sh_nbig, 1u)] = static_cast<uint32_t>(uu);
        __syncthreads();
        const uint32_t nbig = sh_nbig;
        for (uint32_t bi = 0; bi < nbig; bi++) {
        const uint32_t u = sh_big[bi];
        const uint32_t len = g.dl[u];
        uint32_t* adj = g.adj + g.off[u];
        uint32_t* eid = g.eid + g.off[u];
        unsigned long long wp = 0;
        for (uint32_t c = 0; c < len; c += kPeelThreads * 4) {
            uint32_t a[4], e[4];
            uint32_t keep = 0, cnt = 0;
#pragma unroll
            for (int q = 0; q < 4; q++) {
                const uint32_t idx = c + threadIdx.x * 4 + q;  // 4 consecutive: order kept
                a[q] = 0;
                e[q] = 0;
                if (idx < len) {
                    a[q] = adj[idx];
                    e[q] = eid[idx];
                    if (!processed_stamp(ld_relaxed(&stamp[e[q]]), K)) { keep |= 1u << q; cnt++; }
                }
            }
            unsigned long long tot;
            unsigned long long pos = wp + block_excl_scan64(cnt, tot);
#pragma unroll
            for (int q = 0; q < 4; q++)
                if (keep & (1u << q)) { adj[pos] = a[q]; eid[pos] = e[q]; pos++; }
            wp += tot;
            __syncthreads();
        }
        if (threadIdx.x == 0) g.dl[u] = static_cast<uint32_t>(wp);
        }
        __syncthreads();
    }
}

// Pass 2 (short lists): one warp each, ballot compaction in list order.
__device__ void phase_compact_short(const DevGraph& g, const uint32_t* stamp, uint32_t K) {
    const uint32_t lane = lane_id();
    const uint32_t gw = (blockIdx.x * kPeelThreads + threadIdx.x) >> 5, nw = (gridDim.x * kPeelThreads) >> 5;
    for (uint32_t u = gw; u < g.n; u += nw) {
        const uint32_t len = g.dl[u];
        if (len == 0 || len > kBigList) continue;
        uint32_t* adj = g.adj + g.off[u];
        uint32_t* eid = g.eid + g.off[u];
        uint32_t wp = 0;
        for (uint32_t c = 0; c < len; c += 32) {
            const uint32_t idx = c + lane;
            uint32_t a = 0, e = 0;
            bool keep = false;
            if (idx < len) {
                a = adj[idx];
                e = eid[idx];
                keep = !processed_stamp(ld_relaxed(&stamp[e]), K);
            }
            const uint32_t bal = __ballot_sync(kFull, keep);
            if (keep) {
                const uint32_t pos = wp + __popc(bal & lanemask_lt());
                adj[pos] = a;
                eid[pos] = e;
            }
            wp += __popc(bal);
        }
        if (lane == 0) g.dl[u] = wp;
    }
}

__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

__device__ __forceinline__ uint32_t vload(const uint32_t* p) { return *reinterpret_cast<const volatile uint32_t*>(p); }

// The whole truss_parallel level loop (truss_parallel.cpp:119-144) in one launch.
__global__ void __launch_bounds__(kPeelThreads, 4) k_peel(DevGraph g, PeelBufs pb) {
    cg::grid_group grid = cg::this_grid();
    PeelCtl* ctl = pb.ctl;
    const bool leader = blockIdx.x == 0 && threadIdx.x == 0;
    uint32_t j = 0, level = 0, K = 1, nA = g.m, ai = 0, li = 0, live_at_compact = g.m;
    bool implicit = true;
    unsigned long long t_prev = leader ? gtimer() : 0;
    while (true) {
        // ---- scan at `level` (one grid barrier)
        if (leader) { reset_ctr(&ctl->ph[(j + 1) % 3]); ctl->scans++; }
        phase_scan(pb.s, pb.stamp, level, K, pb.A[ai], nA, implicit, pb.A[ai ^ 1], pb.L[li], &ctl->ph[j % 3]);
        grid.sync();
        if (leader) { const unsigned long long t = gtimer(); ctl->scan_ns += t - t_prev; t_prev = t; }
        j++;
        const PhaseCtr* r = &ctl->ph[(j - 1) % 3];
        uint32_t cs = vload(&r->out_size);
        nA = vload(&r->alive_size);
        const uint32_t mins = vload(&r->min_s);
        ai ^= 1;
        implicit = false;
        if (cs == 0) {
            if (nA == 0) break;
            level = mins;  // skip empty levels
            continue;
        }
        // ---- compaction once the live edge count fell below kCompactFrac of the last one
        if (level > 0 && (static_cast<unsigned long long>(cs) + nA) * kCompactDen <
                             static_cast<unsigned long long>(live_at_compact) * kCompactNum) {
            if (leader) { reset_ctr(&ctl->ph[(j + 1) % 3]); ctl->compactions++; }
            phase_compact_long(g, pb.stamp, K);
            grid.sync();
            phase_compact_short(g, pb.stamp, K);
            grid.sync();
            j++;
            live_at_compact = cs + nA;
        }
        // ---- sub-levels: prep + process (two grid barriers each; level 0 one)
        while (true) {
            if (leader) {
                if (level < pb.nsl_cap) pb.nsl[level]++; else ctl->overflow = 1;
                ctl->sublevels++;
                ctl->levels_len = level + 1;
                reset_ctr(&ctl->ph[(j + 1) % 3]);
            }
            if (level > 0) {  // level 0: s[e1] == 0 bounds its live triangles to none
                phase_prep(g, pb.L[li], cs, pb.wpre, pb.bsum);
                grid.sync();
                phase_process(g, pb.s, pb.stamp, level, K, pb.L[li], cs, pb.wpre, pb.bsum, gridDim.x,
                              &ctl->ph[j % 3], pb.L[li ^ 1]);
            }
            grid.sync();
            if (leader) { const unsigned long long t = gtimer(); ctl->proc_ns += t - t_prev; t_prev = t; }
            j++;
            K++;
            r = &ctl->ph[(j - 1) % 3];
            cs = vload(&r->out_size);
            li ^= 1;
            if (cs == 0) break;
        }
        level++;
    }
    if (leader) ctl->final_stamp = K;
}

__global__ void k_peel_init(const uint32_t* __restrict__ off, uint32_t n, uint32_t* __restrict__ dl,
                            PeelCtl* ctl) {
    for (uint32_t u = blockIdx.x * blockDim.x + threadIdx.x; u < n; u += gridDim.x * blockDim.x)
        dl[u] = off[u + 1] - off[u];
    if (blockIdx.x == 0 && threadIdx.x < 3) reset_ctr(&ctl->ph[threadIdx.x]);
}

__global__ void k_finalize(const uint32_t* __restrict__ s, uint32_t m, uint32_t* __restrict__ truss,
                           PeelCtl* ctl) {
    uint32_t mx = 0;
    for (uint32_t e = blockIdx.x * blockDim.x + threadIdx.x; e < m; e += gridDim.x * blockDim.x) {
        const uint32_t t = s[e] + 2;  // truss_parallel.cpp:146-148
        truss[e] = t;
        mx = t > mx ? t : mx;
    }
    for (int o = 16; o > 0; o >>= 1) mx = max(mx, __shfl_xor_sync(kFull, mx, o));
    if (lane_id() == 0 && mx) atomicMax(&ctl->t_max, mx);
}

// ---- step functions on reference-style flag arrays (tests/test_truss_parallel.cpp) ----
__global__ void k_step_stamps(const uint8_t* __restrict__ processed, const uint8_t* __restrict__ in_curr,
                              uint32_t m, uint32_t* __restrict__ stamp, PeelCtl* ctl) {
    for (uint32_t e = blockIdx.x * blockDim.x + threadIdx.x; e < m; e += gridDim.x * blockDim.x)
        stamp[e] = processed[e] ? 1u : ((in_curr && in_curr[e]) ? 2u : 0u);
    if (blockIdx.x == 0 && threadIdx.x < 3) reset_ctr(&ctl->ph[threadIdx.x]);
}

__global__ void __launch_bounds__(kPeelThreads) k_step_scan(PeelBufs pb, uint32_t m, uint32_t level) {
    phase_scan(pb.s, pb.stamp, level, 2, pb.A[0], m, true, pb.A[1], pb.L[0], &pb.ctl->ph[0]);
}

__global__ void k_step_scan_flags(const uint32_t* __restrict__ curr, PeelCtl* ctl, uint8_t* in_curr) {
    const uint32_t cs = ctl->ph[0].out_size;
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < cs; i += gridDim.x * blockDim.x)
        in_curr[curr[i]] = 1;
}

__global__ void __launch_bounds__(kPeelThreads) k_step_prep(DevGraph g, PeelBufs pb, uint32_t cs) {
    phase_prep(g, pb.L[0], cs, pb.wpre, pb.bsum);
}

// Hand-built states may break the level-0 invariant, so the step form always probes.
__global__ void __launch_bounds__(kPeelThreads) k_step_process(DevGraph g, PeelBufs pb, uint32_t cs, uint32_t level,
                                                               uint32_t nchunks) {
    phase_process(g, pb.s, pb.stamp, level, 2, pb.L[0], cs, pb.wpre, pb.bsum, nchunks, &pb.ctl->ph[1], pb.L[1]);
}

// Epilogue (truss_parallel.cpp:97-102) + in_next flags for the appended edges.
__global__ void k_step_process_flags(const uint32_t* __restrict__ curr, uint32_t cs,
                                     const uint32_t* __restrict__ next, PeelCtl* ctl, uint8_t* in_curr,
                                     uint8_t* in_next, uint8_t* processed) {
    const uint32_t ns = ctl->ph[1].out_size;
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < cs || i < ns; i += gridDim.x * blockDim.x) {
        if (i < cs) { processed[curr[i]] = 1; in_curr[curr[i]] = 0; }
        if (i < ns) in_next[next[i]] = 1;
    }
}

}  // namespace

cudaError_t launch_peel(const DevGraph& g, const PeelBufs& p, int sm_count, cudaStream_t st,
                        uint32_t* launches) {
    cudaError_t err = cudaMemsetAsync(p.ctl, 0, sizeof(PeelCtl), st);
    if (err != cudaSuccess) return err;
    if ((err = cudaMemsetAsync(p.nsl, 0, size_t(p.nsl_cap) * sizeof(uint32_t), st)) != cudaSuccess) return err;
    if (g.m == 0) return cudaSuccess;
    if ((err = cudaMemsetAsync(p.stamp, 0, size_t(g.m) * sizeof(uint32_t), st)) != cudaSuccess) return err;
    k_peel_init<<<148 * 4, 256, 0, st>>>(g.off, g.n, g.dl, p.ctl);
    int per_sm = 0;
    err = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_peel, kPeelThreads, 0);
    if (err != cudaSuccess) return err;
    if (per_sm < 1) return cudaErrorLaunchOutOfResources;
    unsigned blocks = static_cast<unsigned>(sm_count * per_sm);
    if (blocks > kMaxChunks) blocks = kMaxChunks;
    DevGraph gg = g;
    PeelBufs pp = p;
    void* args[] = {&gg, &pp};
    err = cudaLaunchCooperativeKernel(reinterpret_cast<void*>(k_peel), dim3(blocks), dim3(kPeelThreads), args, 0, st);
    (*launches) += 2;
    return err;
}

cudaError_t launch_finalize(const uint32_t* s, uint32_t m, uint32_t* truss, PeelCtl* ctl, cudaStream_t st,
                            uint32_t* launches) {
    if (m == 0) return cudaSuccess;
    k_finalize<<<148 * 4, 256, 0, st>>>(s, m, truss, ctl);
    (*launches)++;
    return cudaGetLastError();
}

cudaError_t launch_step_scan(const DevGraph& g, const PeelBufs& p, uint32_t level, const uint8_t* processed,
                             uint8_t* in_curr, int sm_count, cudaStream_t st) {
    k_step_stamps<<<sm_count * 2, 256, 0, st>>>(processed, nullptr, g.m, p.stamp, p.ctl);
    k_step_scan<<<sm_count, kPeelThreads, 0, st>>>(p, g.m, level);
    k_step_scan_flags<<<sm_count, 256, 0, st>>>(p.L[0], p.ctl, in_curr);
    return cudaGetLastError();
}

cudaError_t launch_step_process(const DevGraph& g, const PeelBufs& p, uint32_t level, uint32_t curr_size,
                                uint8_t* in_curr, uint8_t* in_next, uint8_t* processed, int sm_count,
                                cudaStream_t st) {
    const uint32_t nchunks = static_cast<uint32_t>(sm_count);
    k_peel_init<<<sm_count, 256, 0, st>>>(g.off, g.n, g.dl, p.ctl);
    k_step_stamps<<<sm_count * 2, 256, 0, st>>>(processed, in_curr, g.m, p.stamp, p.ctl);
    k_step_prep<<<nchunks, kPeelThreads, 0, st>>>(g, p, curr_size);
    k_step_process<<<sm_count * 2, kPeelThreads, 0, st>>>(g, p, curr_size, level, nchunks);
    k_step_process_flags<<<sm_count, 256, 0, st>>>(p.L[0], curr_size, p.L[1], p.ctl, in_curr, in_next, processed);
    return cudaGetLastError();
}

}  // namespace tdg
