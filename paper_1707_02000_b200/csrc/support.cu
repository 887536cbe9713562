// support.cu — per-edge triangle counts (the support pass).
//
// Reference: support_am4, /root/reference/proj/src/triangle.cpp:26-61 (ordered pivot with a
// dense per-thread mark array X[n] and three relaxed fetch_adds per triangle). B200
// design: every triangle {a,b,c} with a < b < c in the degree order (d, id) is found
// exactly once, at oriented edge a->b, as c in N+(a) ∩ N+(b) (the oriented lists are
// sorted subsequences of the CSR lists, at most sqrt(2m) long). Each oriented edge is a
// task of the shared probe engine (intersect.cuh): the shorter oriented list is walked
// with coalesced loads and every element is binary-searched in the longer one; tasks are
// ordered by the owner of the longer list so its searches hit L1 (ncu on C5: the
// unordered form read 6.8 TB from DRAM for a 2 GB structure); work is balanced over all
// warps. Per triangle: the (a,b) count is aggregated across
// the warp with __match_any_sync and one atomicAdd per group; the other two edges get one
// atomicAdd each. No X[n] scratch.

#include <cstdlib>

#include "intersect.cuh"
#include "tdg_kernels.h"

namespace tdg {

namespace {

constexpr int kThreads = 256;

// Task t = slot j of owner x (build.cu k_svalid): the oriented edge {x, y} whose longer N+
// list is x's. N+(y) (min(d+) elements) is read as 16-byte QUADS — the work items of the
// engine are the aligned 4-element groups that cover the list, one LDG.E.128 per item — and
// every element is looked up in N+(x); tasks are grouped by x. Oriented lists are at most
// sqrt(2m) < 2^16 long, so both lengths share one word: lb = d+(y) << 16 | d+(x).
__device__ __forceinline__ ITask otask(const DevGraph& g, uint32_t t) {
    const uint32_t j = g.stask[t], x = g.sx[t], y = g.adj[j];
    ITask k;
    k.id = g.eid[j];
    k.oa = g.opos[y];
    k.ob = g.opos[x];
    const uint32_t ly = g.opos[y + 1] - k.oa, lx = g.opos[x + 1] - k.ob;
    TDG_CHECK(ly < 65536u && lx < 65536u);
    k.lb = (ly << 16) | lx;
    return k;
}
// Quads covering the list [oa, oa + len) of a 16-byte-aligned array.
__device__ __forceinline__ uint32_t quads_of(uint32_t oa, uint32_t len) {
    return len ? ((oa & 3u) + len + 3u) >> 2 : 0u;
}

// Edge ids are internal (build.cu launch_internal_ids): an edge's id IS its oriented slot
// (position in the N+ arrays). The owner-side slots of a task group are one contiguous
// N+(x) range and the probe-side slots of one task are consecutive, so the per-triangle
// atomics stay out of DRAM (reference-id-indexed atomics were random 2 GB read-modify-writes
// at C5).
// Own-edge counts of one engine step: hq = this lane's hits in its quad of task `id`; one
// atomic per step when every hit belongs to one task (the common case in long lists), else
// one per group of lanes sharing a task (hq <= 4: three bit-plane ballots give a group's sum).
__device__ __forceinline__ void count_own(uint32_t* s, uint32_t id, uint32_t hq) {
    const uint32_t hm = __ballot_sync(kFull, hq != 0);
    if (!hm) return;
    const uint32_t leader = __ffs(hm) - 1;
    const uint32_t id0 = __shfl_sync(kFull, id, leader);
    if (__all_sync(kFull, hq == 0 || id == id0)) {
        const uint32_t tot = __reduce_add_sync(kFull, hq);
        if (lane_id() == leader) atomicAdd(&s[id0], tot);
        return;
    }
    if (hq) {
        const uint32_t grp = __match_any_sync(hm, id);
        const uint32_t b0 = __ballot_sync(hm, hq & 1u), b1 = __ballot_sync(hm, hq & 2u), b2 = __ballot_sync(hm, hq & 4u);
        const uint32_t sum = __popc(b0 & grp) + 2u * __popc(b1 & grp) + 4u * __popc(b2 & grp);
        if (lane_id() == static_cast<uint32_t>(__ffs(grp) - 1)) atomicAdd(&s[id], sum);
    }
}

#ifndef TDG_SUP_U
#define TDG_SUP_U 2  // quads per lane per engine step in the support pass (8 probes per lane)
#endif
// Search form (segments too small to pay for a table): every element of the quad is
// binary-searched in N+(x) in global memory.
struct SupportPolicy {
    const DevGraph& g;
    uint32_t* s;
    const uint32_t* elems;
    static constexpr bool kFast = true;
    static constexpr bool kRunForm = true;
    static constexpr int kUnroll = TDG_SUP_U;
    __device__ ITask load(uint32_t t) const { return otask(g, t); }
    template <int U>
    __device__ void run(const bool (&act)[U], const ITask (&ko)[U], const uint32_t (&ja)[U]) const {
        uint4 v[U];
        uint32_t base[U];
#pragma unroll
        for (int q = 0; q < U; q++) {
            base[q] = (ko[q].oa & ~3u) + 4u * ja[q];
            v[q] = act[q] ? __ldg(reinterpret_cast<const uint4*>(elems + base[q])) : make_uint4(0, 0, 0, 0);
        }
#pragma unroll
        for (int q = 0; q < U; q++) {
            const uint32_t c[4] = {v[q].x, v[q].y, v[q].z, v[q].w};
            const uint32_t ly = ko[q].lb >> 16, lx = ko[q].lb & 0xffffu;
            uint32_t hq = 0;
#pragma unroll
            for (int e = 0; e < 4; e++) {
                const uint32_t idx = base[q] + e;
                if (act[q] && idx - ko[q].oa < ly) {  // (unsigned: also drops idx < oa)
                    const uint32_t p = lower_bound_u32(g.oadj + ko[q].ob, lx, c[e]);
                    if (p < lx && g.oadj[ko[q].ob + p] == c[e]) {
                        atomicAdd(&s[idx], 1u);
                        atomicAdd(&s[ko[q].ob + p], 1u);
                        hq++;
                    }
                }
            }
            count_own(s, ko[q].id, hq);
        }
    }
};

// ---- owner-table form. A block takes a piece of the work axis and walks its owner
// segments (the tasks of one owner x are contiguous, [sbeg[x], sbeg[x+1])). For a segment
// with enough work, N+(x) is loaded once into a shared-memory hash table and the block's 8
// warps split the segment's items evenly; each probe is then a quarter of a coalesced
// 16-byte N+(y) load plus ~1 shared-memory access instead of a log2(d+(x)) chain of L1
// loads. Hub owners whose list exceeds the table (d+ > kSupCap) run several passes, one per
// kSupCap-key slice of the sorted N+(x); a pass skips the elements outside its key range.
// Segments too small to pay for the table are batched and searched in global memory.
// Two block geometries, chosen per graph on the device (k_support_prep measures the share of
// the probe work whose owner list is longer than kSupBigDeg; every block of both launches reads
// the same verdict and the other launch exits at once):
//  * 256 threads x 4096-slot table, 4 blocks/SM: best when owner lists are short (C3, C4);
//  * 512 threads x 8192-slot table, 2 blocks/SM (same warps per SM): owners of 1024 < d+ <= 2048
//    keep the table at load <= 1/4 (fewer bucket walks) and d+ up to 6144 needs no slicing —
//    C5 support 731 -> 680 ms, but C3 55 -> 61 ms (its segments are too small to fill 16 warps).
#ifndef TDG_SUP_TAB
#define TDG_SUP_TAB 4096  // shared-memory table slots (4 B key + 2 B position + 2 B counter) of the small geometry
#endif
constexpr uint32_t kSupTab = TDG_SUP_TAB;
constexpr uint32_t kSupBigDeg = kSupTab / 4;  // owner lists longer than this load a small-geometry table above 1/4
#ifndef TDG_SUP_BIG_PCT
#define TDG_SUP_BIG_PCT 50  // big geometry when more than this share (%) of the probe work has such an owner (101: never)
#endif
#ifndef TDG_SUP_LOAD
#define TDG_SUP_LOAD 4  // table slots per key when the table is not full size (C5: 2 -> 4: 1089 -> 1047 ms)
#endif
constexpr size_t sup_smem(uint32_t tab) { return size_t(tab) * (sizeof(uint32_t) + 2 * sizeof(uint16_t)); }
static_assert(kSupTab % 4 == 0 && 3 * (2 * kSupTab) / 4 < 65536, "bucketed owner table: u16 positions and counters");
#ifndef TDG_SUP_SEGMIN
#define TDG_SUP_SEGMIN 512u  // a segment gets a table if its probes * SEGDIV >= max(d+(x), SEGMIN)
#endif
#ifndef TDG_SUP_SEGDIV
#define TDG_SUP_SEGDIV 1u
#endif
#ifndef TDG_SUP_MINB
#define TDG_SUP_MINB 4  // 64 registers: the 8-probe-per-lane quad step needs them (C5: MINB 5 797 ms, 4 774 ms, 3 878 ms)
#endif
#ifndef TDG_SUP_THREADS
#define TDG_SUP_THREADS 256  // threads of a k_support_tab block (the unit that shares one owner table)
#endif
constexpr int kTabThreads = TDG_SUP_THREADS;

// Shared-memory table slot of key c: multiplicative (Fibonacci) hashing, top bits of
// c * 2^32/phi — one multiply and a shift instead of hmix's five-step mix (the support pass
// is issue-bound).
__device__ __forceinline__ uint32_t tab_hash(uint32_t c, uint32_t mask) {
    return (c * 0x9E3779B1u) >> (__clz(mask) & 31u);
}

// Owner table in shared memory, BUCKETED: 4-key buckets (one 16-byte LDS.128 compares four
// keys), linear probing over buckets, keys claimed in slot order inside a bucket (so a
// bucket whose last slot is empty ends a miss). A hit bumps the slot's 16-bit counter
// (packed pairs, one 32-bit shared-memory atomic; a slot is hit at most once per task of the
// segment, <= d+(x) < 2^16 times); the counters are flushed to s through the slots' u16
// positions in N+(x) once per segment, so a triangle costs one global atomic, not two.
template <bool kRange>
struct SupportTabPolicy {
    const DevGraph& g;
    uint32_t* s;
    const uint32_t* elems;
    const uint4* keys4;      // nb buckets of 4 keys
    uint32_t* cnt2;          // 2 * nb words: u16 hit counters of the 4 * nb slots
    uint32_t cnt2_saddr;     // cnt2 as a shared-window address (for red.shared)
    uint32_t bmask;          // nb - 1
    uint32_t kmin, kmax;     // key range of this pass (kRange)
    static constexpr bool kFast = true;
    static constexpr bool kRunForm = true;
    static constexpr int kUnroll = TDG_SUP_U;
    __device__ ITask load(uint32_t t) const { return otask(g, t); }
    // One-hot match mask of key c in a bucket's key vector (keys are unique: at most one bit).
    // Four compares folded into a mask: no early-exit branch chain (lanes stay converged).
    static __device__ __forceinline__ uint32_t onehot(const uint4& kv, uint32_t c) {
        return (kv.x == c ? 1u : 0u) | (kv.y == c ? 2u : 0u) | (kv.z == c ? 4u : 0u) | (kv.w == c ? 8u : 0u);
    }
    // The two counts of a hit as PREDICATED reductions (no divergent branch around them): the
    // probe-side edge's global counter and the owner-side slot's shared-memory u16 counter.
    static __device__ __forceinline__ void count_hit(bool hit, uint32_t* gs, uint32_t saddr, uint32_t sval) {
        asm volatile(
            "{\n\t.reg .pred p;\n\tsetp.ne.u32 p, %0, 0;\n\t"
            "@p red.global.add.u32 [%1], 1;\n\t"
            "@p red.shared.add.u32 [%2], %3;\n\t}"
            ::"r"(static_cast<uint32_t>(hit)), "l"(gs), "r"(saddr), "r"(sval)
            : "memory");
    }
    template <int U>
    __device__ void run(const bool (&act)[U], const ITask (&ko)[U], const uint32_t (&ja)[U]) const {
        uint4 v[U];
        uint32_t base[U];
#pragma unroll
        for (int q = 0; q < U; q++) {
            base[q] = (ko[q].oa & ~3u) + 4u * ja[q];
            TDG_CHECK(!act[q] || uint64_t(base[q]) + 3 < uint64_t(g.m) + 4);
            v[q] = act[q] ? __ldg(reinterpret_cast<const uint4*>(elems + base[q])) : make_uint4(0, 0, 0, 0);
        }
#pragma unroll
        for (int q = 0; q < U; q++) {
            const uint32_t c[4] = {v[q].x, v[q].y, v[q].z, v[q].w};
            const uint32_t ly = ko[q].lb >> 16;
            uint32_t b[4];
            uint4 kv[4];
#pragma unroll
            for (int e = 0; e < 4; e++) {  // the four home buckets, loaded together
                b[e] = tab_hash(c[e], bmask);
                kv[e] = keys4[b[e]];
            }
            uint32_t hq = 0;
#pragma unroll
            for (int e = 0; e < 4; e++) {
                const uint32_t idx = base[q] + e;
                bool ok = act[q] && idx - ko[q].oa < ly;  // (unsigned: also drops idx < oa)
                if (kRange) ok = ok && c[e] >= kmin && c[e] <= kmax;
                uint32_t oh = onehot(kv[e], c[e]), bb = b[e];
                if (ok && oh == 0u && kv[e].w != kHEmpty) {  // home bucket full (rare at load <= 1/4): walk on
                    uint4 k2;
                    do {
                        bb = (bb + 1) & bmask;
                        k2 = keys4[bb];
                        oh = onehot(k2, c[e]);
                    } while (oh == 0u && k2.w != kHEmpty);
                }
                const bool hit = ok && oh != 0u;
                const uint32_t sl = 4u * bb + ((__ffs(oh) - 1) & 3u);  // slot of the match (any in-table value if !hit)
                count_hit(hit, &s[idx], cnt2_saddr + ((sl >> 1) << 2), 1u << ((sl & 1u) << 4));
                hq += hit ? 1u : 0u;
            }
            count_own(s, ko[q].id, hq);
        }
    }
};

// Last task t in [lo, hi) with start(t) <= x.
__device__ __forceinline__ uint32_t task_in(unsigned long long x, uint32_t lo, uint32_t hi,
                                            const unsigned long long* wpre, const unsigned long long* sboff,
                                            uint32_t CH) {
    while (hi - lo > 1) {
        const uint32_t mid = (lo + hi) >> 1;
        if (sboff[mid / CH] + wpre[mid] <= x) lo = mid; else hi = mid;
    }
    return lo;
}

// kBig: 0 = the small geometry, 1 = the big one (twice the threads and table slots, half the blocks).
template <int kBig>
__global__ void __launch_bounds__(kTabThreads << kBig, TDG_SUP_MINB >> kBig) k_support_tab(
    DevGraph g, uint32_t* __restrict__ s, const unsigned long long* wpre, const unsigned long long* bsum,
    uint32_t nchunks, SupportCtl* ctl, uint32_t shard, uint32_t nshards, int force) {
    constexpr int kTabThreads = tdg::kTabThreads << kBig;
    constexpr uint32_t kSupTab = tdg::kSupTab << kBig;
    constexpr uint32_t kSupCap = 3 * kSupTab / 4;  // keys per table at the full-size load of 3/4
    constexpr uint32_t kSupWarps = kTabThreads / 32;
    extern __shared__ uint4 tab_keys4[];  // kSupTab keys, then kSupTab u16 positions, then kSupTab u16 counters
    __shared__ unsigned long long sboff[kMaxChunks + 1];
    __shared__ uint32_t sh_p;
    const unsigned long long W = chunk_offsets<kTabThreads>(bsum, nchunks, sboff);
    if (W == 0) return;
    // the geometry of this graph (k_support_prep's tally; force: diagnostic override)
    const bool big = force >= 0 ? force != 0 : ctl->big_work * 100ull > W * static_cast<unsigned long long>(TDG_SUP_BIG_PCT);
    if (big != (kBig == 1)) return;
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        ctl->work_items = W;
        ctl->big_geometry = kBig;
    }
    // Shard `shard` of `nshards` (the support pass shards with no exchange but a
    // final sum) owns the contiguous stretch [Wlo, Whi) of the work axis: equal probe work per
    // shard whatever the degree skew; a shard boundary cuts a task like a piece boundary does.
    const unsigned long long Wlo = W / nshards * shard + W % nshards * shard / nshards;
    const unsigned long long Whi = W / nshards * (shard + 1) + W % nshards * (shard + 1) / nshards;
    if (Whi == Wlo) return;
    const uint32_t m = g.m, CH = chunk_len(m, nchunks);
    const uint32_t wid = threadIdx.x >> 5;
    unsigned long long PS = (Whi - Wlo + 4ull * gridDim.x - 1) / (4ull * gridDim.x);
    PS = PS < 1024 ? 1024 : PS;
    const unsigned long long npieces = (Whi - Wlo + PS - 1) / PS;
    auto start = [&](uint32_t t) -> unsigned long long { return t < m ? sboff[t / CH] + wpre[t] : W; };
    uint32_t* keys = reinterpret_cast<uint32_t*>(tab_keys4);
    uint16_t* tpos = reinterpret_cast<uint16_t*>(keys + kSupTab);
    uint32_t* cnt2 = reinterpret_cast<uint32_t*>(tpos + kSupTab);
    const uint32_t cnt2_saddr = static_cast<uint32_t>(__cvta_generic_to_shared(cnt2));
    SupportPolicy SP{g, s, g.oadj};
    while (true) {
        if (threadIdx.x == 0) sh_p = atomicAdd(&ctl->piece_head, 1u);
        __syncthreads();
        const uint32_t p = sh_p;
        __syncthreads();
        if (p >= npieces) break;
        const unsigned long long x0 = Wlo + p * PS, x1 = x0 + PS < Whi ? x0 + PS : Whi;
        uint32_t i = task_at(x0, m, wpre, sboff, nchunks, CH);
        unsigned long long base = x0;
        while (base < x1) {
            // batch of segments searched in global memory, up to the next table segment
            uint32_t j = i, x = 0, dp = 0, tend = 0;
            unsigned long long bend = base, send = 0;
            bool table = false;
            while (bend < x1) {
                x = g.sx[j];
                tend = g.sbeg[x + 1];
                send = start(tend);
                send = send < x1 ? send : x1;
                dp = g.opos[x + 1] - g.opos[x];
                // (items are quads: ~4 probes each; a hub pays one pass per kSupCap keys)
                table = (send - bend) * 4u * TDG_SUP_SEGDIV >= (dp > TDG_SUP_SEGMIN ? dp : TDG_SUP_SEGMIN);
                if (table) break;
                bend = send;
                j = tend;
            }
            if (bend > base) {
                if (threadIdx.x == 0) atomicAdd(&ctl->search_items, bend - base);
                const unsigned long long w0 = base + (bend - base) * wid / kSupWarps;
                const unsigned long long w1 = base + (bend - base) * (wid + 1) / kSupWarps;
                if (w0 < w1) run_items(SP, w0, w1, task_in(w0, i, j, wpre, sboff, CH), m, wpre, sboff, CH);
            }
            if (!table) break;  // bend == x1
            // table segment: owner x, tasks [j, tend), items [bend, send)
            const uint32_t o = g.opos[x];
            const unsigned long long w0 = bend + (send - bend) * wid / kSupWarps;
            const unsigned long long w1 = bend + (send - bend) * (wid + 1) / kSupWarps;
            const uint32_t t0 = w0 < w1 ? task_in(w0, j, tend, wpre, sboff, CH) : 0u;
            if (threadIdx.x == 0) {
                atomicAdd(&ctl->tab_elems, static_cast<unsigned long long>(dp));
                atomicAdd(&ctl->tab_segments, 1ull);
                if (dp > kSupCap) atomicAdd(&ctl->hub_items, (send - bend) * ((dp + kSupCap - 1) / kSupCap));
            }
            for (uint32_t p0 = 0; p0 < dp; p0 += kSupCap) {  // one pass per kSupCap keys of the sorted N+(x)
                const uint32_t nk = dp - p0 < kSupCap ? dp - p0 : kSupCap;
                uint32_t size = 64;
                while (size < TDG_SUP_LOAD * nk && size < kSupTab) size <<= 1;  // load <= 1/LOAD, or <= 3/4 at full size
                const uint32_t bmask = size / 4 - 1;
                for (uint32_t q = threadIdx.x; q < size / 4; q += kTabThreads)
                    tab_keys4[q] = make_uint4(kHEmpty, kHEmpty, kHEmpty, kHEmpty);
                for (uint32_t q = threadIdx.x; q < size / 2; q += kTabThreads) cnt2[q] = 0;
                __syncthreads();
                for (uint32_t q = threadIdx.x; q < nk; q += kTabThreads) {
                    const uint32_t c = g.oadj[o + p0 + q];
                    uint32_t b = tab_hash(c, bmask);
                    while (true) {  // first free slot of the bucket (slots fill in order), else the next bucket
                        uint32_t k = 0;
                        while (k < 4u && atomicCAS(&keys[4u * b + k], kHEmpty, c) != kHEmpty) k++;
                        if (k < 4u) {
                            tpos[4u * b + k] = static_cast<uint16_t>(q);  // position in this slice of N+(x)
                            break;
                        }
                        b = (b + 1) & bmask;
                    }
                }
                __syncthreads();
                if (w0 < w1) {
                    if (dp > kSupCap) {
                        SupportTabPolicy<true> TP{g, s, g.oadj, tab_keys4, cnt2, cnt2_saddr, bmask, g.oadj[o + p0], g.oadj[o + p0 + nk - 1]};
                        run_items(TP, w0, w1, t0, m, wpre, sboff, CH);
                    } else {
                        SupportTabPolicy<false> TP{g, s, g.oadj, tab_keys4, cnt2, cnt2_saddr, bmask, 0u, 0u};
                        run_items(TP, w0, w1, t0, m, wpre, sboff, CH);
                    }
                }
                __syncthreads();
                // flush the slots' hit counters: s[slot of x -> key] += count
                for (uint32_t q = threadIdx.x; q < size / 2; q += kTabThreads) {
                    const uint32_t c2 = cnt2[q];
                    if (c2 & 0xffffu) atomicAdd(&s[o + p0 + tpos[2u * q]], c2 & 0xffffu);
                    if (c2 >> 16) atomicAdd(&s[o + p0 + tpos[2u * q + 1]], c2 >> 16);
                }
                __syncthreads();
            }
            base = send;
            i = tend;
        }
    }
}

// Work of task t: the quads of N+(y) (kQuads) or its elements; the element total is the
// pass's probe count.
template <bool kQuads>
__global__ void __launch_bounds__(kThreads) k_support_prep(DevGraph g, unsigned long long* wpre, unsigned long long* bsum,
                                                           SupportCtl* ctl) {
    unsigned long long elems = 0;
    unsigned long long big = 0;  // work items whose owner list is longer than kSupBigDeg (geometry choice)
    prep_items<kThreads>(g.m, [&](uint32_t t) {
        const uint32_t y = g.adj[g.stask[t]];
        const uint32_t oa = g.opos[y], len = g.opos[y + 1] - oa;
        elems += len;
        const uint32_t items = kQuads ? quads_of(oa, len) : len;
        if (kQuads) {
            const uint32_t x = g.sx[t];
            if (g.opos[x + 1] - g.opos[x] > kSupBigDeg) big += items;
        }
        return items;
    }, wpre, bsum);
    for (int o = 16; o > 0; o >>= 1) {
        elems += shfl64(elems, lane_id() ^ o);
        big += shfl64(big, lane_id() ^ o);
    }
    if (lane_id() == 0 && elems) atomicAdd(&ctl->probes, elems);
    if (lane_id() == 0 && big) atomicAdd(&ctl->big_work, big);
}

// triangle_count (triangle.cpp:90-116): the same task stream with no per-edge writes; each
// warp keeps a register count of its hits and adds it once at the end.
struct CountPolicy {
    const DevGraph& g;
    const uint32_t* elems;
    unsigned long long count = 0;
    static constexpr bool kFast = true;
    static constexpr int kUnroll = 1;
    __device__ ITask load(uint32_t t) const { return otask(g, t); }
    __device__ uint32_t find(const ITask& k, uint32_t x) const {
        const uint32_t lx = k.lb & 0xffffu;
        const uint32_t p = lower_bound_u32(g.oadj + k.ob, lx, x);
        return (p < lx && g.oadj[k.ob + p] == x) ? p : kNone;
    }
    __device__ void visit(bool, bool hit, const ITask&, uint32_t, uint32_t) {
        count += static_cast<unsigned long long>(__popc(__ballot_sync(kFull, hit)));
    }
};

__global__ void __launch_bounds__(kThreads) k_triangle_count(DevGraph g, const unsigned long long* wpre,
                                                             const unsigned long long* bsum, uint32_t nchunks,
                                                             SupportCtl* ctl) {
    __shared__ unsigned long long sboff[kMaxChunks + 1];
    CountPolicy P{g, g.oadj};
    process_items<kThreads>(P, g.m, wpre, bsum, nchunks, &ctl->piece_head, sboff);
    if (lane_id() == 0 && P.count) atomicAdd(&ctl->tri3, P.count);
}

__global__ void __launch_bounds__(kThreads) k_support(DevGraph g, uint32_t* __restrict__ s,
                                                      const unsigned long long* wpre, const unsigned long long* bsum,
                                                      uint32_t nchunks, SupportCtl* ctl) {
    __shared__ unsigned long long sboff[kMaxChunks + 1];
    SupportPolicy P{g, s, g.oadj};
    process_items<kThreads>(P, g.m, wpre, bsum, nchunks, &ctl->piece_head, sboff);
}

__global__ void k_support_sum(const uint32_t* __restrict__ s, uint32_t m, SupportCtl* ctl) {
    unsigned long long sum = 0;
    uint32_t mx = 0;
    for (uint32_t e = blockIdx.x * blockDim.x + threadIdx.x; e < m; e += gridDim.x * blockDim.x) {
        const uint32_t v = s[e];
        sum += v;
        mx = v > mx ? v : mx;
    }
    for (int o = 16; o > 0; o >>= 1) {
        sum += __shfl_xor_sync(kFull, sum, o);
        mx = max(mx, __shfl_xor_sync(kFull, mx, o));
    }
    if (lane_id() == 0) {
        atomicAdd(&ctl->tri3, sum);
        atomicMax(&ctl->smax, mx);
    }
}

}  // namespace

cudaError_t launch_support(const DevGraph& g, uint32_t* s, unsigned long long* wpre,
                           unsigned long long* bsum, SupportCtl* ctl, int sm_count, cudaStream_t st,
                           uint32_t* launches, uint32_t shard, uint32_t nshards) {
    if (nshards == 0 || shard >= nshards) return cudaErrorInvalidValue;
    cudaError_t err = cudaMemsetAsync(ctl, 0, sizeof(SupportCtl), st);
    if (err != cudaSuccess) return err;
    if (g.m == 0) return cudaSuccess;
    if ((err = cudaMemsetAsync(s, 0, size_t(g.m) * sizeof(uint32_t), st)) != cudaSuccess) return err;
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_support, kThreads, 0);
    if (per_sm < 1) per_sm = 1;
    unsigned grid = static_cast<unsigned>(sm_count * per_sm);
    const unsigned nchunks = grid < kMaxChunks ? grid : kMaxChunks;
    k_support_prep<true><<<nchunks, kThreads, 0, st>>>(g, wpre, bsum, ctl);
    static const bool tab_form = [] {
        const char* e = std::getenv("TDG_SUP_FORM");  // diagnostic A/B: "search" = global search only
        return !(e && e[0] == 's');
    }();
    if (tab_form) {
        static const int force = [] {
            const char* e = std::getenv("TDG_SUP_BIG");  // diagnostic A/B: 0 / 1 forces the small / big geometry
            return e ? std::atoi(e) : -1;
        }();
        // both geometries are queued; the one the graph does not want exits at once (the verdict
        // is on the device: no host round trip). Per-device attributes: set on every call.
        const size_t smem0 = sup_smem(kSupTab), smem1 = sup_smem(2 * kSupTab);
        if ((err = cudaFuncSetAttribute(k_support_tab<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem0))) != cudaSuccess) return err;
        if ((err = cudaFuncSetAttribute(k_support_tab<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem1))) != cudaSuccess) return err;
        int tb0 = 0, tb1 = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&tb0, k_support_tab<0>, kTabThreads, smem0);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&tb1, k_support_tab<1>, 2 * kTabThreads, smem1);
        if (tb0 < 1) tb0 = 1;
        if (tb1 < 1) tb1 = 1;
        k_support_tab<0><<<static_cast<unsigned>(sm_count * tb0), kTabThreads, smem0, st>>>(g, s, wpre, bsum, nchunks, ctl, shard,
                                                                                         nshards, force);
        k_support_tab<1><<<static_cast<unsigned>(sm_count * tb1), 2 * kTabThreads, smem1, st>>>(g, s, wpre, bsum, nchunks, ctl,
                                                                                             shard, nshards, force);
        (*launches)++;
    } else {
        if (nshards != 1) return cudaErrorNotSupported;  // the diagnostic search form is unsharded
        k_support<<<grid, kThreads, 0, st>>>(g, s, wpre, bsum, nchunks, ctl);
    }
    k_support_sum<<<grid, kThreads, 0, st>>>(s, g.m, ctl);
    (*launches) += 3;
    return cudaGetLastError();
}

cudaError_t launch_triangle_count(const DevGraph& g, unsigned long long* wpre, unsigned long long* bsum,
                                  SupportCtl* ctl, int sm_count, cudaStream_t st, uint32_t* launches) {
    cudaError_t err = cudaMemsetAsync(ctl, 0, sizeof(SupportCtl), st);
    if (err != cudaSuccess || g.m == 0) return err;
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_triangle_count, kThreads, 0);
    if (per_sm < 1) per_sm = 1;
    const unsigned grid = static_cast<unsigned>(sm_count * per_sm);
    const unsigned nchunks = grid < kMaxChunks ? grid : kMaxChunks;
    k_support_prep<false><<<nchunks, kThreads, 0, st>>>(g, wpre, bsum, ctl);
    k_triangle_count<<<grid, kThreads, 0, st>>>(g, wpre, bsum, nchunks, ctl);
    (*launches) += 2;
    return cudaGetLastError();
}

}  // namespace tdg
