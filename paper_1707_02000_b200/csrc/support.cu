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
// list is x's. Probe N+(y) (coalesced, min(d+) items) and binary-search each element in
// N+(x); tasks are grouped by x, so consecutive tasks search the same L1-resident list.
__device__ __forceinline__ ITask otask(const DevGraph& g, uint32_t t) {
    const uint32_t j = g.stask[t], x = g.sx[t], y = g.adj[j];
    ITask k;
    k.id = g.eid[j];
    k.oa = g.opos[y];
    k.ob = g.opos[x];
    k.lb = g.opos[x + 1] - k.ob;
    return k;
}

// Edge ids are internal (build.cu launch_internal_ids): an edge's id IS its oriented slot
// (position in the N+ arrays). The owner-side slots of a task group are one contiguous,
// L2-resident N+(x) range and the probe-side slots of one task are consecutive, so the
// per-triangle atomics stay out of DRAM (reference-id-indexed atomics were random 2 GB
// read-modify-writes at C5).
// Hits of one engine step (U items per lane): each hit closes triangle {x, y, c} — the
// oriented slots of y->c and x->c get one atomic each; the tasks' own edges are counted
// with one atomic per step when every lane works on the same task (the common case in
// long lists), else per item with one atomic per group of lanes sharing a task.
template <int U>
__device__ __forceinline__ void visit_all(uint32_t* s, const ITask (&ko)[U], const uint32_t (&ja)[U],
                                          const uint32_t (&p)[U]) {
    uint32_t tot = 0;
    bool same = true;
    const uint32_t id0 = __shfl_sync(kFull, ko[0].id, 0);
#pragma unroll
    for (int q = 0; q < U; q++) {
        const bool hit = p[q] != kNone;
        if (hit) {
            atomicAdd(&s[ko[q].oa + ja[q]], 1u);
            atomicAdd(&s[ko[q].ob + p[q]], 1u);
        }
        tot += __popc(__ballot_sync(kFull, hit));
        same = same && (!hit || ko[q].id == id0);
    }
    if (tot == 0) return;
    if (__all_sync(kFull, same)) {
        if (lane_id() == 0) atomicAdd(&s[id0], tot);
        return;
    }
#pragma unroll
    for (int q = 0; q < U; q++) {
        const bool hit = p[q] != kNone;
        const uint32_t fm = __ballot_sync(kFull, hit);
        if (fm && hit) {
            const uint32_t grp = __match_any_sync(fm, ko[q].id);
            if (lane_id() == static_cast<uint32_t>(__ffs(grp) - 1))
                atomicAdd(&s[ko[q].id], static_cast<uint32_t>(__popc(grp)));
        }
    }
}

#ifndef TDG_SUP_U
#define TDG_SUP_U 2  // probe items per lane per engine step in the support pass
#endif
struct SupportPolicy {
    const DevGraph& g;
    uint32_t* s;
    const uint32_t* elems;
    static constexpr bool kFast = true;
    static constexpr int kUnroll = TDG_SUP_U;
    __device__ ITask load(uint32_t t) const { return otask(g, t); }
    __device__ uint32_t find(const ITask& k, uint32_t x) const {
        const uint32_t p = lower_bound_u32(g.oadj + k.ob, k.lb, x);
        return (p < k.lb && g.oadj[k.ob + p] == x) ? p : kNone;
    }
    // U items per lane per engine step: the U list loads and lookups issue together and
    // the engine's per-step bookkeeping is amortised over 32U probes.
    template <int U>
    __device__ void run(const bool (&act)[U], const ITask (&ko)[U], const uint32_t (&ja)[U]) const {
        uint32_t c[U], p[U];
#pragma unroll
        for (int q = 0; q < U; q++) c[q] = act[q] ? elems[ko[q].oa + ja[q]] : 0u;
#pragma unroll
        for (int q = 0; q < U; q++) p[q] = act[q] ? find(ko[q], c[q]) : kNone;
        visit_all<U>(s, ko, ja, p);
    }
};

// ---- owner-table form. A block takes a piece of the work axis and walks its owner
// segments (the tasks of one owner x are contiguous, [sbeg[x], sbeg[x+1])). For a segment
// with enough work, N+(x) is loaded once into a shared-memory hash table (key c -> its
// position in N+(x)) and the block's 8 warps split the segment's items evenly; each probe is then
// one coalesced N+(y) load plus ~1 shared-memory access instead of a log2(d+(x)) chain of
// L1 loads (the search form is issue-bound: ncu C3, 71% issue slots busy). Segments that
// are too small to pay for the table, or whose owner list exceeds the table, are batched
// and searched in global memory as before.
#ifndef TDG_SUP_TAB
#define TDG_SUP_TAB 4096  // shared-memory table slots (4 B key + 2 B position): owners with d+ <= 3/4 TAB
#endif
constexpr uint32_t kSupTab = TDG_SUP_TAB;
#ifndef TDG_SUP_LOAD
#define TDG_SUP_LOAD 4  // table slots per key when the table is not full size (C5: 2 -> 4: 1089 -> 1047 ms)
#endif
constexpr size_t kSupSmem = size_t(kSupTab) * (sizeof(uint32_t) + sizeof(uint16_t));
static_assert(kSupTab % 4 == 0 && 3 * kSupTab / 4 < 65536, "bucketed owner table: u16 positions");
#ifndef TDG_SUP_SEGMIN
#define TDG_SUP_SEGMIN 512u  // a segment gets a table if its probes * SEGDIV >= max(d+(x), SEGMIN)
#endif
#ifndef TDG_SUP_SEGDIV
#define TDG_SUP_SEGDIV 1u
#endif
#ifndef TDG_SUP_MINB
#define TDG_SUP_MINB 5  // 5 blocks/SM (shared memory allows 5; C5 support 1.39 -> 1.20 s)
#endif
constexpr uint32_t kSupWarps = kThreads / 32;

// Shared-memory table slot of key c: multiplicative (Fibonacci) hashing, top bits of
// c * 2^32/phi — one multiply and a shift instead of hmix's five-step mix (the support pass
// is issue-bound).
__device__ __forceinline__ uint32_t tab_hash(uint32_t c, uint32_t mask) {
    return (c * 0x9E3779B1u) >> (__clz(mask) & 31u);
}

// Owner table in shared memory, BUCKETED: 4-key buckets (one 16-byte LDS.128 compares four
// keys), linear probing over buckets, keys claimed in slot order inside a bucket (so a
// bucket whose last slot is empty ends a miss); the position of the key in N+(x) sits in a
// parallel u16 array, read only on a hit. (The previous 8-byte (key, position) slots with
// per-slot probing took ~3-8 dependent shared loads per miss at the 3/4 load of the
// d+ > 1024 owners that carry ~70 % of C5's probes.)
struct SupportTabPolicy {
    const DevGraph& g;
    uint32_t* s;
    const uint32_t* elems;
    const uint4* keys4;      // nb buckets of 4 keys
    const uint16_t* pos;     // 4 * nb positions
    uint32_t bmask;          // nb - 1
    static constexpr bool kFast = true;
    static constexpr int kUnroll = TDG_SUP_U;
    __device__ ITask load(uint32_t t) const { return otask(g, t); }
    __device__ uint32_t find(const ITask&, uint32_t c) const {
        uint32_t b = tab_hash(c, bmask);
        while (true) {
            const uint4 v = keys4[b];
            const uint32_t k = v.x == c ? 0u : v.y == c ? 1u : v.z == c ? 2u : v.w == c ? 3u : 4u;
            if (k < 4u) return pos[4u * b + k];
            if (v.w == kHEmpty) return kNone;
            b = (b + 1) & bmask;
        }
    }
    // U items per lane per engine step: the U list loads and lookups issue together and
    // the engine's per-step bookkeeping is amortised over 32U probes.
    template <int U>
    __device__ void run(const bool (&act)[U], const ITask (&ko)[U], const uint32_t (&ja)[U]) const {
        uint32_t c[U], p[U];
#pragma unroll
        for (int q = 0; q < U; q++) {
            TDG_CHECK(!act[q] || uint64_t(ko[q].oa) + ja[q] < g.m);
            c[q] = act[q] ? elems[ko[q].oa + ja[q]] : 0u;
        }
#pragma unroll
        for (int q = 0; q < U; q++) {
            p[q] = act[q] ? find(ko[q], c[q]) : kNone;
            TDG_CHECK(p[q] == kNone || uint64_t(ko[q].ob) + p[q] < g.m);
        }
        visit_all<U>(s, ko, ja, p);
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

__global__ void __launch_bounds__(kThreads, TDG_SUP_MINB) k_support_tab(DevGraph g, uint32_t* __restrict__ s,
                                                          const unsigned long long* wpre, const unsigned long long* bsum,
                                                          uint32_t nchunks, SupportCtl* ctl) {
    extern __shared__ uint4 tab_keys4[];  // kSupTab keys, then kSupTab u16 positions
    __shared__ unsigned long long sboff[kMaxChunks + 1];
    __shared__ uint32_t sh_p;
    const unsigned long long W = chunk_offsets<kThreads>(bsum, nchunks, sboff);
    if (blockIdx.x == 0 && threadIdx.x == 0) ctl->probes = W;
    if (W == 0) return;
    const uint32_t m = g.m, CH = chunk_len(m, nchunks);
    const uint32_t wid = threadIdx.x >> 5;
    unsigned long long PS = (W + 4ull * gridDim.x - 1) / (4ull * gridDim.x);
    PS = PS < 4096 ? 4096 : PS;
    const unsigned long long npieces = (W + PS - 1) / PS;
    auto start = [&](uint32_t t) -> unsigned long long { return t < m ? sboff[t / CH] + wpre[t] : W; };
    SupportPolicy SP{g, s, g.oadj};
    while (true) {
        if (threadIdx.x == 0) sh_p = atomicAdd(&ctl->piece_head, 1u);
        __syncthreads();
        const uint32_t p = sh_p;
        __syncthreads();
        if (p >= npieces) break;
        const unsigned long long x0 = p * PS, x1 = x0 + PS < W ? x0 + PS : W;
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
                table = 4u * dp <= 3u * kSupTab &&
                        (send - bend) * TDG_SUP_SEGDIV >= (dp > TDG_SUP_SEGMIN ? dp : TDG_SUP_SEGMIN);
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
            uint32_t size = 64;
            while (size < TDG_SUP_LOAD * dp && size < kSupTab) size <<= 1;  // load <= 1/LOAD, or <= 3/4 at full size
            uint32_t* keys = reinterpret_cast<uint32_t*>(tab_keys4);
            uint16_t* tpos = reinterpret_cast<uint16_t*>(keys + kSupTab);
            const uint32_t bmask = size / 4 - 1;
            for (uint32_t q = threadIdx.x; q < size / 4; q += kThreads)
                tab_keys4[q] = make_uint4(kHEmpty, kHEmpty, kHEmpty, kHEmpty);
            if (threadIdx.x == 0) {
                atomicAdd(&ctl->tab_elems, static_cast<unsigned long long>(dp));
                atomicAdd(&ctl->tab_segments, 1ull);
            }
            __syncthreads();
            const uint32_t o = g.opos[x];
            for (uint32_t q = threadIdx.x; q < dp; q += kThreads) {
                const uint32_t c = g.oadj[o + q];
                uint32_t b = tab_hash(c, bmask);
                while (true) {  // first free slot of the bucket (slots fill in order), else the next bucket
                    uint32_t k = 0;
                    while (k < 4u && atomicCAS(&keys[4u * b + k], kHEmpty, c) != kHEmpty) k++;
                    if (k < 4u) {
                        tpos[4u * b + k] = static_cast<uint16_t>(q);  // position in N+(x), as the search form's find returns
                        break;
                    }
                    b = (b + 1) & bmask;
                }
            }
            __syncthreads();
            SupportTabPolicy TP{g, s, g.oadj, tab_keys4, tpos, bmask};
            const unsigned long long w0 = bend + (send - bend) * wid / kSupWarps;
            const unsigned long long w1 = bend + (send - bend) * (wid + 1) / kSupWarps;
            if (w0 < w1) run_items(TP, w0, w1, task_in(w0, j, tend, wpre, sboff, CH), m, wpre, sboff, CH);
            __syncthreads();
            base = send;
            i = tend;
        }
    }
}

__global__ void __launch_bounds__(kThreads) k_support_prep(DevGraph g, unsigned long long* wpre, unsigned long long* bsum) {
    prep_items<kThreads>(g.m, [&](uint32_t t) {
        const uint32_t y = g.adj[g.stask[t]];
        return g.opos[y + 1] - g.opos[y];
    }, wpre, bsum);
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
        const uint32_t p = lower_bound_u32(g.oadj + k.ob, k.lb, x);
        return (p < k.lb && g.oadj[k.ob + p] == x) ? p : kNone;
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
    const unsigned long long W = process_items<kThreads>(P, g.m, wpre, bsum, nchunks, &ctl->piece_head, sboff);
    if (lane_id() == 0 && P.count) atomicAdd(&ctl->tri3, P.count);
    if (blockIdx.x == 0 && threadIdx.x == 0) ctl->probes = W;
}

__global__ void __launch_bounds__(kThreads) k_support(DevGraph g, uint32_t* __restrict__ s,
                                                      const unsigned long long* wpre, const unsigned long long* bsum,
                                                      uint32_t nchunks, SupportCtl* ctl) {
    __shared__ unsigned long long sboff[kMaxChunks + 1];
    SupportPolicy P{g, s, g.oadj};
    const unsigned long long W = process_items<kThreads>(P, g.m, wpre, bsum, nchunks, &ctl->piece_head, sboff);
    if (blockIdx.x == 0 && threadIdx.x == 0) ctl->probes = W;
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
                           uint32_t* launches) {
    cudaError_t err = cudaMemsetAsync(ctl, 0, sizeof(SupportCtl), st);
    if (err != cudaSuccess) return err;
    if (g.m == 0) return cudaSuccess;
    if ((err = cudaMemsetAsync(s, 0, size_t(g.m) * sizeof(uint32_t), st)) != cudaSuccess) return err;
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_support, kThreads, 0);
    if (per_sm < 1) per_sm = 1;
    unsigned grid = static_cast<unsigned>(sm_count * per_sm);
    const unsigned nchunks = grid < kMaxChunks ? grid : kMaxChunks;
    k_support_prep<<<nchunks, kThreads, 0, st>>>(g, wpre, bsum);
    static const bool tab_form = [] {
        const char* e = std::getenv("TDG_SUP_FORM");  // diagnostic A/B: "search" = global search only
        return !(e && e[0] == 's');
    }();
    if (tab_form) {
        const size_t smem = kSupSmem;
        // per-device attribute: set on every call (contexts may sit on different devices)
        err = cudaFuncSetAttribute(k_support_tab, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
        if (err != cudaSuccess) return err;
        int tb = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&tb, k_support_tab, kThreads, smem);
        if (tb < 1) tb = 1;
        k_support_tab<<<static_cast<unsigned>(sm_count * tb), kThreads, smem, st>>>(g, s, wpre, bsum, nchunks, ctl);
    } else {
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
    k_support_prep<<<nchunks, kThreads, 0, st>>>(g, wpre, bsum);
    k_triangle_count<<<grid, kThreads, 0, st>>>(g, wpre, bsum, nchunks, ctl);
    (*launches) += 2;
    return cudaGetLastError();
}

}  // namespace tdg
