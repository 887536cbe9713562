// tdg_common.cuh — shared device helpers and device-side data layout of the B200 PKT path.
//
// Layout in HBM (all 32-bit; the reference is uint32 throughout, graph.hpp:10-11):
//   off[n+1]   CSR offsets (narrowed from the int64 C-ABI input)
//   adj[2m]    working copy of the sorted adjacency (compacted in place by the peel)
//   eid[2m]    reference edge id of every adjacency slot        (graph.cpp:86-99)
//   el[m]      uint2 (u,v), u<v, indexed by edge id             (graph.cpp:98)
//   dl[n]      live length of each adjacency list (peel compaction)
//   opos[n+1], oadj[m], oeid[m], osrc[m]
//              degree-ordered orientation u->v iff (d(u),u) < (d(v),v), each list a
//              sorted subsequence of adj (support pass only)
//   s[m]       support, stamp[m] sub-level stamp (peel)
#pragma once

#include <cstdint>
#include <cuda_runtime.h>
#include <cstdio>

namespace tdg {

constexpr uint32_t kFull = 0xffffffffu;
constexpr uint32_t kNone = 0xffffffffu;
__device__ __forceinline__ uint32_t lane_id() { return threadIdx.x & 31u; }

// Checked builds (-DTDG_CHECKS=1, tests/test_checked_gpu.py): device-side bounds and
// invariant checks on the hot paths; a violation prints its site and traps the kernel.
// (compute-sanitizer is not available on the GPU pool; these are the memory checks.)
#ifndef TDG_CHECKS
#define TDG_CHECKS 0
#endif
#define TDG_CHECK(cond)                                                                          \
    do {                                                                                         \
        if (TDG_CHECKS && !(cond)) {                                                             \
            printf("TDG_CHECK failed %s:%d: %s (block %u thread %u)\n", __FILE__, __LINE__, #cond, \
                   blockIdx.x, threadIdx.x);                                                     \
            __trap();                                                                            \
        }                                                                                        \
    } while (0)

__device__ __forceinline__ uint32_t lanemask_lt() {
    uint32_t r;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(r));
    return r;
}

// Relaxed gpu-scope accesses for words other SMs update inside the same launch
// (supports under atomicSub, sub-level stamps). They bypass the non-coherent L1.
__device__ __forceinline__ uint32_t ld_relaxed(const uint32_t* p) {
    uint32_t v;
    asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p));
    return v;
}
__device__ __forceinline__ void st_relaxed(uint32_t* p, uint32_t v) {
    asm volatile("st.relaxed.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v));
}

// First index in [0,len) with a[i] >= x (len if none). Branch-free halving: every lane
// of a warp runs ceil(log2(len)) steps, so a warp probing one list stays converged.
__device__ __forceinline__ uint32_t lower_bound_u32(const uint32_t* __restrict__ a, uint32_t len,
                                                    uint32_t x) {
    if (len == 0) return 0;
    const uint32_t* base = a;
    uint32_t n = len;
    while (n > 1) {
        uint32_t half = n >> 1;
        base = (base[half] < x) ? base + half : base;
        n -= half;
    }
    return static_cast<uint32_t>(base - a) + (*base < x);
}

// Same for the first index with a[i] > x.
__device__ __forceinline__ uint32_t upper_bound_u32(const uint32_t* __restrict__ a, uint32_t len,
                                                    uint32_t x) {
    if (len == 0) return 0;
    const uint32_t* base = a;
    uint32_t n = len;
    while (n > 1) {
        uint32_t half = n >> 1;
        base = (base[half] <= x) ? base + half : base;
        n -= half;
    }
    return static_cast<uint32_t>(base - a) + (*base <= x);
}

__device__ __forceinline__ uint32_t warp_incl_scan(uint32_t v) {
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        uint32_t t = __shfl_up_sync(kFull, v, o);
        if (lane_id() >= static_cast<uint32_t>(o)) v += t;
    }
    return v;
}

// Warp-aggregated append (the GPU form of BufferedAppender, appender.hpp:12-40): one
// atomicAdd per warp. All 32 lanes must call; returns the slot for lanes with `pred`.
__device__ __forceinline__ uint32_t warp_append(bool pred, uint32_t* counter) {
    uint32_t mask = __ballot_sync(kFull, pred);
    if (mask == 0) return 0;
    uint32_t leader = __ffs(mask) - 1;
    uint32_t base = 0;
    if (lane_id() == leader) base = atomicAdd(counter, static_cast<uint32_t>(__popc(mask)));
    base = __shfl_sync(kFull, base, leader);
    return base + static_cast<uint32_t>(__popc(mask & lanemask_lt()));
}

// ---- per-vertex neighbour -> edge-id hash tables (built once per graph, never compacted)
// BUCKETED: the table of x is nb(x) = ceil(kHF * d(x) / 4) buckets of 32 bytes (one DRAM
// sector) at bucket offset hbo[x] (exclusive scan of nb; the total is bounded by
// kHF * 2m / 4 + n, known before the build — no size readback). A bucket holds 4 keys
// (neighbour ids, kHEmpty = free) then their 4 values (edge id | (neighbour after x in the
// (degree, id) order ? kHUp : 0)). A key lives in its home bucket hbucket(hmix(key), nb) or,
// if that is full, in the following ones (linear probing over buckets); slots fill in order,
// so a lookup reads one 16-byte key vector per bucket and stops at a bucket with a free slot.
#ifndef TDG_HT_FACTOR
#define TDG_HT_FACTOR 2  // table slots per neighbour (load factor 1/kHF): C5 tables 32 B per edge
#endif
constexpr uint32_t kHF = TDG_HT_FACTOR;
constexpr uint32_t kHEmpty = 0xffffffffu;
constexpr uint32_t kHUp = 0x80000000u;

__device__ __forceinline__ uint32_t hmix(uint32_t x) {
    x ^= x >> 16;
    x *= 0x85ebca6bu;
    x ^= x >> 13;
    x *= 0xc2b2ae35u;
    x ^= x >> 16;
    return x;
}
__host__ __device__ __forceinline__ uint32_t hbuckets(uint32_t d) { return (kHF * d + 3u) / 4u; }
// Home bucket of hash h in a table of nb buckets (multiply-high range reduction, any nb).
__device__ __forceinline__ uint32_t hbucket(uint32_t h, uint32_t nb) { return __umulhi(h, nb); }
__device__ __forceinline__ uint32_t hnext(uint32_t i, uint32_t nb) { return i + 1 == nb ? 0u : i + 1; }
// Slot (0..3) of key x in a bucket's key vector, 4 if absent.
__device__ __forceinline__ uint32_t bucket_find(const uint4& k, uint32_t x) {
    return k.x == x ? 0u : k.y == x ? 1u : k.z == x ? 2u : k.w == x ? 3u : 4u;
}
// Insert (key y, value v) into the bucketed table t of nb buckets (global or shared memory).
__device__ __forceinline__ void bucket_insert(uint32_t* t, uint32_t nb, uint32_t y, uint32_t v) {
    uint32_t b = hbucket(hmix(y), nb);
    while (true) {
        uint32_t k = 0;
        while (k < 4u && atomicCAS(&t[8u * b + k], kHEmpty, y) != kHEmpty) k++;
        if (k < 4u) {
            t[8u * b + 4u + k] = v;
            return;
        }
        b = hnext(b, nb);
    }
}

// Table sizes (buckets) up to which a table is built in shared memory by one warp / one
// block and written out with coalesced stores (build.cu, and the peel's rebuilds).
constexpr uint32_t kHSmall = 256;        // buckets (8 KB) per warp
constexpr uint32_t kHMid = 8 * kHSmall;  // block-built tables use the block's whole 64 KB

// ---- per-vertex membership filters (register-blocked Bloom filters) in front of the big
// tables (nb >= kFMin buckets). Vertex x owns the 64-bit words [hbo[x] >> kFShift,
// hbo[x+1] >> kFShift) — disjoint ranges, 2^kFShift buckets (~2^(kFShift+2) / kHF keys) per
// word: 4 bits per key at kHF = 2, kFShift = 3. A key sets TDG_FK bits of one word; a lookup
// whose bits are not all set is a certain miss and skips the table walk, so the misses of a
// sub-level (~3/4 of all probes) mostly hit the L2-resident filters instead of DRAM.
#ifndef TDG_FMIN
#define TDG_FMIN 64  // buckets (256 slots; C5 peel 2150 -> 2127 ms against 256)
#endif
constexpr uint32_t kFMin = TDG_FMIN;
#ifndef TDG_FSHIFT
#define TDG_FSHIFT 2  // 8 bits per key (with hashed word choice 4 bits won: sparser filters stayed L2-resident; with the rank-ordered choice (TDG_FMONO) lanes share sectors and the lower false-positive rate wins: C5 peel 2028 -> 1990 ms)
#endif
#ifndef TDG_FK
#define TDG_FK 3  // bits set per key
#endif
constexpr uint32_t kFShift = TDG_FSHIFT;
#ifndef TDG_FSHIFT_REBUILD
#define TDG_FSHIFT_REBUILD 2  // filters of the tables rebuilt on the live graph: 8 bits per key
#endif
constexpr uint32_t kFShiftRebuild = TDG_FSHIFT_REBUILD;
static_assert(kFShiftRebuild <= kFShift, "rebuilt filters may be denser, never sparser (TDG_FMIN covers both)");
static_assert((kFMin >> kFShift) >= 1, "every filtered vertex owns at least one filter word");

__device__ __forceinline__ unsigned long long fbits(uint32_t h) {  // h = hmix(key)
    unsigned long long b = (1ull << ((h >> 14) & 63)) | (1ull << ((h >> 20) & 63));
    if (TDG_FK > 2) b |= 1ull << ((h >> 26) & 63);
    if (TDG_FK > 3) b |= 1ull << ((h >> 8) & 63);
    return b;
}

// Filter word of key y in the filter of a vertex whose table is buckets [ob, ob + nb).
// (fshift: kFShift for the tables of the input graph; the peel's rebuilds on the live graph
// use the denser kFShiftRebuild — a template parameter of the k_peel segments.)
// The word of a key is umulhi(y * fscale, words of the vertex). Two multipliers (FilterCtl,
// chosen per graph by build.cu, read by the kernels from device memory — no host round trip):
//  * RANK mode, fscale = floor((2^32 - 1) / n): monotone in y, so the sorted list elements a
//    warp probes together fall into neighbouring words and share filter sectors (about
//    d(b)/d(a) sectors per warp step instead of 32). Right when neighbour ids are spread over
//    the id space (permuted / hashed ids): C5 peel 2101 -> 1990 ms.
//  * HASH mode, fscale = 0x9E3779B1 (multiplicative hashing): when ids are clustered (an
//    unpermuted RMAT: hubs and their neighbours sit at low ids) rank mode piles the keys of a
//    vertex into few words, which saturate and pass every probe (measured: peel +21..32 %).
// After a rank-mode fill the build measures the probe-weighted false-positive estimate of the
// filters and refills them in hash mode when it is too high (kFilterFpMax). The bits inside
// the word are hashed in both modes. TDG_FMONO = 0 compiles the rank mode out.
#ifndef TDG_FMONO
#define TDG_FMONO 1
#endif
constexpr uint32_t kFilterHashMul = 0x9E3779B1u;
__host__ __device__ __forceinline__ uint32_t filter_scale(uint32_t n) { return n ? 0xffffffffu / n : 0u; }
struct FilterCtl {
    uint32_t fscale;   // the multiplier in use
    uint32_t hashed;   // 1: hash mode was chosen (filters refilled)
    unsigned long long keys, fp;  // sum over words of set bits, and of set bits x (fill^3) in 2^-18 units
};
__device__ __forceinline__ uint64_t fword_index(uint32_t ob, uint32_t nb, uint32_t y, uint32_t fshift, uint32_t fscale) {
    const uint32_t f0 = ob >> fshift, f1 = (ob + nb) >> fshift;
    return static_cast<uint64_t>(f0) + __umulhi(y * fscale, f1 - f0);
}

struct DevGraph {
    uint32_t n = 0, m = 0;
    uint64_t nbuckets = 0;  // hash-table buckets allocated (bounds for checked builds)
    const uint32_t* htab = nullptr;  // bucketed hash tables: 8 u32 words (4 keys, 4 values) per bucket
    const uint32_t* hbo = nullptr;   // n+1 bucket offsets
    const unsigned long long* filt = nullptr;  // membership filters of the big tables (or null)
    const uint32_t* off = nullptr;
    uint32_t* adj = nullptr;
    uint32_t* eid = nullptr;
    const uint2* el = nullptr;
    uint32_t* dl = nullptr;
    const uint32_t* opos = nullptr;
    const uint32_t* oadj = nullptr;
    const uint32_t* oeid = nullptr;
    const uint32_t* osrc = nullptr;
    const uint32_t* stask = nullptr;  // support tasks (slot index), see build.cu k_svalid
    const uint32_t* sx = nullptr;     // owner vertex of each support task's slot
    const uint32_t* sbeg = nullptr;   // n+1: first support task of each owner
    // (kept LAST: a member in front of the pointers shifted the kernel parameter layout and cost
    // the peel's probe loop 4 %, C5 2101 -> 2186 ms)
    const FilterCtl* fctl = nullptr;  // filter word multiplier of this graph (device memory)
};

}  // namespace tdg
