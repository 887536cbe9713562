// build.cu — edge-id map and degree orientation on the GPU.
//
// Reference: build_truss_graph, /root/reference/proj/src/graph.cpp:73-101. The reference
// walks (u,v) pairs serially and finds mirror slots with a per-vertex cursor; here every
// slot is independent:
//   eo[u]   = first slot of u with neighbour > u                    (graph.cpp:80-84)
//   P       = exclusive scan of up[u] = off[u+1]-eo[u]              (edge-id base per u)
//   upper slot j of u (v>u): eid = P[u] + j - eo[u], el[eid] = (u,v)
//   lower slot j of u (v<u): the mirror's id, read from the upper-slot ids stably sorted by
//                            upper endpoint (a transpose; position j - P[u], k_eid_lower)
// Then the support pass's orientation (north-star item 1): u->v iff
// (d(u),u) < (d(v),v); the oriented lists are order-preserving subsequences of adj,
// compacted with one global scan of per-slot flags. All passes are slot-parallel
// (load-balanced regardless of degree skew) and HBM-streaming plus one radix sort of m
// (key, id) pairs.

#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>

#include "tdg_kernels.h"

namespace tdg {

namespace {

constexpr int kThreads = 256;

inline unsigned grid_for(uint64_t items, int threads = kThreads) {
    uint64_t b = (items + threads - 1) / threads;
    if (b == 0) b = 1;
    if (b > 0x7fffffffull) b = 0x7fffffffull;
    return static_cast<unsigned>(b);
}

__global__ void k_off_to_u32(const int64_t* __restrict__ off64, uint32_t* __restrict__ off, uint32_t n1) {
    for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n1; i += uint64_t(gridDim.x) * blockDim.x)
        off[i] = static_cast<uint32_t>(off64[i]);
}

// src[off[u]] = u for non-empty rows; a max-scan then fills every slot with its row.
__global__ void k_row_start(const uint32_t* __restrict__ off, uint32_t n, uint32_t* __restrict__ src) {
    uint32_t u = blockIdx.x * blockDim.x + threadIdx.x;
    if (u < n && off[u + 1] > off[u]) src[off[u]] = u;
}

__global__ void k_eo(const uint32_t* __restrict__ off, const uint32_t* __restrict__ adj, uint32_t n,
                     uint32_t* __restrict__ eo, uint32_t* __restrict__ up) {
    uint32_t u = blockIdx.x * blockDim.x + threadIdx.x;
    if (u < n) {
        uint32_t o = off[u], d = off[u + 1] - o;
        uint32_t e = o + upper_bound_u32(adj + o, d, u);
        eo[u] = e;
        up[u] = off[u + 1] - e;
    } else if (u == n) {
        up[n] = 0;
    }
}

// Upper slot j of u (v > u): eid = P[u] + j - eo[u], el[eid] = (u,v); the pair (v, eid) is
// emitted for the transpose below. Lower slots are filled by k_eid_lower.
__global__ void k_eid(const uint32_t* __restrict__ off, const uint32_t* __restrict__ adj,
                      const uint32_t* __restrict__ src, const uint32_t* __restrict__ eo,
                      const uint32_t* __restrict__ P, uint64_t slots, uint32_t* __restrict__ eid,
                      uint2* __restrict__ el, uint32_t* __restrict__ flag, uint32_t* __restrict__ tkey,
                      uint32_t* __restrict__ tval) {
    for (uint64_t j = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; j < slots;
         j += uint64_t(gridDim.x) * blockDim.x) {
        const uint32_t u = src[j], v = adj[j];
        TDG_CHECK(u < (1u << 31) && v != u);
        if (v > u) {
            const uint32_t e = P[u] + static_cast<uint32_t>(j - eo[u]);
            TDG_CHECK(j >= eo[u]);
            el[e] = make_uint2(u, v);
            eid[j] = e;
            tkey[e] = v;
            tval[e] = e;
        }
        if (flag) {
            const uint32_t du = off[u + 1] - off[u], dv = off[v + 1] - off[v];
            flag[j] = (du < dv || (du == dv && u < v)) ? 1u : 0u;
        }
    }
}

// Lower slot j of u (v < u). The edge ids sorted (stably) by upper endpoint list, for each
// u, the ids of its edges (v,u), v < u, in ascending v — exactly u's lower slots in order.
// u's group starts at off[u] - P[u] (lower slots of the vertices before u), so slot j
// reads position j - P[u]. Replaces a binary search in N(v) per lower slot.
__global__ void k_eid_lower(const uint32_t* __restrict__ adj, const uint32_t* __restrict__ src,
                            const uint32_t* __restrict__ P, const uint32_t* __restrict__ sorted_ids, uint64_t slots,
                            uint32_t* __restrict__ eid) {
    for (uint64_t j = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; j < slots;
         j += uint64_t(gridDim.x) * blockDim.x) {
        const uint32_t u = src[j];
        if (adj[j] < u) {
            TDG_CHECK(j >= P[u] && j - P[u] < slots / 2);
            eid[j] = sorted_ids[j - P[u]];
        }
    }
}

__global__ void k_orient(const uint32_t* __restrict__ adj, const uint32_t* __restrict__ eid,
                         const uint2* __restrict__ el, const uint32_t* __restrict__ flag,
                         const uint32_t* __restrict__ pos, uint64_t slots, uint32_t* __restrict__ oadj,
                         uint32_t* __restrict__ oeid, uint32_t* __restrict__ osrc) {
    for (uint64_t j = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; j < slots;
         j += uint64_t(gridDim.x) * blockDim.x) {
        if (!flag[j]) continue;
        const uint32_t t = pos[j], v = adj[j], e = eid[j];
        TDG_CHECK(t < slots / 2 && e < slots / 2);
        const uint2 p = el[e];
        oadj[t] = v;
        oeid[t] = e;
        osrc[t] = p.x ^ p.y ^ v;
    }
}

__global__ void k_opos(const uint32_t* __restrict__ off, const uint32_t* __restrict__ pos, uint32_t n,
                       uint32_t* __restrict__ opos) {
    uint32_t u = blockIdx.x * blockDim.x + threadIdx.x;
    if (u <= n) opos[u] = pos[off[u]];
}

// Value stored with neighbour y in x's table: edge id | (y after x in the (degree, id) order).
__device__ __forceinline__ uint32_t htab_value(const uint32_t* __restrict__ off, uint32_t x, uint32_t y, uint32_t e) {
    const uint32_t dx = off[x + 1] - off[x], dy = off[y + 1] - off[y];
    const bool up = dx < dy || (dx == dy && x < y);
    return e | (up ? kHUp : 0u);
}

// Buckets per vertex: hq[x] = nb(x) (hq[n] = 0), scanned into the bucket offsets hbo.
__global__ void k_hsize(const uint32_t* __restrict__ off, uint32_t n, uint32_t* __restrict__ hq) {
    const uint32_t u = blockIdx.x * blockDim.x + threadIdx.x;
    if (u < n) hq[u] = hbuckets(off[u + 1] - off[u]);
    else if (u == n) hq[n] = 0;
}

// Tables of at most kHSmall buckets are built in shared memory, one warp per vertex (up to
// kHMid, one block per vertex), and written out with coalesced stores (random global CAS
// inserts were 1.8 % of a C5 step).
// (kHSmall = 256 buckets, 8 KB, per warp; kHMid = 8 kHSmall: the block's whole 64 KB — tdg_common.cuh)

__global__ void __launch_bounds__(256) k_hbuild_small(const uint32_t* __restrict__ off, const uint32_t* __restrict__ adj,
                                                      const uint32_t* __restrict__ eid, const uint32_t* __restrict__ hbo,
                                                      uint32_t n, uint32_t* __restrict__ htab) {
    extern __shared__ uint32_t htab_smem[];  // 8 warps x kHSmall buckets x 8 words
    const uint32_t lane = threadIdx.x & 31u, w = threadIdx.x >> 5;
    uint32_t* t = htab_smem + w * kHSmall * 8u;
    for (uint32_t x = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; x < n; x += (gridDim.x * blockDim.x) >> 5) {
        const uint32_t b0 = hbo[x], nb = hbo[x + 1] - b0;
        if (nb == 0 || nb > kHSmall) continue;
        for (uint32_t i = lane; i < 8u * nb; i += 32) t[i] = kHEmpty;
        __syncwarp();
        const uint32_t o = off[x], d = off[x + 1] - o;
        for (uint32_t i = lane; i < d; i += 32) {
            const uint32_t y = adj[o + i];
            bucket_insert(t, nb, y, htab_value(off, x, y, eid[o + i]));
        }
        __syncwarp();
        uint32_t* g = htab + 8ull * b0;
        for (uint32_t i = lane; i < 8u * nb; i += 32) g[i] = t[i];
        __syncwarp();
    }
    // Tables of kHSmall < nb <= kHMid buckets: the whole block builds one at a time in the
    // same shared memory. Each block takes 256-vertex chunks and queues their mid-size tables.
    __shared__ uint32_t q[256];
    __shared__ uint32_t qn;
    for (uint64_t c0 = uint64_t(blockIdx.x) * 256; c0 < n; c0 += uint64_t(gridDim.x) * 256) {
        if (threadIdx.x == 0) qn = 0;
        __syncthreads();
        const uint64_t x = c0 + threadIdx.x;
        if (x < n) {
            const uint32_t nb = hbo[x + 1] - hbo[x];
            if (nb > kHSmall && nb <= kHMid) q[atomicAdd(&qn, 1u)] = static_cast<uint32_t>(x);
        }
        __syncthreads();
        const uint32_t cnt = qn;
        for (uint32_t k = 0; k < cnt; k++) {
            const uint32_t v = q[k], b0 = hbo[v], nb = hbo[v + 1] - b0, o = off[v], d = off[v + 1] - o;
            for (uint32_t i = threadIdx.x; i < 8u * nb; i += blockDim.x) htab_smem[i] = kHEmpty;
            __syncthreads();
            for (uint32_t i = threadIdx.x; i < d; i += blockDim.x) {
                const uint32_t y = adj[o + i];
                bucket_insert(htab_smem, nb, y, htab_value(off, v, y, eid[o + i]));
            }
            __syncthreads();
            uint32_t* g = htab + 8ull * b0;
            for (uint32_t i = threadIdx.x; i < 8u * nb; i += blockDim.x) g[i] = htab_smem[i];
            __syncthreads();
        }
    }
}

// Insert every slot (x -> y, eid) of a big table (> kHMid buckets) into x's table in global memory.
__global__ void k_hinsert(const uint32_t* __restrict__ off, const uint32_t* __restrict__ adj,
                          const uint32_t* __restrict__ src, const uint32_t* __restrict__ eid,
                          const uint32_t* __restrict__ hbo, uint64_t slots, uint32_t* __restrict__ htab) {
    for (uint64_t j = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; j < slots;
         j += uint64_t(gridDim.x) * blockDim.x) {
        const uint32_t x = src[j];
        const uint32_t b0 = hbo[x], nb = hbo[x + 1] - b0;
        if (nb <= kHMid) continue;
        const uint32_t y = adj[j];
        bucket_insert(htab + 8ull * b0, nb, y, htab_value(off, x, y, eid[j]));
    }
}

// Filter bits of every slot (x -> y) whose owner table is big enough (tdg_common.cuh). `pass`
// 0: the rank-mode fill; 1: the hash-mode refill, a no-op unless k_fdecide chose it.
__global__ void k_finsert(const uint32_t* __restrict__ hbo, const uint32_t* __restrict__ adj,
                          const uint32_t* __restrict__ src, uint64_t slots, unsigned long long* __restrict__ filt,
                          const FilterCtl* __restrict__ fc, int pass) {
    if (pass == 1 && !fc->hashed) return;
    const uint32_t fscale = fc->fscale;
    for (uint64_t j = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; j < slots;
         j += uint64_t(gridDim.x) * blockDim.x) {
        const uint32_t x = src[j];
        const uint32_t b0 = hbo[x], nb = hbo[x + 1] - b0;
        if (nb < kFMin) continue;
        const uint32_t y = adj[j];
        atomicOr(&filt[fword_index(b0, nb, y, kFShift, fscale)], fbits(hmix(y)));
    }
}

__global__ void k_fctl_init(FilterCtl* fc, uint32_t n) {
    fc->fscale = TDG_FMONO ? filter_scale(n) : kFilterHashMul;
    fc->hashed = TDG_FMONO ? 0u : 1u;
    fc->keys = 0;
    fc->fp = 0;
}

// Probe-weighted false-positive estimate of the rank-mode filters: a word with p bits set
// passes a 3-bit probe with probability ~ (p/64)^3, and receives probes in proportion to the
// keys it holds (the probe lists are neighbour lists of the same id space), ~ p. Sums of p and
// of p * (p/64)^3 (in 2^-18 units) over all words.
__global__ void k_fstat(const unsigned long long* __restrict__ filt, uint64_t words, FilterCtl* fc) {
    unsigned long long keys = 0, fp = 0;
    for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < words; i += uint64_t(gridDim.x) * blockDim.x) {
        const unsigned long long p = static_cast<unsigned long long>(__popcll(filt[i]));
        keys += p;
        fp += p * p * p * p;  // p * (p/64)^3 * 2^18
    }
    for (int o = 16; o > 0; o >>= 1) {
        keys += __shfl_xor_sync(0xffffffffu, keys, o);
        fp += __shfl_xor_sync(0xffffffffu, fp, o);
    }
    if ((threadIdx.x & 31) == 0 && keys) {
        atomicAdd(&fc->keys, keys);
        atomicAdd(&fc->fp, fp);
    }
}

// Hash mode when the estimate exceeds TDG_FILTER_FP_MAX. Balanced 8-bit-per-key words sit at
// 0.046-0.047 (C3, C4, C5; a hashed fill of any graph stays there) and rank order then wins
// 3.5 % of the peel; an unpermuted RMAT sits at 0.24 and rank order loses 21-32 %. Between the
// two points the break-even is near 0.07; every extra point of false positives is one more
// table sector per hundred probes.
#ifndef TDG_FILTER_FP_MAX
#define TDG_FILTER_FP_MAX 0.08
#endif
__global__ void k_fdecide(FilterCtl* fc) {
    const double est = fc->keys ? static_cast<double>(fc->fp) / 262144.0 / static_cast<double>(fc->keys) : 0.0;
    if (TDG_FMONO && est > TDG_FILTER_FP_MAX) {
        fc->hashed = 1;
        fc->fscale = kFilterHashMul;
    }
}

__global__ void k_fclear_if_hashed(unsigned long long* __restrict__ filt, uint64_t words, const FilterCtl* __restrict__ fc) {
    if (!fc->hashed) return;
    for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < words; i += uint64_t(gridDim.x) * blockDim.x)
        filt[i] = 0ull;
}

// Support-pass task list: each oriented edge a->b is owned by the endpoint whose N+ list
// is searched (the longer one; ties -> the source), and tasks are stored grouped by that
// owner so consecutive tasks search the same L1-resident list. Slot j of owner x with
// neighbour y is the task iff (x -> y and d+(x) >= d+(y)) or (y -> x and d+(y) < d+(x)).
__global__ void k_svalid(const uint32_t* __restrict__ adj, const uint32_t* __restrict__ src,
                         const uint32_t* __restrict__ opos, uint32_t* __restrict__ flag, uint64_t slots) {
    for (uint64_t j = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; j < slots;
         j += uint64_t(gridDim.x) * blockDim.x) {
        const uint32_t x = src[j], y = adj[j];
        const uint32_t dx = opos[x + 1] - opos[x], dy = opos[y + 1] - opos[y];
        flag[j] = flag[j] ? (dx >= dy ? 1u : 0u) : (dy < dx ? 1u : 0u);
    }
}

__global__ void k_sscatter(const uint32_t* __restrict__ src, const uint32_t* __restrict__ flag,
                           const uint32_t* __restrict__ pos, uint64_t slots, uint32_t* __restrict__ stask,
                           uint32_t* __restrict__ sx) {
    for (uint64_t j = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; j < slots;
         j += uint64_t(gridDim.x) * blockDim.x) {
        if (!flag[j]) continue;
        const uint32_t t = pos[j];
        stask[t] = static_cast<uint32_t>(j);
        sx[t] = src[j];
    }
}

// ---- internal edge ids (truss / support paths): id of edge {x,y} = its ORIENTED SLOT, the
// position of x->y (x before y in the (degree, id) order) in oadj. Edges of a vertex toward
// higher-ranked neighbours are then consecutive ids in list order, so the per-triangle state
// reads and atomics of a probe walk over a list are coalesced instead of random; results are
// scattered back to reference edge ids (oeid) at the end.
__global__ void k_r2i(const uint32_t* __restrict__ oeid, uint32_t m, uint32_t* __restrict__ r2i) {
    for (uint32_t t = blockIdx.x * blockDim.x + threadIdx.x; t < m; t += gridDim.x * blockDim.x) r2i[oeid[t]] = t;
}

__global__ void k_eid_internal(uint32_t* __restrict__ eid, const uint32_t* __restrict__ r2i, uint64_t slots) {
    for (uint64_t j = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; j < slots;
         j += uint64_t(gridDim.x) * blockDim.x)
        eid[j] = r2i[eid[j]];
}

__global__ void k_el_internal(const uint32_t* __restrict__ osrc, const uint32_t* __restrict__ oadj, uint32_t m,
                              uint2* __restrict__ el) {
    for (uint32_t t = blockIdx.x * blockDim.x + threadIdx.x; t < m; t += gridDim.x * blockDim.x)
        el[t] = make_uint2(osrc[t], oadj[t]);
}

// out[oeid[t]] = in[t] + add: an internal-id array back in reference edge-id order.
__global__ void k_to_ref(const uint32_t* __restrict__ oeid, const uint32_t* __restrict__ in, uint32_t m, uint32_t add,
                         uint32_t* __restrict__ out) {
    for (uint32_t t = blockIdx.x * blockDim.x + threadIdx.x; t < m; t += gridDim.x * blockDim.x)
        out[oeid[t]] = in[t] + add;
}

struct MaxOp {
    __device__ __forceinline__ uint32_t operator()(uint32_t a, uint32_t b) const { return a > b ? a : b; }
};

__global__ void k_stats(const uint32_t* __restrict__ off, const uint32_t* __restrict__ eo,
                        const uint32_t* __restrict__ opos, uint32_t n, StatsAcc* acc) {
    unsigned long long dmax = 0, sdd = 0, sdp = 0, sop = 0, s1 = 0;
    for (uint32_t u = blockIdx.x * blockDim.x + threadIdx.x; u < n; u += gridDim.x * blockDim.x) {
        unsigned long long d = off[u + 1] - off[u];
        unsigned long long dpn = off[u + 1] - eo[u];
        unsigned long long dp = opos[u + 1] - opos[u];
        unsigned long long dm = d - dp;
        dmax = d > dmax ? d : dmax;
        sdd += d * d;
        sdp += dpn * dpn;
        sop += dp * dp;
        s1 += dp * dp + dm * dp;
    }
    for (int o = 16; o > 0; o >>= 1) {
        unsigned long long t = __shfl_xor_sync(kFull, dmax, o);
        dmax = t > dmax ? t : dmax;
        sdd += __shfl_xor_sync(kFull, sdd, o);
        sdp += __shfl_xor_sync(kFull, sdp, o);
        sop += __shfl_xor_sync(kFull, sop, o);
        s1 += __shfl_xor_sync(kFull, s1, o);
    }
    if (lane_id() == 0) {
        atomicMax(&acc->d_max, dmax);
        atomicAdd(&acc->sum_deg_sq, sdd);
        atomicAdd(&acc->sum_dplus_sq, sdp);
        atomicAdd(&acc->deg_sum_dplus_sq, sop);
        atomicAdd(&acc->deg_s1, s1);
    }
}

}  // namespace

size_t build_cub_bytes(uint32_t n, uint32_t m) {
    size_t a = 0, b = 0, c = 0;
    const uint64_t slots = 2ull * m;
    cub::DeviceScan::InclusiveScan(nullptr, a, static_cast<uint32_t*>(nullptr), static_cast<uint32_t*>(nullptr),
                                   MaxOp(), slots > 0 ? slots : 1);
    cub::DeviceScan::ExclusiveSum(nullptr, b, static_cast<uint32_t*>(nullptr), static_cast<uint32_t*>(nullptr),
                                  static_cast<uint64_t>(n) + 1);
    cub::DeviceScan::ExclusiveSum(nullptr, c, static_cast<uint32_t*>(nullptr), static_cast<uint32_t*>(nullptr),
                                  slots + 1);
    size_t d = 0;
    cub::DoubleBuffer<uint32_t> keys(nullptr, nullptr), vals(nullptr, nullptr);
    cub::DeviceRadixSort::SortPairs(nullptr, d, keys, vals, m > 0 ? m : 1);
    c = c > d ? c : d;
    size_t r = a > b ? a : b;
    return r > c ? r : c;
}

cudaError_t launch_build(const BuildBufs& b, uint32_t n, uint32_t m, bool with_orientation,
                         cudaStream_t st, uint32_t* launches) {
    const uint64_t slots = 2ull * m;
    cudaError_t err;
    size_t tmp = b.cub_bytes;
    k_off_to_u32<<<grid_for(uint64_t(n) + 1), kThreads, 0, st>>>(b.off64, b.off, n + 1);
    (*launches)++;
    if (m == 0) return cudaGetLastError();
    if ((err = cudaMemsetAsync(b.src, 0, slots * sizeof(uint32_t), st)) != cudaSuccess) return err;
    k_row_start<<<grid_for(n), kThreads, 0, st>>>(b.off, n, b.src);
    (*launches)++;
    err = cub::DeviceScan::InclusiveScan(b.cub_tmp, tmp, b.src, b.src, MaxOp(), slots, st);
    if (err != cudaSuccess) return err;
    k_eo<<<grid_for(uint64_t(n) + 1), kThreads, 0, st>>>(b.off, b.adj, n, b.eo, b.up);
    (*launches)++;
    tmp = b.cub_bytes;
    err = cub::DeviceScan::ExclusiveSum(b.cub_tmp, tmp, b.up, b.P, static_cast<uint64_t>(n) + 1, st);
    if (err != cudaSuccess) return err;
    const unsigned gs = grid_for(slots) > 148u * 64u ? 148u * 64u : grid_for(slots);
    // transpose scratch: the orientation arrays are free until k_orient
    k_eid<<<gs, kThreads, 0, st>>>(b.off, b.adj, b.src, b.eo, b.P, slots, b.eid, b.el,
                                   with_orientation ? b.flag : nullptr, b.oadj, b.oeid);
    int bits = 1;
    while (bits < 32 && (1ull << bits) < n) bits++;
    tmp = b.cub_bytes;
    // double-buffered (no m-sized temporaries): the sorted ids end in either value buffer
    cub::DoubleBuffer<uint32_t> keys(b.oadj, b.osrc), vals(b.oeid, b.stask);
    err = cub::DeviceRadixSort::SortPairs(b.cub_tmp, tmp, keys, vals, m, 0, bits, st);
    if (err != cudaSuccess) return err;
    k_eid_lower<<<gs, kThreads, 0, st>>>(b.adj, b.src, b.P, vals.Current(), slots, b.eid);
    (*launches) += 2;
    if (!with_orientation) return cudaGetLastError();
    if ((err = cudaMemsetAsync(b.flag + slots, 0, sizeof(uint32_t), st)) != cudaSuccess) return err;
    tmp = b.cub_bytes;
    err = cub::DeviceScan::ExclusiveSum(b.cub_tmp, tmp, b.flag, b.pos, slots + 1, st);
    if (err != cudaSuccess) return err;
    k_orient<<<gs, kThreads, 0, st>>>(b.adj, b.eid, b.el, b.flag, b.pos, slots, b.oadj, b.oeid, b.osrc);
    k_opos<<<grid_for(uint64_t(n) + 1), kThreads, 0, st>>>(b.off, b.pos, n, b.opos);
    (*launches) += 2;
    // support task list (flag/pos reused: orientation flags are consumed above)
    k_svalid<<<gs, kThreads, 0, st>>>(b.adj, b.src, b.opos, b.flag, slots);
    tmp = b.cub_bytes;
    err = cub::DeviceScan::ExclusiveSum(b.cub_tmp, tmp, b.flag, b.pos, slots + 1, st);
    if (err != cudaSuccess) return err;
    k_sscatter<<<gs, kThreads, 0, st>>>(b.src, b.flag, b.pos, slots, b.stask, b.sx);
    k_opos<<<grid_for(uint64_t(n) + 1), kThreads, 0, st>>>(b.off, b.pos, n, b.sbeg);  // first task of each owner
    (*launches) += 3;
    return cudaGetLastError();
}

cudaError_t launch_internal_ids(const BuildBufs& b, uint32_t m, uint32_t* r2i, cudaStream_t st, uint32_t* launches) {
    if (m == 0) return cudaSuccess;
    const unsigned gm = grid_for(m) > 148u * 32u ? 148u * 32u : grid_for(m);
    const unsigned gs = grid_for(2ull * m) > 148u * 64u ? 148u * 64u : grid_for(2ull * m);
    k_r2i<<<gm, kThreads, 0, st>>>(b.oeid, m, r2i);
    k_eid_internal<<<gs, kThreads, 0, st>>>(b.eid, r2i, 2ull * m);
    k_el_internal<<<gm, kThreads, 0, st>>>(b.osrc, b.oadj, m, b.el);
    (*launches) += 3;
    return cudaGetLastError();
}

cudaError_t launch_to_ref(const uint32_t* oeid, const uint32_t* in, uint32_t m, uint32_t add, uint32_t* out,
                          cudaStream_t st, uint32_t* launches) {
    if (m == 0) return cudaSuccess;
    const unsigned gm = grid_for(m) > 148u * 32u ? 148u * 32u : grid_for(m);
    k_to_ref<<<gm, kThreads, 0, st>>>(oeid, in, m, add, out);
    (*launches)++;
    return cudaGetLastError();
}

cudaError_t launch_htab_fill(const uint32_t* off, const uint32_t* adj, const uint32_t* src, const uint32_t* eid,
                             uint32_t n, uint32_t m, uint32_t* hq, uint32_t* hbo, uint32_t* htab, void* cub_tmp,
                             size_t cub_bytes, cudaStream_t st, uint32_t* launches) {
    k_hsize<<<grid_for(uint64_t(n) + 1), kThreads, 0, st>>>(off, n, hq);
    (*launches)++;
    size_t tmp = cub_bytes;
    cudaError_t err = cub::DeviceScan::ExclusiveSum(cub_tmp, tmp, hq, hbo, static_cast<uint64_t>(n) + 1, st);
    if (err != cudaSuccess || m == 0) return err;
    const uint64_t slots = 2ull * m;
    if ((err = cudaMemsetAsync(htab, 0xff, htab_buckets(n, m) * 32, st)) != cudaSuccess) return err;
    const unsigned gs = grid_for(slots) > 148u * 64u ? 148u * 64u : grid_for(slots);
    const size_t smem = 8u * kHSmall * 8u * sizeof(uint32_t);
    // (a per-function attribute of the CURRENT device: set on every call, contexts may sit on
    // different devices)
    err = cudaFuncSetAttribute(k_hbuild_small, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    if (err != cudaSuccess) return err;
    k_hbuild_small<<<148u * 3u, 256, smem, st>>>(off, adj, eid, hbo, n, htab);
    k_hinsert<<<gs, kThreads, 0, st>>>(off, adj, src, eid, hbo, slots, htab);
    (*launches) += 2;
    return cudaGetLastError();
}

cudaError_t launch_filter_fill(const uint32_t* hbo, const uint32_t* adj, const uint32_t* src, uint32_t n, uint32_t m,
                               unsigned long long* filt, FilterCtl* fctl, cudaStream_t st, uint32_t* launches) {
    k_fctl_init<<<1, 1, 0, st>>>(fctl, n);
    (*launches)++;
    if (m == 0) return cudaGetLastError();
    const uint64_t words = filter_words(n, m);
    cudaError_t err = cudaMemsetAsync(filt, 0, words * sizeof(unsigned long long), st);
    if (err != cudaSuccess) return err;
    const uint64_t slots = 2ull * m;
    const unsigned gs = grid_for(slots) > 148u * 64u ? 148u * 64u : grid_for(slots);
    k_finsert<<<gs, kThreads, 0, st>>>(hbo, adj, src, slots, filt, fctl, 0);
    (*launches)++;
    if (TDG_FMONO) {  // rank mode unless the filters it produced pass too much (tdg_common.cuh)
        const unsigned gw = grid_for(words) > 148u * 16u ? 148u * 16u : grid_for(words);
        k_fstat<<<gw, kThreads, 0, st>>>(filt, words, fctl);
        k_fdecide<<<1, 1, 0, st>>>(fctl);
        k_fclear_if_hashed<<<gw, kThreads, 0, st>>>(filt, words, fctl);
        k_finsert<<<gs, kThreads, 0, st>>>(hbo, adj, src, slots, filt, fctl, 1);
        (*launches) += 4;
    }
    return cudaGetLastError();
}

cudaError_t launch_stats(const uint32_t* off, const uint32_t* eo, const uint32_t* opos, uint32_t n,
                         StatsAcc* acc, cudaStream_t st, uint32_t* launches) {
    cudaError_t err = cudaMemsetAsync(acc, 0, sizeof(StatsAcc), st);
    if (err != cudaSuccess) return err;
    unsigned g = grid_for(n) > 148u * 8u ? 148u * 8u : grid_for(n);
    k_stats<<<g, kThreads, 0, st>>>(off, eo, opos, n, acc);
    (*launches)++;
    return cudaGetLastError();
}

}  // namespace tdg
