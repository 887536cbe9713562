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
    k.aux = kNone;
    k.oa = g.opos[y];
    k.la = g.opos[y + 1] - k.oa;
    k.ob = g.opos[x];
    k.lb = g.opos[x + 1] - k.ob;
    return k;
}

// Edge ids are internal (build.cu launch_internal_ids): an edge's id IS its oriented slot
// (position in the N+ arrays). The owner-side slots of a task group are one contiguous,
// L2-resident N+(x) range and the probe-side slots of one task are consecutive, so the
// per-triangle atomics stay out of DRAM (reference-id-indexed atomics were random 2 GB
// read-modify-writes at C5).
struct SupportPolicy {
    const DevGraph& g;
    uint32_t* s;
    const uint32_t* elems;
    static constexpr bool kHasStaged = false;
    static constexpr int kUnroll = 1;
    __device__ ITask load(uint32_t t) const { return otask(g, t); }
    __device__ bool staged(const ITask&) const { return false; }
    __device__ void staged_range(const ITask&, uint32_t, uint32_t) const {}
    __device__ uint32_t find(const ITask& k, uint32_t x) const {
        const uint32_t p = lower_bound_u32(g.oadj + k.ob, k.lb, x);
        return (p < k.lb && g.oadj[k.ob + p] == x) ? p : kNone;
    }
    // A hit closes triangle {x, y, c}: the oriented slots of y->c and x->c get one atomic
    // each, the task's edge one per group of lanes sharing it (__match_any_sync).
    __device__ void visit(bool, bool hit, const ITask& k, uint32_t ja, uint32_t p) const {
        if (hit) {
            atomicAdd(&s[k.oa + ja], 1u);
            atomicAdd(&s[k.ob + p], 1u);
        }
        const uint32_t fm = __ballot_sync(kFull, hit);
        if (fm && hit) {
            const uint32_t grp = __match_any_sync(fm, k.id);
            if (lane_id() == static_cast<uint32_t>(__ffs(grp) - 1)) atomicAdd(&s[k.id], static_cast<uint32_t>(__popc(grp)));
        }
    }
};

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
    static constexpr bool kHasStaged = false;
    static constexpr int kUnroll = 1;
    __device__ ITask load(uint32_t t) const { return otask(g, t); }
    __device__ bool staged(const ITask&) const { return false; }
    __device__ void staged_range(const ITask&, uint32_t, uint32_t) const {}
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
    k_support<<<grid, kThreads, 0, st>>>(g, s, wpre, bsum, nchunks, ctl);
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
