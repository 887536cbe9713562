// support.cu — per-edge triangle counts (the support pass).
//
// Reference: support_am4, /root/reference/proj/src/triangle.cpp:26-61 (ordered pivot with a
// dense per-thread mark array X[n] and three relaxed fetch_adds per triangle). B200
// design: every triangle {a,b,c} with a < b < c in the degree order (d, id) is found
// exactly once, at oriented edge a->b, as c in N+(a) ∩ N+(b). The shorter oriented list
// is walked with coalesced loads and each element is binary-searched in the longer one
// (no X[n] scratch, work min(d+a, d+b)*log). Per triangle: the (a,b) count is
// aggregated across the warp with __match_any_sync and one atomicAdd per group; the
// other two edges get one atomicAdd each. Edges whose probe count exceeds kBigWork are
// split into kPiece-item pieces pulled from a queue so hub-adjacent edges spread over
// all SMs; the rest are packed 32 per warp with an in-warp prefix sum.

#include "tdg_kernels.h"

namespace tdg {

namespace {

constexpr int kThreads = 256;

struct OTask {
    uint32_t euv;          // edge id of a->b
    uint32_t oa, la;       // probe list (shorter)
    uint32_t ob, lb;       // searched list (longer)
};

__device__ __forceinline__ OTask otask(const DevGraph& g, uint32_t t) {
    const uint32_t u = g.osrc[t], v = g.oadj[t];
    const uint32_t ou = g.opos[u], du = g.opos[u + 1] - ou;
    const uint32_t ov = g.opos[v], dv = g.opos[v + 1] - ov;
    OTask k;
    k.euv = g.oeid[t];
    if (du <= dv) { k.oa = ou; k.la = du; k.ob = ov; k.lb = dv; }
    else          { k.oa = ov; k.la = dv; k.ob = ou; k.lb = du; }
    return k;
}

__global__ void k_support_classify(DevGraph g, uint2* __restrict__ queue, SupportCtl* ctl) {
    for (uint32_t t = blockIdx.x * blockDim.x + threadIdx.x; t < g.m; t += gridDim.x * blockDim.x) {
        OTask k = otask(g, t);
        if (k.la > kBigWork)
            if (!queue_push(&ctl->big, queue, t, k.la)) ctl->overflow = 1;
    }
}

// One probe: item j of task k. Returns true if it closed a triangle (and issued the two
// peer-edge increments).
__device__ __forceinline__ bool probe(const DevGraph& g, uint32_t* __restrict__ s, uint32_t oa,
                                      uint32_t ob, uint32_t lb, uint32_t j) {
    const uint32_t x = g.oadj[oa + j];
    const uint32_t p = lower_bound_u32(g.oadj + ob, lb, x);
    if (p < lb && g.oadj[ob + p] == x) {
        atomicAdd(&s[g.oeid[oa + j]], 1u);
        atomicAdd(&s[g.oeid[ob + p]], 1u);
        return true;
    }
    return false;
}

// Add one per found triangle to s[euv], aggregated over lanes sharing euv.
__device__ __forceinline__ void add_own(uint32_t* s, bool found, uint32_t euv) {
    const uint32_t fm = __ballot_sync(kFull, found);
    if (!fm) return;
    if (found) {
        const uint32_t grp = __match_any_sync(fm, euv);
        if (lane_id() == static_cast<uint32_t>(__ffs(grp) - 1)) atomicAdd(&s[euv], static_cast<uint32_t>(__popc(grp)));
    }
}

__global__ void __launch_bounds__(kThreads) k_support(DevGraph g, uint32_t* __restrict__ s,
                                                      const uint2* __restrict__ queue, SupportCtl* ctl) {
    const uint32_t lane = lane_id();
    const unsigned long long big = *reinterpret_cast<volatile unsigned long long*>(&ctl->big);
    const uint32_t nq = static_cast<uint32_t>(big >> 32), npieces = static_cast<uint32_t>(big);

    // 1) pieces of heavy edges
    while (true) {
        uint32_t p = 0;
        if (lane == 0) p = atomicAdd(&ctl->piece_head, 1u);
        p = __shfl_sync(kFull, p, 0);
        if (p >= npieces) break;
        const uint32_t qi = queue_find(queue, nq, p);
        const uint2 qe = queue[qi];
        const OTask k = otask(g, qe.x);
        const uint32_t begin = (p - qe.y) * kPiece;
        const uint32_t end = min(k.la, begin + kPiece);
        for (uint32_t j0 = begin; j0 < end; j0 += 32) {
            const uint32_t j = j0 + lane;
            const bool found = (j < end) && probe(g, s, k.oa, k.ob, k.lb, j);
            add_own(s, found, k.euv);
        }
    }
    // 2) light edges, 32 per warp, `grab` warp-batches per dynamic grab
    const uint32_t nwarps = (gridDim.x * blockDim.x) >> 5;
    uint32_t grab = static_cast<uint32_t>(g.m / (32ull * 8ull * nwarps));
    grab = grab < 1 ? 1 : (grab > 16 ? 16 : grab);
    while (true) {
        uint32_t b = 0;
        if (lane == 0) b = atomicAdd(&ctl->batch_head, 1u);
        b = __shfl_sync(kFull, b, 0);
        const uint64_t tg = uint64_t(b) * 32 * grab;
        if (tg >= g.m) break;
        for (uint32_t sub = 0; sub < grab; sub++) {
            const uint64_t t0 = tg + uint64_t(sub) * 32;
            if (t0 >= g.m) break;
            const uint32_t t = static_cast<uint32_t>(t0) + lane;
            OTask k{0, 0, 0, 0, 0};
            uint32_t w = 0;
            if (t < g.m) {
                k = otask(g, t);
                w = k.la <= kBigWork ? k.la : 0;
            }
            const uint32_t incl = warp_incl_scan(w);
            const uint32_t excl = incl - w;
            const uint32_t total = __shfl_sync(kFull, incl, 31);
            for (uint32_t base = 0; base < total; base += 32) {
                const uint32_t item = base + lane;
                const uint32_t own = warp_owner(excl, item);
                const uint32_t j = item - __shfl_sync(kFull, excl, own);
                const uint32_t oa = __shfl_sync(kFull, k.oa, own);
                const uint32_t ob = __shfl_sync(kFull, k.ob, own);
                const uint32_t lb = __shfl_sync(kFull, k.lb, own);
                const uint32_t euv = __shfl_sync(kFull, k.euv, own);
                const bool found = (item < total) && probe(g, s, oa, ob, lb, j);
                add_own(s, found, euv);
            }
        }
    }
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

cudaError_t launch_support(const DevGraph& g, uint32_t* s, uint2* queue, SupportCtl* ctl,
                           int sm_count, cudaStream_t st, uint32_t* launches) {
    cudaError_t err = cudaMemsetAsync(ctl, 0, sizeof(SupportCtl), st);
    if (err != cudaSuccess) return err;
    if (g.m == 0) return cudaSuccess;
    if ((err = cudaMemsetAsync(s, 0, size_t(g.m) * sizeof(uint32_t), st)) != cudaSuccess) return err;
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_support, kThreads, 0);
    if (per_sm < 1) per_sm = 1;
    const unsigned grid = static_cast<unsigned>(sm_count * per_sm);
    k_support_classify<<<grid, kThreads, 0, st>>>(g, queue, ctl);
    k_support<<<grid, kThreads, 0, st>>>(g, s, queue, ctl);
    k_support_sum<<<grid, kThreads, 0, st>>>(s, g.m, ctl);
    (*launches) += 3;
    return cudaGetLastError();
}

}  // namespace tdg
