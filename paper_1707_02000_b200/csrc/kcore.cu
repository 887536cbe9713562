// kcore.cu — vertex ordering before the path: k-core decomposition,
// coreness order and CSR relabelling on the GPU.
//
// Reference (paths relative to /root/reference/proj):
//   kcore_parallel  src/kcore.cpp:68-127  (ParK: level-synchronous vertex frontiers)
//   coreness_order  src/kcore.cpp:129-138 (stable sort of vertex ids by coreness)
//   reorder         src/graph.cpp:103-133 (relabel by perm, re-sort every adjacency list)
//
// kcore: one persistent cooperative kernel with the peel's structure — scan (live-vertex
// list compaction, level skipping via the minimum live degree), then per sub-level a
// work prefix over the frontier's degrees and the item-balanced engine of intersect.cuh
// (each item = one adjacency slot of a frontier vertex). The decrement rule is the
// reference's (kcore.cpp:105-110): only neighbours with degree > level are decremented; the
// thread that moves one to level+1 -> level appends it (unique); overshoots are repaired.
// Coreness is unique, so the result is bit-exact for any schedule.

#include <cooperative_groups.h>

#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>
#include <cub/device/device_segmented_sort.cuh>

#include "intersect.cuh"
#include "tdg_kernels.h"

namespace cg = cooperative_groups;

namespace tdg {

namespace {

constexpr int kT = 256;

struct KcCtr {
    uint32_t out_size, alive_size, min_d, piece_head;
};
struct KcCtl {
    KcCtr ph[3];
    uint32_t c_max, levels, sublevels, pad;
};

// Engine policy: task = frontier vertex v, items = its adjacency slots; every item is a
// "hit" carrying the neighbour w, and visit applies kcore.cpp:105-110 to it.
struct KcorePolicy {
    const uint32_t* off;
    const uint32_t* adj;
    const uint32_t* curr;
    uint32_t* deg;
    uint32_t level;
    KcCtr* out;
    uint32_t* next;
    const uint32_t* elems;
    static constexpr bool kFast = false;
    static constexpr int kUnroll = 1;
    __device__ ITask load(uint32_t t) const {
        const uint32_t v = curr[t];
        ITask k;
        k.id = v;
        k.oa = off[v];
        k.ob = 0;
        k.lb = 0;
        return k;
    }
    __device__ uint32_t find(const ITask&, uint32_t w) const { return w; }
    __device__ void visit(bool active, bool, const ITask&, uint32_t, uint32_t w) const {
        bool app = false;
        if (active && ld_relaxed(&deg[w]) > level) {
            const uint32_t prev = atomicSub(&deg[w], 1u);
            if (prev == level + 1) app = true;
            else if (prev <= level) atomicAdd(&deg[w], 1u);
        }
        const uint32_t p = warp_append(app, &out->out_size);
        if (app) next[p] = w;
    }
};

__device__ __forceinline__ void kc_reset(KcCtr* c) {
    c->out_size = 0;
    c->alive_size = 0;
    c->min_d = 0xffffffffu;
    c->piece_head = 0;
}

// scan (kcore.cpp:86-95): live vertices with deg == level -> curr (core = level);
// others -> live list, min degree reduced for level skipping.
__device__ void kc_scan(uint32_t* deg, uint32_t* core, uint32_t level, const uint32_t* Ain, uint32_t nA, bool implicit,
                        uint32_t* Aout, uint32_t* curr, KcCtr* ph) {
    const uint32_t lane = lane_id();
    uint32_t local_min = 0xffffffffu;
    for (uint64_t b0 = uint64_t(blockIdx.x) * kT + (threadIdx.x & ~31u); b0 < nA; b0 += uint64_t(gridDim.x) * kT) {
        const uint64_t i = b0 + lane;
        bool c = false, a = false;
        uint32_t v = 0;
        if (i < nA) {
            v = implicit ? static_cast<uint32_t>(i) : Ain[i];
            if (core[v] == kNone) {  // still unassigned (vertices peeled in sub-levels drop out here)
                const uint32_t d = ld_relaxed(&deg[v]);
                if (d == level) { c = true; core[v] = level; }
                else { a = true; local_min = d < local_min ? d : local_min; }
            }
        }
        const uint32_t pc = warp_append(c, &ph->out_size);
        if (c) curr[pc] = v;
        const uint32_t pa = warp_append(a, &ph->alive_size);
        if (a) Aout[pa] = v;
    }
    for (int o = 16; o > 0; o >>= 1) local_min = min(local_min, __shfl_xor_sync(kFull, local_min, o));
    if (lane == 0 && local_min != 0xffffffffu) atomicMin(&ph->min_d, local_min);
}

__device__ __forceinline__ uint32_t vld(const uint32_t* p) { return *reinterpret_cast<const volatile uint32_t*>(p); }

__global__ void __launch_bounds__(kT) k_kcore(const uint32_t* __restrict__ off, const uint32_t* __restrict__ adj,
                                              uint32_t n, uint32_t* deg, uint32_t* core, uint32_t* L0, uint32_t* L1,
                                              uint32_t* A0, uint32_t* A1, unsigned long long* wpre,
                                              unsigned long long* bsum, KcCtl* ctl) {
    cg::grid_group grid = cg::this_grid();
    __shared__ unsigned long long sboff[kMaxChunks + 1];
    const bool leader = blockIdx.x == 0 && threadIdx.x == 0;
    uint32_t* L[2] = {L0, L1};
    uint32_t* A[2] = {A0, A1};
    uint32_t j = 0, level = 0, nA = n, ai = 0, li = 0;
    bool implicit = true;
    while (true) {
        if (leader) kc_reset(&ctl->ph[(j + 1) % 3]);
        kc_scan(deg, core, level, A[ai], nA, implicit, A[ai ^ 1], L[li], &ctl->ph[j % 3]);
        grid.sync();
        j++;
        const KcCtr* r = &ctl->ph[(j - 1) % 3];
        uint32_t cs = vld(&r->out_size);
        nA = vld(&r->alive_size);
        const uint32_t mins = vld(&r->min_d);
        ai ^= 1;
        implicit = false;
        if (cs == 0) {
            if (nA == 0) break;
            level = mins;
            continue;
        }
        if (leader) { ctl->levels++; ctl->c_max = level; }
        while (true) {
            if (leader) { kc_reset(&ctl->ph[(j + 1) % 3]); ctl->sublevels++; }
            const uint32_t* curr = L[li];
            prep_items<kT>(cs, [&](uint32_t t) { const uint32_t v = curr[t]; return off[v + 1] - off[v]; }, wpre, bsum);
            grid.sync();
            KcorePolicy P{off, adj, curr, deg, level, &ctl->ph[j % 3], L[li ^ 1], adj};
            process_items<kT>(P, cs, wpre, bsum, gridDim.x, &ctl->ph[j % 3].piece_head, sboff);
            grid.sync();
            // frontier vertices are done: park them below every future level test
            j++;
            r = &ctl->ph[(j - 1) % 3];
            const uint32_t ns = vld(&r->out_size);
            // appended vertices get core = level now (they join curr at this level)
            for (uint32_t t = blockIdx.x * kT + threadIdx.x; t < ns; t += gridDim.x * kT) core[L[li ^ 1][t]] = level;
            li ^= 1;
            cs = ns;
            if (cs == 0) break;
        }
        level++;
    }
}

__global__ void k_kc_init(const uint32_t* __restrict__ off, uint32_t n, uint32_t* deg, uint32_t* core, KcCtl* ctl) {
    for (uint32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x) {
        deg[v] = off[v + 1] - off[v];
        core[v] = kNone;
    }
    if (blockIdx.x == 0 && threadIdx.x < 3) kc_reset(&ctl->ph[threadIdx.x]);
}

__global__ void k_iota(uint32_t* a, uint32_t n) {
    for (uint32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x) a[v] = v;
}

// perm[by_core[i]] = i (kcore.cpp:135-137)
__global__ void k_perm_from_order(const uint32_t* __restrict__ by_core, uint32_t n, uint32_t* perm) {
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) perm[by_core[i]] = i;
}

// bijection check (graph.cpp:106-113): count[perm[u]]++ must end all ones
__global__ void k_perm_check(const uint32_t* __restrict__ perm, uint32_t n, uint32_t* count, uint32_t* bad) {
    for (uint32_t u = blockIdx.x * blockDim.x + threadIdx.x; u < n; u += gridDim.x * blockDim.x) {
        const uint32_t p = perm[u];
        if (p >= n || atomicAdd(&count[p], 1u) != 0) *bad = 1;
    }
}

__global__ void k_newdeg(const uint32_t* __restrict__ off, const uint32_t* __restrict__ perm, uint32_t n,
                         uint32_t* ndeg) {
    for (uint32_t u = blockIdx.x * blockDim.x + threadIdx.x; u <= n; u += gridDim.x * blockDim.x)
        if (u < n) ndeg[perm[u]] = off[u + 1] - off[u]; else ndeg[n] = 0;
}

// warp per vertex: copy relabelled neighbours into the new row (sorted afterwards)
__global__ void k_relabel(const uint32_t* __restrict__ off, const uint32_t* __restrict__ adj,
                          const uint32_t* __restrict__ perm, const uint32_t* __restrict__ noff, uint32_t n,
                          uint32_t* nadj) {
    const uint32_t lane = threadIdx.x & 31u;
    for (uint32_t u = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; u < n; u += (gridDim.x * blockDim.x) >> 5) {
        const uint32_t o = off[u], d = off[u + 1] - o, no = noff[perm[u]];
        for (uint32_t j = lane; j < d; j += 32) nadj[no + j] = perm[adj[o + j]];
    }
}

}  // namespace

size_t kcore_cub_bytes(uint32_t n, uint32_t m) {
    size_t a = 0, b = 0, c = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, a, static_cast<uint32_t*>(nullptr), static_cast<uint32_t*>(nullptr),
                                    static_cast<uint32_t*>(nullptr), static_cast<uint32_t*>(nullptr), n > 0 ? n : 1);
    cub::DeviceScan::ExclusiveSum(nullptr, b, static_cast<uint32_t*>(nullptr), static_cast<uint32_t*>(nullptr),
                                  static_cast<uint64_t>(n) + 1);
    cub::DeviceSegmentedSort::SortKeys(nullptr, c, static_cast<uint32_t*>(nullptr), static_cast<uint32_t*>(nullptr),
                                       2 * static_cast<int64_t>(m) > 0 ? 2 * static_cast<int64_t>(m) : 1, n > 0 ? n : 1,
                                       static_cast<uint32_t*>(nullptr), static_cast<uint32_t*>(nullptr) + 1);
    size_t r = a > b ? a : b;
    return r > c ? r : c;
}

cudaError_t launch_kcore(const uint32_t* off, const uint32_t* adj, uint32_t n, const KcoreBufs& b, int sm_count,
                         cudaStream_t st, uint32_t* launches, uint32_t* c_max_dev) {
    cudaError_t err = cudaMemsetAsync(b.ctl, 0, sizeof(KcCtl), st);
    if (err != cudaSuccess || n == 0) return err;
    k_kc_init<<<148 * 4, kT, 0, st>>>(off, n, b.deg, b.core, static_cast<KcCtl*>(b.ctl));
    int per_sm = 0;
    err = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_kcore, kT, 0);
    if (err != cudaSuccess) return err;
    unsigned blocks = static_cast<unsigned>(sm_count * (per_sm < 1 ? 1 : per_sm));
    if (blocks > kMaxChunks) blocks = kMaxChunks;
    KcCtl* ctl = static_cast<KcCtl*>(b.ctl);
    void* args[] = {const_cast<uint32_t**>(&off), const_cast<uint32_t**>(&adj), &n, const_cast<uint32_t**>(&b.deg),
                    const_cast<uint32_t**>(&b.core), const_cast<uint32_t**>(&b.L0), const_cast<uint32_t**>(&b.L1),
                    const_cast<uint32_t**>(&b.A0), const_cast<uint32_t**>(&b.A1),
                    const_cast<unsigned long long**>(&b.wpre), const_cast<unsigned long long**>(&b.bsum), &ctl};
    err = cudaLaunchCooperativeKernel(reinterpret_cast<void*>(k_kcore), dim3(blocks), dim3(kT), args, 0, st);
    (*launches) += 2;
    if (err != cudaSuccess) return err;
    return cudaMemcpyAsync(c_max_dev, &ctl->c_max, 4, cudaMemcpyDeviceToDevice, st);
}

cudaError_t launch_coreness_order(const uint32_t* core, uint32_t n, const KcoreBufs& b, uint32_t* perm,
                                  cudaStream_t st, uint32_t* launches) {
    if (n == 0) return cudaSuccess;
    k_iota<<<148 * 4, kT, 0, st>>>(b.L0, n);
    size_t tmp = b.cub_bytes;
    // radix sort is stable: ids that tie on coreness keep ascending order (std::stable_sort)
    cudaError_t err = cub::DeviceRadixSort::SortPairs(b.cub_tmp, tmp, core, b.A0, b.L0, b.L1, n, 0, 32, st);
    if (err != cudaSuccess) return err;
    k_perm_from_order<<<148 * 4, kT, 0, st>>>(b.L1, n, perm);
    (*launches) += 2;
    return cudaGetLastError();
}

cudaError_t launch_reorder(const uint32_t* off, const uint32_t* adj, const uint32_t* perm, uint32_t n, uint32_t m,
                           const KcoreBufs& b, uint32_t* noff, uint32_t* nadj, uint32_t* bad, cudaStream_t st,
                           uint32_t* launches) {
    cudaError_t err = cudaMemsetAsync(b.deg, 0, size_t(n + 1) * 4, st);
    if (err != cudaSuccess) return err;
    if ((err = cudaMemsetAsync(bad, 0, 4, st)) != cudaSuccess) return err;
    if (n == 0) return cudaMemsetAsync(noff, 0, 4, st);
    k_perm_check<<<148 * 4, kT, 0, st>>>(perm, n, b.deg, bad);
    k_newdeg<<<148 * 4, kT, 0, st>>>(off, perm, n, b.core);
    size_t tmp = b.cub_bytes;
    err = cub::DeviceScan::ExclusiveSum(b.cub_tmp, tmp, b.core, noff, static_cast<uint64_t>(n) + 1, st);
    if (err != cudaSuccess) return err;
    (*launches) += 2;
    if (m == 0) return cudaGetLastError();
    k_relabel<<<148 * 16, kT, 0, st>>>(off, adj, perm, noff, n, b.tmp_adj);
    tmp = b.cub_bytes;
    err = cub::DeviceSegmentedSort::SortKeys(b.cub_tmp, tmp, b.tmp_adj, nadj, 2 * static_cast<int64_t>(m), n, noff,
                                             noff + 1, st);
    (*launches) += 1;
    if (err != cudaSuccess) return err;
    return cudaGetLastError();
}

}  // namespace tdg
