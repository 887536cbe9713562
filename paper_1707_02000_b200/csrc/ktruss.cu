// ktruss.cu — maximal k-trusses as connected components.
//
// Reference: ktruss_subgraphs, /root/reference/proj/src/truss_serial.cpp:176-210: union-find
// over vertices joined by edges with truss >= k; components are then numbered in the order
// their first qualifying edge appears in edge-id order, and each lists its edges ascending.
// B200 form: lock-free union-find with atomicCAS hooking of the larger root under the
// smaller (ECL-CC style) over all qualifying edges in parallel, pointer jumping, then the
// component order is recovered exactly: first[root] = atomicMin(edge id), one scan over the
// "edge is its component's first edge" flags ranks the components. Output: comp[e] per edge
// (kNone below k); the host groups edges ascending per component.

#include <cub/device/device_scan.cuh>

#include "tdg_kernels.h"

namespace tdg {

namespace {

constexpr int kThreads = 256;

__device__ __forceinline__ uint32_t uf_find(uint32_t* parent, uint32_t x) {
    uint32_t p = ld_relaxed(&parent[x]);
    while (p != x) {
        const uint32_t gp = ld_relaxed(&parent[p]);
        if (gp != p) atomicCAS(&parent[x], p, gp);  // path halving (benign race)
        x = p;
        p = gp;
    }
    return x;
}

__global__ void k_kt_init(uint32_t* parent, uint32_t n, uint32_t* first) {
    for (uint32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x) {
        parent[v] = v;
        first[v] = kNone;
    }
}

__global__ void k_kt_hook(const uint2* __restrict__ el, const uint32_t* __restrict__ truss, uint32_t m, uint32_t k,
                          uint32_t* parent) {
    for (uint32_t e = blockIdx.x * blockDim.x + threadIdx.x; e < m; e += gridDim.x * blockDim.x) {
        if (truss[e] < k) continue;
        const uint2 p = el[e];
        uint32_t ru = uf_find(parent, p.x), rv = uf_find(parent, p.y);
        while (ru != rv) {
            if (ru > rv) { const uint32_t t = ru; ru = rv; rv = t; }
            const uint32_t old = atomicCAS(&parent[rv], rv, ru);  // hook larger root under smaller
            if (old == rv) break;
            rv = uf_find(parent, old);
            ru = uf_find(parent, ru);
        }
    }
}

__global__ void k_kt_first(const uint2* __restrict__ el, const uint32_t* __restrict__ truss, uint32_t m, uint32_t k,
                           uint32_t* parent, uint32_t* first, uint32_t* root_of_edge) {
    for (uint32_t e = blockIdx.x * blockDim.x + threadIdx.x; e < m; e += gridDim.x * blockDim.x) {
        uint32_t r = kNone;
        if (truss[e] >= k) {
            r = uf_find(parent, el[e].x);
            atomicMin(&first[r], e);
        }
        root_of_edge[e] = r;
    }
}

__global__ void k_kt_flag(const uint32_t* __restrict__ root_of_edge, const uint32_t* __restrict__ first, uint32_t m,
                          uint32_t* flag) {
    for (uint32_t e = blockIdx.x * blockDim.x + threadIdx.x; e <= m; e += gridDim.x * blockDim.x) {
        const uint32_t r = e < m ? root_of_edge[e] : kNone;
        flag[e] = (r != kNone && first[r] == e) ? 1u : 0u;
    }
}

__global__ void k_kt_label(const uint32_t* __restrict__ root_of_edge, const uint32_t* __restrict__ first,
                           const uint32_t* __restrict__ rank, uint32_t m, uint32_t* comp) {
    for (uint32_t e = blockIdx.x * blockDim.x + threadIdx.x; e < m; e += gridDim.x * blockDim.x) {
        const uint32_t r = root_of_edge[e];
        comp[e] = r == kNone ? kNone : rank[first[r]];
    }
}

}  // namespace

size_t ktruss_cub_bytes(uint32_t m) {
    size_t b = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, b, static_cast<uint32_t*>(nullptr), static_cast<uint32_t*>(nullptr),
                                  static_cast<uint64_t>(m) + 1);
    return b;
}

cudaError_t launch_ktruss(const uint2* el, const uint32_t* truss, uint32_t n, uint32_t m, uint32_t k,
                          const KtrussBufs& b, cudaStream_t st, uint32_t* launches) {
    const unsigned g = 148 * 8;
    k_kt_init<<<g, kThreads, 0, st>>>(b.parent, n, b.first);
    k_kt_hook<<<g, kThreads, 0, st>>>(el, truss, m, k, b.parent);
    k_kt_first<<<g, kThreads, 0, st>>>(el, truss, m, k, b.parent, b.first, b.root_of_edge);
    k_kt_flag<<<g, kThreads, 0, st>>>(b.root_of_edge, b.first, m, b.flag);
    size_t tmp = b.cub_bytes;
    cudaError_t err = cub::DeviceScan::ExclusiveSum(b.cub_tmp, tmp, b.flag, b.rank, static_cast<uint64_t>(m) + 1, st);
    if (err != cudaSuccess) return err;
    k_kt_label<<<g, kThreads, 0, st>>>(b.root_of_edge, b.first, b.rank, m, b.comp);
    (*launches) += 5;
    return cudaGetLastError();
}

}  // namespace tdg
