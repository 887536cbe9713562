// ingest.cu — edge-list ingest on the GPU.
//
// Reference: canonicalize, /root/reference/proj/src/graph.cpp:19-71: labels are interned in
// first-appearance order over the raw stream (a then b for every pair), self loops are
// dropped, (min,max) pairs are sorted and deduplicated, and the CSR is filled so every
// list is ascending. B200 form, all sort/scan based (no hash map):
//   1. radix-sort the 2N label occurrences with their stream positions (stable, so each
//      label group starts with its first appearance);
//   2. group heads -> distinct labels; radix-sort the groups by first position -> the
//      reference's dense ids (rank of first appearance);
//   3. scatter ids back to stream positions, build canonical 64-bit keys, sort + unique;
//   4. degrees by atomics, scan -> offsets, scatter both directions, segmented sort of
//      every list (same CSR as the reference's ordered fill).

#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>
#include <cub/device/device_segmented_sort.cuh>
#include <cub/device/device_select.cuh>

#include "tdg_kernels.h"

namespace tdg {

namespace {

constexpr int kT = 256;

inline unsigned gfor(uint64_t items) {
    uint64_t b = (items + kT - 1) / kT;
    if (b == 0) b = 1;
    return static_cast<unsigned>(b > 148ull * 64 ? 148ull * 64 : b);
}

#define GRID_STRIDE(i, N) for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < (N); i += uint64_t(gridDim.x) * blockDim.x)

__global__ void k_iota_u32(uint32_t* a, uint64_t n) {
    GRID_STRIDE(i, n) a[i] = static_cast<uint32_t>(i);
}

__global__ void k_heads(const unsigned long long* __restrict__ key, uint64_t n, uint32_t* head) {
    GRID_STRIDE(i, n + 1) head[i] = (i < n && (i == 0 || key[i] != key[i - 1])) ? 1u : 0u;
}

// group g = gidx[i] (exclusive scan of heads); for heads: first position and label
__global__ void k_groups(const unsigned long long* __restrict__ key, const uint32_t* __restrict__ pos,
                         const uint32_t* __restrict__ head, const uint32_t* __restrict__ gidx, uint64_t n,
                         uint32_t* first_pos, unsigned long long* glabel, uint32_t* gid_seq) {
    GRID_STRIDE(i, n) {
        if (head[i]) {
            const uint32_t g = gidx[i];
            first_pos[g] = pos[i];
            glabel[g] = key[i];
            gid_seq[g] = g;
        }
    }
}

// rank of group g in first-appearance order: rank_of[gsorted[r]] = r; labels_out[r] = label
__global__ void k_rank(const uint32_t* __restrict__ gsorted, const unsigned long long* __restrict__ glabel,
                       uint64_t ng, uint32_t* rank_of, unsigned long long* labels_out) {
    GRID_STRIDE(r, ng) {
        const uint32_t g = gsorted[r];
        rank_of[g] = static_cast<uint32_t>(r);
        labels_out[r] = glabel[g];
    }
}

__global__ void k_ids(const uint32_t* __restrict__ pos, const uint32_t* __restrict__ gidx,
                      const uint32_t* __restrict__ rank_of, uint64_t n, uint32_t* vid) {
    GRID_STRIDE(i, n) vid[pos[i]] = rank_of[gidx[i + 1] - 1];  // group = inclusive head count - 1
}

// canonical keys; self loops become ~0 (sorted last, dropped by the count)
__global__ void k_keys(const uint32_t* __restrict__ vid, uint64_t npairs, unsigned long long* keys) {
    GRID_STRIDE(e, npairs) {
        const uint32_t a = vid[2 * e], b = vid[2 * e + 1];
        keys[e] = a == b ? ~0ull
                         : ((static_cast<unsigned long long>(a < b ? a : b) << 32) | (a < b ? b : a));
    }
}

__global__ void k_degrees(const unsigned long long* __restrict__ keys, const unsigned long long* __restrict__ nuniq,
                          uint32_t* deg) {
    const uint64_t m = *nuniq;
    GRID_STRIDE(k, m) {
        const unsigned long long key = keys[k];
        if (key == ~0ull) continue;
        atomicAdd(&deg[key >> 32], 1u);
        atomicAdd(&deg[key & 0xffffffffu], 1u);
    }
}

__global__ void k_fill(const unsigned long long* __restrict__ keys, const unsigned long long* __restrict__ nuniq,
                       uint32_t* cursor, uint32_t* nb) {
    const uint64_t m = *nuniq;
    GRID_STRIDE(k, m) {
        const unsigned long long key = keys[k];
        if (key == ~0ull) continue;
        const uint32_t u = static_cast<uint32_t>(key >> 32), v = static_cast<uint32_t>(key);
        nb[atomicAdd(&cursor[u], 1u)] = v;
        nb[atomicAdd(&cursor[v], 1u)] = u;
    }
}

}  // namespace

const char* g_ingest_step = "";

size_t ingest_cub_bytes(uint64_t npairs) {
    const uint64_t N = 2 * npairs > 0 ? 2 * npairs : 1;
    size_t a = 0, b = 0, c = 0, d = 0, e = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, a, static_cast<unsigned long long*>(nullptr),
                                    static_cast<unsigned long long*>(nullptr), static_cast<uint32_t*>(nullptr),
                                    static_cast<uint32_t*>(nullptr), N);
    cub::DeviceScan::ExclusiveSum(nullptr, b, static_cast<uint32_t*>(nullptr), static_cast<uint32_t*>(nullptr), N + 1);
    cub::DeviceRadixSort::SortKeys(nullptr, c, static_cast<unsigned long long*>(nullptr),
                                   static_cast<unsigned long long*>(nullptr), N);
    cub::DeviceSelect::Unique(nullptr, d, static_cast<unsigned long long*>(nullptr),
                              static_cast<unsigned long long*>(nullptr), static_cast<unsigned long long*>(nullptr), N);
    cub::DeviceSegmentedSort::SortKeys(nullptr, e, static_cast<uint32_t*>(nullptr), static_cast<uint32_t*>(nullptr),
                                       static_cast<int64_t>(N), static_cast<int64_t>(N),
                                       static_cast<uint32_t*>(nullptr), static_cast<uint32_t*>(nullptr) + 1);
    size_t r = a;
    for (size_t x : {b, c, d, e}) r = x > r ? x : r;
    return r;
}

// Phase 1: ids. Returns the number of distinct labels in *ng_host (synchronises).
cudaError_t launch_ingest(const IngestBufs& B, uint64_t npairs, cudaStream_t st, uint64_t* n_out, uint64_t* m_out,
                          uint32_t* launches) {
    const uint64_t N = 2 * npairs;
    cudaError_t err;
    size_t tmp;
    *n_out = 0;
    *m_out = 0;
    if (npairs == 0) return cudaSuccess;
// launch-error check per step (no sync); the name tells the caller where a failure surfaced
#define STEP(name) do { g_ingest_step = name; if ((err = cudaGetLastError()) != cudaSuccess) return err; } while (0)
    k_iota_u32<<<gfor(N), kT, 0, st>>>(B.pos_in, N);
    STEP("iota");
    tmp = B.cub_bytes;
    if ((err = cub::DeviceRadixSort::SortPairs(B.cub_tmp, tmp, B.labels_in, B.key_sorted, B.pos_in, B.pos_sorted, N, 0,
                                               64, st)) != cudaSuccess)
        return err;
    STEP("sort labels");
    k_heads<<<gfor(N + 1), kT, 0, st>>>(B.key_sorted, N, B.head);
    STEP("heads");
    tmp = B.cub_bytes;
    if ((err = cub::DeviceScan::ExclusiveSum(B.cub_tmp, tmp, B.head, B.gidx, N + 1, st)) != cudaSuccess) return err;
    uint32_t ng = 0;
    if ((err = cudaMemcpyAsync(&ng, B.gidx + N, 4, cudaMemcpyDeviceToHost, st)) != cudaSuccess) return err;
    if ((err = cudaStreamSynchronize(st)) != cudaSuccess) return err;
    k_groups<<<gfor(N), kT, 0, st>>>(B.key_sorted, B.pos_sorted, B.head, B.gidx, N, B.first_pos, B.glabel, B.gseq);
    tmp = B.cub_bytes;
    if ((err = cub::DeviceRadixSort::SortPairs(B.cub_tmp, tmp, B.first_pos, B.first_sorted, B.gseq, B.gsorted, ng, 0,
                                               32, st)) != cudaSuccess)
        return err;
    STEP("sort groups");
    k_rank<<<gfor(ng), kT, 0, st>>>(B.gsorted, B.glabel, ng, B.rank_of, B.labels_out);
    STEP("rank");
    k_ids<<<gfor(N), kT, 0, st>>>(B.pos_sorted, B.gidx, B.rank_of, N, B.vid);
    STEP("ids");
    k_keys<<<gfor(npairs), kT, 0, st>>>(B.vid, npairs, B.keys);
    STEP("keys");
    tmp = B.cub_bytes;
    if ((err = cub::DeviceRadixSort::SortKeys(B.cub_tmp, tmp, B.keys, B.keys_sorted, npairs, 0, 64, st)) != cudaSuccess)
        return err;
    tmp = B.cub_bytes;
    if ((err = cub::DeviceSelect::Unique(B.cub_tmp, tmp, B.keys_sorted, B.keys, B.nuniq, npairs, st)) != cudaSuccess)
        return err;
    STEP("unique");
    if ((err = cudaMemsetAsync(B.deg, 0, (uint64_t(ng) + 1) * 4, st)) != cudaSuccess) return err;
    k_degrees<<<gfor(npairs), kT, 0, st>>>(B.keys, B.nuniq, B.deg);
    tmp = B.cub_bytes;
    if ((err = cub::DeviceScan::ExclusiveSum(B.cub_tmp, tmp, B.deg, B.off, uint64_t(ng) + 1, st)) != cudaSuccess)
        return err;
    if ((err = cudaMemcpyAsync(B.cursor, B.off, uint64_t(ng) * 4 + 4, cudaMemcpyDeviceToDevice, st)) != cudaSuccess)
        return err;
    STEP("degrees");
    k_fill<<<gfor(npairs), kT, 0, st>>>(B.keys, B.nuniq, B.cursor, B.nb_tmp);
    STEP("fill");
    uint32_t slots = 0;
    if ((err = cudaMemcpyAsync(&slots, B.off + ng, 4, cudaMemcpyDeviceToHost, st)) != cudaSuccess) return err;
    if ((err = cudaStreamSynchronize(st)) != cudaSuccess) return err;
    if (slots) {
        tmp = B.cub_bytes;
        if ((err = cub::DeviceSegmentedSort::SortKeys(B.cub_tmp, tmp, B.nb_tmp, B.nb, slots, ng, B.off, B.off + 1,
                                                      st)) != cudaSuccess)
            return err;
    }
    (*launches) += 9;
    *n_out = ng;
    *m_out = slots / 2;
    return cudaGetLastError();
}

}  // namespace tdg
