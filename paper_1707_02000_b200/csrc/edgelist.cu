// edgelist.cu — text edge-list parsing on the GPU (the on-disk side of
// ingest).
//
// Reference: read_edge_list, /root/reference/proj/src/graph.cpp:152-200. Per physical line
// (1-based line numbers, blank lines counted): skip leading whitespace; blank lines and
// lines starting with '#' or '%' are skipped; otherwise exactly two unsigned decimal
// integers separated by whitespace (u64 arithmetic, wrapping like the reference's
// `v = v * 10 + digit`), then only whitespace. The first failing line in file order is
// reported: '-' where a number starts -> "negative vertex label"; anything else that is not
// a digit -> "expected two nonnegative integers"; text after the second number -> "trailing
// characters after edge". (A NUL byte is an ordinary non-digit character here; the
// reference's C-string appends of gzgets buffers would splice lines at it — binary input is
// outside both parsers' contract.)
//
// B200 form: the host inflates / reads the bytes (zlib, as the reference) and the GPU
// parses them. The text is cut into 256-byte segments, one thread each; a line belongs to
// the segment holding its first byte and is parsed whole by that thread (pass 1 counts the
// edges of every segment and the first error position; pass 2, after an exclusive scan of
// the counts, writes the (u, v) pairs in file order).

#include <cub/device/device_scan.cuh>

#include "tdg_kernels.h"

namespace tdg {

namespace {

constexpr int kT = 256;
constexpr uint32_t kSeg = 256;  // bytes per thread segment

__device__ __forceinline__ bool is_space(unsigned char c) { return c == ' ' || (c >= '\t' && c <= '\r'); }
__device__ __forceinline__ bool is_digit(unsigned char c) { return c >= '0' && c <= '9'; }

// Parse the line starting at `p` (its content ends at the first '\n' or `end`).
// Returns 0 = skipped, 1 = edge (a, b), 2 + ParseError = error; *next = start of the next line.
__device__ uint32_t parse_line(const unsigned char* __restrict__ t, uint64_t p, uint64_t end, uint64_t* next,
                               unsigned long long* a, unsigned long long* b) {
    uint64_t e = p;  // content end
    while (e < end && t[e] != '\n') e++;
    *next = e < end ? e + 1 : end;
    // (the reference's line includes its '\n', which is whitespace: same as ending here)
    uint64_t i = p;
    while (i < e && is_space(t[i])) i++;
    if (i == e || t[i] == '#' || t[i] == '%') return 0;
    unsigned long long v[2];
    for (int k = 0; k < 2; k++) {
        while (i < e && is_space(t[i])) i++;
        if (i < e && t[i] == '-') return 2 + kParseNegative;
        if (i == e || !is_digit(t[i])) return 2 + kParseExpected;
        unsigned long long x = 0;
        while (i < e && is_digit(t[i])) x = x * 10ull + static_cast<unsigned long long>(t[i++] - '0');
        v[k] = x;
    }
    while (i < e && is_space(t[i])) i++;
    if (i != e) return 2 + kParseTrailing;
    *a = v[0];
    *b = v[1];
    return 1;
}

// First line start inside segment [s0, s1): s0 itself if it starts a line, else after the
// first '\n' in the segment (or s1 if none: the segment lies inside one line).
__device__ __forceinline__ uint64_t first_line(const unsigned char* __restrict__ t, uint64_t s0, uint64_t s1) {
    if (s0 == 0 || t[s0 - 1] == '\n') return s0;
    uint64_t i = s0;
    while (i < s1 && t[i] != '\n') i++;
    return i < s1 ? i + 1 : s1;
}

// Pass 1: edges per segment; first error as atomicMin of (line start << 2 | code).
__global__ void k_parse_count(const unsigned char* __restrict__ t, uint64_t N, uint64_t nseg, uint32_t* __restrict__ cnt,
                              unsigned long long* err) {
    for (uint64_t sgi = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; sgi < nseg; sgi += uint64_t(gridDim.x) * blockDim.x) {
        const uint64_t s0 = sgi * kSeg, s1 = s0 + kSeg < N ? s0 + kSeg : N;
        uint32_t c = 0;
        for (uint64_t p = first_line(t, s0, s1); p < s1;) {
            uint64_t nx;
            unsigned long long a, b;
            const uint32_t r = parse_line(t, p, N, &nx, &a, &b);
            if (r == 1) c++;
            else if (r >= 2) {
                atomicMin(err, (static_cast<unsigned long long>(p) << 2) | (r - 2));
                break;
            }
            p = nx;
        }
        cnt[sgi] = c;
    }
}

// Pass 2: write the pairs of every segment at its exclusive-scan offset (file order).
__global__ void k_parse_write(const unsigned char* __restrict__ t, uint64_t N, uint64_t nseg,
                              const uint32_t* __restrict__ off, unsigned long long* __restrict__ pairs) {
    for (uint64_t sgi = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; sgi < nseg; sgi += uint64_t(gridDim.x) * blockDim.x) {
        const uint64_t s0 = sgi * kSeg, s1 = s0 + kSeg < N ? s0 + kSeg : N;
        uint64_t o = off[sgi];
        for (uint64_t p = first_line(t, s0, s1); p < s1;) {
            uint64_t nx;
            unsigned long long a, b;
            if (parse_line(t, p, N, &nx, &a, &b) == 1) {
                pairs[2 * o] = a;
                pairs[2 * o + 1] = b;
                o++;
            }
            p = nx;
        }
    }
}

inline unsigned grid_of(uint64_t items) {
    uint64_t b = (items + kT - 1) / kT;
    if (b == 0) b = 1;
    return static_cast<unsigned>(b > 148ull * 32 ? 148ull * 32 : b);
}

}  // namespace

size_t parse_scratch_bytes(uint64_t nbytes) {
    const uint64_t nseg = (nbytes + kSeg - 1) / kSeg + 1;
    size_t tmp = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, tmp, static_cast<uint32_t*>(nullptr), static_cast<uint32_t*>(nullptr), nseg);
    return 2 * nseg * sizeof(uint32_t) + tmp + 512;
}

cudaError_t launch_parse_count(const unsigned char* text, uint64_t nbytes, void* scratch, size_t scratch_bytes,
                               unsigned long long* err, cudaStream_t st, uint32_t* launches) {
    const uint64_t nseg = (nbytes + kSeg - 1) / kSeg;
    uint32_t* cnt = static_cast<uint32_t*>(scratch);
    uint32_t* off = cnt + nseg + 1;
    void* tmp = reinterpret_cast<void*>((reinterpret_cast<uintptr_t>(off + nseg + 1) + 255) & ~uintptr_t(255));
    size_t tb = scratch_bytes - 2 * (nseg + 1) * sizeof(uint32_t) - 256;
    cudaError_t e = cudaMemsetAsync(err, 0xff, sizeof(unsigned long long), st);
    if (e != cudaSuccess) return e;
    if (nseg == 0) return cudaSuccess;
    k_parse_count<<<grid_of(nseg), kT, 0, st>>>(text, nbytes, nseg, cnt, err);
    if ((e = cudaMemsetAsync(cnt + nseg, 0, sizeof(uint32_t), st)) != cudaSuccess) return e;
    e = cub::DeviceScan::ExclusiveSum(tmp, tb, cnt, off, nseg + 1, st);
    (*launches) += 2;
    return e;
}

cudaError_t launch_parse_write(const unsigned char* text, uint64_t nbytes, void* scratch, unsigned long long* pairs,
                               cudaStream_t st, uint32_t* launches) {
    const uint64_t nseg = (nbytes + kSeg - 1) / kSeg;
    if (nseg == 0) return cudaSuccess;
    const uint32_t* off = static_cast<const uint32_t*>(scratch) + nseg + 1;
    k_parse_write<<<grid_of(nseg), kT, 0, st>>>(text, nbytes, nseg, off, pairs);
    (*launches)++;
    return cudaGetLastError();
}

}  // namespace tdg
