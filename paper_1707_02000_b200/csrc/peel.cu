// peel.cu — the level-synchronous PKT peel as ONE persistent cooperative kernel.
//
// Reference (paths relative to /root/reference/proj):
//   scan              src/truss_parallel.cpp:21-37
//   process_sublevel  src/truss_parallel.cpp:39-104 (try_decrement :49-63)
//   truss_parallel    src/truss_parallel.cpp:106-150 (level / sub-level driver)
//   BufferedAppender  include/trussdec/appender.hpp:12-40
//
// Semantics kept exactly: level = support value; curr(l) =
// {unprocessed e : s[e]==l}; each e1=(u,v) in curr visits every w in N(u)∩N(v),
// skips triangles with a processed peer, and for each peer target decrements only if
// s[target] > l and (other peer not in curr or e1 < other); the thread whose atomicSub
// returns l+1 appends target to next; a return <= l is repaired with +1; trussness =
// final support + 2. Sub-level sets (hence nsl) and results are therefore identical to
// the reference for any schedule.
//
// B200 design differences:
//  * Device-resident loop: all levels and sub-levels run inside one cooperative launch;
//    a sub-level costs one grid barrier (the reference pays 2 OpenMP barriers + a fork).
//  * Flags -> stamps: stamp[e] = index of the sub-level in which e is (or was) curr.
//    processed(e) <=> 0 < stamp < K, in_curr(e) <=> stamp == K, next <=> stamp == K+1.
//    Entering next is the single stamp store by the appending thread, so the
//    reference's epilogue pass over curr (:97-102) and the flag swaps vanish.
//  * No dense X[n] mark array (MarkScratchPool, truss_parallel.hpp:55-59): N(u)∩N(v) is
//    computed by walking the shorter live list and binary-searching the longer one.
//  * Level 0 needs no intersections: s[e1] >= #live triangles of e1, so s==0 edges have
//    none (the reference still marks/scans their lists).
//  * Levels with no edges are skipped: the scan that finds curr empty also returns the
//    minimum live support, which is the next non-empty level. Each scan compacts the
//    live-edge list, so later levels stream only survivors.
//  * Load balance: edges with more than kBigWork probes are split into kPiece pieces in a
//    queue built while the edge is appended; the rest are packed 32 per warp.

#include <cooperative_groups.h>

#include "tdg_kernels.h"

namespace cg = cooperative_groups;

namespace tdg {

namespace {

constexpr int kPeelThreads = 256;
constexpr int kScanItems = 8;

struct PTask {
    uint32_t e1;
    uint32_t oa, la;  // probe list (shorter live list)
    uint32_t ob, lb;  // searched list
    uint32_t b;       // vertex owning the searched list
};

__device__ __forceinline__ PTask ptask(const DevGraph& g, uint32_t e1) {
    const uint2 p = g.el[e1];
    const uint32_t du = g.dl[p.x], dv = g.dl[p.y];
    PTask k;
    k.e1 = e1;
    if (du <= dv) { k.oa = g.off[p.x]; k.la = du; k.ob = g.off[p.y]; k.lb = dv; k.b = p.y; }
    else          { k.oa = g.off[p.y]; k.la = dv; k.ob = g.off[p.x]; k.lb = du; k.b = p.x; }
    return k;
}

__device__ __forceinline__ void reset_ctr(PhaseCtr* c) {
    c->big = 0;
    c->out_size = 0;
    c->alive_size = 0;
    c->min_s = 0xffffffffu;
    c->piece_head = 0;
    c->batch_head = 0;
}

// try_decrement, truss_parallel.cpp:49-63. Returns target if this thread moved it to the
// level (it then owns the append), else kNone.
__device__ __forceinline__ uint32_t try_dec(uint32_t* s, uint32_t* stamp, uint32_t level, uint32_t K,
                                            uint32_t e1, uint32_t target, uint32_t other,
                                            bool other_in_curr) {
    if (ld_relaxed(&s[target]) <= level) return kNone;   // :52
    if (other_in_curr && e1 >= other) return kNone;      // :53 ownership
    const uint32_t prev = atomicSub(&s[target], 1u);     // :54
    if (prev == level + 1) {                             // :55-57
        st_relaxed(&stamp[target], K + 1);
        return target;
    }
    if (prev <= level) atomicAdd(&s[target], 1u);        // :58-62 repair
    return kNone;
}

// One triangle probe of e1 (truss_parallel.cpp:80-88): x = item j of the probe list.
__device__ __forceinline__ void peel_probe(const DevGraph& g, uint32_t* s, uint32_t* stamp,
                                           uint32_t level, uint32_t K, uint32_t e1, uint32_t oa,
                                           uint32_t ob, uint32_t lb, uint32_t b, uint32_t j,
                                           uint32_t& out0, uint32_t& out1) {
    const uint32_t x = g.adj[oa + j];
    if (x == b) return;
    const uint32_t p = lower_bound_u32(g.adj + ob, lb, x);
    if (p >= lb || g.adj[ob + p] != x) return;
    const uint32_t ea = g.eid[oa + j], eb = g.eid[ob + p];
    const uint32_t sa = ld_relaxed(&stamp[ea]), sb = ld_relaxed(&stamp[eb]);
    if ((sa != 0 && sa < K) || (sb != 0 && sb < K)) return;  // :85 processed peer
    out0 = try_dec(s, stamp, level, K, e1, ea, eb, sb == K);  // :86
    out1 = try_dec(s, stamp, level, K, e1, eb, ea, sa == K);  // :87
}

__device__ __forceinline__ void classify_push(const DevGraph& g, uint32_t e, PhaseCtr* out, uint2* q,
                                              PeelCtl* ctl) {
    const PTask k = ptask(g, e);
    if (k.la > kBigWork)
        if (!queue_push(&out->big, q, e, k.la)) ctl->overflow = 1;
}

// Append up to two targets per lane to next (warp-aggregated) and queue heavy ones.
__device__ __forceinline__ void emit(const DevGraph& g, uint32_t o0, uint32_t o1, PhaseCtr* out,
                                     uint32_t* next, uint2* qnext, PeelCtl* ctl) {
    const uint32_t p0 = warp_append(o0 != kNone, &out->out_size);
    if (o0 != kNone) { next[p0] = o0; classify_push(g, o0, out, qnext, ctl); }
    const uint32_t p1 = warp_append(o1 != kNone, &out->out_size);
    if (o1 != kNone) { next[p1] = o1; classify_push(g, o1, out, qnext, ctl); }
}

// scan (truss_parallel.cpp:21-37) over the live-edge list A: survivors with s==level
// become curr (stamp K), the others are compacted into Aout and their minimum support is
// reduced for level skipping. Block-aggregated appends: 2 atomics per 2048 edges.
__device__ void phase_scan(const DevGraph& g, uint32_t* s, uint32_t* stamp, uint32_t level,
                           uint32_t K, const uint32_t* Ain, uint32_t nA, bool implicit,
                           uint32_t* Aout, uint32_t* curr, uint2* q, PhaseCtr* ph, PeelCtl* ctl,
                           bool classify) {
    __shared__ uint32_t sh_c[kPeelThreads / 32], sh_a[kPeelThreads / 32];
    __shared__ uint32_t sh_bc, sh_ba;
    const uint32_t tid = threadIdx.x, lane = lane_id(), wid = tid >> 5;
    const uint64_t tile = uint64_t(kPeelThreads) * kScanItems;
    uint32_t local_min = 0xffffffffu;
    for (uint64_t t0 = uint64_t(blockIdx.x) * tile; t0 < nA; t0 += uint64_t(gridDim.x) * tile) {
        uint32_t es[kScanItems];
        uint32_t kind = 0;  // 2 bits per item: 1 = curr, 2 = alive
        uint32_t cc = 0, ca = 0;
#pragma unroll
        for (int k = 0; k < kScanItems; k++) {
            const uint64_t i = t0 + uint64_t(k) * kPeelThreads + tid;
            es[k] = 0;
            if (i < nA) {
                const uint32_t e = implicit ? static_cast<uint32_t>(i) : Ain[i];
                es[k] = e;
                if (ld_relaxed(&stamp[e]) == 0) {
                    const uint32_t sv = ld_relaxed(&s[e]);
                    if (sv == level) {
                        st_relaxed(&stamp[e], K);
                        kind |= 1u << (2 * k);
                        cc++;
                    } else {
                        kind |= 2u << (2 * k);
                        ca++;
                        local_min = sv < local_min ? sv : local_min;
                    }
                }
            }
        }
        const uint32_t ic = warp_incl_scan(cc), ia = warp_incl_scan(ca);
        if (lane == 31) { sh_c[wid] = ic; sh_a[wid] = ia; }
        __syncthreads();
        if (tid == 0) {
            uint32_t rc = 0, ra = 0;
            for (int w = 0; w < kPeelThreads / 32; w++) {
                uint32_t c = sh_c[w], a = sh_a[w];
                sh_c[w] = rc; sh_a[w] = ra;
                rc += c; ra += a;
            }
            sh_bc = rc ? atomicAdd(&ph->out_size, rc) : 0;
            sh_ba = ra ? atomicAdd(&ph->alive_size, ra) : 0;
        }
        __syncthreads();
        uint32_t pc = sh_bc + sh_c[wid] + ic - cc, pa = sh_ba + sh_a[wid] + ia - ca;
#pragma unroll
        for (int k = 0; k < kScanItems; k++) {
            const uint32_t f = (kind >> (2 * k)) & 3u;
            if (f == 1u) {
                curr[pc++] = es[k];
                if (classify && level > 0) classify_push(g, es[k], ph, q, ctl);
            } else if (f == 2u) {
                Aout[pa++] = es[k];
            }
        }
        __syncthreads();
    }
    for (int o = 16; o > 0; o >>= 1) local_min = min(local_min, __shfl_xor_sync(kFull, local_min, o));
    if (lane == 0 && local_min != 0xffffffffu) atomicMin(&ph->min_s, local_min);
}

// process_sublevel (truss_parallel.cpp:39-104) for curr[0..cs): heavy edges from the
// piece queue first, then light edges 32 per warp, `grab` batches per dynamic grab.
__device__ void phase_process(const DevGraph& g, uint32_t* s, uint32_t* stamp, uint32_t level,
                              uint32_t K, const uint32_t* curr, uint32_t cs, const uint2* q,
                              uint32_t nq, uint32_t npieces, PhaseCtr* ph, uint32_t* next,
                              uint2* qnext, uint32_t grab, PeelCtl* ctl, bool l0_shortcut) {
    const uint32_t lane = lane_id();
    while (true) {
        uint32_t p = 0;
        if (lane == 0) p = atomicAdd(&ph->piece_head, 1u);
        p = __shfl_sync(kFull, p, 0);
        if (p >= npieces) break;
        const uint2 qe = q[queue_find(q, nq, p)];
        const PTask k = ptask(g, qe.x);
        const uint32_t begin = (p - qe.y) * kPiece;
        const uint32_t end = min(k.la, begin + kPiece);
        for (uint32_t j0 = begin; j0 < end; j0 += 32) {
            const uint32_t j = j0 + lane;
            uint32_t o0 = kNone, o1 = kNone;
            if (j < end) peel_probe(g, s, stamp, level, K, k.e1, k.oa, k.ob, k.lb, k.b, j, o0, o1);
            emit(g, o0, o1, ph, next, qnext, ctl);
        }
    }
    if (l0_shortcut && level == 0) return;  // s[e1]==0 => no live triangle on e1
    const uint32_t span = 32u * grab;
    while (true) {
        uint32_t b = 0;
        if (lane == 0) b = atomicAdd(&ph->batch_head, 1u);
        b = __shfl_sync(kFull, b, 0);
        const uint64_t t0 = uint64_t(b) * span;
        if (t0 >= cs) break;
        for (uint32_t sub = 0; sub < grab; sub++) {
            const uint64_t tb = t0 + uint64_t(sub) * 32;
            if (tb >= cs) break;
            const uint64_t i = tb + lane;
            PTask k{0, 0, 0, 0, 0, 0};
            uint32_t w = 0;
            if (i < cs) {
                k = ptask(g, curr[i]);
                w = k.la <= kBigWork ? k.la : 0;
            }
            const uint32_t incl = warp_incl_scan(w);
            const uint32_t excl = incl - w;
            const uint32_t total = __shfl_sync(kFull, incl, 31);
            for (uint32_t base = 0; base < total; base += 32) {
                const uint32_t item = base + lane;
                const uint32_t own = warp_owner(excl, item);
                const uint32_t j = item - __shfl_sync(kFull, excl, own);
                const uint32_t e1 = __shfl_sync(kFull, k.e1, own);
                const uint32_t oa = __shfl_sync(kFull, k.oa, own);
                const uint32_t ob = __shfl_sync(kFull, k.ob, own);
                const uint32_t lb = __shfl_sync(kFull, k.lb, own);
                const uint32_t bv = __shfl_sync(kFull, k.b, own);
                uint32_t o0 = kNone, o1 = kNone;
                if (item < total) peel_probe(g, s, stamp, level, K, e1, oa, ob, lb, bv, j, o0, o1);
                emit(g, o0, o1, ph, next, qnext, ctl);
            }
        }
    }
}

__device__ __forceinline__ uint32_t grab_for(uint32_t cs, uint32_t nwarps) {
    uint32_t g = cs / (32u * 8u * (nwarps ? nwarps : 1u));
    return g < 1 ? 1 : (g > 16 ? 16 : g);
}

__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

__device__ __forceinline__ uint32_t vload(const uint32_t* p) { return *reinterpret_cast<const volatile uint32_t*>(p); }
__device__ __forceinline__ unsigned long long vload64(const unsigned long long* p) {
    return *reinterpret_cast<const volatile unsigned long long*>(p);
}

// The whole truss_parallel level loop (truss_parallel.cpp:119-144) in one launch.
__global__ void __launch_bounds__(kPeelThreads) k_peel(DevGraph g, PeelBufs pb) {
    cg::grid_group grid = cg::this_grid();
    PeelCtl* ctl = pb.ctl;
    const bool leader = blockIdx.x == 0 && threadIdx.x == 0;
    const uint32_t nwarps = (gridDim.x * blockDim.x) >> 5;
    uint32_t j = 0, level = 0, K = 1, nA = g.m, ai = 0, li = 0;
    bool implicit = true;
    unsigned long long t_prev = leader ? gtimer() : 0;
    while (true) {
        // ---- scan at `level` (one grid barrier)
        if (leader) { reset_ctr(&ctl->ph[(j + 1) % 3]); ctl->scans++; }
        phase_scan(g, pb.s, pb.stamp, level, K, pb.A[ai], nA, implicit, pb.A[ai ^ 1], pb.L[li], pb.Q[li],
                   &ctl->ph[j % 3], ctl, true);
        grid.sync();
        if (leader) { const unsigned long long t = gtimer(); ctl->scan_ns += t - t_prev; t_prev = t; }
        j++;
        const PhaseCtr* r = &ctl->ph[(j - 1) % 3];
        uint32_t cs = vload(&r->out_size);
        nA = vload(&r->alive_size);
        const uint32_t mins = vload(&r->min_s);
        unsigned long long big = vload64(&r->big);
        ai ^= 1;
        implicit = false;
        if (cs == 0) {
            if (nA == 0) break;
            level = mins;  // skip empty levels
            continue;
        }
        // ---- sub-levels (one grid barrier each)
        while (true) {
            if (leader) {
                reset_ctr(&ctl->ph[(j + 1) % 3]);
                if (level < pb.nsl_cap) pb.nsl[level]++; else ctl->overflow = 1;
                ctl->sublevels++;
                ctl->levels_len = level + 1;
            }
            phase_process(g, pb.s, pb.stamp, level, K, pb.L[li], cs, pb.Q[li], static_cast<uint32_t>(big >> 32),
                          static_cast<uint32_t>(big), &ctl->ph[j % 3], pb.L[li ^ 1], pb.Q[li ^ 1],
                          grab_for(cs, nwarps), ctl, true);
            grid.sync();
            if (leader) { const unsigned long long t = gtimer(); ctl->proc_ns += t - t_prev; t_prev = t; }
            j++;
            K++;
            r = &ctl->ph[(j - 1) % 3];
            cs = vload(&r->out_size);
            big = vload64(&r->big);
            li ^= 1;
            if (cs == 0) break;
        }
        level++;
    }
    if (leader) ctl->final_stamp = K;
}

__global__ void k_peel_init(const uint32_t* __restrict__ off, uint32_t n, uint32_t* __restrict__ dl,
                            PeelCtl* ctl) {
    for (uint32_t u = blockIdx.x * blockDim.x + threadIdx.x; u < n; u += gridDim.x * blockDim.x)
        dl[u] = off[u + 1] - off[u];
    if (blockIdx.x == 0 && threadIdx.x < 3) reset_ctr(&ctl->ph[threadIdx.x]);
}

__global__ void k_finalize(const uint32_t* __restrict__ s, uint32_t m, uint32_t* __restrict__ truss,
                           PeelCtl* ctl) {
    uint32_t mx = 0;
    for (uint32_t e = blockIdx.x * blockDim.x + threadIdx.x; e < m; e += gridDim.x * blockDim.x) {
        const uint32_t t = s[e] + 2;  // truss_parallel.cpp:146-148
        truss[e] = t;
        mx = t > mx ? t : mx;
    }
    for (int o = 16; o > 0; o >>= 1) mx = max(mx, __shfl_xor_sync(kFull, mx, o));
    if (lane_id() == 0 && mx) atomicMax(&ctl->t_max, mx);
}

// ---- step functions on reference-style flag arrays (tests/test_truss_parallel.cpp) ----
__global__ void k_step_stamps(const uint8_t* __restrict__ processed, const uint8_t* __restrict__ in_curr,
                              uint32_t m, uint32_t* __restrict__ stamp, PeelCtl* ctl) {
    for (uint32_t e = blockIdx.x * blockDim.x + threadIdx.x; e < m; e += gridDim.x * blockDim.x)
        stamp[e] = processed[e] ? 1u : ((in_curr && in_curr[e]) ? 2u : 0u);
    if (blockIdx.x == 0 && threadIdx.x < 3) reset_ctr(&ctl->ph[threadIdx.x]);
}

__global__ void k_step_scan(DevGraph g, PeelBufs pb, uint32_t level) {
    phase_scan(g, pb.s, pb.stamp, level, 2, pb.A[0], g.m, true, pb.A[1], pb.L[0], pb.Q[0], &pb.ctl->ph[0], pb.ctl,
               false);
}

__global__ void k_step_scan_flags(const uint32_t* __restrict__ curr, PeelCtl* ctl, uint8_t* in_curr) {
    const uint32_t cs = ctl->ph[0].out_size;
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < cs; i += gridDim.x * blockDim.x)
        in_curr[curr[i]] = 1;
}

__global__ void k_step_classify(DevGraph g, PeelBufs pb, uint32_t cs) {
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < cs; i += gridDim.x * blockDim.x)
        classify_push(g, pb.L[0][i], &pb.ctl->ph[0], pb.Q[0], pb.ctl);
}

__global__ void k_step_process(DevGraph g, PeelBufs pb, uint32_t cs, uint32_t level) {
    const unsigned long long big = pb.ctl->ph[0].big;
    phase_process(g, pb.s, pb.stamp, level, 2, pb.L[0], cs, pb.Q[0], static_cast<uint32_t>(big >> 32),
                  static_cast<uint32_t>(big), &pb.ctl->ph[1], pb.L[1], pb.Q[1], 1, pb.ctl, false);
}

// Epilogue (truss_parallel.cpp:97-102) + in_next flags for the appended edges.
__global__ void k_step_process_flags(const uint32_t* __restrict__ curr, uint32_t cs,
                                     const uint32_t* __restrict__ next, PeelCtl* ctl, uint8_t* in_curr,
                                     uint8_t* in_next, uint8_t* processed) {
    const uint32_t ns = ctl->ph[1].out_size;
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < cs || i < ns; i += gridDim.x * blockDim.x) {
        if (i < cs) { processed[curr[i]] = 1; in_curr[curr[i]] = 0; }
        if (i < ns) in_next[next[i]] = 1;
    }
}

}  // namespace

cudaError_t launch_peel(const DevGraph& g, const PeelBufs& p, int sm_count, cudaStream_t st,
                        uint32_t* launches) {
    cudaError_t err = cudaMemsetAsync(p.ctl, 0, sizeof(PeelCtl), st);
    if (err != cudaSuccess) return err;
    if ((err = cudaMemsetAsync(p.nsl, 0, size_t(p.nsl_cap) * sizeof(uint32_t), st)) != cudaSuccess) return err;
    if (g.m == 0) return cudaSuccess;
    if ((err = cudaMemsetAsync(p.stamp, 0, size_t(g.m) * sizeof(uint32_t), st)) != cudaSuccess) return err;
    k_peel_init<<<148 * 4, 256, 0, st>>>(g.off, g.n, g.dl, p.ctl);
    int per_sm = 0;
    err = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_peel, kPeelThreads, 0);
    if (err != cudaSuccess) return err;
    if (per_sm < 1) return cudaErrorLaunchOutOfResources;
    dim3 grid(static_cast<unsigned>(sm_count * per_sm)), block(kPeelThreads);
    DevGraph gg = g;
    PeelBufs pp = p;
    void* args[] = {&gg, &pp};
    err = cudaLaunchCooperativeKernel(reinterpret_cast<void*>(k_peel), grid, block, args, 0, st);
    (*launches) += 2;
    return err;
}

cudaError_t launch_finalize(const uint32_t* s, uint32_t m, uint32_t* truss, PeelCtl* ctl, cudaStream_t st,
                            uint32_t* launches) {
    if (m == 0) return cudaSuccess;
    k_finalize<<<148 * 4, 256, 0, st>>>(s, m, truss, ctl);
    (*launches)++;
    return cudaGetLastError();
}

cudaError_t launch_step_scan(const DevGraph& g, const PeelBufs& p, uint32_t level, const uint8_t* processed,
                             uint8_t* in_curr, int sm_count, cudaStream_t st) {
    k_step_stamps<<<sm_count * 2, 256, 0, st>>>(processed, nullptr, g.m, p.stamp, p.ctl);
    k_step_scan<<<sm_count, kPeelThreads, 0, st>>>(g, p, level);
    k_step_scan_flags<<<sm_count, 256, 0, st>>>(p.L[0], p.ctl, in_curr);
    return cudaGetLastError();
}

cudaError_t launch_step_process(const DevGraph& g, const PeelBufs& p, uint32_t level, uint32_t curr_size,
                                uint8_t* in_curr, uint8_t* in_next, uint8_t* processed, int sm_count,
                                cudaStream_t st) {
    k_peel_init<<<sm_count, 256, 0, st>>>(g.off, g.n, g.dl, p.ctl);
    k_step_stamps<<<sm_count * 2, 256, 0, st>>>(processed, in_curr, g.m, p.stamp, p.ctl);
    k_step_classify<<<sm_count, 256, 0, st>>>(g, p, curr_size);
    k_step_process<<<sm_count * 2, kPeelThreads, 0, st>>>(g, p, curr_size, level);
    k_step_process_flags<<<sm_count, 256, 0, st>>>(p.L[0], curr_size, p.L[1], p.ctl, in_curr, in_next, processed);
    return cudaGetLastError();
}

}  // namespace tdg
