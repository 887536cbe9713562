// intersect.cuh — work-balanced, warp-cooperative probe engine shared by the support pass
// (support.cu) and the peel's sub-levels (peel.cu).
//
// A "task" probes every element x of its list A = elems[oa .. oa+la) against the
// neighbour -> edge-id hash table of one vertex (tdg_common.cuh: 1-2 dependent accesses
// per probe instead of a log2(d)-step binary search). The tasks' la items are laid out on
// one global axis by a chunked exclusive prefix sum (prep_items); process_items cuts the
// axis into equal pieces pulled dynamically by warps, so skew in list lengths never leaves
// a warp with a long tail. Inside a piece a warp walks 32-item windows over consecutive
// tasks: lane k holds task i+k and each lane finds its item's owner with a 5-step shuffle
// search. Policy (per caller) supplies `load(t)`, `elems`, `kUnroll` (U items per lane per
// step) and either `run<U>(act, task, ja)` (U > 1: the policy issues the U probe chains'
// loads together) or, for U = 1, `find(task, x)` (edge id of the searched side or kNone) and
// `visit(active, hit, task, ja, e)`; all 32 lanes call them together (warp collectives ok).
#pragma once

#include <type_traits>

#include "tdg_common.cuh"

namespace tdg {

// Policy::flush() (optional): called by process_items after every piece, so a policy may
// buffer work across engine steps (the peel's candidate queue).
template <class P, class = void>
struct has_flush : std::false_type {};
template <class P>
struct has_flush<P, std::void_t<decltype(std::declval<P&>().flush())>> : std::true_type {};

// Policy::kRunForm (optional, true): the policy takes whole steps through run<U> even at U = 1.
template <class P, class = void>
struct has_run_form : std::false_type {};
template <class P>
struct has_run_form<P, std::enable_if_t<P::kRunForm>> : std::true_type {};

// A task as the engine carries it between lanes (its item count lives in the work prefix).
struct ITask {
    uint32_t id;      // peel: e1 ; support: edge id of the oriented edge a->b
    uint32_t oa;      // probe list A = elems[oa ..)
    uint32_t ob, lb;  // searched side (peel: table bucket offset / count; support: N+ list)
};

__device__ __forceinline__ ITask shfl_task(const ITask& k, uint32_t src) {
    ITask r;
    r.id = __shfl_sync(kFull, k.id, src);
    r.oa = __shfl_sync(kFull, k.oa, src);
    r.ob = __shfl_sync(kFull, k.ob, src);
    r.lb = __shfl_sync(kFull, k.lb, src);
    return r;
}

__device__ __forceinline__ unsigned long long shfl64(unsigned long long v, uint32_t src) {
    const uint32_t lo = __shfl_sync(kFull, static_cast<uint32_t>(v), src);
    const uint32_t hi = __shfl_sync(kFull, static_cast<uint32_t>(v >> 32), src);
    return (static_cast<unsigned long long>(hi) << 32) | lo;
}

// Largest lane t with held_t <= key (held non-decreasing over lanes); 0 if none.
__device__ __forceinline__ uint32_t warp_search_le(uint32_t held, uint32_t key) {
    uint32_t lo = 0;
#pragma unroll
    for (uint32_t step = 16; step > 0; step >>= 1) {
        const uint32_t v = __shfl_sync(kFull, held, lo + step);
        if (v <= key) lo += step;
    }
    return lo;
}

template <int kThreads>
__device__ __forceinline__ unsigned long long block_excl_scan64(unsigned long long v, unsigned long long& total) {
    constexpr int kW = kThreads / 32;
    __shared__ unsigned long long sh[kW];
    const uint32_t lane = lane_id(), wid = threadIdx.x >> 5;
    unsigned long long x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const unsigned long long t = shfl64(x, lane >= static_cast<uint32_t>(o) ? lane - o : lane);
        if (lane >= static_cast<uint32_t>(o)) x += t;
    }
    if (lane == 31) sh[wid] = x;
    __syncthreads();
    unsigned long long woff = 0, tot = 0;
#pragma unroll
    for (int w = 0; w < kW; w++) {
        const unsigned long long t = sh[w];
        if (w < static_cast<int>(wid)) woff += t;
        tot += t;
    }
    __syncthreads();
    total = tot;
    return woff + x - v;
}

__device__ __forceinline__ uint32_t chunk_len(uint32_t ntasks, uint32_t nchunks) {
    return (ntasks + nchunks - 1) / nchunks;
}

// Block b of a gridDim.x-block grid owns task chunk b: writes the chunk-local exclusive
// prefix of the tasks' work (probe counts) and the chunk total bsum[b].
template <int kThreads, class WorkF>
__device__ void prep_items(uint32_t ntasks, WorkF&& work, unsigned long long* wpre, unsigned long long* bsum) {
    const uint32_t CH = chunk_len(ntasks, gridDim.x);
    const uint64_t lo = uint64_t(blockIdx.x) * CH;
    const uint64_t hi = lo + CH < ntasks ? lo + CH : ntasks;
    unsigned long long run = 0;
    for (uint64_t t0 = lo; t0 < hi; t0 += kThreads) {
        const uint64_t t = t0 + threadIdx.x;
        const unsigned long long w = t < hi ? static_cast<unsigned long long>(work(static_cast<uint32_t>(t))) : 0ull;
        unsigned long long tot;
        const unsigned long long ex = block_excl_scan64<kThreads>(w, tot);
        if (t < hi) wpre[t] = run + ex;
        run += tot;
    }
    if (threadIdx.x == 0) bsum[blockIdx.x] = run;
}

// Largest task t with start(t) <= x (start = sboff[t / CH] + wpre[t]).
__device__ __forceinline__ uint32_t task_at(unsigned long long x, uint32_t ntasks, const unsigned long long* wpre,
                                            const unsigned long long* sboff, uint32_t nchunks, uint32_t CH) {
    uint32_t clo = 0, chi = nchunks;
    while (chi - clo > 1) {
        const uint32_t mid = (clo + chi) >> 1;
        if (sboff[mid] <= x) clo = mid; else chi = mid;
    }
    uint32_t ilo = clo * CH, ihi = min(ntasks, (clo + 1) * CH);
    const unsigned long long rel = x - sboff[clo];
    while (ihi - ilo > 1) {
        const uint32_t mid = (ilo + ihi) >> 1;
        if (wpre[mid] <= rel) ilo = mid; else ihi = mid;
    }
    return ilo;
}

// One warp processes work items [x0, x1) of the global axis, starting at the task i that
// contains x0 (see the file comment).
template <class Policy>
__device__ __forceinline__ void run_items(Policy& P, unsigned long long x0, unsigned long long x1, uint32_t i0,
                                          uint32_t ntasks, const unsigned long long* wpre,
                                          const unsigned long long* sboff, uint32_t CH) {
    const uint32_t lane = lane_id();
    uint32_t i = i0;
    // lanes hold tasks i..i+31 (start st); end_held = start of task i+32
    uint32_t held = kNone;
    ITask k{0, 0, 0, 0};
    unsigned long long st = ~0ull, end_held = ~0ull;
    // fast-path cache: lane 0's task broadcast to every lane, valid while i == c_task
    ITask c0{0, 0, 0, 0};
    unsigned long long c_st = 0;
    uint32_t c_task = kNone;
    for (unsigned long long base = x0; base < x1;) {
        if (held != i) {
            // Slide the held window: tasks already held move down by `adv` lanes with
            // shuffles; only the lanes past the old window load (each task descriptor
            // costs ~6 random loads, so reloading all 32 per step dominated traffic).
            const uint32_t adv = (held != kNone && i > held) ? i - held : 32u;
            if (adv < 32) {
                k.id = __shfl_down_sync(kFull, k.id, adv);
                k.oa = __shfl_down_sync(kFull, k.oa, adv);
                k.ob = __shfl_down_sync(kFull, k.ob, adv);
                k.lb = __shfl_down_sync(kFull, k.lb, adv);
                const uint32_t lo = __shfl_down_sync(kFull, static_cast<uint32_t>(st), adv);
                const uint32_t hi = __shfl_down_sync(kFull, static_cast<uint32_t>(st >> 32), adv);
                st = (static_cast<unsigned long long>(hi) << 32) | lo;
            }
            const uint32_t t = i + lane;
            if (lane + adv >= 32) {
                if (t < ntasks) {
                    k = P.load(t);
                    st = sboff[t / CH] + wpre[t];
                } else {
                    st = ~0ull;
                }
            }
            unsigned long long s32 = ~0ull;
            if (lane == 31 && t + 1 < ntasks) s32 = sboff[(t + 1) / CH] + wpre[t + 1];
            end_held = shfl64(s32, 31);
            held = i;
        }
        const unsigned long long limit = x1 < end_held ? x1 : end_held;
        const uint32_t relk = st <= base ? 0u
                              : (st - base > 0xffffffffull ? 0xffffffffu : static_cast<uint32_t>(st - base));
        constexpr int U = Policy::kUnroll;
        // Fast path (Policy::kFast): when lane 0's task covers the whole step (the next task
        // starts at least 32U items on), every item belongs to it and its descriptor, broadcast
        // once, is reused while the warp stays inside it — no per-item owner search. (The
        // peel's U = 3 probe loop is register-bound and loses more to the cache than it saves.)
        const uint32_t r1 = Policy::kFast ? __shfl_sync(kFull, relk, 1) : 0u;
        const bool one = Policy::kFast && r1 >= 32u * U;
        if constexpr (U > 1 || has_run_form<Policy>::value) {
            // U items per lane per step (item base + lane + 32q): the policy issues their
            // independent loads together, so each lane keeps U probe chains in flight.
            ITask ko[U];
            uint32_t ja[U];
            bool act[U];
            if (one) {
                if (c_task != i) { c0 = shfl_task(k, 0); c_st = shfl64(st, 0); c_task = i; }
#pragma unroll
                for (int q = 0; q < U; q++) {
                    const unsigned long long x = base + lane + 32u * q;
                    ko[q] = c0;
                    act[q] = x < limit;
                    ja[q] = act[q] ? static_cast<uint32_t>(x - c_st) : 0u;
                }
            } else {
#pragma unroll
                for (int q = 0; q < U; q++) {
                    const uint32_t key = lane + 32u * q;
                    const uint32_t own = warp_search_le(relk, key);
                    const unsigned long long so = shfl64(st, own);
                    ko[q] = shfl_task(k, own);
                    const unsigned long long x = base + key;
                    act[q] = x < limit;
                    ja[q] = act[q] ? static_cast<uint32_t>(x - so) : 0u;
                }
            }
            P.template run<U>(act, ko, ja);
        } else {
            if (one && c_task != i) { c0 = shfl_task(k, 0); c_st = shfl64(st, 0); c_task = i; }
            const uint32_t own = one ? 0u : warp_search_le(relk, lane);
            const unsigned long long so = one ? c_st : shfl64(st, own);
            const ITask ko = one ? c0 : shfl_task(k, own);
            const unsigned long long x = base + lane;
            uint32_t ja = 0, e = kNone;
            const bool active = x < limit;
            if (active) {
                ja = static_cast<uint32_t>(x - so);
                e = P.find(ko, P.elems[ko.oa + ja]);
            }
            P.visit(active, e != kNone, ko, ja, e);
        }
        const unsigned long long nb = base + 32u * U < limit ? base + 32u * U : limit;
        i = (nb >= end_held) ? i + 32
            : (one && nb - base < r1) ? i  // still inside lane 0's task
                                      : i + warp_search_le(relk, static_cast<uint32_t>(nb - base));
        base = nb;
    }
}

#ifndef TDG_PIECE_ROUND
#define TDG_PIECE_ROUND 1  // round pieces to whole 32*U-item steps
#endif
#ifndef TDG_MIN_PIECE
#define TDG_MIN_PIECE 32ull  // smallest piece (items): bounds per-piece overhead in small phases
#endif
#ifndef TDG_PIECES
#define TDG_PIECES 4ull  // work pieces per warp in process_items (dynamic; smaller = shorter tail)
#endif
#ifndef TDG_GUIDED
#define TDG_GUIDED 1  // guided pieces: tiers of nwarps pieces whose size halves per tier (short tail)
#endif

// Guided piece schedule over W items for nw warps: tier t holds nw pieces of S0 >> t items
// (S0 = W / 2nw, whole engine steps), so each tier covers about half of what the previous
// one left; pieces never shrink below `minp` and the last tier repeats that size. Piece p ->
// [*x0, *x1) (*x0 >= W: no piece). Dynamic pulling of a piece counter keeps it balanced; the
// phase tail is one minimum piece instead of one W / (4 nw) piece.
__device__ __forceinline__ void guided_piece(unsigned long long p, unsigned long long W, uint32_t nw,
                                             unsigned long long S0, unsigned long long minp,
                                             unsigned long long* x0, unsigned long long* x1) {
    unsigned long long base = 0, S = S0 > minp ? S0 : minp;
    while (S > minp && p >= nw) {
        base += nw * S;
        p -= nw;
        S = (S >> 1) > minp ? (S >> 1) : minp;
    }
    *x0 = base + p * S;
    *x1 = *x0 + S < W ? *x0 + S : W;
}

// sboff[c] = exclusive prefix of the chunk totals bsum[0..nchunks) (block-wide; smem
// sboff holds >= nchunks+1 entries); returns the total work.
template <int kThreads>
__device__ unsigned long long chunk_offsets(const unsigned long long* bsum, uint32_t nchunks, unsigned long long* sboff) {
    const uint32_t per = (nchunks + kThreads - 1) / kThreads;
    const uint32_t c0 = threadIdx.x * per;
    unsigned long long loc = 0;
    for (uint32_t c = c0; c < c0 + per && c < nchunks; c++) loc += bsum[c];
    unsigned long long tot;
    unsigned long long run = block_excl_scan64<kThreads>(loc, tot);
    for (uint32_t c = c0; c < c0 + per && c < nchunks; c++) {
        sboff[c] = run;
        run += bsum[c];
    }
    if (threadIdx.x == 0) sboff[nchunks] = tot;
    __syncthreads();
    return sboff[nchunks];
}

// Process all work of tasks [0, ntasks) (see file comment). `piece_head` must be 0 on
// entry; bsum/wpre come from prep_items over a `nchunks`-block grid. smem: sboff holds
// >= nchunks+1 entries. Returns the total work W.
template <int kThreads, class Policy>
__device__ unsigned long long process_items(Policy& P, uint32_t ntasks, const unsigned long long* wpre,
                              const unsigned long long* bsum, uint32_t nchunks, uint32_t* piece_head,
                              unsigned long long* sboff) {
    chunk_offsets<kThreads>(bsum, nchunks, sboff);
    const unsigned long long W = sboff[nchunks];
    if (W == 0) return 0;
    const uint32_t CH = chunk_len(ntasks, nchunks);
    const uint32_t nwarps = (gridDim.x * kThreads) >> 5;
    constexpr unsigned long long kStep = TDG_PIECE_ROUND ? 32ull * Policy::kUnroll : 32ull;
    const uint32_t lane = lane_id();
    if (TDG_GUIDED) {
        unsigned long long S0 = (W + 2ull * nwarps - 1) / (2ull * nwarps);
        S0 = (S0 + kStep - 1) / kStep * kStep;
        const unsigned long long minp = kStep > TDG_MIN_PIECE ? kStep : TDG_MIN_PIECE;
        // Every piece is pulled from the counter in arrival order, so concurrently running
        // warps work on neighbouring stretches of the (sorted) task axis. (A static first tier
        // — piece = warp index, no atomics in one-tier phases — was measured: C1 peel 16.1 vs
        // 15.6 ms, C5 2.66 vs 2.40 s; removed.)
        while (true) {
            uint32_t p = 0;
            if (lane == 0) p = atomicAdd(piece_head, 1u);
            p = __shfl_sync(kFull, p, 0);
            unsigned long long x0, x1;
            guided_piece(p, W, nwarps, S0, minp, &x0, &x1);
            if (x0 >= W) break;
            run_items(P, x0, x1, task_at(x0, ntasks, wpre, sboff, nchunks, CH), ntasks, wpre, sboff, CH);
            if constexpr (has_flush<Policy>::value) P.flush();
        }
        return W;
    }
    unsigned long long PS = (W + TDG_PIECES * nwarps - 1) / (TDG_PIECES * nwarps);
    PS = (PS + kStep - 1) / kStep * kStep;  // whole engine steps per piece
    if (PS < TDG_MIN_PIECE) PS = TDG_MIN_PIECE;
    const unsigned long long npieces = (W + PS - 1) / PS;

    while (true) {
        uint32_t p = 0;
        if (lane == 0) p = atomicAdd(piece_head, 1u);
        p = __shfl_sync(kFull, p, 0);
        if (p >= npieces) break;
        const unsigned long long x0 = p * PS;
        const unsigned long long x1 = x0 + PS < W ? x0 + PS : W;
        run_items(P, x0, x1, task_at(x0, ntasks, wpre, sboff, nchunks, CH), ntasks, wpre, sboff, CH);
        if constexpr (has_flush<Policy>::value) P.flush();
    }
    return W;
}

}  // namespace tdg
