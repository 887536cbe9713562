// graphgen.cpp — seeded config generator (host C++/OpenMP). See include/tdg_gen.h for
// the exact rules. Test/bench infrastructure: it produces the CSR the GPU path and the
// CPU reference both consume; it is not on the decomposition path.
//
// RMAT follows /root/reference/proj/src/generate.cpp:58-92 (draw loop) and :13-15
// (uniform01). The permutation / G(n,m) / planted-clique rules are SURVEY.md
// Appendix B.2-B.4 (the reference has no such generators).

#include "tdg_gen.h"

#include <omp.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <new>
#include <random>
#include <stdexcept>
#include <string>
#include <vector>

struct tdg_gen_graph {
    int64_t n = 0;
    std::vector<uint64_t> keys;  // sorted unique (u << 32 | v), u < v
};

namespace {

thread_local std::string g_err;

// TDG_GEN_VERBOSE=1 prints per-step wall times to stderr.
void tick(const char* what) {
    static const bool on = std::getenv("TDG_GEN_VERBOSE") != nullptr;
    static auto last = std::chrono::steady_clock::now();
    auto now = std::chrono::steady_clock::now();
    if (on) std::fprintf(stderr, "[graphgen] %-10s %.3f s\n", what, std::chrono::duration<double>(now - last).count());
    last = now;
}

// std::mt19937_64, bit-identical output, generated 312 words per twist with the
// tempering done in a separate (vectorisable) pass. tests/test_generator.py pins it
// against std::mt19937_64 through the oracle's restatement.
struct FastMT64 {
    static constexpr int N = 312, M = 156;
    uint64_t mt[N];
    uint64_t out[N];
    int idx = N;
    explicit FastMT64(uint64_t seed) {
        mt[0] = seed;
        for (int i = 1; i < N; i++) mt[i] = 6364136223846793005ull * (mt[i - 1] ^ (mt[i - 1] >> 62)) + uint64_t(i);
    }
    static inline uint64_t mix(uint64_t hi, uint64_t lo, uint64_t far) {
        const uint64_t x = (hi & 0xFFFFFFFF80000000ull) | (lo & 0x7FFFFFFFull);
        return far ^ (x >> 1) ^ ((0ull - (x & 1ull)) & 0xB5026F5AA96619E9ull);
    }
    __attribute__((target_clones("avx2", "default"))) void refill() {
        for (int i = 0; i < N - M; i++) mt[i] = mix(mt[i], mt[i + 1], mt[i + M]);
        for (int i = N - M; i < N - 1; i++) mt[i] = mix(mt[i], mt[i + 1], mt[i + M - N]);
        mt[N - 1] = mix(mt[N - 1], mt[0], mt[M - 1]);
        for (int i = 0; i < N; i++) {
            uint64_t x = mt[i];
            x ^= (x >> 29) & 0x5555555555555555ull;
            x ^= (x << 17) & 0x71D67FFFEDA60000ull;
            x ^= (x << 37) & 0xFFF7EEE000000000ull;
            x ^= (x >> 43);
            out[i] = x;
        }
        idx = 0;
    }
    inline uint64_t operator()() {
        if (idx == N) refill();
        return out[idx++];
    }
};

double uniform01(FastMT64& rng) {  // generate.cpp:13-15
    return static_cast<double>(rng() >> 11) * 0x1.0p-53;
}

inline uint64_t make_key(uint64_t u, uint64_t v) {
    if (u > v) std::swap(u, v);
    return (u << 32) | v;
}

// LSD radix sort on u64 keys whose significant bits are < `bits`. OpenMP, 11-bit digits.
void radix_sort(std::vector<uint64_t>& a, int bits) {
    const size_t n = a.size();
    if (n < 2) return;
    constexpr int D = 11;
    constexpr size_t B = size_t(1) << D;
    std::vector<uint64_t> tmp(n);
    const int nthreads = std::max(1, omp_get_max_threads());
    std::vector<size_t> hist(static_cast<size_t>(nthreads) * B);
    uint64_t* src = a.data();
    uint64_t* dst = tmp.data();
    int passes = (bits + D - 1) / D;
    for (int p = 0; p < passes; p++) {
        const int shift = p * D;
        std::fill(hist.begin(), hist.end(), 0);
#pragma omp parallel num_threads(nthreads)
        {
            const int t = omp_get_thread_num();
            const int nt = omp_get_num_threads();
            const size_t lo = n * t / nt, hi = n * (t + 1) / nt;
            size_t* h = &hist[static_cast<size_t>(t) * B];
            for (size_t i = lo; i < hi; i++) h[(src[i] >> shift) & (B - 1)]++;
#pragma omp barrier
#pragma omp single
            {
                size_t run = 0;
                for (size_t d = 0; d < B; d++)
                    for (int tt = 0; tt < nt; tt++) {
                        size_t c = hist[static_cast<size_t>(tt) * B + d];
                        hist[static_cast<size_t>(tt) * B + d] = run;
                        run += c;
                    }
            }
            for (size_t i = lo; i < hi; i++) {
                uint64_t k = src[i];
                dst[h[(k >> shift) & (B - 1)]++] = k;
            }
        }
        std::swap(src, dst);
    }
    if (src != a.data()) std::memcpy(a.data(), src, n * sizeof(uint64_t));
}

int key_bits(int64_t n) {
    int b = 1;
    while ((int64_t(1) << b) < n) b++;
    return 32 + b;  // u occupies the high word
}

void sort_unique(tdg_gen_graph& g) {
    radix_sort(g.keys, key_bits(std::max<int64_t>(g.n, 2)));
    g.keys.erase(std::unique(g.keys.begin(), g.keys.end()), g.keys.end());
}

// Open-addressing set of canonical keys (0 = empty; canonical keys are never 0).
struct KeySet {
    std::vector<uint64_t> slot;
    uint64_t mask;
    explicit KeySet(uint64_t expect) {
        uint64_t cap = 16;
        while (cap < expect * 2) cap <<= 1;
        slot.assign(cap, 0);
        mask = cap - 1;
    }
    static uint64_t mix(uint64_t x) {
        x ^= x >> 30; x *= 0xbf58476d1ce4e5b9ull;
        x ^= x >> 27; x *= 0x94d049bb133111ebull;
        return x ^ (x >> 31);
    }
    bool insert(uint64_t k) {
        uint64_t h = mix(k) & mask;
        while (true) {
            if (slot[h] == 0) { slot[h] = k; return true; }
            if (slot[h] == k) return false;
            h = (h + 1) & mask;
        }
    }
};

// G(n,m) draw loop (Appendix B.3): first m distinct non-loop canonical pairs.
void draw_gnm(FastMT64& rng, int64_t n, int64_t m, std::vector<uint64_t>& out) {
    const uint64_t total = static_cast<uint64_t>(n) * static_cast<uint64_t>(n - 1) / 2;
    if (static_cast<uint64_t>(m) > total) throw std::invalid_argument("gnm: m exceeds n(n-1)/2");
    KeySet set(static_cast<uint64_t>(m));
    out.reserve(out.size() + static_cast<size_t>(m));
    int64_t have = 0;
    while (have < m) {
        uint64_t u = rng() % static_cast<uint64_t>(n);
        uint64_t v = rng() % static_cast<uint64_t>(n);
        if (u == v) continue;
        uint64_t k = make_key(u, v);
        if (set.insert(k)) {
            out.push_back(k);
            have++;
        }
    }
}

template <typename F>
int guarded(F&& f) {
    try {
        f();
        return 0;
    } catch (const std::bad_alloc&) {
        g_err = "out of host memory";
        return -3;
    } catch (const std::exception& e) {
        g_err = e.what();
        return -1;
    }
}

}  // namespace

extern "C" {

int tdg_gen_rmat(uint32_t scale, uint32_t edge_factor, uint64_t seed, double a, double b,
                 double c, double d, int permute, tdg_gen_graph** out) {
    return guarded([&] {
        if (std::abs(a + b + c + d - 1.0) > 1e-9)
            throw std::invalid_argument("rmat: quadrant probabilities must sum to 1");
        if (a < 0 || b < 0 || c < 0 || d < 0)
            throw std::invalid_argument("rmat: quadrant probabilities must be nonnegative");
        if (scale == 0 || scale > 31) throw std::invalid_argument("rmat: scale must be in [1, 31]");
        auto g = new tdg_gen_graph;
        FastMT64 rng(seed);
        const uint64_t n = 1ull << scale;
        const uint64_t draws = n * edge_factor;
        const double t1 = a, t2 = a + b, t3 = a + b + c;  // generate.cpp:75-81 thresholds
        // r = k * 2^-53 with k = rng() >> 11 (generate.cpp:13-15), so r < t <=> k < t*2^53
        // <=> k < ceil(t*2^53) exactly (scaling by 2^53 is exact): integer compares only.
        auto kth = [](double t) {
            const double T = std::ceil(std::ldexp(t, 53));
            return T <= 0 ? 0ull : (T >= 0x1p63 ? ~0ull : static_cast<uint64_t>(T));
        };
        const uint64_t k1 = kth(t1), k2 = kth(t2), k3 = kth(t3);
        std::vector<uint64_t> raw(draws);
        for (uint64_t e = 0; e < draws; e++) {
            uint64_t u = 0, v = 0;
            for (uint32_t bit = 0; bit < scale; bit++) {
                // Branch-free form of generate.cpp:73-86: q = #thresholds <= r selects
                // the quadrant (0: none, 1: v, 2: u, 3: both); t1 <= t2 <= t3.
                const uint64_t k = rng() >> 11;
                const uint32_t q = uint32_t(k >= k1) + uint32_t(k >= k2) + uint32_t(k >= k3);
                u = (u << 1) | uint64_t(q >= 2);
                v = (v << 1) | uint64_t(q & 1);
            }
            raw[e] = (u << 32) | v;
        }
        tick("draws");
        std::vector<uint32_t> p(n);
        for (uint64_t i = 0; i < n; i++) p[i] = static_cast<uint32_t>(i);
        if (permute)
            for (uint64_t i = n - 1; i >= 1; i--) {
                uint64_t j = rng() % (i + 1);
                std::swap(p[i], p[j]);
            }
        // map, drop self loops, canonicalise (parallel, order-preserving compaction)
        const int64_t nd = static_cast<int64_t>(draws);
#pragma omp parallel for schedule(static)
        for (int64_t e = 0; e < nd; e++) {
            uint64_t u = p[raw[e] >> 32], v = p[raw[e] & 0xffffffffu];
            raw[e] = (u == v) ? ~0ull : make_key(u, v);
        }
        g->n = static_cast<int64_t>(n);
        g->keys.swap(raw);
        tick("permute");
        radix_sort(g->keys, 64);
        tick("sort");
        while (!g->keys.empty() && g->keys.back() == ~0ull) g->keys.pop_back();
        g->keys.erase(std::unique(g->keys.begin(), g->keys.end()), g->keys.end());
        *out = g;
    });
}

int tdg_gen_gnm(int64_t n, int64_t m, uint64_t seed, tdg_gen_graph** out) {
    return guarded([&] {
        if (n < 2 || m < 0) throw std::invalid_argument("gnm: need n >= 2 and m >= 0");
        auto g = new tdg_gen_graph;
        FastMT64 rng(seed);
        g->n = n;
        draw_gnm(rng, n, m, g->keys);
        sort_unique(*g);
        *out = g;
    });
}

int tdg_gen_planted(int64_t n, int64_t m_bg, uint32_t cliques, uint32_t smin, uint32_t smax,
                    uint64_t seed, tdg_gen_graph** out) {
    return guarded([&] {
        if (n < 2 || smin < 2 || smax < smin || static_cast<int64_t>(smax) > n)
            throw std::invalid_argument("planted: bad parameters");
        auto g = new tdg_gen_graph;
        FastMT64 rng(seed);
        g->n = n;
        draw_gnm(rng, n, m_bg, g->keys);
        std::vector<uint32_t> pool(static_cast<size_t>(n));
        for (int64_t i = 0; i < n; i++) pool[i] = static_cast<uint32_t>(i);
        for (uint32_t q = 0; q < cliques; q++) {
            uint32_t size = smin + static_cast<uint32_t>(rng() % (smax - smin + 1));
            for (uint32_t i = 0; i < size; i++) {
                uint64_t j = i + rng() % static_cast<uint64_t>(n - i);
                std::swap(pool[i], pool[j]);
            }
            for (uint32_t i = 0; i < size; i++)
                for (uint32_t k = i + 1; k < size; k++) g->keys.push_back(make_key(pool[i], pool[k]));
        }
        sort_unique(*g);
        *out = g;
    });
}

int tdg_gen_config(int config, int scale_override, tdg_gen_graph** out) {
    switch (config) {
        case 1: return tdg_gen_rmat(scale_override > 0 ? scale_override : 16, 16, 1, 0.57, 0.19, 0.19, 0.05, 1, out);
        case 2: return tdg_gen_gnm(int64_t(1) << 22, int64_t(32) << 20, 2, out);
        case 3: return tdg_gen_rmat(scale_override > 0 ? scale_override : 22, 16, 3, 0.57, 0.19, 0.19, 0.05, 1, out);
        case 4: return tdg_gen_planted(int64_t(1) << 21, int64_t(5) << 21, 2000, 8, 256, 4, out);
        case 5: return tdg_gen_rmat(scale_override > 0 ? scale_override : 25, 16, 5, 0.57, 0.19, 0.19, 0.05, 1, out);
        default: g_err = "config must be 1..5"; return -1;
    }
}

int tdg_gen_from_pairs(const int64_t* pairs, int64_t npairs, int64_t n_hint, tdg_gen_graph** out) {
    return guarded([&] {
        auto g = new tdg_gen_graph;
        int64_t mx = -1;
        for (int64_t i = 0; i < npairs; i++) {
            int64_t u = pairs[2 * i], v = pairs[2 * i + 1];
            if (u < 0 || v < 0 || u > 0xffffffffll || v > 0xffffffffll)
                throw std::invalid_argument("from_pairs: vertex id out of range");
            mx = std::max(mx, std::max(u, v));
            if (u != v) g->keys.push_back(make_key(static_cast<uint64_t>(u), static_cast<uint64_t>(v)));
        }
        g->n = std::max<int64_t>(n_hint, mx + 1);
        radix_sort(g->keys, 64);
        g->keys.erase(std::unique(g->keys.begin(), g->keys.end()), g->keys.end());
        *out = g;
    });
}

int64_t tdg_gen_n(const tdg_gen_graph* g) { return g ? g->n : -1; }
int64_t tdg_gen_m(const tdg_gen_graph* g) { return g ? static_cast<int64_t>(g->keys.size()) : -1; }

int tdg_gen_fill_csr(const tdg_gen_graph* g, int64_t* offsets, int32_t* neighbors) {
    return guarded([&] {
        const int64_t n = g->n;
        const int64_t m = static_cast<int64_t>(g->keys.size());
        const uint64_t* K = g->keys.data();
        std::vector<uint32_t> lo(static_cast<size_t>(n), 0), up(static_cast<size_t>(n), 0);
        // up[u]: run length of keys with first == u; lo[v]: count of keys with second == v
        for (int64_t k = 0; k < m; k++) {
            up[K[k] >> 32]++;
            lo[K[k] & 0xffffffffu]++;
        }
        offsets[0] = 0;
        for (int64_t u = 0; u < n; u++) offsets[u + 1] = offsets[u] + lo[u] + up[u];
        // Upper parts: keys sorted by (u, v) -> contiguous per u, ascending v.
        std::vector<int64_t> first(static_cast<size_t>(n) + 1, 0);
        for (int64_t u = 0; u < n; u++) first[u + 1] = first[u] + up[u];
#pragma omp parallel for schedule(static)
        for (int64_t k = 0; k < m; k++) {
            uint64_t u = K[k] >> 32;
            neighbors[offsets[u] + lo[u] + (k - first[u])] = static_cast<int32_t>(K[k] & 0xffffffffu);
        }
        // Lower parts: sort swapped keys (v, u) -> contiguous per v, ascending u.
        std::vector<uint64_t> sw(static_cast<size_t>(m));
#pragma omp parallel for schedule(static)
        for (int64_t k = 0; k < m; k++) sw[k] = (K[k] << 32) | (K[k] >> 32);
        radix_sort(sw, key_bits(std::max<int64_t>(n, 2)));
        std::vector<int64_t> firstv(static_cast<size_t>(n) + 1, 0);
        for (int64_t v = 0; v < n; v++) firstv[v + 1] = firstv[v] + lo[v];
#pragma omp parallel for schedule(static)
        for (int64_t k = 0; k < m; k++) {
            uint64_t v = sw[k] >> 32;
            neighbors[offsets[v] + (k - firstv[v])] = static_cast<int32_t>(sw[k] & 0xffffffffu);
        }
    });
}

void tdg_gen_free(tdg_gen_graph* g) { delete g; }

const char* tdg_gen_last_error(void) { return g_err.c_str(); }

}  // extern "C"
