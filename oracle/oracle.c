/*
 * oracle.c — CPU restatement of the reference PKT path (TEST INFRASTRUCTURE ONLY;
 * see oracle.h). Citations are relative to /root/reference/.
 */
#include "oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

/* ---------------------------------------------------------------- mt19937_64 */
#define MT_NN 312
#define MT_MM 156
#define MT_A 0xB5026F5AA96619E9ull
#define MT_UM 0xFFFFFFFF80000000ull
#define MT_LM 0x7FFFFFFFull

void or_mt64_seed(or_mt64* r, uint64_t seed) {
    r->mt[0] = seed;
    for (int i = 1; i < MT_NN; i++)
        r->mt[i] = 6364136223846793005ull * (r->mt[i - 1] ^ (r->mt[i - 1] >> 62)) + (uint64_t)i;
    r->mti = MT_NN;
}

uint64_t or_mt64_next(or_mt64* r) {
    uint64_t x;
    if (r->mti >= MT_NN) {
        int i;
        for (i = 0; i < MT_NN - MT_MM; i++) {
            x = (r->mt[i] & MT_UM) | (r->mt[i + 1] & MT_LM);
            r->mt[i] = r->mt[i + MT_MM] ^ (x >> 1) ^ ((x & 1ull) ? MT_A : 0ull);
        }
        for (; i < MT_NN - 1; i++) {
            x = (r->mt[i] & MT_UM) | (r->mt[i + 1] & MT_LM);
            r->mt[i] = r->mt[i + (MT_MM - MT_NN)] ^ (x >> 1) ^ ((x & 1ull) ? MT_A : 0ull);
        }
        x = (r->mt[MT_NN - 1] & MT_UM) | (r->mt[0] & MT_LM);
        r->mt[MT_NN - 1] = r->mt[MT_MM - 1] ^ (x >> 1) ^ ((x & 1ull) ? MT_A : 0ull);
        r->mti = 0;
    }
    x = r->mt[r->mti++];
    x ^= (x >> 29) & 0x5555555555555555ull;
    x ^= (x << 17) & 0x71D67FFFEDA60000ull;
    x ^= (x << 37) & 0xFFF7EEE000000000ull;
    x ^= (x >> 43);
    return x;
}

/* generate.cpp:13-15 */
static double uniform01(or_mt64* r) { return (double)(or_mt64_next(r) >> 11) * 0x1.0p-53; }

/* ---------------------------------------------------------------- generators */
/* generate.cpp:19-56 */
int64_t or_generate_er(uint32_t n, double p, uint64_t seed, uint64_t* pairs, int64_t cap) {
    int64_t cnt = 0;
    if (n == 0 || p <= 0.0) return 0;
    if (p >= 1.0) {
        for (uint32_t u = 0; u < n; u++)
            for (uint32_t v = u + 1; v < n; v++) {
                if (cnt < cap) { pairs[2 * cnt] = u; pairs[2 * cnt + 1] = v; }
                cnt++;
            }
        return cnt;
    }
    or_mt64 rng;
    or_mt64_seed(&rng, seed);
    const uint64_t total = (uint64_t)n * (n - 1) / 2;
    const double log1mp = log1p(-p);
    uint64_t idx = 0;
    for (;;) {
        double r = uniform01(&rng);
        uint64_t skip = (uint64_t)floor(log1p(-r) / log1mp);
        idx += skip;
        if (idx >= total) break;
        uint64_t i = idx, row = n - 1;
        uint32_t u = 0;
        while (i >= row) { i -= row; row--; u++; }
        if (cnt < cap) { pairs[2 * cnt] = u; pairs[2 * cnt + 1] = u + 1 + i; }
        cnt++;
        idx++;
    }
    return cnt;
}

/* generate.cpp:58-92 */
int64_t or_generate_rmat(uint32_t scale, uint32_t ef, uint64_t seed, double a, double b,
                         double c, double d, uint64_t* pairs, int64_t cap) {
    (void)d;
    or_mt64 rng;
    or_mt64_seed(&rng, seed);
    const uint64_t n = 1ull << scale;
    const int64_t edges = (int64_t)(n * ef);
    for (int64_t e = 0; e < edges; e++) {
        uint64_t u = 0, v = 0;
        for (uint32_t bit = 0; bit < scale; bit++) {
            double r = uniform01(&rng);
            u <<= 1;
            v <<= 1;
            if (r < a) {
            } else if (r < a + b) {
                v |= 1;
            } else if (r < a + b + c) {
                u |= 1;
            } else {
                u |= 1;
                v |= 1;
            }
        }
        if (e < cap) { pairs[2 * e] = u; pairs[2 * e + 1] = v; }
    }
    return edges;
}

/* ---------------------------------------------------------------- canonicalize */
static int cmp_u64(const void* a, const void* b) {
    uint64_t x = *(const uint64_t*)a, y = *(const uint64_t*)b;
    return x < y ? -1 : (x > y);
}

static uint64_t mix64(uint64_t x) {
    x ^= x >> 30; x *= 0xbf58476d1ce4e5b9ull;
    x ^= x >> 27; x *= 0x94d049bb133111ebull;
    return x ^ (x >> 31);
}

/* graph.cpp:19-71: intern labels in first-appearance order (a then b per edge),
 * drop loops, sort + unique canonical (u<v) pairs, count degrees, fill in (u,v) order. */
int or_canonicalize(const uint64_t* pairs, int64_t npairs, int64_t* offsets, int32_t* neighbors,
                    uint64_t* labels, int64_t* n_out, int64_t* m_out) {
    uint64_t cap = 16;
    while (cap < (uint64_t)npairs * 4 + 4) cap <<= 1;
    uint64_t* hk = (uint64_t*)malloc(cap * sizeof(uint64_t));
    uint32_t* hv = (uint32_t*)malloc(cap * sizeof(uint32_t));
    uint8_t* used = (uint8_t*)calloc(cap, 1);
    uint64_t* keys = (uint64_t*)malloc(((size_t)npairs + 1) * sizeof(uint64_t));
    if (!hk || !hv || !used || !keys) { free(hk); free(hv); free(used); free(keys); return -3; }
    int64_t n = 0, k = 0;
    for (int64_t i = 0; i < npairs; i++) {
        uint32_t id[2];
        for (int t = 0; t < 2; t++) {
            uint64_t lab = pairs[2 * i + t];
            uint64_t h = mix64(lab) & (cap - 1);
            while (used[h] && hk[h] != lab) h = (h + 1) & (cap - 1);
            if (!used[h]) { used[h] = 1; hk[h] = lab; hv[h] = (uint32_t)n; labels[n] = lab; n++; }
            id[t] = hv[h];
        }
        if (id[0] == id[1]) continue;
        uint32_t u = id[0] < id[1] ? id[0] : id[1], v = id[0] < id[1] ? id[1] : id[0];
        keys[k++] = ((uint64_t)u << 32) | v;
    }
    qsort(keys, (size_t)k, sizeof(uint64_t), cmp_u64);
    int64_t m = 0;
    for (int64_t i = 0; i < k; i++)
        if (i == 0 || keys[i] != keys[i - 1]) keys[m++] = keys[i];
    for (int64_t u = 0; u <= n; u++) offsets[u] = 0;
    for (int64_t i = 0; i < m; i++) {
        offsets[(keys[i] >> 32) + 1]++;
        offsets[(keys[i] & 0xffffffffu) + 1]++;
    }
    for (int64_t u = 0; u < n; u++) offsets[u + 1] += offsets[u];
    int64_t* cur = (int64_t*)malloc(((size_t)n + 1) * sizeof(int64_t));
    if (!cur) { free(hk); free(hv); free(used); free(keys); return -3; }
    memcpy(cur, offsets, (size_t)n * sizeof(int64_t));
    for (int64_t i = 0; i < m; i++) {
        uint32_t u = (uint32_t)(keys[i] >> 32), v = (uint32_t)keys[i];
        neighbors[cur[u]++] = (int32_t)v;
        neighbors[cur[v]++] = (int32_t)u;
    }
    free(cur); free(hk); free(hv); free(used); free(keys);
    *n_out = n;
    *m_out = m;
    return 0;
}

/* ---------------------------------------------------------------- truss graph */
static int64_t upper_bound_i32(const int32_t* a, int64_t lo, int64_t hi, uint32_t x) {
    while (lo < hi) {
        int64_t mid = lo + (hi - lo) / 2;
        if ((uint32_t)a[mid] <= x) lo = mid + 1; else hi = mid;
    }
    return lo;
}
static int64_t lower_bound_i32(const int32_t* a, int64_t lo, int64_t hi, uint32_t x) {
    while (lo < hi) {
        int64_t mid = lo + (hi - lo) / 2;
        if ((uint32_t)a[mid] < x) lo = mid + 1; else hi = mid;
    }
    return lo;
}

/* graph.cpp:73-101 */
void or_build_truss_graph(int64_t n, int64_t m, const int64_t* offsets, const int32_t* neighbors,
                          uint32_t* eo, uint32_t* eid, uint32_t* el) {
    (void)m;
    for (int64_t u = 0; u < n; u++)
        eo[u] = (uint32_t)upper_bound_i32(neighbors, offsets[u], offsets[u + 1], (uint32_t)u);
    uint32_t* cursor = (uint32_t*)malloc(((size_t)n + 1) * sizeof(uint32_t));
    for (int64_t u = 0; u < n; u++) cursor[u] = (uint32_t)offsets[u];
    uint32_t next_id = 0;
    for (int64_t u = 0; u < n; u++)
        for (int64_t j = eo[u]; j < offsets[u + 1]; j++) {
            uint32_t v = (uint32_t)neighbors[j];
            eid[j] = next_id;
            eid[cursor[v]++] = next_id;
            el[2 * (size_t)next_id] = (uint32_t)u;
            el[2 * (size_t)next_id + 1] = v;
            next_id++;
        }
    free(cursor);
}

/* graph.cpp:135-150, plus the degree-order (deg, id) terms of SURVEY §8(d). */
void or_stats_compute(int64_t n, int64_t m, const int64_t* offsets, const int32_t* neighbors,
                      or_stats* st) {
    memset(st, 0, sizeof(*st));
    for (int64_t u = 0; u < n; u++) {
        uint64_t d = (uint64_t)(offsets[u + 1] - offsets[u]);
        if (d > st->d_max) st->d_max = d;
        st->sum_deg_sq += d * d;
        uint64_t dplus = (uint64_t)(offsets[u + 1] -
                                    upper_bound_i32(neighbors, offsets[u], offsets[u + 1], (uint32_t)u));
        st->sum_dplus_sq += dplus * dplus;
    }
    st->wedge_count = (st->sum_deg_sq - 2ull * (uint64_t)m) / 2;
    uint64_t* dp = (uint64_t*)calloc((size_t)n + 1, sizeof(uint64_t));
    uint64_t* dm = (uint64_t*)calloc((size_t)n + 1, sizeof(uint64_t));
    for (int64_t u = 0; u < n; u++) {
        uint64_t du = (uint64_t)(offsets[u + 1] - offsets[u]);
        for (int64_t j = offsets[u]; j < offsets[u + 1]; j++) {
            uint32_t v = (uint32_t)neighbors[j];
            uint64_t dv = (uint64_t)(offsets[v + 1] - offsets[v]);
            if (du < dv || (du == dv && (uint64_t)u < v)) dp[u]++; else dm[u]++;
        }
    }
    for (int64_t u = 0; u < n; u++) {
        st->deg_order_sum_dplus_sq += dp[u] * dp[u];
        st->deg_order_s1 += dp[u] * dp[u] + dm[u] * dp[u];
    }
    free(dp);
    free(dm);
}

/* ---------------------------------------------------------------- support */
/* triangle.cpp:26-61 (serial schedule: relaxed atomics become plain increments). */
void or_support_am4(int64_t n, int64_t m, const int64_t* offsets, const int32_t* neighbors,
                    const uint32_t* eo, const uint32_t* eid, uint32_t* s) {
    uint32_t* x = (uint32_t*)calloc((size_t)n + 1, sizeof(uint32_t));
    memset(s, 0, (size_t)m * sizeof(uint32_t));
    for (int64_t u = 0; u < n; u++) {
        for (int64_t j = eo[u]; j < offsets[u + 1]; j++) x[neighbors[j]] = (uint32_t)j + 1;
        for (int64_t j = offsets[u]; j < eo[u]; j++) {
            uint32_t v = (uint32_t)neighbors[j];
            for (int64_t k = offsets[v + 1]; k-- > (int64_t)eo[v];) {
                uint32_t w = (uint32_t)neighbors[k];
                if (w < (uint32_t)u) break;
                if (x[w] == 0) continue;
                s[eid[k]]++;
                s[eid[j]]++;
                s[eid[x[w] - 1]]++;
            }
        }
        for (int64_t j = eo[u]; j < offsets[u + 1]; j++) x[neighbors[j]] = 0;
    }
    free(x);
}

/* triangle.cpp:118-150 */
int64_t or_triangle_oracle(int64_t n, int64_t m, const int64_t* offsets, const int32_t* neighbors,
                           uint32_t* s) {
    if (n > 512) return -1;
    uint32_t* eo = (uint32_t*)malloc(((size_t)n + 1) * sizeof(uint32_t));
    uint32_t* eid = (uint32_t*)malloc(((size_t)2 * m + 1) * sizeof(uint32_t));
    uint32_t* el = (uint32_t*)malloc(((size_t)2 * m + 1) * sizeof(uint32_t));
    or_build_truss_graph(n, m, offsets, neighbors, eo, eid, el);
    memset(s, 0, (size_t)m * sizeof(uint32_t));
    int64_t count = 0;
#define HAS(a, b) (lower_bound_i32(neighbors, offsets[a], offsets[(a) + 1], (uint32_t)(b)) < offsets[(a) + 1] && \
                   (uint32_t)neighbors[lower_bound_i32(neighbors, offsets[a], offsets[(a) + 1], (uint32_t)(b))] == (uint32_t)(b))
#define EID(a, b) eid[lower_bound_i32(neighbors, offsets[a], offsets[(a) + 1], (uint32_t)(b))]
    for (int64_t u = 0; u < n; u++)
        for (int64_t v = u + 1; v < n; v++) {
            if (!HAS(u, v)) continue;
            for (int64_t w = v + 1; w < n; w++)
                if (HAS(u, w) && HAS(v, w)) {
                    count++;
                    s[EID(u, v)]++;
                    s[EID(u, w)]++;
                    s[EID(v, w)]++;
                }
        }
#undef HAS
#undef EID
    free(eo); free(eid); free(el);
    return count;
}

/* ---------------------------------------------------------------- PKT peel */
/* truss_parallel.cpp:21-37 */
void or_scan(int64_t m, const uint32_t* s, uint32_t level, const uint8_t* processed,
             uint8_t* in_curr, uint32_t* curr, uint64_t* curr_size) {
    uint64_t cs = 0;
    for (int64_t e = 0; e < m; e++)
        if (!processed[e] && s[e] == level) {
            in_curr[e] = 1;
            curr[cs++] = (uint32_t)e;
        }
    *curr_size = cs;
}

/* truss_parallel.cpp:49-63 (try_decrement; serial, so prev <= level cannot occur). */
static void try_decrement(uint32_t e1, uint32_t target, uint32_t other, uint32_t* s, uint32_t level,
                          const uint8_t* in_curr, uint8_t* in_next, uint32_t* next, uint64_t* ns) {
    if (s[target] <= level) return;
    if (in_curr[other] && e1 >= other) return;
    uint32_t prev = s[target]--;
    if (prev == level + 1) {
        in_next[target] = 1;
        next[(*ns)++] = target;
    } else if (prev <= level) {
        s[target]++;
    }
}

/* truss_parallel.cpp:39-104 */
void or_process_sublevel(int64_t n, const int64_t* offsets, const int32_t* neighbors,
                         const uint32_t* eid, const uint32_t* el, uint32_t* s, uint32_t level,
                         const uint32_t* curr, uint64_t curr_size, uint8_t* in_curr,
                         uint8_t* in_next, uint8_t* processed, uint32_t* next,
                         uint64_t* next_size, uint32_t* x) {
    (void)n;
    for (uint64_t i = 0; i < curr_size; i++) {
        const uint32_t e1 = curr[i];
        const uint32_t u = el[2 * (size_t)e1], v = el[2 * (size_t)e1 + 1];
        for (int64_t j = offsets[u]; j < offsets[u + 1]; j++) x[neighbors[j]] = (uint32_t)j + 1;
        for (int64_t j = offsets[v]; j < offsets[v + 1]; j++) {
            const uint32_t w = (uint32_t)neighbors[j];
            if (x[w] == 0) continue;
            const uint32_t e2 = eid[j];
            const uint32_t e3 = eid[x[w] - 1];
            if (processed[e2] || processed[e3]) continue;
            try_decrement(e1, e2, e3, s, level, in_curr, in_next, next, next_size);
            try_decrement(e1, e3, e2, s, level, in_curr, in_next, next, next_size);
        }
        for (int64_t j = offsets[u]; j < offsets[u + 1]; j++) x[neighbors[j]] = 0;
    }
    for (uint64_t i = 0; i < curr_size; i++) {
        processed[curr[i]] = 1;
        in_curr[curr[i]] = 0;
    }
}

/* truss_parallel.cpp:106-150 */
int or_truss_pkt(int64_t n, int64_t m, const int64_t* offsets, const int32_t* neighbors,
                 uint32_t* truss, uint32_t* support_out, uint32_t* nsl, uint64_t nsl_cap,
                 uint64_t* nsl_len, uint64_t* barriers) {
    size_t M = (size_t)m + 1;
    uint32_t* eo = (uint32_t*)malloc(((size_t)n + 1) * sizeof(uint32_t));
    uint32_t* eid = (uint32_t*)malloc(2 * M * sizeof(uint32_t));
    uint32_t* el = (uint32_t*)malloc(2 * M * sizeof(uint32_t));
    uint32_t* s = (uint32_t*)malloc(M * sizeof(uint32_t));
    uint32_t* curr = (uint32_t*)malloc(M * sizeof(uint32_t));
    uint32_t* next = (uint32_t*)malloc(M * sizeof(uint32_t));
    uint8_t* in_curr = (uint8_t*)calloc(M, 1);
    uint8_t* in_next = (uint8_t*)calloc(M, 1);
    uint8_t* processed = (uint8_t*)calloc(M, 1);
    uint32_t* x = (uint32_t*)calloc((size_t)n + 1, sizeof(uint32_t));
    if (!eo || !eid || !el || !s || !curr || !next || !in_curr || !in_next || !processed || !x) return -3;
    or_build_truss_graph(n, m, offsets, neighbors, eo, eid, el);
    or_support_am4(n, m, offsets, neighbors, eo, eid, s);
    if (support_out) memcpy(support_out, s, (size_t)m * sizeof(uint32_t));
    uint64_t bar = 1; /* after support, :113 */
    uint64_t len = 0, todo = (uint64_t)m, cs = 0, ns = 0;
    uint32_t level = 0;
    while (todo > 0) {
        or_scan(m, s, level, processed, in_curr, curr, &cs);
        bar++;
        while (cs > 0) {
            if (len <= level) {
                for (uint64_t l = len; l <= level; l++) if (l < nsl_cap) nsl[l] = 0;
                len = (uint64_t)level + 1;
            }
            if (level < nsl_cap) nsl[level]++;
            todo -= cs;
            ns = 0;
            or_process_sublevel(n, offsets, neighbors, eid, el, s, level, curr, cs, in_curr, in_next,
                                processed, next, &ns, x);
            bar++;
            uint32_t* t = curr; curr = next; next = t;
            uint8_t* tf = in_curr; in_curr = in_next; in_next = tf;
            cs = ns;
            bar++;
        }
        level++;
    }
    for (int64_t e = 0; e < m; e++) truss[e] = s[e] + 2;
    *nsl_len = len;
    if (barriers) *barriers = bar;
    free(eo); free(eid); free(el); free(s); free(curr); free(next);
    free(in_curr); free(in_next); free(processed); free(x);
    return 0;
}

/* ---------------------------------------------------------------- WC (serial) */
/* truss_serial.cpp:23-54 (EdgeBucketOrder) and :62-112 (truss_wc). The edge lookup of
 * {v,w} uses binary search in the sorted CSR instead of a hash map (same function). */
int or_truss_wc(int64_t n, int64_t m, const int64_t* offsets, const int32_t* neighbors,
                uint32_t* truss) {
    size_t M = (size_t)m + 1;
    uint32_t* eo = (uint32_t*)malloc(((size_t)n + 1) * sizeof(uint32_t));
    uint32_t* eid = (uint32_t*)malloc(2 * M * sizeof(uint32_t));
    uint32_t* el = (uint32_t*)malloc(2 * M * sizeof(uint32_t));
    uint32_t* s = (uint32_t*)malloc(M * sizeof(uint32_t));
    uint32_t* sorted = (uint32_t*)malloc(M * sizeof(uint32_t));
    uint32_t* pos = (uint32_t*)malloc(M * sizeof(uint32_t));
    uint8_t* deleted = (uint8_t*)calloc(M, 1);
    if (!eo || !eid || !el || !s || !sorted || !pos || !deleted) return -3;
    or_build_truss_graph(n, m, offsets, neighbors, eo, eid, el);
    or_support_am4(n, m, offsets, neighbors, eo, eid, s);
    uint32_t maxs = 0;
    for (int64_t e = 0; e < m; e++) if (s[e] > maxs) maxs = s[e];
    uint32_t* bstart = (uint32_t*)calloc((size_t)maxs + 2, sizeof(uint32_t));
    uint32_t* cursor = (uint32_t*)calloc((size_t)maxs + 2, sizeof(uint32_t));
    for (int64_t e = 0; e < m; e++) bstart[s[e] + 1]++;
    for (uint32_t b = 0; b <= maxs; b++) bstart[b + 1] += bstart[b];
    memcpy(cursor, bstart, ((size_t)maxs + 1) * sizeof(uint32_t));
    for (int64_t e = 0; e < m; e++) { pos[e] = cursor[s[e]]++; sorted[pos[e]] = (uint32_t)e; }
#define DECR(e_, b_) do { uint32_t pe = pos[e_], pf = bstart[b_], first = sorted[pf]; \
        if (first != (e_)) { sorted[pe] = first; sorted[pf] = (e_); pos[e_] = pf; pos[first] = pe; } \
        bstart[b_]++; } while (0)
    for (int64_t i = 0; i < m; i++) {
        const uint32_t e = sorted[i];
        const uint32_t k = s[e];
        const uint32_t u = el[2 * (size_t)e], v = el[2 * (size_t)e + 1];
        for (int64_t j = offsets[u]; j < offsets[u + 1]; j++) {
            const uint32_t w = (uint32_t)neighbors[j];
            if (w == v) continue;
            const uint32_t euw = eid[j];
            if (deleted[euw]) continue;
            int64_t p = lower_bound_i32(neighbors, offsets[v], offsets[v + 1], w);
            if (p >= offsets[v + 1] || (uint32_t)neighbors[p] != w) continue;
            const uint32_t evw = eid[p];
            if (deleted[evw]) continue;
            if (s[euw] > k) { DECR(euw, s[euw]); s[euw]--; }
            if (s[evw] > k) { DECR(evw, s[evw]); s[evw]--; }
        }
        deleted[e] = 1;
        truss[e] = k + 2;
    }
#undef DECR
    free(eo); free(eid); free(el); free(s); free(sorted); free(pos); free(deleted);
    free(bstart); free(cursor);
    return 0;
}
