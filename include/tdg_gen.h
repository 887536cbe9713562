/*
 * tdg_gen.h — seeded synthetic graph generator for the five BASELINE.json configs.
 *
 * Host-only C-ABI (no CUDA). This is benchmark/test infrastructure, not the
 * decomposition product: it produces the undirected CSR (int64 offsets, int32
 * sorted neighbours, isolated vertices kept) that both the GPU path and the CPU
 * reference consume byte-identically.
 *
 * Rules:
 *   RMAT   : reference generate_rmat semantics, /root/reference/proj/src/generate.cpp:58-92
 *            (std::mt19937_64(seed), uniform01 = (rng()>>11)*2^-53, generate.cpp:13-15),
 *            then (optionally) a Fisher-Yates vertex permutation drawn from the SAME
 *            continuing stream: for i=N-1..1, j = rng() % (i+1), swap(p[i], p[j]).
 *   G(n,m) : draws u = rng() % n, v = rng() % n; rejects u==v and repeats until m
 *            distinct canonical pairs exist (first m distinct pairs in draw order).
 *   planted: G(n, m_bg) background as above, then `cliques` cliques from the same
 *            stream: size = smin + rng() % (smax-smin+1); members by partial
 *            Fisher-Yates over a persistent pool: j = i + rng() % (n-i).
 *   CSR    : sorted unique (u<v) keys, symmetric adjacency, each list ascending.
 */
#ifndef TDG_GEN_H
#define TDG_GEN_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct tdg_gen_graph tdg_gen_graph; /* opaque: sorted unique edge keys */

/* Each returns 0 on success, <0 on error (message via tdg_gen_last_error). */
int tdg_gen_rmat(uint32_t scale, uint32_t edge_factor, uint64_t seed, double a, double b,
                 double c, double d, int permute, tdg_gen_graph** out);
int tdg_gen_gnm(int64_t n, int64_t m, uint64_t seed, tdg_gen_graph** out);
int tdg_gen_planted(int64_t n, int64_t m_bg, uint32_t cliques, uint32_t smin, uint32_t smax,
                    uint64_t seed, tdg_gen_graph** out);
/* Config presets 1..5 of BASELINE.json (C1 RMAT-16, C2 ER, C3 RMAT-22, C4 planted,
 * C5 RMAT-25). `scale_override` > 0 replaces the RMAT scale (bounded CPU samples). */
int tdg_gen_config(int config, int scale_override, tdg_gen_graph** out);
/* Arbitrary edge list (u,v pairs, any order, duplicates/self loops dropped), vertex ids
 * kept as given; n = max(id)+1 unless n_hint is larger. */
int tdg_gen_from_pairs(const int64_t* pairs, int64_t npairs, int64_t n_hint, tdg_gen_graph** out);

int64_t tdg_gen_n(const tdg_gen_graph* g);
int64_t tdg_gen_m(const tdg_gen_graph* g);
/* Fill caller buffers: offsets[n+1], neighbors[2m]. */
int tdg_gen_fill_csr(const tdg_gen_graph* g, int64_t* offsets, int32_t* neighbors);
void tdg_gen_free(tdg_gen_graph* g);
const char* tdg_gen_last_error(void);

#ifdef __cplusplus
}
#endif

#endif /* TDG_GEN_H */
