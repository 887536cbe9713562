/*
 * oracle.h — CPU restatement of the reference PKT truss-decomposition path.
 *
 * TEST INFRASTRUCTURE ONLY. Nothing in paper_1707_02000_b200/ links, imports or
 * calls this; only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs use it, and only as the checker.
 *
 * Plain C, single-threaded, uint32 vertex/edge ids. Each function cites the reference
 * file:line it restates (paths relative to /root/reference/). Pinned against the
 * reference library itself (oracle/_ref, built from the reference sources by
 * oracle/Makefile) and the reference tests' known answers: tests/test_oracle_pins.py.
 */
#ifndef TDG_ORACLE_H
#define TDG_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* std::mt19937_64 restated (Matsumoto & Nishimura's published MT19937-64). */
typedef struct or_mt64 { uint64_t mt[312]; int mti; } or_mt64;
void or_mt64_seed(or_mt64* r, uint64_t seed);
uint64_t or_mt64_next(or_mt64* r);

/* generate.cpp:19-56 — G(n,p) by geometric skipping. Writes up to cap pairs (u,v)
 * into pairs[2*i], returns the number of pairs generated (may exceed cap: call again). */
int64_t or_generate_er(uint32_t n, double p, uint64_t seed, uint64_t* pairs, int64_t cap);
/* generate.cpp:58-92 — RMAT raw draws (2^scale * ef pairs, duplicates/loops included). */
int64_t or_generate_rmat(uint32_t scale, uint32_t ef, uint64_t seed, double a, double b,
                         double c, double d, uint64_t* pairs, int64_t cap);

/* graph.cpp:19-71 — dedupe, drop loops, first-appearance relabel, CSR.
 * offsets[n+1] (caller sizes it n_cap+1 with n_cap >= distinct labels), neighbors[2m],
 * labels[n]. Returns 0 on success; *n_out, *m_out set. */
int or_canonicalize(const uint64_t* pairs, int64_t npairs, int64_t* offsets, int32_t* neighbors,
                    uint64_t* labels, int64_t* n_out, int64_t* m_out);

/* graph.cpp:73-101 — eo[n], eid[2m], el[2m] (pairs u<v) in ascending (u,v) scan order. */
void or_build_truss_graph(int64_t n, int64_t m, const int64_t* offsets, const int32_t* neighbors,
                          uint32_t* eo, uint32_t* eid, uint32_t* el);

/* graph.cpp:135-150 (+ degree-order terms used by the roofline model). */
typedef struct or_stats {
    uint64_t d_max, sum_deg_sq, sum_dplus_sq, wedge_count;
    uint64_t deg_order_sum_dplus_sq, deg_order_s1; /* orientation (deg, id) ascending */
} or_stats;
void or_stats_compute(int64_t n, int64_t m, const int64_t* offsets, const int32_t* neighbors,
                      or_stats* out);

/* triangle.cpp:26-61 — support_am4 (serial): s[m] = triangles per edge. */
void or_support_am4(int64_t n, int64_t m, const int64_t* offsets, const int32_t* neighbors,
                    const uint32_t* eo, const uint32_t* eid, uint32_t* s);

/* triangle.cpp:118-150 — brute-force triangle oracle (n <= 512). Returns count or -1. */
int64_t or_triangle_oracle(int64_t n, int64_t m, const int64_t* offsets, const int32_t* neighbors,
                           uint32_t* s);

/* truss_parallel.cpp:21-37 — scan. */
void or_scan(int64_t m, const uint32_t* s, uint32_t level, const uint8_t* processed,
             uint8_t* in_curr, uint32_t* curr, uint64_t* curr_size);
/* truss_parallel.cpp:39-104 — process_sublevel, serial schedule. mark[n] zero scratch. */
void or_process_sublevel(int64_t n, const int64_t* offsets, const int32_t* neighbors,
                         const uint32_t* eid, const uint32_t* el, uint32_t* s, uint32_t level,
                         const uint32_t* curr, uint64_t curr_size, uint8_t* in_curr,
                         uint8_t* in_next, uint8_t* processed, uint32_t* next,
                         uint64_t* next_size, uint32_t* mark);

/* truss_parallel.cpp:106-150 — full PKT decomposition. truss[m]; nsl written up to
 * nsl_cap entries, *nsl_len = full trace length; *barriers per the reference tally.
 * Returns 0, or -3 on allocation failure. */
int or_truss_pkt(int64_t n, int64_t m, const int64_t* offsets, const int32_t* neighbors,
                 uint32_t* truss, uint32_t* support_out, uint32_t* nsl, uint64_t nsl_cap,
                 uint64_t* nsl_len, uint64_t* barriers);

/* truss_serial.cpp:62-112 — serial WC engine (independent cross-check). */
int or_truss_wc(int64_t n, int64_t m, const int64_t* offsets, const int32_t* neighbors,
                uint32_t* truss);

#ifdef __cplusplus
}
#endif

#endif
