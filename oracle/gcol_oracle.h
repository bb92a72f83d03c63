/*
 * gcol_oracle.h -- CPU restatement of the reference RSOC coloring path.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this code, and
 * only as the checker or the timed CPU baseline -- never as the product
 * path.  The product (paper_1505_04086_b200/, libgcol_cuda.so) has no CPU
 * fallback and never links or loads anything under oracle/.
 *
 * Every function restates one reference function; the citation is
 * /root/reference/proj/include/gcol/<file>:<line>.  Parity is pinned two
 * ways (see tests/test_oracle.py): against the known-answer tests of the
 * reference's own test suite (proj/tests/test_coloring.cpp,
 * test_parallel.cpp, test_graph.cpp, test_lockstep.cpp) and against the
 * reference itself, compiled from its headers into oracle/_ref/ by
 * oracle/Makefile (fixtures in tests/golden/, made by
 * tests/golden/make_golden.py).
 *
 * Layout: CSR with uint64 row offsets (n+1) and uint32 column ids (m),
 * rows sorted ascending, symmetric, no self loops (graph.hpp:15-19).
 * Colors are int32, -1 = uncolored (types.hpp:8-12).
 */
#ifndef GCOL_ORACLE_H
#define GCOL_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define ORACLE_UNCOLORED (-1)
#define ORACLE_NO_VERTEX 0xFFFFFFFFu

/* Algorithm ids follow gcol::Algorithm (parallel.hpp:21). */
enum { ORACLE_ALG_SEQ = 0, ORACLE_ALG_CATALYUREK = 1, ORACLE_ALG_RSOC = 2 };

/* Mirrors gcol::ColoringStats (parallel.hpp:47-57).  conflicts_per_round is
 * written into a caller buffer of capacity cpr_cap; cpr_len is the true
 * length (== rounds). */
typedef struct {
  int32_t algorithm;
  uint32_t thread_count;
  uint64_t rounds;
  uint64_t conflicts_total;
  uint64_t barrier_events;
  uint32_t num_colors;
  uint32_t fallback_triggered;
  uint64_t wall_time_ns;
  uint64_t cpr_len;
  uint64_t* conflicts_per_round;
  uint64_t cpr_cap;
} oracle_stats;

/* build_graph (graph.hpp:98-138): canonical CSR from an unordered edge list
 * (pairs[2*i], pairs[2*i+1]).  Self-loops dropped, duplicates in either
 * orientation collapsed, rows sorted.  offsets_out has n+1 entries; cols_out
 * capacity cols_cap (2 * num_pairs always suffices).  Returns m (directed
 * entries), -1 if an id is >= n (input_error), -2 if cols_cap is too small.
 */
int64_t oracle_build_graph(const uint32_t* pairs, int64_t num_pairs, uint32_t n,
                           uint64_t* offsets_out, uint32_t* cols_out, int64_t cols_cap,
                           uint32_t* max_degree_out);

/* smallest_available_color (coloring.hpp:95-106). */
int32_t oracle_smallest_available_color(const uint64_t* off, const uint32_t* cols,
                                        const int32_t* colors, uint32_t v);

/* Snapshot-mode tentative pass: out[wl[i]] = smallest_available_color over
 * the frozen colors_in (no in-place visibility).  The GPU K1 snapshot mode is
 * checked bit-exactly against this. */
void oracle_tentative_snapshot(const uint64_t* off, const uint32_t* cols,
                               const int32_t* colors_in, const uint32_t* wl, int64_t nwl,
                               int32_t* colors_out);

/* first_fit_sequential (coloring.hpp:110-116). */
void oracle_first_fit_sequential(const uint64_t* off, const uint32_t* cols, uint32_t n,
                                 int32_t* colors_out);

/* has_conflicting_higher_neighbor (coloring.hpp:121-129). */
int oracle_has_conflicting_higher_neighbor(const uint64_t* off, const uint32_t* cols,
                                           const int32_t* colors, uint32_t v);

/* detect_conflicts (coloring.hpp:133-141): writes the defective subset of
 * pending, in pending order; returns its length. */
int64_t oracle_detect_conflicts(const uint64_t* off, const uint32_t* cols,
                                const int32_t* colors, const uint32_t* pending,
                                int64_t npending, uint32_t* out);

/* verify_coloring (coloring.hpp:159-177): reports violations in the
 * reference order (v ascending, then neighbour ascending).  Up to cap
 * violations are written; the return value is the total count. */
int64_t oracle_verify_coloring(const uint64_t* off, const uint32_t* cols, uint32_t n,
                               const int32_t* colors, uint32_t* out_u, uint32_t* out_v,
                               int32_t* out_c, int64_t cap);

/* count_colors (coloring.hpp:181-196): distinct colors; -1 if incomplete,
 * -2 if a negative color other than -1 is present (both input_error). */
int64_t oracle_count_colors(const int32_t* colors, int64_t n);

/* color_rsoc (parallel.hpp:253-319) with POSIX threads.  chunk_size 0 =
 * auto (parallel.hpp:83-88).  Returns 0, or -1 for thread_count < 1
 * (input_error), -3 if the final coloring is improper (logic_error). */
int oracle_color_rsoc(const uint64_t* off, const uint32_t* cols, uint32_t n,
                      uint32_t max_degree, uint32_t thread_count, uint64_t chunk_size,
                      uint64_t min_chunk_size, uint64_t round_cap, int32_t* colors_out,
                      oracle_stats* stats);

/* color_catalyurek (parallel.hpp:184-246), same conventions. */
int oracle_color_catalyurek(const uint64_t* off, const uint32_t* cols, uint32_t n,
                            uint32_t max_degree, uint32_t thread_count, uint64_t chunk_size,
                            uint64_t min_chunk_size, uint64_t round_cap,
                            int32_t* colors_out, oracle_stats* stats);

/* lockstep_color (lockstep.hpp:37-78): trace_out holds round_cap * n
 * colors (one snapshot per executed round).  Returns rounds executed, and
 * *converged.  -1 on bad arguments (input_error). */
int64_t oracle_lockstep_color(const uint64_t* off, const uint32_t* cols, uint32_t n,
                              const uint32_t* lane_of, uint64_t round_cap,
                              int32_t* trace_out, int32_t* converged);

#ifdef __cplusplus
}
#endif
#endif
