/*
 * gcol_oracle.c -- CPU restatement of the reference RSOC path (TEST
 * INFRASTRUCTURE ONLY; see gcol_oracle.h for the rules and the pinning).
 *
 * Own code.  Each function names the reference function it restates.
 */
#define _GNU_SOURCE
#include "gcol_oracle.h"

#include <pthread.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>

/* ------------------------------------------------------------------ */
/* build_graph (graph.hpp:98-138)                                       */
/* ------------------------------------------------------------------ */

static int cmp_u64(const void* a, const void* b) {
  uint64_t x = *(const uint64_t*)a, y = *(const uint64_t*)b;
  return (x > y) - (x < y);
}

int64_t oracle_build_graph(const uint32_t* pairs, int64_t num_pairs, uint32_t n,
                           uint64_t* offsets_out, uint32_t* cols_out, int64_t cols_cap,
                           uint32_t* max_degree_out) {
  for (int64_t i = 0; i < 2 * num_pairs; ++i)
    if (pairs[i] >= n) return -1; /* graph.hpp:100-104 input_error */
  uint64_t* keys = (uint64_t*)malloc(sizeof(uint64_t) * (size_t)(num_pairs > 0 ? num_pairs : 1));
  int64_t kept = 0;
  for (int64_t i = 0; i < num_pairs; ++i) {
    uint32_t u = pairs[2 * i], v = pairs[2 * i + 1];
    if (u == v) continue; /* self-loops dropped (:108) */
    uint32_t a = u < v ? u : v, b = u < v ? v : u;
    keys[kept++] = ((uint64_t)a << 32) | b; /* normalised (min,max) (:109) */
  }
  qsort(keys, (size_t)kept, sizeof(uint64_t), cmp_u64);
  int64_t uniq = 0;
  for (int64_t i = 0; i < kept; ++i)
    if (i == 0 || keys[i] != keys[i - 1]) keys[uniq++] = keys[i]; /* unique (:113) */
  if (2 * uniq > cols_cap) {
    free(keys);
    return -2;
  }
  memset(offsets_out, 0, sizeof(uint64_t) * ((size_t)n + 1));
  for (int64_t i = 0; i < uniq; ++i) {
    offsets_out[(keys[i] >> 32) + 1]++;
    offsets_out[(keys[i] & 0xFFFFFFFFu) + 1]++;
  }
  for (uint64_t i = 1; i <= n; ++i) offsets_out[i] += offsets_out[i - 1];
  uint64_t* cursor = (uint64_t*)malloc(sizeof(uint64_t) * ((size_t)n + 1));
  memcpy(cursor, offsets_out, sizeof(uint64_t) * ((size_t)n + 1));
  /* (u,v) sorted, so both directions fill each row ascending (:126-130). */
  for (int64_t i = 0; i < uniq; ++i) {
    uint32_t u = (uint32_t)(keys[i] >> 32), v = (uint32_t)(keys[i] & 0xFFFFFFFFu);
    cols_out[cursor[u]++] = v;
    cols_out[cursor[v]++] = u;
  }
  uint32_t maxd = 0;
  for (uint32_t v = 0; v < n; ++v) {
    uint32_t d = (uint32_t)(offsets_out[v + 1] - offsets_out[v]);
    if (d > maxd) maxd = d;
  }
  if (max_degree_out) *max_degree_out = maxd;
  free(cursor);
  free(keys);
  return 2 * uniq;
}

/* ------------------------------------------------------------------ */
/* Forbidden-color scratch (ForbiddenMarks, coloring.hpp:41-76)          */
/* ------------------------------------------------------------------ */

typedef struct {
  uint32_t* stamps;
  uint64_t cap;
  uint32_t epoch;
} marks_t;

static void marks_init(marks_t* m, uint64_t cap) {
  m->stamps = (uint32_t*)calloc((size_t)(cap ? cap : 1), sizeof(uint32_t));
  m->cap = cap;
  m->epoch = 0;
}
static void marks_free(marks_t* m) { free(m->stamps); }
static void marks_next_epoch(marks_t* m) {
  if (++m->epoch == 0) { /* wrap: clear (coloring.hpp:47-52) */
    memset(m->stamps, 0, sizeof(uint32_t) * (size_t)m->cap);
    m->epoch = 1;
  }
}

static inline int32_t load_relaxed(const int32_t* p) { return __atomic_load_n(p, __ATOMIC_RELAXED); }
static inline void store_relaxed(int32_t* p, int32_t v) { __atomic_store_n(p, v, __ATOMIC_RELAXED); }

/* smallest_available_color (coloring.hpp:95-106): limit = deg(v); mark each
 * neighbour color c with 0 <= c <= limit; smallest unmarked in [0, limit]. */
static int32_t sac(const uint64_t* off, const uint32_t* cols, const int32_t* colors, uint32_t v,
                   marks_t* m) {
  const uint64_t b = off[v], e = off[v + 1];
  const int32_t limit = (int32_t)(e - b);
  marks_next_epoch(m);
  for (uint64_t i = b; i < e; ++i) {
    const int32_t cw = load_relaxed(&colors[cols[i]]);
    if (cw >= 0 && cw <= limit) m->stamps[cw] = m->epoch;
  }
  for (int32_t c = 0; c <= limit; ++c)
    if (m->stamps[c] != m->epoch) return c;
  return limit + 1; /* unreachable: at most `limit` marks below limit+1 */
}

int32_t oracle_smallest_available_color(const uint64_t* off, const uint32_t* cols,
                                        const int32_t* colors, uint32_t v) {
  marks_t m;
  marks_init(&m, off[v + 1] - off[v] + 1);
  int32_t c = sac(off, cols, colors, v, &m);
  marks_free(&m);
  return c;
}

void oracle_tentative_snapshot(const uint64_t* off, const uint32_t* cols,
                               const int32_t* colors_in, const uint32_t* wl, int64_t nwl,
                               int32_t* colors_out) {
  uint64_t maxd = 0;
  for (int64_t i = 0; i < nwl; ++i) {
    uint64_t d = off[wl[i] + 1] - off[wl[i]];
    if (d > maxd) maxd = d;
  }
  marks_t m;
  marks_init(&m, maxd + 1);
  for (int64_t i = 0; i < nwl; ++i) colors_out[wl[i]] = sac(off, cols, colors_in, wl[i], &m);
  marks_free(&m);
}

/* first_fit_sequential (coloring.hpp:110-116) */
void oracle_first_fit_sequential(const uint64_t* off, const uint32_t* cols, uint32_t n,
                                 int32_t* colors_out) {
  uint64_t maxd = 0;
  for (uint32_t v = 0; v < n; ++v)
    if (off[v + 1] - off[v] > maxd) maxd = off[v + 1] - off[v];
  for (uint32_t v = 0; v < n; ++v) colors_out[v] = ORACLE_UNCOLORED;
  marks_t m;
  marks_init(&m, maxd + 1);
  for (uint32_t v = 0; v < n; ++v) colors_out[v] = sac(off, cols, colors_out, v, &m);
  marks_free(&m);
}

/* Index of the first entry of row v with id > v (std::upper_bound). */
static uint64_t upper_bound_row(const uint64_t* off, const uint32_t* cols, uint32_t v) {
  uint64_t lo = off[v], hi = off[v + 1];
  while (lo < hi) {
    uint64_t mid = lo + (hi - lo) / 2;
    if (cols[mid] <= v) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}

/* has_conflicting_higher_neighbor (coloring.hpp:121-129): the LOWER-id
 * endpoint of a monochromatic edge is the defective one. */
int oracle_has_conflicting_higher_neighbor(const uint64_t* off, const uint32_t* cols,
                                           const int32_t* colors, uint32_t v) {
  const int32_t cv = load_relaxed(&colors[v]);
  if (cv == ORACLE_UNCOLORED) return 0;
  for (uint64_t i = upper_bound_row(off, cols, v); i < off[v + 1]; ++i)
    if (load_relaxed(&colors[cols[i]]) == cv) return 1;
  return 0;
}

/* defective_relaxed (parallel.hpp:105-111): same scan, but no uncolored
 * shortcut (every vertex is colored after the initial pass). */
static int defective_relaxed(const uint64_t* off, const uint32_t* cols, const int32_t* colors,
                             uint32_t v) {
  const int32_t cv = load_relaxed(&colors[v]);
  for (uint64_t i = upper_bound_row(off, cols, v); i < off[v + 1]; ++i)
    if (load_relaxed(&colors[cols[i]]) == cv) return 1;
  return 0;
}

int64_t oracle_detect_conflicts(const uint64_t* off, const uint32_t* cols,
                                const int32_t* colors, const uint32_t* pending,
                                int64_t npending, uint32_t* out) {
  int64_t k = 0;
  for (int64_t i = 0; i < npending; ++i)
    if (oracle_has_conflicting_higher_neighbor(off, cols, colors, pending[i])) out[k++] = pending[i];
  return k;
}

/* verify_coloring (coloring.hpp:159-177) */
int64_t oracle_verify_coloring(const uint64_t* off, const uint32_t* cols, uint32_t n,
                               const int32_t* colors, uint32_t* out_u, uint32_t* out_v,
                               int32_t* out_c, int64_t cap) {
  int64_t k = 0;
  for (uint32_t v = 0; v < n; ++v) {
    const int32_t cv = colors[v];
    if (cv == ORACLE_UNCOLORED) {
      if (k < cap) { out_u[k] = v; out_v[k] = ORACLE_NO_VERTEX; out_c[k] = ORACLE_UNCOLORED; }
      ++k;
      continue;
    }
    for (uint64_t i = upper_bound_row(off, cols, v); i < off[v + 1]; ++i)
      if (colors[cols[i]] == cv) {
        if (k < cap) { out_u[k] = v; out_v[k] = cols[i]; out_c[k] = cv; }
        ++k;
      }
  }
  return k;
}

/* count_colors (coloring.hpp:181-196): number of DISTINCT colors. */
int64_t oracle_count_colors(const int32_t* colors, int64_t n) {
  int32_t maxc = -1;
  for (int64_t i = 0; i < n; ++i) {
    if (colors[i] == ORACLE_UNCOLORED) return -1;
    if (colors[i] < 0) return -2;
    if (colors[i] > maxc) maxc = colors[i];
  }
  if (maxc < 0) return 0;
  unsigned char* used = (unsigned char*)calloc((size_t)maxc + 1, 1);
  for (int64_t i = 0; i < n; ++i) used[colors[i]] = 1;
  int64_t d = 0;
  for (int32_t c = 0; c <= maxc; ++c) d += used[c];
  free(used);
  return d;
}

/* ------------------------------------------------------------------ */
/* Parallel drivers (parallel.hpp:76-319)                               */
/* ------------------------------------------------------------------ */

/* A barrier whose completion step runs on the last arriving thread while all
 * others are still blocked -- the std::barrier(completion) semantics the
 * reference relies on (parallel.hpp:213, :281). */
typedef struct {
  pthread_mutex_t mu;
  pthread_cond_t cv;
  uint32_t expected, arrived;
  uint64_t generation;
  void (*completion)(void*);
  void* ctx;
} cbarrier_t;

static void cbarrier_init(cbarrier_t* b, uint32_t n, void (*fn)(void*), void* ctx) {
  pthread_mutex_init(&b->mu, NULL);
  pthread_cond_init(&b->cv, NULL);
  b->expected = n;
  b->arrived = 0;
  b->generation = 0;
  b->completion = fn;
  b->ctx = ctx;
}
static void cbarrier_destroy(cbarrier_t* b) {
  pthread_mutex_destroy(&b->mu);
  pthread_cond_destroy(&b->cv);
}
static void cbarrier_arrive_and_wait(cbarrier_t* b) {
  pthread_mutex_lock(&b->mu);
  uint64_t gen = b->generation;
  if (++b->arrived == b->expected) {
    b->completion(b->ctx);
    b->arrived = 0;
    b->generation++;
    pthread_cond_broadcast(&b->cv);
  } else {
    while (gen == b->generation) pthread_cond_wait(&b->cv, &b->mu);
  }
  pthread_mutex_unlock(&b->mu);
}

/* pick_chunk_size (parallel.hpp:83-88) */
static uint64_t pick_chunk_size(uint64_t items, uint32_t threads, uint64_t chunk, uint64_t minc) {
  if (chunk > 0) return chunk;
  uint64_t t = items / (8ull * threads);
  if (t < minc) t = minc;
  if (t < 1) t = 1;
  return t;
}

typedef struct {
  /* inputs */
  const uint64_t* off;
  const uint32_t* cols;
  uint32_t n, maxdeg, threads;
  uint64_t chunk_opt, min_chunk, round_cap;
  int algorithm;
  int32_t* colors;
  /* round state (RoundState, parallel.hpp:115-138) */
  uint32_t* worklist;
  uint64_t wl_len;
  uint32_t** local;   /* per-worker defect lists */
  uint64_t* local_len;
  uint64_t chunk_size;
  uint64_t next_chunk; /* atomic cursor */
  int done, capped, phase_flag;
  /* stats */
  oracle_stats* st;
} run_t;

static void stats_push(oracle_stats* st, uint64_t found) {
  if (st->conflicts_per_round && st->cpr_len < st->cpr_cap) st->conflicts_per_round[st->cpr_len] = found;
  st->cpr_len++;
}

/* merge_defects + finish_round (parallel.hpp:128-154) */
static void finish_round(run_t* r) {
  uint64_t found = 0;
  r->wl_len = 0;
  for (uint32_t w = 0; w < r->threads; ++w) {
    memcpy(r->worklist + r->wl_len, r->local[w], sizeof(uint32_t) * (size_t)r->local_len[w]);
    r->wl_len += r->local_len[w];
    found += r->local_len[w];
    r->local_len[w] = 0;
  }
  r->st->rounds += 1;
  stats_push(r->st, found);
  r->st->conflicts_total += found;
  if (r->wl_len == 0) {
    r->done = 1;
  } else if (r->st->rounds >= r->round_cap) {
    r->done = 1;
    r->capped = 1;
  } else {
    r->chunk_size = pick_chunk_size(r->wl_len, r->threads, r->chunk_opt, r->min_chunk);
  }
}

static void rsoc_completion(void* ctx) {
  run_t* r = (run_t*)ctx;
  r->st->barrier_events += 1;
  if (!r->phase_flag) { /* initial pass done: worklist = iota(n) (:272-275) */
    r->phase_flag = 1;
    for (uint32_t v = 0; v < r->n; ++v) r->worklist[v] = v;
    r->wl_len = r->n;
  } else {
    finish_round(r);
  }
  __atomic_store_n(&r->next_chunk, 0, __ATOMIC_RELAXED);
}

static void cat_completion(void* ctx) {
  run_t* r = (run_t*)ctx;
  r->st->barrier_events += 1;
  if (!r->phase_flag) {
    r->phase_flag = 1; /* tentative phase ended (:205-206) */
  } else {
    r->phase_flag = 0;
    finish_round(r);
  }
  __atomic_store_n(&r->next_chunk, 0, __ATOMIC_RELAXED);
}

typedef struct {
  run_t* r;
  cbarrier_t* bar;
  uint32_t wid;
} worker_arg_t;

/* Claim contiguous chunks in ascending order (for_claimed_chunks,
 * parallel.hpp:90-102); returns 0 when exhausted. */
static int claim(run_t* r, uint64_t total, uint64_t* b, uint64_t* e) {
  if (total == 0) return 0;
  const uint64_t nch = (total + r->chunk_size - 1) / r->chunk_size;
  uint64_t k = __atomic_fetch_add(&r->next_chunk, 1, __ATOMIC_RELAXED);
  if (k >= nch) return 0;
  *b = k * r->chunk_size;
  *e = *b + r->chunk_size < total ? *b + r->chunk_size : total;
  return 1;
}

static void push_local(run_t* r, uint32_t wid, uint32_t v) { r->local[wid][r->local_len[wid]++] = v; }

/* Worker body of color_rsoc (parallel.hpp:283-314). */
static void* rsoc_worker(void* p) {
  worker_arg_t* a = (worker_arg_t*)p;
  run_t* r = a->r;
  marks_t m;
  marks_init(&m, (uint64_t)r->maxdeg + 1);
  uint64_t b, e;
  while (claim(r, r->n, &b, &e))
    for (uint64_t i = b; i < e; ++i)
      store_relaxed(&r->colors[i], sac(r->off, r->cols, r->colors, (uint32_t)i, &m));
  cbarrier_arrive_and_wait(a->bar);
  for (;;) {
    while (claim(r, r->wl_len, &b, &e))
      for (uint64_t i = b; i < e; ++i) {
        const uint32_t v = r->worklist[i];
        if (defective_relaxed(r->off, r->cols, r->colors, v)) {
          store_relaxed(&r->colors[v], sac(r->off, r->cols, r->colors, v, &m));
          push_local(r, a->wid, v);
        }
      }
    cbarrier_arrive_and_wait(a->bar);
    if (r->done) break;
  }
  marks_free(&m);
  return NULL;
}

/* Worker body of color_catalyurek (parallel.hpp:215-241). */
static void* cat_worker(void* p) {
  worker_arg_t* a = (worker_arg_t*)p;
  run_t* r = a->r;
  marks_t m;
  marks_init(&m, (uint64_t)r->maxdeg + 1);
  uint64_t b, e;
  for (;;) {
    while (claim(r, r->wl_len, &b, &e))
      for (uint64_t i = b; i < e; ++i) {
        const uint32_t v = r->worklist[i];
        store_relaxed(&r->colors[v], sac(r->off, r->cols, r->colors, v, &m));
      }
    cbarrier_arrive_and_wait(a->bar);
    while (claim(r, r->wl_len, &b, &e))
      for (uint64_t i = b; i < e; ++i) {
        const uint32_t v = r->worklist[i];
        if (oracle_has_conflicting_higher_neighbor(r->off, r->cols, r->colors, v))
          push_local(r, a->wid, v);
      }
    cbarrier_arrive_and_wait(a->bar);
    if (r->done) break;
  }
  marks_free(&m);
  return NULL;
}

/* repair_coloring (coloring.hpp:203-216): only reached on round_cap. */
static void repair(const uint64_t* off, const uint32_t* cols, uint32_t n, uint32_t maxdeg,
                   int32_t* colors) {
  marks_t m;
  marks_init(&m, (uint64_t)maxdeg + 1);
  for (uint32_t v = 0; v < n; ++v)
    if (colors[v] == ORACLE_UNCOLORED || oracle_has_conflicting_higher_neighbor(off, cols, colors, v))
      colors[v] = sac(off, cols, colors, v, &m);
  marks_free(&m);
}

static uint64_t now_ns(void) {
  struct timespec ts;
  clock_gettime(CLOCK_MONOTONIC, &ts);
  return (uint64_t)ts.tv_sec * 1000000000ull + (uint64_t)ts.tv_nsec;
}

static int run_parallel(int alg, const uint64_t* off, const uint32_t* cols, uint32_t n,
                        uint32_t max_degree, uint32_t threads, uint64_t chunk_size,
                        uint64_t min_chunk, uint64_t round_cap, int32_t* colors,
                        oracle_stats* st) {
  if (threads < 1) return -1; /* parallel.hpp:186, :255 */
  for (uint32_t v = 0; v < n; ++v) colors[v] = ORACLE_UNCOLORED;
  st->algorithm = alg;
  st->thread_count = threads;
  st->rounds = st->conflicts_total = st->barrier_events = 0;
  st->cpr_len = 0;
  st->num_colors = 0;
  st->fallback_triggered = 0;

  run_t r;
  memset(&r, 0, sizeof r);
  r.off = off; r.cols = cols; r.n = n; r.maxdeg = max_degree; r.threads = threads;
  r.chunk_opt = chunk_size; r.min_chunk = min_chunk; r.round_cap = round_cap;
  r.algorithm = alg; r.colors = colors; r.st = st;
  r.worklist = (uint32_t*)malloc(sizeof(uint32_t) * ((size_t)n + 1));
  r.local = (uint32_t**)malloc(sizeof(uint32_t*) * threads);
  r.local_len = (uint64_t*)calloc(threads, sizeof(uint64_t));
  for (uint32_t w = 0; w < threads; ++w) r.local[w] = (uint32_t*)malloc(sizeof(uint32_t) * ((size_t)n + 1));
  if (alg == ORACLE_ALG_CATALYUREK) {
    for (uint32_t v = 0; v < n; ++v) r.worklist[v] = v;
    r.wl_len = n;
  }
  r.chunk_size = pick_chunk_size(n, threads, chunk_size, min_chunk);

  cbarrier_t bar;
  cbarrier_init(&bar, threads, alg == ORACLE_ALG_RSOC ? rsoc_completion : cat_completion, &r);
  worker_arg_t* args = (worker_arg_t*)malloc(sizeof(worker_arg_t) * threads);
  pthread_t* tids = (pthread_t*)malloc(sizeof(pthread_t) * threads);
  void* (*body)(void*) = alg == ORACLE_ALG_RSOC ? rsoc_worker : cat_worker;

  const uint64_t t0 = now_ns(); /* timer excludes allocation (:267) */
  for (uint32_t w = 0; w < threads; ++w) {
    args[w].r = &r; args[w].bar = &bar; args[w].wid = w;
    if (w > 0) pthread_create(&tids[w], NULL, body, &args[w]);
  }
  body(&args[0]); /* the caller is worker 0 (parallel.hpp:156-162) */
  for (uint32_t w = 1; w < threads; ++w) pthread_join(tids[w], NULL);

  /* finalize_run (parallel.hpp:164-177) */
  if (r.capped) {
    st->fallback_triggered = 1;
    repair(off, cols, n, max_degree, colors);
  }
  st->wall_time_ns = now_ns() - t0;
  int rc = 0;
  uint32_t u, vv;
  int32_t c;
  if (oracle_verify_coloring(off, cols, n, colors, &u, &vv, &c, 0) != 0) rc = -3;
  else st->num_colors = (uint32_t)oracle_count_colors(colors, n);

  cbarrier_destroy(&bar);
  for (uint32_t w = 0; w < threads; ++w) free(r.local[w]);
  free(r.local); free(r.local_len); free(r.worklist); free(args); free(tids);
  return rc;
}

int oracle_color_rsoc(const uint64_t* off, const uint32_t* cols, uint32_t n, uint32_t max_degree,
                      uint32_t thread_count, uint64_t chunk_size, uint64_t min_chunk_size,
                      uint64_t round_cap, int32_t* colors_out, oracle_stats* stats) {
  return run_parallel(ORACLE_ALG_RSOC, off, cols, n, max_degree, thread_count, chunk_size,
                      min_chunk_size, round_cap, colors_out, stats);
}

int oracle_color_catalyurek(const uint64_t* off, const uint32_t* cols, uint32_t n,
                            uint32_t max_degree, uint32_t thread_count, uint64_t chunk_size,
                            uint64_t min_chunk_size, uint64_t round_cap, int32_t* colors_out,
                            oracle_stats* stats) {
  return run_parallel(ORACLE_ALG_CATALYUREK, off, cols, n, max_degree, thread_count, chunk_size,
                      min_chunk_size, round_cap, colors_out, stats);
}

/* ------------------------------------------------------------------ */
/* lockstep_color (lockstep.hpp:37-78)                                  */
/* ------------------------------------------------------------------ */

static int proper_complete(const uint64_t* off, const uint32_t* cols, uint32_t n,
                           const int32_t* c) {
  uint32_t u, v;
  int32_t cc;
  return oracle_verify_coloring(off, cols, n, c, &u, &v, &cc, 0) == 0;
}

int64_t oracle_lockstep_color(const uint64_t* off, const uint32_t* cols, uint32_t n,
                              const uint32_t* lane_of, uint64_t round_cap, int32_t* trace_out,
                              int32_t* converged) {
  if (round_cap < 1) return -1;
  *converged = 0;
  int32_t* cur = (int32_t*)malloc(sizeof(int32_t) * ((size_t)n + 1));
  int32_t* nxt = (int32_t*)malloc(sizeof(int32_t) * ((size_t)n + 1));
  for (uint32_t v = 0; v < n; ++v) cur[v] = ORACLE_UNCOLORED;
  int64_t rounds = 0;
  if (proper_complete(off, cols, n, cur)) { /* vacuously proper (:47-50) */
    *converged = 1;
    free(cur); free(nxt);
    return 0;
  }
  uint64_t maxd = 0;
  for (uint32_t v = 0; v < n; ++v)
    if (off[v + 1] - off[v] > maxd) maxd = off[v + 1] - off[v];
  marks_t m;
  marks_init(&m, maxd + 1);
  for (uint64_t round = 1; round <= round_cap; ++round) {
    memcpy(nxt, cur, sizeof(int32_t) * n);
    for (uint32_t v = 0; v < n; ++v) {
      const int32_t limit = (int32_t)(off[v + 1] - off[v]);
      marks_next_epoch(&m);
      for (uint64_t i = off[v]; i < off[v + 1]; ++i) {
        const uint32_t w = cols[i];
        /* a lane sees its own earlier writes, others only at commit (:63-66) */
        const int32_t cw = (lane_of[w] == lane_of[v] && w < v) ? nxt[w] : cur[w];
        if (cw >= 0 && cw <= limit) m.stamps[cw] = m.epoch;
      }
      int32_t c = 0;
      while (c <= limit && m.stamps[c] == m.epoch) ++c;
      nxt[v] = c;
    }
    int32_t* t = cur; cur = nxt; nxt = t;
    memcpy(trace_out + (size_t)(round - 1) * n, cur, sizeof(int32_t) * n);
    rounds = (int64_t)round;
    if (proper_complete(off, cols, n, cur)) {
      *converged = 1;
      break;
    }
  }
  marks_free(&m);
  free(cur); free(nxt);
  return rounds;
}
