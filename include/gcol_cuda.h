/*
 * gcol_cuda.h -- C ABI of the B200 (sm_100a) RSOC graph-coloring library.
 *
 * Drop-in boundary for the reference's coloring entry points
 * (/root/reference/proj/include/gcol/...):
 *
 *   reference                                  replaced by
 *   ---------------------------------------    ---------------------------------
 *   Graph / build_graph   graph.hpp:20-138     gcol_cuda_graph_create (uploads a
 *                                              canonical CSR once; the graph is
 *                                              immutable like gcol::Graph)
 *   color_rsoc            parallel.hpp:253-319 gcol_cuda_color_rsoc
 *   run_coloring          bench.hpp:35-60      gcol_cuda_run_coloring (seq | rsoc)
 *   first_fit_sequential  coloring.hpp:110-116 gcol_cuda_first_fit_sequential
 *   smallest_available_color coloring.hpp:95-106
 *                                              gcol_cuda_tentative_snapshot
 *   detect_conflicts      coloring.hpp:133-141 gcol_cuda_detect_conflicts
 *   verify_coloring       coloring.hpp:159-177 gcol_cuda_verify_coloring
 *   count_colors          coloring.hpp:181-196 gcol_cuda_count_colors
 *   ColoringStats         parallel.hpp:47-57   gcol_cuda_stats
 *   ParallelOptions       parallel.hpp:64-72   gcol_cuda_options
 *   errors.hpp exception taxonomy              gcol_status codes (below)
 *
 * Plain C types only: int64 row offsets (n+1), int32 column ids (m), int32
 * colors (-1 = uncolored).  Pointers may be host or device memory; the
 * `memory` arguments say which.  Nothing here falls back to the CPU: with no
 * usable CUDA device every call returns GCOL_ERR_NO_DEVICE.
 * A graph handle is not thread-safe (one stream per handle); separate
 * handles may be used concurrently.
 */
#ifndef GCOL_CUDA_H
#define GCOL_CUDA_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define GCOL_CUDA_ABI_VERSION 2

/* Status codes.  The C++ adapter (gcol_cuda.hpp) rethrows them as the
 * reference's exceptions (errors.hpp:11-52). */
typedef enum {
  GCOL_OK = 0,
  GCOL_ERR_INVALID_ARGUMENT = 1, /* gcol::input_error */
  GCOL_ERR_CAPACITY = 2,         /* gcol::capacity_error */
  GCOL_ERR_CUDA = 3,             /* CUDA runtime failure (message in last_error) */
  GCOL_ERR_NCCL = 4,             /* collective failure (multi-GPU) */
  GCOL_ERR_ROUND_CAP = 5,        /* round_cap reached; the reference would run its
                                    sequential repair here -- we never fall back
                                    to the CPU, so this is an error */
  GCOL_ERR_VERIFY = 6,           /* improper result (gcol::verification_error /
                                    the logic_error of parallel.hpp:174-175) */
  GCOL_ERR_NO_DEVICE = 7         /* no CUDA device: there is no CPU fallback */
} gcol_status;

/* Where a pointer lives. */
typedef enum { GCOL_MEM_HOST = 0, GCOL_MEM_DEVICE = 1 } gcol_memory;

/* Which endpoint of a monochromatic edge recolors.  Any strict total order
 * terminates; ID_LOW is the reference rule
 * (coloring.hpp:118-120: "the lower-indexed endpoint is the one that
 * recolors") and the default. */
typedef enum {
  GCOL_PRIORITY_DEFAULT = 0,   /* library default: DEGREE_ID (the rule that keeps the
                                  colour count inside the reference's band at GPU
                                  concurrency) */
  GCOL_PRIORITY_ID_LOW = 1,    /* reference: lower id recolors (full neighbourhood) */
  GCOL_PRIORITY_ID_HIGH = 2,   /* mirror: higher id recolors (full neighbourhood) */
  GCOL_PRIORITY_DEGREE_ID = 3, /* lower (degree, id) recolors (full neighbourhood) */
  GCOL_PRIORITY_ORDERED = 4    /* higher id recolors -- "only if it loses a tie to a
                                  lower-id neighbour" -- with First-Fit over its lower
                                  neighbours, pushing higher neighbours it now collides
                                  with; converges towards sequential First-Fit quality */
} gcol_priority;

/* Algorithm ids follow gcol::Algorithm (parallel.hpp:21). */
typedef enum { GCOL_ALG_SEQ = 0, GCOL_ALG_CATALYUREK = 1, GCOL_ALG_RSOC = 2 } gcol_algorithm;

/* ParallelOptions (parallel.hpp:64-72) plus device knobs.  Zero-initialise
 * and set struct_size = sizeof(gcol_cuda_options); zero fields = defaults. */
typedef struct {
  uint32_t struct_size;
  uint32_t thread_count;     /* recorded in stats only (the GPU has no threads knob) */
  uint64_t chunk_size;       /* accepted for API parity; ignored on the GPU */
  uint64_t min_chunk_size;   /* accepted for API parity; ignored on the GPU */
  uint64_t round_cap;        /* 0 -> 1000 (parallel.hpp:71) */
  int32_t priority;          /* gcol_priority; 0 = library default */
  int32_t k1_blocks_per_sm;  /* K1 residency (in-flight window) knob, 0 = auto */
  int32_t k1_read_all;       /* 0 (default): the initial pass gathers only the
                                lower-id neighbours' colours; 1: every neighbour,
                                like smallest_available_color (coloring.hpp:95-106).
                                Both are valid RSOC initial passes. */
  int32_t k1_split_min_degree; /* rows at least this long are split into 1024-entry
                                  pieces that every warp helps colour; 0 = default
                                  (1024) */
  int32_t k1_wide;           /* initial-pass kernel: 0 auto (the waiting pass K1W when every
                                row has degree <= 63, else the class-split pass K1H + K1L),
                                1 narrow k1_pipe (8 consumer warps per SM), 2 wide k1_pipe
                                (16), 3 K1W where it applies, 4 class split (waiting heavy pass: exact
                                once the colour array exceeds L2, else with a short budget of
                                polls after which a row colours past a pending neighbour and the
                                rounds repair it), 5 class split with the speculative heavy pass,
                                6 class split with the waiting heavy pass (the result is then
                                sequential First-Fit in the order "rows of degree >= 64
                                ascending, then the others ascending", bit for bit) */
  int32_t k1_wait_polls;     /* K1W: re-checks of a row's in-flight lower neighbours before
                                it colours past them and logs the reads for round 1;
                                0 default (4096), < 0 none (purely optimistic) */
  int32_t reserved[2];
} gcol_cuda_options;

/* ColoringStats (parallel.hpp:47-57) + device-side instrumentation. */
typedef struct {
  int32_t algorithm;
  uint32_t thread_count;
  uint64_t rounds;
  uint64_t conflicts_total;
  uint64_t barrier_events;     /* rounds + 1 for rsoc (kernel boundaries) */
  uint32_t num_colors;         /* distinct colors (count_colors semantics) */
  uint32_t fallback_triggered; /* always 0: no CPU repair exists here */
  uint64_t wall_time_ns;       /* device time of the coloring graph (CUDA events) */
  uint64_t initial_pass_ns;    /* device time of the tentative-color kernel (K1) */
  uint64_t cpr_len;            /* == rounds */
  uint64_t* conflicts_per_round; /* caller buffer (may be NULL) */
  uint64_t cpr_cap;            /* its capacity */
  uint64_t pairs_logged;       /* K1 in-flight (u,v) observations */
  uint64_t round1_candidates;  /* vertices re-checked in round 1 */
  uint32_t pair_overflow;      /* 1 if round 1 had to scan all of V */
  int32_t priority;
  uint64_t k1_gathers;         /* neighbour-colour loads issued by K1 */
  uint64_t h2d_bytes;          /* bytes copied host -> device by this call (the first call
                                  on a handle also counts its graph upload: for
                                  gcol_cuda_color_rsoc_csr, everything that crossed PCIe up) */
  uint64_t d2h_bytes;          /* bytes copied device -> host by this call */
  uint64_t heavy_pass_ns;      /* class-split initial pass (skewed degree): device time of
                                  the heavy-row pass K1H (0 when the pass is not split) */
  uint64_t heavy_rows;         /* rows of that pass (degree >= 64) */
} gcol_cuda_stats;

/* verify_coloring (coloring.hpp:159-177) summary + color bound check. */
typedef struct {
  uint64_t violations;     /* == reference ConflictReport.violations.size() */
  uint64_t uncolored;      /* vertices with color -1 */
  uint64_t conflict_edges; /* monochromatic undirected edges */
  uint64_t out_of_bound;   /* vertices with color < -1 or color > degree */
  uint64_t negative;       /* vertices with color < -1 */
  uint32_t num_colors;     /* distinct non-negative colors (count_colors) */
  int32_t max_color;
} gcol_cuda_verify_report;

typedef struct gcol_cuda_graph gcol_cuda_graph;

/* Library / device queries. */
int gcol_cuda_abi_version(void);
int gcol_cuda_device_count(int32_t* count);
/* Thread-local message for the last failing call on this thread. */
const char* gcol_cuda_last_error(void);

/* Uploads (memory == HOST) or borrows (memory == DEVICE, caller keeps the
 * buffers alive and unchanged) a canonical CSR: offsets[0] == 0,
 * offsets[n] == m, rows sorted ascending, symmetric, no self loops
 * (graph.hpp:15-19; not re-validated beyond cheap checks).  n < 2^31 and
 * column ids < n.  m may exceed 2^31 (int64 offsets).  device < 0 selects
 * the current device. */
int gcol_cuda_graph_create(const int64_t* offsets, const int32_t* cols, int64_t n, int64_t m,
                           int32_t memory, int32_t device, gcol_cuda_graph** out);
int gcol_cuda_graph_destroy(gcol_cuda_graph* g);
int gcol_cuda_graph_info(const gcol_cuda_graph* g, int64_t* n, int64_t* m, int32_t* max_degree);

/* color_rsoc (parallel.hpp:253-319).  colors_out (n entries, host or
 * device per colors_memory) receives the final proper coloring; stats may be
 * NULL.  The run is verified on the device after the timed region (like
 * finalize_run, parallel.hpp:164-177); an improper result is
 * GCOL_ERR_VERIFY. */
int gcol_cuda_color_rsoc(gcol_cuda_graph* g, const gcol_cuda_options* opt, int32_t* colors_out,
                         int32_t colors_memory, gcol_cuda_stats* stats);

/* color_rsoc on a HOST CSR in one call (gcol::color_rsoc(g, T, opt) with a
 * host gcol::Graph, parallel.hpp:253): graph_create + color_rsoc +
 * graph_destroy, except that the adjacency is uploaded in pieces on a second
 * stream while the initial pass colours the rows already resident, so the
 * PCIe transfer and the coloring overlap.  Same checks and errors as
 * graph_create and color_rsoc; stats->wall_time_ns runs from the start of
 * the initial pass and so includes its waits for the upload. */
int gcol_cuda_color_rsoc_csr(const int64_t* offsets, const int32_t* cols, int64_t n, int64_t m,
                             int32_t device, const gcol_cuda_options* opt, int32_t* colors_out,
                             gcol_cuda_stats* stats);

/* color_catalyurek (parallel.hpp:180-246): rounds of a tentative First-Fit
 * phase over the worklist (in place, stale reads allowed) and a detection
 * phase whose defective vertices form the next worklist; W_1 = V.  Stats as
 * the reference's: barrier_events = 2 * rounds, conflicts_per_round[r] =
 * defective vertices found in round r (last entry 0).  `priority` picks the
 * endpoint that retries (ID_LOW is the reference's
 * has_conflicting_higher_neighbor). */
int gcol_cuda_color_catalyurek(gcol_cuda_graph* g, const gcol_cuda_options* opt,
                               int32_t* colors_out, int32_t colors_memory,
                               gcol_cuda_stats* stats);

/* run_coloring (bench.hpp:35-60) dispatch: GCOL_ALG_SEQ -> the exact
 * sequential First-Fit on the device, GCOL_ALG_RSOC -> color_rsoc,
 * GCOL_ALG_CATALYUREK -> color_catalyurek. */
int gcol_cuda_run_coloring(gcol_cuda_graph* g, int32_t algorithm, const gcol_cuda_options* opt,
                           int32_t* colors_out, int32_t colors_memory, gcol_cuda_stats* stats);

/* first_fit_sequential (coloring.hpp:110-116), bit-identical output. */
int gcol_cuda_first_fit_sequential(gcol_cuda_graph* g, int32_t* colors_out, int32_t colors_memory);

/* Snapshot-mode tentative pass (the production K1 with its in-place reads
 * redirected to a frozen snapshot): for every v in worklist (or all v when
 * worklist == NULL), colors_out[v] = smallest_available_color(v) computed
 * over colors_in (coloring.hpp:95-106).  lower_only != 0 restricts the
 * neighbourhood to ids < v (the initial-pass variant).  Deterministic.
 * All buffers in `memory`. */
int gcol_cuda_tentative_snapshot(gcol_cuda_graph* g, const int32_t* colors_in,
                                 const int32_t* worklist, int64_t nwl, int32_t lower_only,
                                 int32_t* colors_out, int32_t memory);

/* detect_conflicts (coloring.hpp:133-141) under a priority rule:
 * flags_out[i] = 1 iff pending[i] is defective.  ID_LOW reproduces the
 * reference predicate exactly.  pending == NULL means all vertices. */
int gcol_cuda_detect_conflicts(gcol_cuda_graph* g, const int32_t* colors, const int32_t* pending,
                               int64_t npending, int32_t priority, int32_t* flags_out,
                               int32_t memory);

/* One fused detect-and-recolor step (the K2 round body, parallel.hpp:297-313)
 * over `pending`, in place on `colors`; recolored ids are returned in
 * recolored_out (capacity npending), their number in *nrecolored.
 * Deterministic when `pending` is an independent set. */
int gcol_cuda_detect_and_recolor(gcol_cuda_graph* g, int32_t* colors, const int32_t* pending,
                                 int64_t npending, int32_t priority, int32_t* recolored_out,
                                 int64_t* nrecolored, int32_t memory);

/* verify_coloring (coloring.hpp:159-177).  Up to cap violations are written
 * (u, v, color) in the reference order; report may be NULL.  colors in
 * `memory`; out_* are host arrays (may be NULL when cap == 0). */
int gcol_cuda_verify_coloring(gcol_cuda_graph* g, const int32_t* colors, int64_t ncolors,
                              int32_t memory, gcol_cuda_verify_report* report, uint32_t* out_u,
                              uint32_t* out_v, int32_t* out_c, int64_t cap);

/* count_colors (coloring.hpp:181-196): distinct colors.  Incomplete or
 * negative colorings are GCOL_ERR_INVALID_ARGUMENT (input_error). */
int gcol_cuda_count_colors(gcol_cuda_graph* g, const int32_t* colors, int64_t ncolors,
                           int32_t memory, uint32_t* num_colors);

/* ---- Multi-GPU building blocks (one process and one handle per GPU) ----
 * Every rank keeps a full replica of the colour array on its device.  All
 * pointers are device pointers on the handle's device.  The host
 * orchestration is paper_1505_04086_b200/dist.py.
 *
 * Push mode (the product): ids are dealt out in 256-id
 * chunks, chunk c to rank c mod world, so all GPUs sweep the ids in one
 * ascending front; every colour a rank commits (initial pass and rounds)
 * is stored into its own replica AND into every peer's replica through
 * peer-mapped memory (NVLink), so other GPUs see it within the round. */

/* Registers this GPU as `rank` of `world` (<= 8) with the peers' replicas
 * (world device pointers, mapped into this process, e.g. by CUDA IPC;
 * entry `rank` is ignored).  Used by k1_owned and round_list. */
int gcol_cuda_partition_set(gcol_cuda_graph* g, int32_t rank, int32_t world,
                            int32_t* const* peer_colors);

/* Peer mapping of a replica between processes (CUDA IPC): export gives the
 * 64-byte handle of the allocation holding dev_ptr and dev_ptr's offset in
 * it; import maps a peer's handle into this process (peer access enabled)
 * and returns base + offset; close unmaps it. */
int gcol_cuda_ipc_export(const void* dev_ptr, uint8_t handle_out[64], uint64_t* offset_out);
int gcol_cuda_ipc_import(const uint8_t handle[64], uint64_t offset, void** dev_ptr_out);
int gcol_cuda_ipc_close(void* dev_ptr, uint64_t offset);

/* Initial pass over the owned chunks, in place on colors_dev, pushing every
 * committed colour to the peers.  Call after every replica is initialised
 * to -1 (barrier). */
int gcol_cuda_k1_owned(gcol_cuda_graph* g, const gcol_cuda_options* opt, int32_t* colors_dev,
                       gcol_cuda_stats* stats);

/* Round-1 candidates from the observation log of the last k1_owned: the
 * losers (under `priority`) of logged pairs whose colours are now equal,
 * owned or not -> cand_out (device, capacity n), count in *ncand.  Call
 * after every rank's k1_owned has completed (barrier), so the remote
 * endpoints' colours have arrived. */
int gcol_cuda_candidates(gcol_cuda_graph* g, int32_t priority, const int32_t* colors_dev,
                         int32_t* cand_out, int64_t* ncand);

/* Baseline mode (contiguous ranges, NCCL exchange at round boundaries):
 * each rank owns [lo, hi). */

/* Initial pass (K1) over the owned rows [lo, hi) in place on colors_dev
 * (lo a multiple of 256).  Colours of rows outside the range are read as
 * they are in the replica. */
int gcol_cuda_k1_range(gcol_cuda_graph* g, const gcol_cuda_options* opt, int32_t* colors_dev,
                       int64_t lo, int64_t hi, gcol_cuda_stats* stats);

/* Owned vertices of [lo, hi) defective under `priority` -> out_dev
 * (capacity hi - lo), count in *nout. */
int gcol_cuda_detect_range(gcol_cuda_graph* g, int32_t priority, const int32_t* colors_dev,
                           int64_t lo, int64_t hi, int32_t* out_dev, int64_t* nout);

/* One fused detect-and-recolor round over a device worklist, in place on
 * colors_dev; recoloured ids -> out_dev (capacity nin), count in *nout.
 * After gcol_cuda_partition_set the recolours are pushed to the peers. */
int gcol_cuda_round_list(gcol_cuda_graph* g, int32_t priority, int32_t* colors_dev,
                         const int32_t* in_dev, int64_t nin, int32_t* out_dev, int64_t* nout);

/* colors_dev[ids_dev[i]] = vals_dev[i] for i < count. */
int gcol_cuda_scatter_colors(gcol_cuda_graph* g, int32_t* colors_dev, const int32_t* ids_dev,
                             const int32_t* vals_dev, int64_t count);

#ifdef __cplusplus
}
#endif
#endif /* GCOL_CUDA_H */
