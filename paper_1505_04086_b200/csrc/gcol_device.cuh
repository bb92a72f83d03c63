// gcol_device.cuh -- device building blocks of the sm_100a RSOC path.
//
// Memory model.  Colours are read with ld.relaxed.gpu and written with
// st.relaxed.gpu: the CUDA counterpart of the reference's std::atomic_ref
// relaxed accesses (coloring.hpp:80-88).  Stale reads inside a round are
// allowed by the algorithm; kernel boundaries give the round-boundary
// visibility the termination argument needs.  CSR arrays are
// read-only and streamed with L1::no_allocate + an L2 evict_first policy so
// the colour array stays L2-resident while the adjacency streams past it.
#pragma once
#include <cstdint>
#include <climits>
#include <cuda_runtime.h>

namespace gcol {
namespace dev {

constexpr int kBlock = 256;             // threads per CTA everywhere
constexpr int kWarps = kBlock / 32;
constexpr int kSmallMax = 63;           // deg <= 63: thread-per-row, 64-bit register mask
constexpr int kWarpMax = 1023;          // 64..1023: warp per row, 1024-colour smem window
constexpr int kStage = 1024;            // staged adjacency entries per warp (4 KB)
constexpr int kStageStep = kStage - 64; // rows starting in a batch always fit the stage
constexpr int kBWinWords = 512;         // block window: 16384 colours (2 KB)
constexpr int kHPiece = 4096;           // entries per piece of a heavy row in the rounds
constexpr int kHeavyGridPerSM = 2;      // k_heavy CTAs per SM
constexpr int kMaxRoundsRecorded = 1 << 16;
constexpr unsigned kFull = 0xffffffffu;

// Who recolours on a monochromatic edge, and with which neighbourhood:
//   kIdLow   lower id recolours, full neighbourhood (reference/paper rule,
//            coloring.hpp:118-120, Alg. 3)
//   kIdHigh  higher id recolours, full neighbourhood (mirror)
//   kDegId   lower (degree, id) recolours, full neighbourhood
//   kOrdered higher id recolours ("a vertex recolours only if it loses a tie
//            to a lower-id neighbour", BASELINE north_star) with First-Fit over
//            its LOWER neighbours only, and pushes any higher neighbour its new
//            colour collides with.  Converges towards sequential First-Fit;
//            terminates because the minimum id recoloured strictly increases
//            round over round.
enum Rule : int { kIdLow = 0, kIdHigh = 1, kDegId = 2, kOrdered = 3 };

// Multi-GPU: every GPU keeps a full replica of the
// colours; a partitioned run commits each colour to the local replica and
// pushes it into every peer's replica (peer-mapped HBM over NVLink), so the
// other GPUs see it within the round.  The peer set is per launch: it lives
// in the handle's control block (Ctrl::peers, empty outside partitioned
// calls) and each kernel copies it into shared memory at entry
// (init_peers), so concurrent handles -- even several partitioned ones on
// one device -- never see each other's peers.
constexpr int kMaxPeers = 7;  // 8 GPUs per node
struct PeerSet {
  int* ptr[kMaxPeers];        // peer replicas (this GPU's own excluded)
  int n;
};

// Device control block: round state of the on-device round loop (the GPU
// RoundState of parallel.hpp:115-138).
struct Ctrl {
  unsigned long long ord_ticket;    // ordered round 1: members handed out in priority order
  unsigned long long pair_len;      // K1 in-flight observations logged
  unsigned long long k1_gathers;    // neighbour-colour loads issued by K1
  int* in_list;                     // current round's worklist
  int* out_list;                    // next round's worklist (R_r)
  int* flags;                       // detect-only API mode: per-position result
  int in_len;
  int out_len;
  int heavy_len;
  int recolored;                    // vertices recoloured in the current round
  int round;                        // completed detect-and-recolor rounds
  int round_cap;
  int pair_overflow;
  int capped;
  int cand_total;                   // round-1 candidates
  int ord_sorted;                   // ordered round 1: the worklist is in priority order
  int done;                         // loop exit flag (eager mode reads it)
  // heavy rows (deg > kWarpMax) of a round, split into kHPiece-entry pieces
  // spread over the whole grid (k_heavy); slots are per heavy row
  int heavy_slots;                  // slots used this round
  int heavy_pieces;                 // pieces queued this round
  int hslots;                       // slot capacity (0: split path off)
  int hq_cap;                       // piece capacity
  int2* hq;                         // (slot, first entry) per piece
  int* hslot_v;                     // row of a slot
  int* hslot_i;                     // its worklist position
  int* hslot_left;                  // pieces not finished yet
  int* hslot_flag;                  // 1: the row is defective
  unsigned* hslot_bm;               // [hslots][kBWinWords] colours seen, 0..16383
  unsigned k1_ctas_done;            // K1W: CTAs finished (the last one may end the run)
  unsigned long long prof[24];      // K1 phase cycle counters (GCOL_K1_PROFILE)
  PeerSet peers;                    // peer replicas of this launch (n = 0: none)
  unsigned long long cpr[kMaxRoundsRecorded];  // conflicts_per_round
};

// K1 observation log: every read of a lower neighbour that was still
// uncoloured (in flight) is recorded as (u, v).  Each CTA appends to its own
// slice of the log with a shared-memory counter, so logging never contends
// on a global atomic; an overflowing slice sets *overflow and round 1 scans
// all of V instead.
struct PairLog {
  int2* region;   // this CTA's slice
  int cap;        // slice capacity
  int* s_count;   // shared-memory fill counter
  int* overflow;  // global flag
};

// Kernel-argument form of the log (the per-CTA slice is derived in-kernel).
struct PairLogArgs {
  int2* pairs;
  int region_cap;
  int* counts;      // per-CTA fill counts (written at K1 exit)
  int* overflow;
};

__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}

__device__ __forceinline__ int ld_col(const int* p, uint64_t pol) {
  int r;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.b32 %0, [%1], %2;"
               : "=r"(r) : "l"(p), "l"(pol));
  return r;
}

__device__ __forceinline__ long long ld_off(const long long* p, uint64_t pol) {
  long long r;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.b64 %0, [%1], %2;"
               : "=l"(r) : "l"(p), "l"(pol));
  return r;
}

__device__ __forceinline__ int ld_color(const int* p) {
  int r;
  asm volatile("ld.relaxed.gpu.global.b32 %0, [%1];" : "=r"(r) : "l"(p) : "memory");
  return r;
}

__device__ __forceinline__ void st_color(int* p, int v) {
  asm volatile("st.relaxed.gpu.global.b32 [%0], %1;" :: "l"(p), "r"(v) : "memory");
}

// This CTA's copy of the launch's peer set (namespace-scope shared memory:
// one instance per CTA of every kernel that uses it).  init_peers must run
// before any commit_color, followed by a CTA barrier.
__shared__ PeerSet s_peers;

__device__ __forceinline__ void init_peers(const Ctrl* ctrl) {
  if (threadIdx.x == 0) s_peers = ctrl->peers;
}

__device__ __forceinline__ void st_color_sys(int* p, int v) {
  asm volatile("st.relaxed.sys.global.b32 [%0], %1;" :: "l"(p), "r"(v) : "memory");
}

__device__ __forceinline__ void commit_color(int* base, int v, int c) {
  st_color(base + v, c);
  const int np = s_peers.n;
  for (int q = 0; q < np; ++q) st_color_sys(s_peers.ptr[q] + v, c);
}

// Before a pushing kernel's threads exit: their peer stores are performed.
__device__ __forceinline__ void peers_fence() {
  if (s_peers.n) __threadfence_system();
}

// kSnap: snapshot mode reads a frozen, never-written array with plain loads.
template <bool kSnap>
__device__ __forceinline__ int read_color(const int* c, int w) {
  if (kSnap) return __ldg(c + w);
  return ld_color(c + w);
}

__device__ __forceinline__ int lane_id() { return threadIdx.x & 31; }

// Warp-aggregated append of (u, v) observations: one atomicAdd per warp.
// Must be called by all 32 lanes.
// The append itself is out of line: it is rare, and inlined at every call
// site it would swell the K1 kernel past the instruction cache.
__device__ __noinline__ void log_pairs_append(int2* region, int cap, int* s_count, int* overflow,
                                              unsigned m, bool pred, int u, int v) {
  const int lane = lane_id();
  const int leader = __ffs(m) - 1;
  int base = 0;
  if (lane == leader) base = atomicAdd(s_count, __popc(m));
  base = __shfl_sync(kFull, base, leader);
  if (pred) {
    const int idx = base + __popc(m & ((1u << lane) - 1u));
    if (idx < cap) region[idx] = make_int2(u, v);
    else *overflow = 1;
  }
}

__device__ __forceinline__ void log_pairs(const PairLog& L, bool pred, int u, int v) {
  const unsigned m = __ballot_sync(kFull, pred);
  if (m) log_pairs_append(L.region, L.cap, L.s_count, L.overflow, m, pred, u, v);
}

// The same log with the append inlined: for kernels whose register budget
// cannot afford an out-of-line call (the wide K1, 96 registers per thread).
struct PairLogInl : PairLog {};

__device__ __forceinline__ void log_pairs(const PairLogInl& L, bool pred, int u, int v) {
  const unsigned m = __ballot_sync(kFull, pred);
  if (!m) return;
  const int lane = lane_id();
  const int leader = __ffs(m) - 1;
  int base = 0;
  if (lane == leader) base = atomicAdd(L.s_count, __popc(m));
  base = __shfl_sync(kFull, base, leader);
  if (pred) {
    const int idx = base + __popc(m & ((1u << lane) - 1u));
    if (idx < L.cap) L.region[idx] = make_int2(u, v);
    else *L.overflow = 1;
  }
}

// Warp-aggregated append of ids to a list: one atomicAdd per warp.
__device__ __forceinline__ void append_warp(int* list, int* len, bool pred, int v) {
  const unsigned m = __ballot_sync(kFull, pred);
  if (!m) return;
  const int lane = lane_id();
  const int leader = __ffs(m) - 1;
  int base = 0;
  if (lane == leader) base = atomicAdd(len, __popc(m));
  base = __shfl_sync(kFull, base, leader);
  if (pred) list[base + __popc(m & ((1u << lane) - 1u))] = v;
}

// Priority order behind "who recolors": true iff v must yield to w on a
// monochromatic edge {v, w}.  Any strict total order terminates.
template <int R>
__device__ __forceinline__ bool yields_to(int v, int dv, int w, int dw) {
  if (R == kIdLow) return v < w;             // coloring.hpp:118-120
  if (R == kIdHigh || R == kOrdered) return v > w;
  return dv < dw || (dv == dw && v < w);      // lower (degree, id) yields
}

// Neighbours w a defect test of v has to look at under rule R.
template <int R>
__device__ __forceinline__ bool considers(int v, int w) {
  if (R == kIdLow) return w > v;
  if (R == kIdHigh || R == kOrdered) return w < v;
  return true;
}

// ---------------------------------------------------------------------------
// First-Fit over one row, warp-cooperative (deg <= kWarpMax).
// smallest colour in [0, deg] not carried by a (considered) neighbour
// (smallest_available_color, coloring.hpp:95-106).  kLower: consider only
// neighbours w < v (the initial-pass variant; rows are sorted, so the scan
// stops at the first chunk that reaches past v).  win: 32 smem words owned
// by this warp.  Returns the colour in every lane.
// ---------------------------------------------------------------------------
template <bool kSnap, bool kLower, bool kLog>
__device__ int warp_first_fit(const int* __restrict__ cols, const int* csrc, int v, long long b,
                              int deg, unsigned* win, uint64_t pol, const PairLog& L,
                              unsigned& gathers) {
  constexpr int U = 4;
  const int lane = lane_id();
  win[lane] = 0u;
  __syncwarp();
  unsigned long long reg = 0ull;
  for (int base = 0; base < deg; base += 32 * U) {
    int w[U];
    bool take[U];
    bool past = false;
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int i = base + u * 32 + lane;
      const bool in = i < deg;
      w[u] = in ? ld_col(cols + b + i, pol) : 0;
      take[u] = in && (!kLower || w[u] < v);
      past |= kLower && in && w[u] > v;
    }
    int c[U];
#pragma unroll
    for (int u = 0; u < U; ++u) c[u] = take[u] ? read_color<kSnap>(csrc, w[u]) : -2;
#pragma unroll
    for (int u = 0; u < U; ++u) {
      gathers += take[u];
      if (c[u] >= 0 && c[u] <= deg) {
        if (c[u] < 64) reg |= 1ull << c[u];
        else atomicOr(&win[c[u] >> 5], 1u << (c[u] & 31));
      }
      if (kLog) log_pairs(L, take[u] && c[u] == -1, w[u], v);
    }
    if (kLower && __any_sync(kFull, past)) break;
  }
  const unsigned lo = __reduce_or_sync(kFull, (unsigned)reg);
  const unsigned hi = __reduce_or_sync(kFull, (unsigned)(reg >> 32));
  __syncwarp();
  unsigned word = win[lane];
  if (lane == 0) word |= lo;
  if (lane == 1) word |= hi;
  // At most deg marks among deg+1 candidates, none above deg: a zero exists
  // at a position <= deg <= 1023, inside this single window.
  const unsigned nf = __ballot_sync(kFull, word != kFull);
  const int j = __ffs(nf) - 1;
  const unsigned wj = __shfl_sync(kFull, word, j);
  __syncwarp();
  return j * 32 + __ffs(~wj) - 1;
}

// ---------------------------------------------------------------------------
// First-Fit over one row, block-cooperative (any degree).  All threads of
// the CTA must call it with the same v.  bwin: kBWinWords smem words;
// sred: one smem int.  Windows of 16384 colours; a further window needs a
// rescan and can only happen with >= 16384 distinct neighbour colours.
// ---------------------------------------------------------------------------
template <bool kSnap, bool kLower, bool kLog>
__device__ int block_first_fit(const int* __restrict__ cols, const int* csrc, int v, long long b,
                               int deg, unsigned* bwin, int* sred, uint64_t pol,
                               const PairLog& L, unsigned& gathers) {
  constexpr int U = 4;
  const int tid = threadIdx.x;
  for (int wb = 0;; wb += kBWinWords * 32) {
    for (int i = tid; i < kBWinWords; i += kBlock) bwin[i] = 0u;
    if (tid == 0) *sred = INT_MAX;
    __syncthreads();
    unsigned long long reg = 0ull;
    for (int base = 0; base < deg; base += kBlock * U) {
      int w[U];
      bool take[U];
      bool past = false;
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int i = base + u * kBlock + tid;
        const bool in = i < deg;
        w[u] = in ? ld_col(cols + b + i, pol) : 0;
        take[u] = in && (!kLower || w[u] < v);
        past |= kLower && in && w[u] > v;
      }
      int c[U];
#pragma unroll
      for (int u = 0; u < U; ++u) c[u] = take[u] ? read_color<kSnap>(csrc, w[u]) : -2;
#pragma unroll
      for (int u = 0; u < U; ++u) {
        if (wb == 0) gathers += take[u];
        const int cc = c[u] - wb;
        if (c[u] >= wb && c[u] <= deg && cc < kBWinWords * 32) {
          if (cc < 64) reg |= 1ull << cc;
          else atomicOr(&bwin[cc >> 5], 1u << (cc & 31));
        }
        if (kLog) log_pairs(L, wb == 0 && take[u] && c[u] == -1, w[u], v);
      }
      if (kLower) {
        if (__syncthreads_or(past)) break;
      }
    }
    const unsigned lo = __reduce_or_sync(kFull, (unsigned)reg);
    const unsigned hi = __reduce_or_sync(kFull, (unsigned)(reg >> 32));
    if (lane_id() == 0) {
      if (lo) atomicOr(&bwin[0], lo);
      if (hi) atomicOr(&bwin[1], hi);
    }
    __syncthreads();
    // candidates in this window: positions [0, min(deg - wb, bits - 1)]
    const long long span = (long long)deg - wb + 1;
    const int nbits = span < kBWinWords * 32 ? (int)span : kBWinWords * 32;
    for (int i = tid; i * 32 < nbits; i += kBlock) {
      const int valid = nbits - i * 32;
      const unsigned vm = valid >= 32 ? kFull : ((1u << valid) - 1u);
      const unsigned fr = ~bwin[i] & vm;
      if (fr) atomicMin(sred, i * 32 + __ffs(fr) - 1);
    }
    __syncthreads();
    const int p = *sred;
    __syncthreads();
    if (p != INT_MAX) return wb + p;
  }
}

// ---------------------------------------------------------------------------
// Defect test of v under rule R, warp-cooperative (any degree).  Same
// predicate as has_conflicting_higher_neighbor (coloring.hpp:121-129) for
// R == kIdLow, including its uncoloured shortcut.
// ---------------------------------------------------------------------------
template <int R>
__device__ bool warp_defective(const long long* __restrict__ off, const int* __restrict__ cols,
                               const int* colors, int v, long long b, int deg, uint64_t pol) {
  constexpr int U = 4;
  const int lane = lane_id();
  const int cv = ld_color(colors + v);
  if (cv == -1) return false;
  for (int base = 0; base < deg; base += 32 * U) {
    int w[U];
    bool cons[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int i = base + u * 32 + lane;
      const bool in = i < deg;
      w[u] = in ? ld_col(cols + b + i, pol) : 0;
      cons[u] = in && considers<R>(v, w[u]);
    }
    bool hit = false;
#pragma unroll
    for (int u = 0; u < U; ++u) {
      if (cons[u] && ld_color(colors + w[u]) == cv) {
        if (R == kDegId) {
          const int dw = (int)(ld_off(off + w[u] + 1, pol) - ld_off(off + w[u], pol));
          hit |= yields_to<R>(v, deg, w[u], dw);
        } else {
          hit = true;
        }
      }
    }
    if (__any_sync(kFull, hit)) return true;
  }
  return false;
}

template <int R>
__device__ bool block_defective(const long long* __restrict__ off, const int* __restrict__ cols,
                                const int* colors, int v, long long b, int deg, uint64_t pol) {
  constexpr int U = 4;
  const int tid = threadIdx.x;
  const int cv = ld_color(colors + v);
  if (cv == -1) return false;
  for (int base = 0; base < deg; base += kBlock * U) {
    bool hit = false;
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int i = base + u * kBlock + tid;
      if (i < deg) {
        const int w = ld_col(cols + b + i, pol);
        const bool cons = considers<R>(v, w);
        if (cons && ld_color(colors + w) == cv) {
          if (R == kDegId) {
            const int dw = (int)(ld_off(off + w + 1, pol) - ld_off(off + w, pol));
            hit |= yields_to<R>(v, deg, w, dw);
          } else {
            hit = true;
          }
        }
      }
    }
    if (__syncthreads_or(hit)) return true;
  }
  return false;
}

// Thread-level defect test (fallback scan of all vertices).
template <int R>
__device__ bool thread_defective(const long long* __restrict__ off, const int* __restrict__ cols,
                                 const int* colors, int v, uint64_t pol) {
  const long long b = ld_off(off + v, pol), e = ld_off(off + v + 1, pol);
  const int cv = ld_color(colors + v);
  if (cv == -1) return false;
  const int dv = (int)(e - b);
  for (long long i = b; i < e; ++i) {
    const int w = ld_col(cols + i, pol);
    const bool cons = considers<R>(v, w);
    if (cons && ld_color(colors + w) == cv) {
      if (R != kDegId) return true;
      const int dw = (int)(ld_off(off + w + 1, pol) - ld_off(off + w, pol));
      if (yields_to<R>(v, dv, w, dw)) return true;
    }
  }
  return false;
}

// ---------------------------------------------------------------------------
// kOrdered push step: after v took colour c (First-Fit over its lower
// neighbours), every higher neighbour now carrying c is appended to the next
// worklist (once per round: marks[w] holds the round stamp of its last
// insertion).  Warp- and CTA-cooperative versions.
// ---------------------------------------------------------------------------
__device__ __forceinline__ bool claim_slot(int* marks, int w, int stamp) {
  return atomicMax(marks + w, stamp) < stamp;
}

__device__ void warp_push_higher(const int* __restrict__ cols, const int* colors, int v,
                                 long long b, int deg, int c, int* marks, int stamp, int* out,
                                 int* out_len, uint64_t pol) {
  const int lane = lane_id();
  for (int base = 0; base < deg; base += 32) {
    const int i = base + lane;
    bool pred = false;
    int w = 0;
    if (i < deg) {
      w = ld_col(cols + b + i, pol);
      if (w > v && ld_color(colors + w) == c) pred = claim_slot(marks, w, stamp);
    }
    append_warp(out, out_len, pred, w);
  }
}

__device__ void block_push_higher(const int* __restrict__ cols, const int* colors, int v,
                                  long long b, int deg, int c, int* marks, int stamp, int* out,
                                  int* out_len, uint64_t pol) {
  for (int base = 0; base < deg; base += kBlock) {
    const int i = base + threadIdx.x;
    bool pred = false;
    int w = 0;
    if (i < deg) {
      w = ld_col(cols + b + i, pol);
      if (w > v && ld_color(colors + w) == c) pred = claim_slot(marks, w, stamp);
    }
    append_warp(out, out_len, pred, w);
  }
}

}  // namespace dev
}  // namespace gcol
