// gcol_k1w.cuh -- K1W, the waiting tentative-colour pass for graphs whose
// rows are all small (max degree <= kSmallMax = 63: thread per row,
// 64-bit register mask).
//
// Same contract as the in-place k1_pipe (parallel.hpp:286-296 with the
// lower-id neighbourhood): each vertex takes the smallest
// colour not carried by a lower-id neighbour, colours are written once, and
// every read of a still-uncoloured lower neighbour that is not resolved is
// logged for round 1.  What changes is how a stale read is treated: instead
// of colouring past it, the row WAITS for that neighbour (polling only its
// in-flight neighbours, up to `max_polls` times) and then commits.  Lower
// neighbours form a DAG and every warp of the grid is resident (the grid is
// sized to the occupancy), so the lowest pending row can always finish and
// waits resolve; the poll bound only guards against a warp that is not
// resident.  Because waiting -- not a small in-flight window -- is what keeps
// the colouring close to sequential First-Fit, the kernel can keep the
// whole GPU's worth of rows in flight: every warp of a fully occupied grid
// colours 32-row tiles independently (tile t -> warp t mod #warps), with
// the next tile's offsets prefetched while the current one is gathered.
//
// Per row (one lane): the lower-id prefix of the row is scanned kW = 4
// entries per step, the colours seen form a 32-bit forbidden mask when
// every degree is <= 31 (colours <= degree) and a 64-bit one otherwise, and
// the in-flight neighbours are remembered by their positions in the row (a
// 64-bit mask, deg <= 63) and re-read from the row when re-checked.
//
// Measured on B200 (profiles/r01/k1w_sweeps.md): the kernel is bound by the
// L1 wavefronts of its thread-per-row loads and by per-warp latency, not by
// the waits -- reading a frozen colour array (no in-flight reads at all)
// makes it only 15-30 % faster; staging the tile's adjacency in shared
// memory, 16-byte vector loads of aligned row chunks (1.4-1.8x slower),
// prefetching the next tile's adjacency (L2 or registers), parking pending
// rows while the next tile is scanned, and 8-wide steps all lost or
// tied.  48 resident warps per SM (40 registers) is the best occupancy.
#pragma once
#include "gcol_device.cuh"
#include "gcol_k1.cuh"

namespace gcol {
namespace dev {

constexpr int kWaitBlock = 256;        // threads per K1W CTA
constexpr int kWaitPollsDefault = 4096;

struct WaitArgs {
  const unsigned* piece_ready;  // streamed upload: flag per 2^piece_shift adjacency entries
  int piece_shift;              //   (null: the whole CSR is resident)
  int max_polls;                // re-checks of a pending row before it is logged
  int cstride, coffset;         // interleaved partition: 256-id chunks coffset + cstride*i
  int sleep_ns;                 // back-off between re-checks of a pending row
  unsigned long long* trace;    // GCOL_K1W_TRACE (tooling): per tile {start, end} ns
  unsigned long long loop;      // the round loop's WHILE handle (0: none)
  int close_round;              // the last CTA closes round 1 when nothing was logged
  int light_lim;                // class-split light pass: rows of degree >= light_lim are
                                //   the heavy pass's (already coloured, skipped)
  int light_coop;               // light pass: long rows scanned warp-cooperatively
  // light pass with compact heavy colours (class split on graphs whose colour array exceeds
  // L2, gcol_k1hw.cuh): the heavy-rank table ({bits, base} per 32 ids) and the heavy rows'
  // colours by rank, all final before this pass starts
  const uint2* rank;
  const int* hcol;
};

// Colour of neighbour w of light row v in the light pass, compact variant:
// the rank word says whether w is heavy (then its colour comes from the
// compact array, L2-resident) or light (a lower one is read from the colour
// array and may be in flight; a higher one has not started and is not read
// at all).  Two phases so that a step's rank loads are all in flight together.
__device__ __forceinline__ uint2 k1l_rank_word(const WaitArgs& A, int w) {
  uint2 r;
  asm volatile("ld.global.nc.v2.u32 {%0, %1}, [%2];" : "=r"(r.x), "=r"(r.y) : "l"(A.rank + (w >> 5)));
  return r;
}
__device__ __forceinline__ int k1l_colour(const WaitArgs& A, const int* colors, uint2 e, int w, int v) {
  const unsigned bit = 1u << (w & 31);
  if (e.x & bit) {
    int c;
    asm volatile("ld.global.nc.L1::no_allocate.b32 %0, [%1];"
                 : "=r"(c) : "l"(A.hcol + ((int)e.y + __popc(e.x & (bit - 1u)))));
    return c;
  }
  return w < v ? ld_color(colors + w) : -2;
}

__device__ __forceinline__ unsigned long long globaltimer_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

// Adjacency loads: read-only, L1-allocating (a warp's rows are contiguous,
// so successive entries of neighbouring lanes share sectors), L2 evict_first.
__device__ __forceinline__ int ld_col_l1(const int* p, uint64_t pol) {
  int r;
  asm volatile("ld.global.nc.L2::cache_hint.b32 %0, [%1], %2;" : "=r"(r) : "l"(p), "l"(pol));
  return r;
}

// Where a tile's adjacency entries are read from (thread per row).
struct ColsGlobal {
  const int* cols;
  uint64_t pol;
  __device__ __forceinline__ int operator()(long long i) const { return ld_col_l1(cols + i, pol); }
};

template <class Mask>
__device__ __forceinline__ Mask bit_of(int c) { return Mask(1) << c; }

template <class Mask>
__device__ __forceinline__ int first_free(Mask m) {
  if (sizeof(Mask) == 4) return __ffs(~static_cast<unsigned>(m)) - 1;
  return __ffsll(static_cast<long long>(~static_cast<unsigned long long>(m))) - 1;
}

// Scan of the lane's lower-id prefix (sorted row: stops at the first entry
// above v), warp-collective: mask = colours seen (<= deg), pp = positions of
// the neighbours read while still uncoloured (in flight).
// kClass (light pass of the class-split initial pass, gcol_k1c.cuh): the
// WHOLE row is read -- its heavy neighbours of any id were coloured by the
// heavy pass and must be avoided -- and only an uncoloured LOWER neighbour
// is in flight (an uncoloured higher one is a light row that reads this one).
template <int kW, class Mask, bool kClass = false>
__device__ __forceinline__ void k1w_scan(const ColsGlobal& src, const int* colors, int v,
                                         bool valid, long long b, int deg, unsigned& gathers,
                                         Mask& mask, unsigned long long& pp) {
  mask = 0;
  pp = 0ull;  // positions of in-flight lower neighbours
  bool active = valid && deg > 0;
  for (int k = 0; __any_sync(kFull, active); k += kW) {
    int w[kW];
#pragma unroll
    for (int j = 0; j < kW; ++j) w[j] = (active && k + j < deg) ? src(b + k + j) : 0x7fffffff;
    int c[kW];
#pragma unroll
    for (int j = 0; j < kW; ++j)
      c[j] = (kClass ? w[j] != 0x7fffffff : w[j] < v) ? ld_color(colors + w[j]) : -2;
#pragma unroll
    for (int j = 0; j < kW; ++j) {
      gathers += kClass ? w[j] != 0x7fffffff : w[j] < v;
      if (static_cast<unsigned>(c[j]) <= static_cast<unsigned>(deg)) mask |= bit_of<Mask>(c[j]);
      if (c[j] == -1 && (!kClass || w[j] < v)) pp |= 1ull << (k + j);
    }
    // sorted row: once an entry above v (or the row end) is reached, done
    active = active && k + kW < deg && (kClass || w[kW - 1] < v);
  }
}

// The light pass's scan (kClass): the WHOLE row, kW entries per step, with
// the next step's adjacency loads issued before this step's colour gathers,
// so a step costs one dependent round trip instead of two (light rows reach
// degree 63: up to 8 steps, and the slowest lane sets the tile's time).
template <int kW, class Mask>
__device__ __forceinline__ void k1l_scan(const ColsGlobal& src, const int* colors, int v,
                                         bool valid, long long b, int deg, unsigned& gathers,
                                         Mask& mask, unsigned long long& pp) {
  mask = 0;
  pp = 0ull;
  const int steps = valid ? (deg + kW - 1) / kW : 0;
  const int maxs = (int)__reduce_max_sync(kFull, (unsigned)steps);
  int wn[kW];
#pragma unroll
  for (int j = 0; j < kW; ++j) wn[j] = (valid && j < deg) ? src(b + j) : 0x7fffffff;
  for (int s = 0; s < maxs; ++s) {
    const int k = s * kW;
    int w[kW];
#pragma unroll
    for (int j = 0; j < kW; ++j) w[j] = wn[j];
    if (s + 1 < maxs) {
#pragma unroll
      for (int j = 0; j < kW; ++j) wn[j] = (valid && k + kW + j < deg) ? src(b + k + kW + j) : 0x7fffffff;
    }
    int c[kW];
#pragma unroll
    for (int j = 0; j < kW; ++j) c[j] = w[j] != 0x7fffffff ? ld_color(colors + w[j]) : -2;
#pragma unroll
    for (int j = 0; j < kW; ++j) {
      gathers += w[j] != 0x7fffffff;
      if (static_cast<unsigned>(c[j]) <= static_cast<unsigned>(deg)) mask |= bit_of<Mask>(c[j]);
      if (c[j] == -1 && w[j] < v) pp |= 1ull << (k + j);
    }
  }
}

// The light pass's tile scan, warp-cooperative for the long rows: rows of
// degree <= kLightShort are scanned by their own lane in one step; the
// tile's longer rows (R-MAT: ~3 per tile, degree up to 63) are scanned by
// the whole warp over their concatenated entries, 128 per step, the
// colours OR-ed into per-row masks in shared memory.  A tile then costs
// about two round trips instead of (its longest row / kW) of them.
constexpr int kLightShort = 8;
template <class Mask, bool kC = false>
__device__ __forceinline__ void k1l_scan_coop(const ColsGlobal& src, const int* colors, int v,
                                              bool valid, long long b, int deg, unsigned& gathers,
                                              Mask& mask, unsigned long long& pp,
                                              unsigned long long* smask, unsigned long long* spp,
                                              const WaitArgs& A) {
  const int lane = lane_id();
  mask = 0;
  pp = 0ull;
  // short rows: one step, every load in flight at once
  {
    const bool sh = valid && deg <= kLightShort;
    int w[kLightShort], c[kLightShort];
#pragma unroll
    for (int j = 0; j < kLightShort; ++j) w[j] = (sh && j < deg) ? src(b + j) : 0x7fffffff;
    if (kC) {
      uint2 e[kLightShort];
#pragma unroll
      for (int j = 0; j < kLightShort; ++j) e[j] = w[j] != 0x7fffffff ? k1l_rank_word(A, w[j]) : make_uint2(0u, 0u);
#pragma unroll
      for (int j = 0; j < kLightShort; ++j) c[j] = w[j] != 0x7fffffff ? k1l_colour(A, colors, e[j], w[j], v) : -2;
    } else {
#pragma unroll
      for (int j = 0; j < kLightShort; ++j) c[j] = w[j] != 0x7fffffff ? ld_color(colors + w[j]) : -2;
    }
#pragma unroll
    for (int j = 0; j < kLightShort; ++j) {
      gathers += w[j] != 0x7fffffff;
      if (static_cast<unsigned>(c[j]) <= static_cast<unsigned>(deg)) mask |= bit_of<Mask>(c[j]);
      if (c[j] == -1 && w[j] < v) pp |= 1ull << j;
    }
  }
  // long rows: warp-cooperative
  const bool lg = valid && deg > kLightShort;
  if (!__any_sync(kFull, lg)) return;
  smask[lane] = 0ull;
  spp[lane] = 0ull;
  const int len = lg ? deg : 0;
  int incl = len;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const int y = __shfl_up_sync(kFull, incl, d);
    if (lane >= d) incl += y;
  }
  const int eoff = incl - len;
  const int E = __shfl_sync(kFull, incl, 31);
  __syncwarp();
  constexpr int U = 4;
  for (int i0 = 0; i0 < E; i0 += 32 * U) {
    int w[U], r[U], jj[U], vr[U], dr[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int i = i0 + u * 32 + lane;
      const int rr = row_of(eoff, i);
      r[u] = rr;
      const long long br = __shfl_sync(kFull, b, rr);
      const int er = __shfl_sync(kFull, eoff, rr);
      vr[u] = __shfl_sync(kFull, v, rr);
      dr[u] = __shfl_sync(kFull, deg, rr);
      jj[u] = i - er;
      w[u] = i < E ? src(br + jj[u]) : 0x7fffffff;
    }
    int c[U];
    if (kC) {
      uint2 e[U];
#pragma unroll
      for (int u = 0; u < U; ++u) e[u] = w[u] != 0x7fffffff ? k1l_rank_word(A, w[u]) : make_uint2(0u, 0u);
#pragma unroll
      for (int u = 0; u < U; ++u) c[u] = w[u] != 0x7fffffff ? k1l_colour(A, colors, e[u], w[u], vr[u]) : -2;
    } else {
#pragma unroll
      for (int u = 0; u < U; ++u) c[u] = w[u] != 0x7fffffff ? ld_color(colors + w[u]) : -2;
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      gathers += w[u] != 0x7fffffff;
      if (static_cast<unsigned>(c[u]) <= static_cast<unsigned>(dr[u]))
        atomicOr(smask + r[u], 1ull << c[u]);
      if (c[u] == -1 && w[u] < vr[u]) atomicOr(spp + r[u], 1ull << jj[u]);
    }
  }
  __syncwarp();
  if (lg) {
    mask = static_cast<Mask>(smask[lane]);
    pp = spp[lane];
  }
  __syncwarp();
}

// Commit the row if nothing it read was in flight; else re-check the
// in-flight ones until they are coloured (after max_polls: log the rest for
// round 1) and commit.  Warp-collective.
template <class Mask>
__device__ __forceinline__ void k1w_wait(const ColsGlobal& src, int* colors, int v, bool valid,
                                         long long b, int deg, int max_polls, int sleep_ns,
                                         Mask mask, unsigned long long pp, const PairLogInl& L) {
  bool pend = pp != 0ull;
  if (valid && !pend) commit_color(colors, v, first_free(mask));
  for (int polls = 0; __any_sync(kFull, pend); ++polls) {
    if (polls >= max_polls) {
      // give up: log the still-uncoloured ones for round 1, commit
      while (__any_sync(kFull, pp != 0ull)) {
        const bool has = pp != 0ull;
        const int j = has ? __ffsll(static_cast<long long>(pp)) - 1 : 0;
        if (has) pp &= pp - 1;
        const int wj = has ? src(b + j) : 0;
        const int cj = has ? ld_color(colors + wj) : 0;
        if (has && static_cast<unsigned>(cj) <= static_cast<unsigned>(deg)) mask |= bit_of<Mask>(cj);
        log_pairs(L, has && cj == -1, wj, v);
      }
      if (pend) commit_color(colors, v, first_free(mask));
      break;
    }
    if (sleep_ns) __nanosleep(sleep_ns);
    if (pend) {
      for (unsigned long long q = pp; q; q &= q - 1) {
        const int j = __ffsll(static_cast<long long>(q)) - 1;
        const int cj = ld_color(colors + src(b + j));
        if (cj != -1) {
          pp &= ~(1ull << j);
          if (static_cast<unsigned>(cj) <= static_cast<unsigned>(deg)) mask |= bit_of<Mask>(cj);
        }
      }
      if (pp == 0ull) {
        commit_color(colors, v, first_free(mask));
        pend = false;
      }
    }
  }
}

constexpr int kWaitScanW = 4;   // adjacency entries per scan step
#ifndef GCOL_K1L_W
#define GCOL_K1L_W 8
#endif
constexpr int kLightScanW = GCOL_K1L_W;  // light pass (kClass): entries per pipelined step
#ifndef GCOL_K1L_MINB
#define GCOL_K1L_MINB 4
#endif
constexpr int kLightMinBlocks = GCOL_K1L_MINB;  // light pass: 32 resident warps per SM (64 registers)
constexpr int kWaitMinBlocks = 6;  // 48 resident warps per SM: 40 registers

// kM32: every degree is <= 31, so the forbidden set fits 32 bits.
// kClass: the light pass of the class-split initial pass (gcol_k1c.cuh):
// rows of degree >= A.light_lim are skipped and whole rows are scanned.
// kLC (with kClass): heavy neighbours' colours come from the compact array (A.rank, A.hcol).
template <bool kStream, bool kM32, bool kClass = false, bool kLC = false>
__global__ void __launch_bounds__(kWaitBlock, kClass ? kLightMinBlocks : kWaitMinBlocks)
    k1_wait(const long long* __restrict__ off, const int* __restrict__ cols, int n, int* colors,
            Ctrl* ctrl, PairLogArgs LA, WaitArgs A) {
  using Mask = typename std::conditional<kM32, unsigned, unsigned long long>::type;
  __shared__ unsigned long long s_lmask[kWaitBlock / 32][32], s_lpp[kWaitBlock / 32][32];
  __shared__ int s_npairs;
  __shared__ unsigned s_gathers;
  if (threadIdx.x == 0) {
    s_npairs = 0;
    s_gathers = 0;
  }
  init_peers(ctrl);
  __syncthreads();
  const int lane = lane_id();
  const int wpb = blockDim.x >> 5;
  const int gw = blockIdx.x * wpb + (threadIdx.x >> 5);
  const int NW = gridDim.x * wpb;
  const uint64_t pol = policy_evict_first();
  const ColsGlobal src{cols, pol};
  PairLogInl L;
  L.region = LA.pairs + (size_t)blockIdx.x * LA.region_cap;
  L.cap = LA.region_cap;
  L.s_count = &s_npairs;
  L.overflow = LA.overflow;
  unsigned gathers = 0;
  // local tile lt -> ids: chunk (lt / 8) of this partition, 32-id tile lt % 8
  const int nchunks_all = (n + 255) >> 8;
  const int nchunks = nchunks_all > A.coffset ? (nchunks_all - A.coffset + A.cstride - 1) / A.cstride : 0;
  const int ntiles = nchunks * 8;
  auto tile_v0 = [&](int lt) { return ((lt >> 3) * A.cstride + A.coffset) * 256 + (lt & 7) * 32; };
  int t = gw;
  long long b = 0;
  if (t < ntiles) b = ld_off(off + min(tile_v0(t) + lane, n), pol);
  for (; t < ntiles; t += NW) {
    const int v = tile_v0(t) + lane;
    const bool valid = v < n;
    long long e = __shfl_down_sync(kFull, b, 1);
    if (lane == 31) e = ld_off(off + min(v + 1, n), pol);
    // next tile's offsets in flight while this one is coloured
    const int tn = t + NW;
    long long nb = 0;
    if (tn < ntiles) nb = ld_off(off + min(tile_v0(tn) + lane, n), pol);
    const int deg0 = valid ? (int)(e - b) : 0;
    const bool mine = valid && (!kClass || deg0 < A.light_lim);
    const int deg = mine ? deg0 : 0;
    if (kStream) {  // streamed upload: the tile's adjacency must be resident
      const long long lo = __shfl_sync(kFull, b, 0), hi = __shfl_sync(kFull, e, 31);
      if (lane == 0 && hi > lo)
        for (long long p = lo >> A.piece_shift; p <= (hi - 1) >> A.piece_shift; ++p)
          while (ld_acquire_u32(A.piece_ready + p) == 0u) __nanosleep(256);
      __syncwarp();
    }
    unsigned long long t0 = 0;
    if (A.trace && lane == 0) t0 = globaltimer_ns();
    Mask mask;
    unsigned long long pp;
    if (kClass && (kLC || A.light_coop))
      k1l_scan_coop<Mask, kLC>(src, colors, v, mine, b, deg, gathers, mask, pp,
                               s_lmask[threadIdx.x >> 5], s_lpp[threadIdx.x >> 5], A);
    else if (kClass)
      k1l_scan<kLightScanW, Mask>(src, colors, v, mine, b, deg, gathers, mask, pp);
    else
      k1w_scan<kWaitScanW, Mask>(src, colors, v, mine, b, deg, gathers, mask, pp);
    k1w_wait<Mask>(src, colors, v, mine, b, deg, A.max_polls, A.sleep_ns, mask, pp, L);
    if (A.trace && lane == 0) {
      A.trace[2 * (size_t)t] = t0;
      A.trace[2 * (size_t)t + 1] = globaltimer_ns();
    }
    b = nb;
  }
  peers_fence();
  const unsigned g = __reduce_add_sync(kFull, gathers);
  if (lane == 0 && g) atomicAdd(&s_gathers, g);
  __syncthreads();
  if (threadIdx.x == 0) {
    if (s_gathers) atomicAdd(&ctrl->k1_gathers, (unsigned long long)s_gathers);
    LA.counts[blockIdx.x] = min(s_npairs, LA.region_cap);
    atomicAdd(&ctrl->pair_len, (unsigned long long)s_npairs);
    if (A.close_round) {
      // The last CTA to finish: with nothing logged (every in-flight read was
      // waited for -- the usual case) round 1's worklist is empty, so it
      // closes round 1 with no conflicts as k_control would
      // (finish_round, parallel.hpp:140-154) and the graph skips the loop
      // (k_candidates finds nothing to do).
      __threadfence();
      if (atomicAdd(&ctrl->k1_ctas_done, 1u) == gridDim.x - 1) {
        __threadfence();
        const unsigned long long pairs = atomicAdd(&ctrl->pair_len, 0ull);
        const int ovf = atomicAdd(&ctrl->pair_overflow, 0);
        if (pairs == 0ull && ovf == 0) {
          ctrl->round = 1;
          ctrl->cpr[0] = 0ull;
          ctrl->done = 1;
          if (A.loop) cudaGraphSetConditional(static_cast<cudaGraphConditionalHandle>(A.loop), 0u);
        }
      }
    }
  }
}

}  // namespace dev
}  // namespace gcol
