// gcol_kernels.cuh -- the sm_100a kernels of the RSOC path.
//
//   K1 k1_tentative   initial tentative pass (parallel.hpp:286-296)
//   K2 k_candidates   round-1 worklist from K1's in-flight observations
//      k_list/k_heavy fused detect-and-recolor over a worklist
//                     (parallel.hpp:297-313 + defective_relaxed :105-111)
//   K3 k_control      round bookkeeping + CUDA-graph WHILE condition
//                     (barrier completion + finish_round, parallel.hpp:140-154)
//   K4 k_verify_*     verify_coloring / count_colors (coloring.hpp:159-196)
#pragma once
#include "gcol_device.cuh"

namespace gcol {
namespace dev {

// ---------------------------------------------------------------------------
// Deferred commit (K1, in-place mode).  A small row that read a lower
// neighbour still uncoloured does not commit at once: it parks its partial
// forbidden mask and the ids of the in-flight neighbours in a per-CTA table,
// and one tile later re-reads only those neighbours, which by then have
// almost always committed.  What is still uncoloured then is logged for
// round 1 exactly like an immediate stale read.  This keeps the initial
// pass close to sequential First-Fit even with ~10^5 vertices in flight.
// ---------------------------------------------------------------------------
constexpr int kDeferPairs = 384;

struct DeferTable {
  int* dv;           // [kBlock] vertex parked in this slot, -1 = none
  unsigned* dmask;   // [kBlock][2] 64-bit partial forbidden mask
  unsigned char* ddeg;  // [kBlock] degree (<= 63)
  int* du;           // [kDeferPairs] in-flight neighbour
  unsigned char* dslot; // [kDeferPairs] owning slot
  int* np;           // fill counter
};

// Warp-aggregated record of stale (u, slot) observations; overflow goes
// straight to the round-1 log.  All lanes must call.
__device__ __forceinline__ void defer_pairs(const DeferTable& D, const PairLog& L, bool pred,
                                            int u, int v, int slot) {
  const unsigned m = __ballot_sync(kFull, pred);
  if (!m) return;
  const int lane = lane_id();
  const int leader = __ffs(m) - 1;
  int base = 0;
  if (lane == leader) base = atomicAdd(D.np, __popc(m));
  base = __shfl_sync(kFull, base, leader);
  const int idx = base + __popc(m & ((1u << lane) - 1u));
  const bool spill = pred && idx >= kDeferPairs;
  if (pred && !spill) {
    D.du[idx] = u;
    D.dslot[idx] = (unsigned char)slot;
  }
  log_pairs(L, spill, u, v);
}

// ---------------------------------------------------------------------------
// Small rows (1 <= deg <= 63) of one warp's 32 consecutive items: the rows'
// adjacency is staged in shared memory with coalesced loads, then each lane
// runs First-Fit over its own row with a 64-bit register mask.  All lanes
// must call.  Items are rows of consecutive ids (or worklist entries).
// ---------------------------------------------------------------------------
template <bool kSnap, bool kLower, bool kLog>
__device__ void small_rows(const int* __restrict__ cols, const int* csrc, int* cdst, int v,
                           long long b, int deg, bool small, int* stage, uint64_t pol,
                           const PairLog& L, const DeferTable& D, unsigned& gathers) {
  const int lane = lane_id();
  const int len = small ? deg : 0;
  int incl = len;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const int y = __shfl_up_sync(kFull, incl, d);
    if (lane >= d) incl += y;
  }
  const int excl = incl - len;
  const int total = __shfl_sync(kFull, incl, 31);
  if (total == 0) return;
  // contiguous: every small row r is followed in memory by row r+1's start
  const long long nb = __shfl_down_sync(kFull, b, 1);
  const bool all_small_contig = __all_sync(kFull, (len == deg) && (lane == 31 || nb == b + deg));
  const long long b0 = __shfl_sync(kFull, b, 0);
  const int nbatch = (total + kStageStep - 1) / kStageStep;
  for (int bt = 0; bt < nbatch; ++bt) {
    const int lo = bt * kStageStep;
    const bool mine = small && excl >= lo && excl < lo + kStageStep;
    // ---- stage ----
    if (all_small_contig) {
      const int hi = min(total, lo + kStage);
      for (int i = lo + lane; i < hi; i += 32 * 4) {
        int x[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int j = i + u * 32;
          x[u] = j < hi ? ld_col(cols + b0 + j, pol) : 0;
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int j = i + u * 32;
          if (j < hi) stage[j - lo] = x[u];
        }
      }
    } else {
      unsigned rows = __ballot_sync(kFull, mine);
      while (rows) {
        const int r = __ffs(rows) - 1;
        rows &= rows - 1;
        const int lr = __shfl_sync(kFull, len, r);
        const int er = __shfl_sync(kFull, excl, r);
        const long long br = __shfl_sync(kFull, b, r);
        for (int t = lane; t < lr; t += 32) stage[er - lo + t] = ld_col(cols + br + t, pol);
      }
    }
    __syncwarp();
    // ---- First-Fit, thread per row ----
    const int myk = mine ? len : 0;
    const int maxk = __reduce_max_sync(kFull, (unsigned)myk);
    bool active = mine;
    bool stale_me = false;
    unsigned long long mask = 0ull;
    const int* row = stage + (excl - lo);
    for (int k = 0; k < maxk; k += 4) {
      int w[4];
      bool take[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const bool in = active && (k + u) < len;
        w[u] = in ? row[k + u] : 0;
        take[u] = in && (!kLower || w[u] < v);
        if (kLower && in && w[u] > v) active = false;  // sorted row: rest is > v
      }
      int c[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) c[u] = take[u] ? read_color<kSnap>(csrc, w[u]) : -2;
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        gathers += take[u];
        if (c[u] >= 0 && c[u] <= deg) mask |= 1ull << c[u];
        if (kLog) {
          const bool st = take[u] && c[u] == -1 && w[u] < v;
          stale_me |= st;
          defer_pairs(D, L, st, w[u], v, threadIdx.x);
        }
      }
      if (kLower && !__any_sync(kFull, active)) break;
    }
    if (mine) {
      if (kLog && stale_me) {  // park: commit after the recheck one tile later
        D.dv[threadIdx.x] = v;
        D.dmask[2 * threadIdx.x] = (unsigned)mask;
        D.dmask[2 * threadIdx.x + 1] = (unsigned)(mask >> 32);
        D.ddeg[threadIdx.x] = (unsigned char)deg;
      } else {
        st_color(cdst + v, __ffsll((long long)~mask) - 1);
      }
    }
    __syncwarp();
  }
}

// Recheck and commit the rows parked in table D (all CTA threads call).
__device__ void drain_deferred(const DeferTable& D, const PairLog& L, int* cdst) {
  const int np = min(*D.np, kDeferPairs);
  for (int p0 = (threadIdx.x & ~31); p0 < np; p0 += kBlock) {
    const int p = p0 + lane_id();
    bool still = false;
    int u = 0, v = 0;
    if (p < np) {
      u = D.du[p];
      const int slot = D.dslot[p];
      v = D.dv[slot];
      const int c = ld_color(cdst + u);
      if (c >= 0 && c <= (int)D.ddeg[slot]) atomicOr(&D.dmask[2 * slot + (c >> 5)], 1u << (c & 31));
      still = c == -1;
    }
    log_pairs(L, still, u, v);
  }
  __syncthreads();
  const int v = D.dv[threadIdx.x];
  if (v >= 0) {
    const unsigned long long mask =
        (unsigned long long)D.dmask[2 * threadIdx.x] |
        ((unsigned long long)D.dmask[2 * threadIdx.x + 1] << 32);
    st_color(cdst + v, __ffsll((long long)~mask) - 1);
  }
}

// ---------------------------------------------------------------------------
// K1: tentative First-Fit for every item, CTAs claiming 256-item tiles in
// ascending order from a device cursor (the GPU analog of the reference's
// ascending chunk claiming, parallel.hpp:76-102).  Per item the width is
// chosen by degree: thread (<= 63), warp (<= 1023), CTA (larger).
// In-place mode (kSnap = false) reads and writes the live colour array,
// defers small rows that saw an in-flight lower neighbour (above) and logs
// every still-stale read so round 1 only re-checks those edges.  Snapshot
// mode reads csrc, writes cdst.
// ---------------------------------------------------------------------------
template <bool kSnap, bool kLower, bool kLog>
__global__ void __launch_bounds__(kBlock) k1_tentative(const long long* __restrict__ off,
                                                       const int* __restrict__ cols, int n,
                                                       int nitems, const int* worklist,
                                                       const int* csrc, int* cdst, Ctrl* ctrl,
                                                       PairLogArgs LA) {
  __shared__ int s_stage[kWarps][kStage];
  __shared__ unsigned s_win[kWarps][32];
  __shared__ unsigned s_bwin[kBWinWords];
  __shared__ int s_heavy[kBlock];
  __shared__ int s_nheavy, s_tile, s_red, s_npairs;
  __shared__ unsigned s_gathers;
  // deferral tables (ping-pong: filled in tile t, drained at the end of t+1)
  __shared__ int s_dv[2][kBlock];
  __shared__ unsigned s_dmask[2][2 * kBlock];
  __shared__ unsigned char s_ddeg[2][kBlock];
  __shared__ int s_du[2][kDeferPairs];
  __shared__ unsigned char s_dslot[2][kDeferPairs];
  __shared__ int s_dnp[2];
  const uint64_t pol = policy_evict_first();
  const int warp = threadIdx.x >> 5, lane = lane_id();
  const int ntiles = (nitems + kBlock - 1) / kBlock;
  PairLog L{LA.pairs + (size_t)blockIdx.x * LA.region_cap, LA.region_cap, &s_npairs, LA.overflow};
  auto table = [&](int i) {
    return DeferTable{s_dv[i], s_dmask[i], s_ddeg[i], s_du[i], s_dslot[i], &s_dnp[i]};
  };
  unsigned gathers = 0;
  if (threadIdx.x == 0) {
    s_gathers = 0;
    s_npairs = 0;
  }
  int it = 0;
  for (;; ++it) {
    const DeferTable D = table(it & 1);
    if (threadIdx.x == 0) {
      s_tile = (int)atomicAdd(&ctrl->tile_cursor, 1ull);
      s_nheavy = 0;
      s_dnp[it & 1] = 0;
    }
    D.dv[threadIdx.x] = -1;
    __syncthreads();
    const int tile = s_tile;
    if (tile >= ntiles) break;
    const int item = tile * kBlock + threadIdx.x;
    const bool valid = item < nitems;
    const int v = valid ? (worklist ? worklist[item] : item) : n;
    const long long b = ld_off(off + v, pol);
    const long long e = valid ? ld_off(off + v + 1, pol) : b;
    const int deg = (int)(e - b);
    if (valid && deg == 0) st_color(cdst + v, 0);  // limit 0: only colour 0 (coloring.hpp:98-105)
    const bool small = valid && deg >= 1 && deg <= kSmallMax;
    const bool medium = valid && deg > kSmallMax && deg <= kWarpMax;
    if (valid && deg > kWarpMax) s_heavy[atomicAdd(&s_nheavy, 1)] = v;

    small_rows<kSnap, kLower, kLog>(cols, csrc, cdst, v, b, deg, small, s_stage[warp], pol, L, D,
                                    gathers);

    unsigned med = __ballot_sync(kFull, medium);
    while (med) {
      const int r = __ffs(med) - 1;
      med &= med - 1;
      const int vr = __shfl_sync(kFull, v, r);
      const long long br = __shfl_sync(kFull, b, r);
      const int dr = __shfl_sync(kFull, deg, r);
      const int c = warp_first_fit<kSnap, kLower, kLog>(cols, csrc, vr, br, dr, s_win[warp], pol,
                                                        L, gathers);
      if (lane == 0) st_color(cdst + vr, c);
    }
    __syncthreads();
    const int nh = s_nheavy;
    for (int h = 0; h < nh; ++h) {
      const int vh = s_heavy[h];
      const long long bh = ld_off(off + vh, pol);
      const int dh = (int)(ld_off(off + vh + 1, pol) - bh);
      const int c = block_first_fit<kSnap, kLower, kLog>(cols, csrc, vh, bh, dh, s_bwin, &s_red,
                                                         pol, L, gathers);
      if (threadIdx.x == 0) st_color(cdst + vh, c);
    }
    if (kLog && it > 0) drain_deferred(table((it + 1) & 1), L, cdst);  // rows parked in tile t-1
    __syncthreads();
  }
  if (kLog && it > 0) drain_deferred(table((it + 1) & 1), L, cdst);  // the last tile's rows
  const unsigned g = __reduce_add_sync(kFull, gathers);
  if (lane == 0 && g) atomicAdd(&s_gathers, g);
  __syncthreads();
  if (threadIdx.x == 0) {
    if (s_gathers) atomicAdd(&ctrl->k1_gathers, (unsigned long long)s_gathers);
    if (kLog) {
      LA.counts[blockIdx.x] = min(s_npairs, LA.region_cap);
      atomicAdd(&ctrl->pair_len, (unsigned long long)s_npairs);
    }
  }
}

// ---------------------------------------------------------------------------
// Round-1 worklist.  A monochromatic edge {u < v} after K1 implies v read u
// while u was still uncoloured (u is written once; v avoided every colour
// it saw), and every such read was logged.  So the defective set at the
// start of round 1 is contained in {loser of a logged pair with equal
// colours}.  Overflowed logs fall back to scanning all of V on the device.
// ---------------------------------------------------------------------------
template <int R>
__global__ void __launch_bounds__(kBlock) k_candidates(const long long* __restrict__ off,
                                                       const int* __restrict__ cols, int n,
                                                       const int* colors, Ctrl* ctrl,
                                                       PairLogArgs LA, int nregions, int* marks) {
  const uint64_t pol = policy_evict_first();
  int* list = ctrl->in_list;
  int* len = &ctrl->in_len;
  const int lane = lane_id();
  const unsigned long long stride = (unsigned long long)gridDim.x * blockDim.x;
  if (!ctrl->pair_overflow) {
    for (int rg = blockIdx.x; rg < nregions; rg += gridDim.x) {
      const int cnt = LA.counts[rg];
      const int2* pairs = LA.pairs + (size_t)rg * LA.region_cap;
      for (int i0 = (threadIdx.x & ~31); i0 < cnt; i0 += blockDim.x) {
        const int i = i0 + lane;
        bool pred = false;
        int loser = 0;
        if (i < cnt) {
          const int2 p = pairs[i];
          const int u = min(p.x, p.y), v = max(p.x, p.y);
          if (ld_color(colors + u) == ld_color(colors + v)) {
            if (R == kIdLow) {
              loser = u;
            } else if (R == kIdHigh || R == kOrdered) {
              loser = v;
            } else {
              const int du = (int)(ld_off(off + u + 1, pol) - ld_off(off + u, pol));
              const int dv = (int)(ld_off(off + v + 1, pol) - ld_off(off + v, pol));
              loser = yields_to<R>(u, du, v, dv) ? u : v;
            }
            pred = atomicExch(marks + loser, 1) == 0;
          }
        }
        append_warp(list, len, pred, loser);
      }
    }
  } else {
    for (long long v0 = (long long)blockIdx.x * blockDim.x + (threadIdx.x & ~31u); v0 < n;
         v0 += (long long)stride) {
      const int v = (int)(v0 + lane);
      const bool pred = v < n && thread_defective<R>(off, cols, colors, v, pol);
      append_warp(list, len, pred, v);
    }
  }
}

// ---------------------------------------------------------------------------
// Fused detect-and-recolor over ctrl->in_list, one warp per vertex
// (deg <= 1023; larger ones are queued for k_heavy).  A defective vertex
// is recoloured in place and appended to ctrl->out_list.  kDetectOnly:
// only write ctrl->flags[i] (detect_conflicts parity mode).
// ---------------------------------------------------------------------------
template <int R, bool kDetectOnly>
__global__ void __launch_bounds__(kBlock) k_list(const long long* __restrict__ off,
                                                 const int* __restrict__ cols, int* colors,
                                                 Ctrl* ctrl, int* heavy, int* marks) {
  __shared__ unsigned s_win[kWarps][32];
  const uint64_t pol = policy_evict_first();
  const int warp = threadIdx.x >> 5, lane = lane_id();
  const int* in = ctrl->in_list;
  const int nin = ctrl->in_len;
  int* out = ctrl->out_list;
  int* flags = ctrl->flags;
  PairLog L{};
  unsigned dummy = 0;
  for (int i = blockIdx.x * kWarps + warp; i < nin; i += gridDim.x * kWarps) {
    const int v = in[i];
    const long long b = ld_off(off + v, pol);
    const int deg = (int)(ld_off(off + v + 1, pol) - b);
    if (deg > kWarpMax) {
      if (lane == 0) heavy[atomicAdd(&ctrl->heavy_len, 1)] = i;
      continue;
    }
    const bool d = warp_defective<R>(off, cols, colors, v, b, deg, pol);
    if (kDetectOnly) {
      if (lane == 0) flags[i] = d ? 1 : 0;
      continue;
    }
    if (d) {
      if (R == kOrdered) {
        const int stamp = ctrl->round + 2;  // insertion into W_{r+1}
        const int c = warp_first_fit<false, true, false>(cols, colors, v, b, deg, s_win[warp],
                                                         pol, L, dummy);
        if (lane == 0) {
          st_color(colors + v, c);
          atomicAdd(&ctrl->recolored, 1);
          if (claim_slot(marks, v, stamp)) out[atomicAdd(&ctrl->out_len, 1)] = v;
        }
        __syncwarp();
        warp_push_higher(cols, colors, v, b, deg, c, marks, stamp, out, &ctrl->out_len, pol);
      } else {
        const int c = warp_first_fit<false, false, false>(cols, colors, v, b, deg, s_win[warp],
                                                          pol, L, dummy);
        if (lane == 0) {
          st_color(colors + v, c);
          atomicAdd(&ctrl->recolored, 1);
          out[atomicAdd(&ctrl->out_len, 1)] = v;
        }
      }
    }
  }
}

template <int R, bool kDetectOnly>
__global__ void __launch_bounds__(kBlock) k_heavy(const long long* __restrict__ off,
                                                  const int* __restrict__ cols, int* colors,
                                                  Ctrl* ctrl, const int* heavy, int* marks) {
  __shared__ unsigned s_bwin[kBWinWords];
  __shared__ int s_red;
  const uint64_t pol = policy_evict_first();
  const int nh = ctrl->heavy_len;
  const int* in = ctrl->in_list;
  PairLog L{};
  unsigned dummy = 0;
  for (int h = blockIdx.x; h < nh; h += gridDim.x) {
    const int i = heavy[h];
    const int v = in[i];
    const long long b = ld_off(off + v, pol);
    const int deg = (int)(ld_off(off + v + 1, pol) - b);
    const bool d = block_defective<R>(off, cols, colors, v, b, deg, pol);
    if (kDetectOnly) {
      if (threadIdx.x == 0) ctrl->flags[i] = d ? 1 : 0;
      continue;
    }
    if (d) {
      if (R == kOrdered) {
        const int stamp = ctrl->round + 2;
        const int c = block_first_fit<false, true, false>(cols, colors, v, b, deg, s_bwin, &s_red,
                                                          pol, L, dummy);
        if (threadIdx.x == 0) {
          st_color(colors + v, c);
          atomicAdd(&ctrl->recolored, 1);
          if (claim_slot(marks, v, stamp)) ctrl->out_list[atomicAdd(&ctrl->out_len, 1)] = v;
        }
        __syncthreads();
        block_push_higher(cols, colors, v, b, deg, c, marks, stamp, ctrl->out_list,
                          &ctrl->out_len, pol);
      } else {
        const int c = block_first_fit<false, false, false>(cols, colors, v, b, deg, s_bwin,
                                                           &s_red, pol, L, dummy);
        if (threadIdx.x == 0) {
          st_color(colors + v, c);
          atomicAdd(&ctrl->recolored, 1);
          ctrl->out_list[atomicAdd(&ctrl->out_len, 1)] = v;
        }
      }
    }
  }
}

// K3: one thread closes the round (finish_round, parallel.hpp:140-154) and
// drives the graph's WHILE node.
__global__ void k_control(Ctrl* ctrl, cudaGraphConditionalHandle handle, int in_graph) {
  const int r = ctrl->round + 1;
  ctrl->round = r;
  const int found = ctrl->out_len;  // next worklist (recoloured + pushed)
  if (r == 1) ctrl->cand_total = ctrl->in_len;
  if (r - 1 < kMaxRoundsRecorded) ctrl->cpr[r - 1] = (unsigned long long)ctrl->recolored;
  ctrl->recolored = 0;
  int* t = ctrl->in_list;
  ctrl->in_list = ctrl->out_list;
  ctrl->out_list = t;
  ctrl->in_len = found;
  ctrl->out_len = 0;
  ctrl->heavy_len = 0;
  unsigned cont = 0;
  if (found > 0) {
    if (r >= ctrl->round_cap) ctrl->capped = 1;
    else cont = 1;
  }
  ctrl->done = cont ? 0 : 1;
  if (in_graph) cudaGraphSetConditional(handle, cont);
}

// ---------------------------------------------------------------------------
// K4: verification (verify_coloring, coloring.hpp:159-177) + colour census.
// ---------------------------------------------------------------------------
struct VerifyAcc {
  unsigned long long violations;
  unsigned long long uncolored;
  unsigned long long conflict_edges;
  unsigned long long out_of_bound;
  unsigned long long negative;
  int max_color;
  int pad;
};

__global__ void __launch_bounds__(kBlock) k_verify_count(const long long* __restrict__ off,
                                                         const int* __restrict__ cols, int n,
                                                         const int* colors, VerifyAcc* acc,
                                                         int* vcount) {
  __shared__ unsigned long long s_acc[4];
  __shared__ int s_max;
  const uint64_t pol = policy_evict_first();
  const int lane = lane_id();
  if (threadIdx.x < 4) s_acc[threadIdx.x] = 0ull;
  if (threadIdx.x == 0) s_max = -1;
  __syncthreads();
  unsigned long long unc = 0, conf = 0, oob = 0, neg = 0;
  int mx = -1;
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long v0 = (long long)blockIdx.x * blockDim.x + (threadIdx.x & ~31u); v0 < n;
       v0 += stride) {
    const int v = (int)(v0 + lane);
    const bool valid = v < n;
    int c = -1;
    long long b = 0;
    int deg = 0;
    int cnt = 0;
    bool big = false;
    if (valid) {
      c = colors[v];
      b = ld_off(off + v, pol);
      deg = (int)(ld_off(off + v + 1, pol) - b);
      if (c == -1) {
        unc++;
        cnt = 1;
      } else {
        if (c < -1 || c > deg) oob++;
        if (c < -1) neg++;
        if (c > mx) mx = c;
        if (deg <= 32) {
          for (int k = 0; k < deg; ++k) {
            const int w = ld_col(cols + b + k, pol);
            if (w > v && colors[w] == c) cnt++;
          }
        } else {
          big = true;
        }
      }
    }
    unsigned bigm = __ballot_sync(kFull, big);
    while (bigm) {
      const int r = __ffs(bigm) - 1;
      bigm &= bigm - 1;
      const int vr = __shfl_sync(kFull, v, r);
      const int cr = __shfl_sync(kFull, c, r);
      const long long br = __shfl_sync(kFull, b, r);
      const int dr = __shfl_sync(kFull, deg, r);
      int hits = 0;
      for (int k = lane; k < dr; k += 32) {
        const int w = ld_col(cols + br + k, pol);
        if (w > vr && colors[w] == cr) hits++;
      }
      hits = __reduce_add_sync(kFull, (unsigned)hits);
      if (lane == r) cnt += hits;
    }
    if (valid) {
      if (c != -1) conf += cnt;
      if (vcount) vcount[v] = cnt;
    }
  }
  atomicAdd(&s_acc[0], unc);
  atomicAdd(&s_acc[1], conf);
  atomicAdd(&s_acc[2], oob);
  atomicAdd(&s_acc[3], neg);
  atomicMax(&s_max, mx);
  __syncthreads();
  if (threadIdx.x == 0) {
    atomicAdd(&acc->uncolored, s_acc[0]);
    atomicAdd(&acc->conflict_edges, s_acc[1]);
    atomicAdd(&acc->out_of_bound, s_acc[2]);
    atomicAdd(&acc->negative, s_acc[3]);
    atomicAdd(&acc->violations, s_acc[0] + s_acc[1]);
    atomicMax(&acc->max_color, s_max);
  }
}

// Colour census (count_colors, coloring.hpp:181-196): one bit per colour in
// [0, max_color]; colours below 4096 are aggregated in shared memory first.
__global__ void __launch_bounds__(kBlock) k_census(const int* colors, int n, unsigned* bitmap,
                                                   int max_color) {
  constexpr int kLocalWords = 128;
  __shared__ unsigned s_bits[kLocalWords];
  for (int i = threadIdx.x; i < kLocalWords; i += blockDim.x) s_bits[i] = 0u;
  __syncthreads();
  for (long long v = (long long)blockIdx.x * blockDim.x + threadIdx.x; v < n;
       v += (long long)gridDim.x * blockDim.x) {
    const int c = colors[v];
    if (c >= 0 && c <= max_color) {
      if (c < kLocalWords * 32) atomicOr(&s_bits[c >> 5], 1u << (c & 31));
      else atomicOr(&bitmap[c >> 5], 1u << (c & 31));
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < kLocalWords && i * 32 <= max_color; i += blockDim.x)
    if (s_bits[i]) atomicOr(&bitmap[i], s_bits[i]);
}

// Writes each violation at its exact position in reference order
// (pos = exclusive prefix sum of per-vertex counts).
__global__ void __launch_bounds__(kBlock) k_verify_write(const long long* __restrict__ off,
                                                         const int* __restrict__ cols, int n,
                                                         const int* colors, const int* vcount,
                                                         const long long* pos, int3* out,
                                                         long long cap) {
  for (long long v0 = (long long)blockIdx.x * blockDim.x + threadIdx.x; v0 < n;
       v0 += (long long)gridDim.x * blockDim.x) {
    const int v = (int)v0;
    if (vcount[v] == 0) continue;
    long long p = pos[v];
    if (p >= cap) continue;
    const int c = colors[v];
    if (c == -1) {
      out[p] = make_int3(v, -1, -1);
      continue;
    }
    for (long long k = off[v]; k < off[v + 1] && p < cap; ++k) {
      const int w = cols[k];
      if (w > v && colors[w] == c) out[p++] = make_int3(v, w, c);
    }
  }
}

// Sequential First-Fit (first_fit_sequential, coloring.hpp:110-116) on one
// CTA: ascending ids, each vertex coloured with every earlier colour visible.
__global__ void __launch_bounds__(kBlock) k_first_fit_seq(const long long* __restrict__ off,
                                                          const int* __restrict__ cols, int n,
                                                          int* colors) {
  __shared__ unsigned s_win[32];
  __shared__ unsigned s_bwin[kBWinWords];
  __shared__ int s_red;
  const uint64_t pol = policy_evict_first();
  const int warp = threadIdx.x >> 5, lane = lane_id();
  PairLog L{};
  unsigned dummy = 0;
  for (int v = 0; v < n; ++v) {
    const long long b = ld_off(off + v, pol);
    const int deg = (int)(ld_off(off + v + 1, pol) - b);
    if (deg <= kWarpMax) {
      if (warp == 0) {
        const int c = warp_first_fit<false, false, false>(cols, colors, v, b, deg, s_win, pol, L,
                                                          dummy);
        if (lane == 0) st_color(colors + v, c);
        __syncwarp();
      }
    } else {
      const int c = block_first_fit<false, false, false>(cols, colors, v, b, deg, s_bwin, &s_red,
                                                         pol, L, dummy);
      if (threadIdx.x == 0) st_color(colors + v, c);
      __syncthreads();
    }
  }
}

__global__ void k_max_degree(const long long* __restrict__ off, int n, int* out) {
  int mx = 0;
  for (long long v = (long long)blockIdx.x * blockDim.x + threadIdx.x; v < n;
       v += (long long)gridDim.x * blockDim.x)
    mx = max(mx, (int)(off[v + 1] - off[v]));
  mx = (int)__reduce_max_sync(kFull, (unsigned)mx);
  if (lane_id() == 0) atomicMax(out, mx);
}

__global__ void k_fill(int* p, long long n, int value) {
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    p[i] = value;
}

}  // namespace dev
}  // namespace gcol
