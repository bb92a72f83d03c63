// gcol_kernels.cuh -- the sm_100a kernels of the RSOC path.
//
//   K1 k1_light/k1_mega  initial tentative pass (parallel.hpp:286-296), gcol_k1.cuh
//   K2 k_candidates   round-1 worklist from K1's in-flight observations
//      k_list/k_heavy fused detect-and-recolor over a worklist
//                     (parallel.hpp:297-313 + defective_relaxed :105-111)
//   K3 k_control      round bookkeeping + CUDA-graph WHILE condition
//                     (barrier completion + finish_round, parallel.hpp:140-154)
//   K4 k_verify_*     verify_coloring / count_colors (coloring.hpp:159-196)
#pragma once
#include "gcol_device.cuh"
#include "gcol_k1.cuh"

namespace gcol {
namespace dev {

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
                                                       PairLogArgs LA, int nregions, int* marks,
                                                       PairLogArgs LB = PairLogArgs{},
                                                       int nregionsB = 0) {
  const uint64_t pol = policy_evict_first();
  int* list = ctrl->in_list;
  int* len = &ctrl->in_len;
  const int lane = lane_id();
  const unsigned long long stride = (unsigned long long)gridDim.x * blockDim.x;
  if (!ctrl->pair_overflow) {
    // two slice sets (the class-split pass: heavy CTAs' slices, light CTAs')
    for (int rg = blockIdx.x; rg < nregions + nregionsB; rg += gridDim.x) {
      const bool a = rg < nregions;
      const int r = a ? rg : rg - nregions;
      const int cnt = a ? LA.counts[r] : LB.counts[r];
      const int2* pairs = a ? LA.pairs + (size_t)r * LA.region_cap : LB.pairs + (size_t)r * LB.region_cap;
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
  } else {  // the log overflowed: test every vertex (rows above 32 entries warp-wide)
    for (long long v0 = (long long)blockIdx.x * blockDim.x + (threadIdx.x & ~31u); v0 < n;
         v0 += (long long)stride) {
      const int v = (int)(v0 + lane);
      long long b = 0;
      int deg = 0;
      if (v < n) {
        b = ld_off(off + v, pol);
        deg = (int)(ld_off(off + v + 1, pol) - b);
      }
      bool pred = v < n && deg <= 32 && thread_defective<R>(off, cols, colors, v, pol);
      unsigned big = __ballot_sync(kFull, v < n && deg > 32);
      while (big) {
        const int r = __ffs(big) - 1;
        big &= big - 1;
        const int vr = __shfl_sync(kFull, v, r);
        const long long br = __shfl_sync(kFull, b, r);
        const int dr = __shfl_sync(kFull, deg, r);
        const bool d = warp_defective<R>(off, cols, colors, vr, br, dr, pol);
        if (lane == r) pred = d;
      }
      if (pred) marks[v] = 1;  // a member of round 1 (the ordered round waits on members)
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
  init_peers(ctrl);
  __syncthreads();
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
      int slot = -1;
      if (!kDetectOnly && R != kOrdered && ctrl->hslots > 0) {
        if (lane == 0) {
          slot = atomicAdd(&ctrl->heavy_slots, 1);
          if (slot >= ctrl->hslots) slot = -1;  // out of slots: one block per row below
        }
        slot = __shfl_sync(kFull, slot, 0);
      }
      if (slot >= 0) {  // split over the grid: kHPiece-entry pieces for k_heavy
        const int np = (deg + kHPiece - 1) / kHPiece;
        int p0 = 0;
        if (lane == 0) {
          p0 = atomicAdd(&ctrl->heavy_pieces, np);
          ctrl->hslot_v[slot] = v;
          ctrl->hslot_i[slot] = i;
          ctrl->hslot_left[slot] = np;
        }
        p0 = __shfl_sync(kFull, p0, 0);
        for (int j = lane; j < np; j += 32) ctrl->hq[p0 + j] = make_int2(slot, j * kHPiece);
      } else if (lane == 0) {
        heavy[atomicAdd(&ctrl->heavy_len, 1)] = i;
      }
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
          commit_color(colors, v, c);
          atomicAdd(&ctrl->recolored, 1);
          if (claim_slot(marks, v, stamp)) out[atomicAdd(&ctrl->out_len, 1)] = v;
        }
        __syncwarp();
        warp_push_higher(cols, colors, v, b, deg, c, marks, stamp, out, &ctrl->out_len, pol);
      } else {
        const int c = warp_first_fit<false, false, false>(cols, colors, v, b, deg, s_win[warp],
                                                          pol, L, dummy);
        if (lane == 0) {
          commit_color(colors, v, c);
          atomicAdd(&ctrl->recolored, 1);
          out[atomicAdd(&ctrl->out_len, 1)] = v;
        }
      }
    }
  }
  peers_fence();
}

// One piece of a split heavy row (block-wide): detect its conflicts and
// OR the colours it sees into the row's slot bitmap; the block finishing the
// row's last piece recolours it when defective (First-Fit over the bitmap).
template <int R>
__device__ __forceinline__ void heavy_piece(const long long* __restrict__ off,
                                            const int* __restrict__ cols, int* colors, Ctrl* ctrl,
                                            int slot, int start, unsigned* s_bwin, int* s_red,
                                            uint64_t pol) {
  constexpr int U = 4;
  const int tid = threadIdx.x;
  const int v = ctrl->hslot_v[slot];
  const long long b = ld_off(off + v, pol);
  const int deg = (int)(ld_off(off + v + 1, pol) - b);
  const int cv = ld_color(colors + v);
  const int end = min(deg, start + kHPiece);
  for (int k = tid; k < kBWinWords; k += kBlock) s_bwin[k] = 0u;
  __syncthreads();
  bool hit = false;
  unsigned long long reg = 0ull;
  for (int base = start; base < end; base += kBlock * U) {
    int w[U], c[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int i = base + u * kBlock + tid;
      w[u] = i < end ? ld_col(cols + b + i, pol) : -1;
    }
#pragma unroll
    for (int u = 0; u < U; ++u) c[u] = w[u] >= 0 ? ld_color(colors + w[u]) : -2;
#pragma unroll
    for (int u = 0; u < U; ++u) {
      if (c[u] >= 0 && c[u] <= deg && c[u] < kBWinWords * 32) {
        if (c[u] < 64) reg |= 1ull << c[u];
        else atomicOr(&s_bwin[c[u] >> 5], 1u << (c[u] & 31));
      }
      if (cv >= 0 && c[u] == cv && considers<R>(v, w[u])) {
        if (R == kDegId) {
          const int dw = (int)(ld_off(off + w[u] + 1, pol) - ld_off(off + w[u], pol));
          hit |= yields_to<R>(v, deg, w[u], dw);
        } else {
          hit = true;
        }
      }
    }
  }
  const unsigned lo = __reduce_or_sync(kFull, (unsigned)reg);
  const unsigned hi = __reduce_or_sync(kFull, (unsigned)(reg >> 32));
  if (lane_id() == 0) {
    if (lo) atomicOr(&s_bwin[0], lo);
    if (hi) atomicOr(&s_bwin[1], hi);
  }
  const int any = __syncthreads_or(hit);
  unsigned* gbm = ctrl->hslot_bm + (size_t)slot * kBWinWords;
  for (int k = tid; k < kBWinWords; k += kBlock)
    if (s_bwin[k]) atomicOr(gbm + k, s_bwin[k]);
  if (tid == 0 && any) atomicOr(ctrl->hslot_flag + slot, 1);
  __syncthreads();
  if (tid == 0) *s_red = atom_add_acq_rel(ctrl->hslot_left + slot, -1) == 1 ? 1 : 0;
  __syncthreads();
  if (!*s_red) return;
  // last piece of the row
  const bool defective = ld_acquire_u32(reinterpret_cast<const unsigned*>(ctrl->hslot_flag + slot)) != 0u;
  __syncthreads();
  if (tid == 0) *s_red = INT_MAX;
  __syncthreads();
  if (defective) {
    const int lim = min(deg, kBWinWords * 32 - 1);  // candidates 0..lim
    for (int k = tid; k * 32 <= lim; k += kBlock) {
      unsigned fr = ~ld_acquire_u32(gbm + k);
      const int top = lim - k * 32;  // valid bits 0..top of this word
      if (top < 31) fr &= (2u << top) - 1u;
      if (fr) atomicMin(s_red, k * 32 + __ffs(fr) - 1);
    }
  }
  __syncthreads();
  int c = *s_red;
  __syncthreads();
  if (defective && c == INT_MAX) {  // 16384 colours all seen: the next windows, the slow way
    PairLog L{};
    unsigned dummy = 0;
    c = block_first_fit<false, false, false>(cols, colors, v, b, deg, s_bwin, s_red, pol, L,
                                              dummy);
  }
  if (tid == 0) {
    if (defective) {
      commit_color(colors, v, c);
      atomicAdd(&ctrl->recolored, 1);
      ctrl->out_list[atomicAdd(&ctrl->out_len, 1)] = v;
    }
    ctrl->hslot_flag[slot] = 0;
  }
  for (int k = tid; k < kBWinWords; k += kBlock) gbm[k] = 0u;  // clean for the next round
}

template <int R, bool kDetectOnly>
__global__ void __launch_bounds__(kBlock) k_heavy(const long long* __restrict__ off,
                                                  const int* __restrict__ cols, int* colors,
                                                  Ctrl* ctrl, const int* heavy, int* marks) {
  __shared__ unsigned s_bwin[kBWinWords];
  __shared__ int s_red;
  init_peers(ctrl);
  __syncthreads();
  const uint64_t pol = policy_evict_first();
  if (!kDetectOnly && R != kOrdered) {
    const int npc = ctrl->heavy_pieces;
    for (int p = blockIdx.x; p < npc; p += gridDim.x) {
      const int2 e = ctrl->hq[p];
      heavy_piece<R>(off, cols, colors, ctrl, e.x, e.y, s_bwin, &s_red, pol);
      __syncthreads();
    }
  }
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
          commit_color(colors, v, c);
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
          commit_color(colors, v, c);
          atomicAdd(&ctrl->recolored, 1);
          ctrl->out_list[atomicAdd(&ctrl->out_len, 1)] = v;
        }
      }
    }
  }
  peers_fence();
}

// K3: one thread closes the round (finish_round, parallel.hpp:140-154) and
// drives the graph's WHILE node.
__global__ void k_control(Ctrl* ctrl, cudaGraphConditionalHandle handle, int in_graph) {
  const int r = ctrl->round + 1;
  ctrl->round = r;
#ifdef GCOL_DEBUG_HEAVY  // experiments: GCOL_NVCC_EXTRA=-DGCOL_DEBUG_HEAVY
  printf("round %d in_len %d heavy_slots %d heavy_len %d pieces %d recolored %d\n", r, ctrl->in_len,
         ctrl->heavy_slots, ctrl->heavy_len, ctrl->heavy_pieces, ctrl->recolored);
#endif
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
  ctrl->heavy_slots = 0;
  ctrl->heavy_pieces = 0;
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
                                                         int* vcount, int big_min,
                                                         unsigned* census, int census_max) {
  // rows with deg >= big_min (a piece plan exists) are left to k_verify_big;
  // colours 0..census_max are also marked in `census` (count_colors)
  constexpr int U = 4;
  constexpr int kLocalWords = 128;
  __shared__ unsigned long long s_acc[4];
  __shared__ int s_max;
  __shared__ unsigned s_bits[kLocalWords];
  const int lane = lane_id();
  if (threadIdx.x < 4) s_acc[threadIdx.x] = 0ull;
  if (threadIdx.x == 0) s_max = -1;
  for (int i = threadIdx.x; i < kLocalWords; i += blockDim.x) s_bits[i] = 0u;
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
      b = __ldg(off + v);
      deg = (int)(__ldg(off + v + 1) - b);
      if (c == -1) {
        unc++;
        cnt = 1;
      } else {
        if (c < -1 || c > deg) oob++;
        if (c < -1) neg++;
        if (c > mx) mx = c;
        if (census && c >= 0 && c <= census_max) {
          if (c < kLocalWords * 32) atomicOr(&s_bits[c >> 5], 1u << (c & 31));
          else atomicOr(&census[c >> 5], 1u << (c & 31));
        }
        big = deg > 32;
      }
    }
    // thread per row: independent loads, U entries at a time
    const int lim = valid && c != -1 && !big ? deg : 0;
    const int maxk = (int)__reduce_max_sync(kFull, (unsigned)lim);
    for (int k = 0; k < maxk; k += U) {
      int w[U], cw[U];
#pragma unroll
      for (int u = 0; u < U; ++u) w[u] = k + u < lim ? __ldg(cols + b + k + u) : -1;
#pragma unroll
      for (int u = 0; u < U; ++u) cw[u] = w[u] > v ? colors[w[u]] : -3;
#pragma unroll
      for (int u = 0; u < U; ++u) cnt += cw[u] == c;
    }
    // warp per row
    unsigned bigm = __ballot_sync(kFull, big && deg < big_min);
    while (bigm) {
      const int r = __ffs(bigm) - 1;
      bigm &= bigm - 1;
      const int vr = __shfl_sync(kFull, v, r);
      const int cr = __shfl_sync(kFull, c, r);
      const long long br = __shfl_sync(kFull, b, r);
      const int dr = __shfl_sync(kFull, deg, r);
      int hits = 0;
      for (int k0 = 0; k0 < dr; k0 += 32 * U) {
        int w[U], cw[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int k = k0 + u * 32 + lane;
          w[u] = k < dr ? __ldg(cols + br + k) : -1;
        }
#pragma unroll
        for (int u = 0; u < U; ++u) cw[u] = w[u] > vr ? colors[w[u]] : -3;
#pragma unroll
        for (int u = 0; u < U; ++u) hits += cw[u] == cr;
      }
      hits = (int)__reduce_add_sync(kFull, (unsigned)hits);
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
  if (census)
    for (int i = threadIdx.x; i < kLocalWords && i * 32 <= census_max; i += blockDim.x)
      if (s_bits[i]) atomicOr(&census[i], s_bits[i]);
  if (threadIdx.x == 0) {
    atomicAdd(&acc->uncolored, s_acc[0]);
    atomicAdd(&acc->conflict_edges, s_acc[1]);
    atomicAdd(&acc->out_of_bound, s_acc[2]);
    atomicAdd(&acc->negative, s_acc[3]);
    atomicAdd(&acc->violations, s_acc[0] + s_acc[1]);
    atomicMax(&acc->max_color, s_max);
  }
}

// The rows k_verify_count left out (deg >= big_min), as kHPiece-entry pieces
// spread over the grid: piece p belongs to rows[j] with pre[j] <= p < pre[j+1].
__global__ void __launch_bounds__(kBlock) k_verify_big(const long long* __restrict__ off,
                                                       const int* __restrict__ cols,
                                                       const int* colors, const int* rows,
                                                       const int* pre, int nrows, VerifyAcc* acc,
                                                       int* vcount) {
  constexpr int U = 4;
  __shared__ int s_hits;
  const int npieces = pre[nrows];
  for (int p = blockIdx.x; p < npieces; p += gridDim.x) {
    int lo = 0, hi = nrows - 1;  // last j with pre[j] <= p
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (__ldg(pre + mid) <= p) lo = mid;
      else hi = mid - 1;
    }
    const int v = rows[lo];
    const int c = colors[v];
    if (c == -1) continue;  // counted once by k_verify_count
    const long long b = __ldg(off + v);
    const int deg = (int)(__ldg(off + v + 1) - b);
    const int start = (p - pre[lo]) * kHPiece;
    const int end = min(deg, start + kHPiece);
    if (threadIdx.x == 0) s_hits = 0;
    __syncthreads();
    int hits = 0;
    for (int k0 = start; k0 < end; k0 += kBlock * U) {
      int w[U], cw[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int k = k0 + u * kBlock + threadIdx.x;
        w[u] = k < end ? __ldg(cols + b + k) : -1;
      }
#pragma unroll
      for (int u = 0; u < U; ++u) cw[u] = w[u] > v ? colors[w[u]] : -3;
#pragma unroll
      for (int u = 0; u < U; ++u) hits += cw[u] == c;
    }
    hits = (int)__reduce_add_sync(kFull, (unsigned)hits);
    if (lane_id() == 0 && hits) atomicAdd(&s_hits, hits);
    __syncthreads();
    if (threadIdx.x == 0 && s_hits) {
      atomicAdd(&acc->conflict_edges, (unsigned long long)s_hits);
      atomicAdd(&acc->violations, (unsigned long long)s_hits);
      if (vcount) atomicAdd(vcount + v, s_hits);
    }
    __syncthreads();
  }
}

// Rows with deg >= min_deg, appended in any order, and their piece counts.
__global__ void k_collect_big(const long long* __restrict__ off, int n, int min_deg, int* rows,
                              int* pieces, int* len) {
  for (long long v = (long long)blockIdx.x * blockDim.x + threadIdx.x; v < n;
       v += (long long)gridDim.x * blockDim.x) {
    const long long d = off[v + 1] - off[v];
    if (d >= min_deg) {
      const int j = atomicAdd(len, 1);
      rows[j] = (int)v;
      pieces[j] = (int)((d + kHPiece - 1) / kHPiece);
    }
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

// Degree statistics every run plan needs, in one pass over the offsets
// (on the host while validating a host CSR, or by k_graph_stats):
//   [0] rows K1 splits into kPiece pieces (deg >= kSplitDefault)
//   [1] rows the rounds split into kHPiece pieces (deg > kWarpMax)
//   [2] rows verified in kHPiece pieces (deg >= kHPiece)
struct GraphStats {
  unsigned long long rows[3];
  unsigned long long pieces[3];
  int max_degree;
  int pad;
};

__host__ __device__ inline void gs_add(GraphStats& s, long long d) {
  if (d > s.max_degree) s.max_degree = (int)d;
  if (d >= kSplitDefault) {
    s.rows[0]++;
    s.pieces[0] += (unsigned long long)((d + kPiece - 1) / kPiece);
  }
  if (d > kWarpMax) {
    s.rows[1]++;
    s.pieces[1] += (unsigned long long)((d + kHPiece - 1) / kHPiece);
  }
  if (d >= kHPiece) {
    s.rows[2]++;
    s.pieces[2] += (unsigned long long)((d + kHPiece - 1) / kHPiece);
  }
}

__global__ void k_graph_stats(const long long* __restrict__ off, int n, GraphStats* out) {
  GraphStats s{};
  for (long long v = (long long)blockIdx.x * blockDim.x + threadIdx.x; v < n;
       v += (long long)gridDim.x * blockDim.x)
    gs_add(s, off[v + 1] - off[v]);
  const int mx = (int)__reduce_max_sync(kFull, (unsigned)s.max_degree);
  if (lane_id() == 0) atomicMax(&out->max_degree, mx);
  for (int k = 0; k < 3; ++k) {
    if (__any_sync(kFull, s.rows[k] != 0)) {
      // few rows qualify: plain atomics from the lanes that saw some
      if (s.rows[k]) {
        atomicAdd(&out->rows[k], s.rows[k]);
        atomicAdd(&out->pieces[k], s.pieces[k]);
      }
    }
  }
}

__global__ void k_fill(int* p, long long n, int value) {
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    p[i] = value;
}

}  // namespace dev
}  // namespace gcol

namespace gcol {
namespace dev {

// Multi-GPU round 1: defective owned vertices in [lo, hi) under rule R.
template <int R>
__global__ void __launch_bounds__(kBlock) k_detect_range(const long long* __restrict__ off,
                                                         const int* __restrict__ cols, int lo,
                                                         int hi, const int* colors, int* out,
                                                         int* count) {
  const uint64_t pol = policy_evict_first();
  for (long long v0 = lo + (long long)blockIdx.x * blockDim.x + (threadIdx.x & ~31u); v0 < hi;
       v0 += (long long)gridDim.x * blockDim.x) {
    const int v = (int)(v0 + lane_id());
    const bool pred = v < hi && thread_defective<R>(off, cols, colors, v, pol);
    append_warp(out, count, pred, v);
  }
}

// Çatalyürek's detection phase output: the flagged worklist entries,
// appended to ctrl->out_list (warp-aggregated).
__global__ void __launch_bounds__(kBlock) k_compact_flags(Ctrl* ctrl, const int* in, int nin,
                                                          const int* flags) {
  for (long long i0 = (long long)blockIdx.x * blockDim.x + (threadIdx.x & ~31u); i0 < nin;
       i0 += (long long)gridDim.x * blockDim.x) {
    const long long i = i0 + lane_id();
    const bool pred = i < nin && flags[i] != 0;
    append_warp(ctrl->out_list, &ctrl->out_len, pred, pred ? in[i] : 0);
  }
}

// Colours narrowed to `width` bytes for the copy to the host (all colours
// are <= the maximum degree < 2^(8 width)).
__global__ void k_pack_colors(const int* colors, long long n, int width, int* out) {
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    const int c = colors[i];
    if (width == 1) reinterpret_cast<unsigned char*>(out)[i] = (unsigned char)c;
    else reinterpret_cast<unsigned short*>(out)[i] = (unsigned short)c;
  }
}

__global__ void k_iota(int* p, int n) {
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    p[i] = (int)i;
}

// Apply (id, colour) deltas received from other ranks.
__global__ void k_scatter_colors(int* colors, const int* ids, const int* vals, long long count) {
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < count;
       i += (long long)gridDim.x * blockDim.x)
    colors[ids[i]] = vals[i];
}

}  // namespace dev
}  // namespace gcol
