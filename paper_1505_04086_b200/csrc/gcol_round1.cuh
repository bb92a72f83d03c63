// gcol_round1.cuh -- round 1 in priority order (the "ordered round").
//
// Round 1's worklist W (the losers of logged pairs with equal colours,
// k_candidates) is recoloured as the reference's fused detect-and-recolor
// does (parallel.hpp:297-313: a member that is still defective recolours
// with First-Fit over its whole neighbourhood), but in descending priority
// order, each member first WAITING for its higher-priority neighbours in W
// to finish.  Every member then sees the final colours of everything it must
// avoid: a member conflicts neither with stable vertices (it read them) nor
// with other members (the lower-priority one of any adjacent pair read the
// other's final colour), so round 1 leaves no conflict and the round loop
// that follows (k_list/k_heavy, which re-checks the recoloured set) ends at
// once.  Without the order, adjacent hubs that lose in the same round read
// each other's old colours, pick the same smallest free colour, and collide
// again round after round (R-MAT: 19-22 rounds, each pushing some hubs to a
// new top colour).
//
// Priority: the rule's total order (yields_to, gcol_device.cuh) as a 64-bit
// key; larger = higher priority = processed first.  A member yields to every
// neighbour of larger key.
//
// Progress: members are handed out (one per CTA, ascending ticket) in
// descending key order by a co-resident (cooperative) grid, so the member
// with the smallest unfinished ticket waits only on members with smaller
// tickets -- all handed out, each being processed by a resident CTA or done.
// A list too long to sort in one CTA is processed in list order with the
// waits bounded; anything left defective is caught by the round loop.
#pragma once
#include "gcol_device.cuh"
#include "gcol_k1.cuh"

namespace gcol {
namespace dev {

constexpr int kSortCap = 16384;          // members sorted in one CTA (128 KB of keys)
constexpr int kOrdWaitPolls = 1 << 16;   // bounded waits (only bind on the unsorted path)
constexpr int kMemberPending = 1;        // marks[]: member not finished
constexpr int kMemberDone = 2;

template <int R>
__device__ __forceinline__ unsigned long long prio_key(int v, int deg) {
  if (R == kIdLow) return (unsigned)v;                          // lower id yields
  if (R == kIdHigh || R == kOrdered) return (unsigned)(INT_MAX - v);
  return ((unsigned long long)(unsigned)deg << 32) | (unsigned)v;  // lower (deg, id) yields
}

template <int R>
__device__ __forceinline__ int key_vertex(unsigned long long k) {
  if (R == kIdLow) return (int)k;
  if (R == kIdHigh || R == kOrdered) return INT_MAX - (int)k;
  return (int)(unsigned)k;
}

// One CTA (1024 threads): sort ctrl->in_list by descending priority key
// (bitonic, shared memory).  Lists above kSortCap are left as they are.
template <int R>
__global__ void __launch_bounds__(1024) k_sort_members(const long long* __restrict__ off,
                                                       Ctrl* ctrl) {
  extern __shared__ unsigned long long s_key[];
  const int n = ctrl->in_len;
  int* list = ctrl->in_list;
  if (n > kSortCap || n <= 1) {
    if (threadIdx.x == 0) ctrl->ord_sorted = n <= 1 ? 1 : 0;
    return;
  }
  int P = 1;
  while (P < n) P <<= 1;
  for (int i = threadIdx.x; i < P; i += blockDim.x) {
    unsigned long long k = 0ull;  // padding sorts last
    if (i < n) {
      const int v = list[i];
      const int d = (int)(off[v + 1] - off[v]);
      k = prio_key<R>(v, d) | (1ull << 63);
    }
    s_key[i] = k;
  }
  __syncthreads();
  for (int size = 2; size <= P; size <<= 1) {
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      for (int i = threadIdx.x; i < P; i += blockDim.x) {
        const int j = i ^ stride;
        if (j > i) {
          const bool desc = (i & size) == 0;  // descending overall
          const unsigned long long a = s_key[i], b = s_key[j];
          if (desc ? a < b : a > b) {
            s_key[i] = b;
            s_key[j] = a;
          }
        }
      }
      __syncthreads();
    }
  }
  for (int i = threadIdx.x; i < n; i += blockDim.x) list[i] = key_vertex<R>(s_key[i] & ~(1ull << 63));
  if (threadIdx.x == 0) ctrl->ord_sorted = 1;
}

// The ordered round: one member per CTA at a time (ascending tickets).
template <int R>
__global__ void __launch_bounds__(kBlock) k_ordered_round(const long long* __restrict__ off,
                                                          const int* __restrict__ cols,
                                                          int* colors, Ctrl* ctrl, int* marks) {
  constexpr int U = 4;
  __shared__ unsigned s_bm[kBWinWords];
  __shared__ int s_i, s_red;
  const uint64_t pol = policy_evict_first();
  const int tid = threadIdx.x;
  const int n = ctrl->in_len;
  const int* list = ctrl->in_list;
  const int polls_max = ctrl->ord_sorted ? INT_MAX : kOrdWaitPolls;
  init_peers(ctrl);  // (the loop's first barrier orders it)
  for (;;) {
    if (tid == 0) s_i = (int)atomicAdd(&ctrl->ord_ticket, 1ull);
    for (int k = tid; k < kBWinWords; k += kBlock) s_bm[k] = 0u;
    __syncthreads();
    const int i = s_i;
    if (i >= n) break;
    const int v = list[i];
    const long long b = ld_off(off + v, pol);
    const int deg = (int)(ld_off(off + v + 1, pol) - b);
    const unsigned long long kv = prio_key<R>(v, deg);
    const int cv = ld_color(colors + v);
    bool defect = false;
    unsigned long long reg = 0ull;
    for (int base = 0; base < deg; base += kBlock * U) {
      int w[U], c[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int k = base + u * kBlock + tid;
        w[u] = k < deg ? ld_col(cols + b + k, pol) : -1;
      }
      int mk[U];
#pragma unroll
      for (int u = 0; u < U; ++u) mk[u] = w[u] >= 0 ? ld_color(marks + w[u]) : 0;
#pragma unroll
      for (int u = 0; u < U; ++u) {
        if (mk[u] == kMemberPending) {  // a member: wait for it if it outranks v
          const int dw = (int)(ld_off(off + w[u] + 1, pol) - ld_off(off + w[u], pol));
          if (prio_key<R>(w[u], dw) > kv)
            for (int p = 0; p < polls_max && ld_acquire_u32(reinterpret_cast<const unsigned*>(marks + w[u])) ==
                                                 (unsigned)kMemberPending; ++p)
              __nanosleep(64);
        }
      }
#pragma unroll
      for (int u = 0; u < U; ++u) c[u] = w[u] >= 0 ? ld_color(colors + w[u]) : -1;
#pragma unroll
      for (int u = 0; u < U; ++u) {
        if (w[u] < 0) continue;
        if (c[u] == cv && cv >= 0) {
          // a conflict v must resolve: the neighbour outranks v
          if (R == kDegId) {
            const int dw = (int)(ld_off(off + w[u] + 1, pol) - ld_off(off + w[u], pol));
            defect |= yields_to<R>(v, deg, w[u], dw);
          } else {
            defect |= yields_to<R>(v, deg, w[u], 0);
          }
        }
        if (c[u] >= 0 && c[u] <= deg && c[u] < kBWinWords * 32) {
          if (c[u] < 64) reg |= 1ull << c[u];
          else atomicOr(&s_bm[c[u] >> 5], 1u << (c[u] & 31));
        }
      }
    }
    const unsigned lo = __reduce_or_sync(kFull, (unsigned)reg);
    const unsigned hi = __reduce_or_sync(kFull, (unsigned)(reg >> 32));
    if (lane_id() == 0) {
      if (lo) atomicOr(&s_bm[0], lo);
      if (hi) atomicOr(&s_bm[1], hi);
    }
    if (tid == 0) s_red = INT_MAX;
    defect = __syncthreads_or(defect);
    if (defect) {
      const int lim = min(deg, kBWinWords * 32 - 1);
      for (int k = tid; k * 32 <= lim; k += kBlock) {
        unsigned fr = ~s_bm[k];
        const int top = lim - k * 32;
        if (top < 31) fr &= (2u << top) - 1u;
        if (fr) atomicMin(&s_red, k * 32 + __ffs(fr) - 1);
      }
      __syncthreads();
      int c = s_red;
      __syncthreads();
      if (c == INT_MAX) {  // every colour below 16384 taken: the next windows
        PairLog L{};
        unsigned dummy = 0;
        c = block_first_fit<false, false, false>(cols, colors, v, b, deg, s_bm, &s_red, pol, L,
                                                  dummy);
      }
      if (tid == 0) {
        commit_color(colors, v, c);
        atomicAdd(&ctrl->recolored, 1);
        ctrl->out_list[atomicAdd(&ctrl->out_len, 1)] = v;
      }
    }
    __syncthreads();
    if (tid == 0) {
      __threadfence();  // the colour before the done mark
      asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(marks + v), "r"((unsigned)kMemberDone)
                   : "memory");
    }
  }
  peers_fence();
}

}  // namespace dev
}  // namespace gcol
