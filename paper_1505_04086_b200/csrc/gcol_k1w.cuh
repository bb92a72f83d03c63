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
};

// Adjacency loads: read-only, L1-allocating (a warp's rows are contiguous,
// so successive entries of neighbouring lanes share sectors), L2 evict_first.
__device__ __forceinline__ int ld_col_l1(const int* p, uint64_t pol) {
  int r;
  asm volatile("ld.global.nc.L2::cache_hint.b32 %0, [%1], %2;" : "=r"(r) : "l"(p), "l"(pol));
  return r;
}

// One pass over the lower-id prefix of the row (sorted: stops at the first
// entry above v), warp-collective.  mask |= colours seen (<= deg); the first
// four still-uncoloured neighbours land in u[], their count in ns (may be
// > 4).  kLogAll: log every uncoloured one instead (the final pass).
template <bool kLogAll>
__device__ __forceinline__ void k1w_scan(const int* __restrict__ cols, const int* colors, int v,
                                         long long b, int deg, bool need, uint64_t pol,
                                         unsigned long long& mask, int (&u)[4], int& ns,
                                         unsigned& gathers, const PairLogInl& L) {
  bool active = need && deg > 0;
  for (int k = 0; __any_sync(kFull, active); k += 4) {
    int w[4];
    bool take[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const bool in = active && k + j < deg;
      w[j] = in ? ld_col_l1(cols + b + k + j, pol) : 0;
      take[j] = in && w[j] < v;
    }
    int c[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) c[j] = take[j] ? ld_color(colors + w[j]) : -2;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      if (!kLogAll) gathers += take[j];
      if (c[j] >= 0 && c[j] <= deg) mask |= 1ull << c[j];
      const bool st = take[j] && c[j] == -1;
      if (kLogAll) {
        log_pairs(L, st, w[j], v);
      } else if (st) {
        if (ns == 0) u[0] = w[j];
        else if (ns == 1) u[1] = w[j];
        else if (ns == 2) u[2] = w[j];
        else if (ns == 3) u[3] = w[j];
        ++ns;
      }
    }
    // sorted row: once an entry above v (or the row end) is reached, done
    if (active && (k + 4 >= deg || !take[3])) active = false;
  }
}

template <bool kStream>
__global__ void __launch_bounds__(kWaitBlock) k1_wait(const long long* __restrict__ off,
                                                      const int* __restrict__ cols, int n,
                                                      int* colors, Ctrl* ctrl, PairLogArgs LA,
                                                      WaitArgs A) {
  __shared__ int s_npairs;
  __shared__ unsigned s_gathers;
  if (threadIdx.x == 0) {
    s_npairs = 0;
    s_gathers = 0;
  }
  __syncthreads();
  const int lane = lane_id();
  const int wpb = blockDim.x >> 5;
  const int gw = blockIdx.x * wpb + (threadIdx.x >> 5);
  const int NW = gridDim.x * wpb;
  const uint64_t pol = policy_evict_first();
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
    const int deg = valid ? (int)(e - b) : 0;
    if (kStream) {  // streamed upload: the tile's adjacency must be resident
      const long long lo = __shfl_sync(kFull, b, 0), hi = __shfl_sync(kFull, e, 31);
      if (lane == 0 && hi > lo)
        for (long long p = lo >> A.piece_shift; p <= (hi - 1) >> A.piece_shift; ++p)
          while (ld_acquire_u32(A.piece_ready + p) == 0u) __nanosleep(256);
      __syncwarp();
    }
    unsigned long long mask = 0ull;
    int u[4] = {0, 0, 0, 0};
    int ns = 0;
    k1w_scan<false>(cols, colors, v, b, deg, valid, pol, mask, u, ns, gathers, L);
    // pending: bit j = u[j] still uncoloured; `more`: > 4 were, rescan later
    unsigned pm = ns >= 4 ? 15u : ((1u << ns) - 1u);
    bool more = ns > 4;
    bool done = valid && ns == 0;
    if (done) commit_color(colors, v, __ffsll((long long)~mask) - 1);
    bool pend = valid && !done;
    for (int polls = 0; __any_sync(kFull, pend); ++polls) {
      if (polls >= A.max_polls) {
        // give up: log every still-uncoloured lower neighbour for round 1
        unsigned long long m2 = 0ull;
        int ns2 = 0;
        k1w_scan<true>(cols, colors, v, b, deg, pend, pol, m2, u, ns2, gathers, L);
        if (pend) commit_color(colors, v, __ffsll((long long)~m2) - 1);
        break;
      }
      __nanosleep(128);
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        if (pend && ((pm >> j) & 1u)) {
          const int c = ld_color(colors + u[j]);
          if (c != -1) {
            pm &= ~(1u << j);
            if (c >= 0 && c <= deg) mask |= 1ull << c;
          }
        }
      }
      // the four tracked ones resolved but more were pending: scan again
      const bool again = pend && pm == 0u && more;
      if (__any_sync(kFull, again)) {
        int ns2 = 0;
        unsigned g2 = 0;
        if (again) mask = 0ull;
        k1w_scan<false>(cols, colors, v, b, deg, again, pol, mask, u, ns2, g2, L);
        if (again) {
          pm = ns2 >= 4 ? 15u : ((1u << ns2) - 1u);
          more = ns2 > 4;
        }
      }
      if (pend && pm == 0u) {
        commit_color(colors, v, __ffsll((long long)~mask) - 1);
        pend = false;
      }
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
  }
}

}  // namespace dev
}  // namespace gcol
