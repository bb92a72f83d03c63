// gcol_k1hw.cuh -- K1HW: the WAITING heavy pass of the class split
// (k1_wide 6, or chosen by graph size; gcol_k1c.cuh holds k1_heavy and everything shared).
//
// Same place in the pass as k1_heavy: heavy rows (degree >= T) in ascending id
// order, each First-Fit over its LOWER heavy neighbours, before the light pass
// K1L.  What changes is what a row does with a lower neighbour it reads as
// pending (-2): k1_heavy colours past it (re-reads it once, then logs it for
// round 1), so the rows in flight together must stay few or the hubs collide
// and the colour count leaves the reference's band -- that cap
// (~1.2k rows on the GPU) is what made K1H latency-bound at 25 % of the warp
// slots.  Here a row WAITS for it, as K1W does for bounded degree
// (gcol_k1w.cuh): every heavy row ends with the smallest colour not carried by
// the FINAL colours of its lower heavy neighbours, i.e. the heavy subgraph is
// coloured exactly as sequential First-Fit in id order would
// (coloring.hpp:110-116 restricted to the heavy rows), nothing is logged, no
// heavy row is ever defective, and the number of rows in flight no longer
// touches the colour count -- the SM can be filled.
//
// Waiting without a list: rows are sorted and commits run roughly in id
// order, so the pending neighbours of a row sit in a suffix of its lower
// prefix.  The first scan records the POSITION of the first pending entry;
// everything before it is final and marked.  The wait re-gathers a window of
// the row from that position, marks what became final, moves the position to
// the first entry still pending, and sleeps only when it did not move.
//
// Split rows (degree >= 1024): the owner warp publishes the pieces (as
// k1_heavy) and keeps the row.  Piece warps never wait (they are a shared
// service: a waiting piece could sit in front of the pieces of the row it
// waits for); a piece that reads a pending neighbour records its position
// (atomicMax of INT_MAX - position into the slot's word).  Once the slot's
// piece count is back to zero the owner runs the same wait from that
// position over its own row, merges the slot's bitmap, and commits.
//
// Progress: rows are claimed in ascending order and a row waits only for
// lower heavy rows, so the lowest uncommitted row never waits; its warp is
// resident (cooperative launch).  H.polls bounds the polls that make no
// progress: past it the row logs what is still pending and colours past it,
// exactly as k1_heavy does -- round 1 then repairs it.
#pragma once
#include "gcol_k1c.cuh"

namespace gcol {
namespace dev {

#ifndef GCOL_K1HW_WARPS
#define GCOL_K1HW_WARPS 24
#endif
constexpr int kHwWarps = GCOL_K1HW_WARPS;    // warps per CTA: row warps + piece warps
constexpr int kHwThreads = kHwWarps * 32;
constexpr int kHwBatch = 8;                  // heavy rows per cursor claim (per CTA)
constexpr int kHwBufs = 8;                   // claimed-batch records kept
constexpr int kHwWin = 4;                    // entries per lane per wait window
constexpr size_t kHwSmem = sizeof(int) * kHvPieceWarps * kHvPieceBuf;  // dynamic: piece buffers

// Where a neighbour's colour is read.  Plain variant: the colour array, index
// w.  Compact variant (kC): the heavy colours by rank -- one 8-byte load of
// the rank word, then rank = base + popc(bits below w); -1 for a light row
// (its colour is not read at all: it has not started and reads this row
// itself later).
__device__ __forceinline__ uint2 ld_nc_u32x2(const void* p) {
  uint2 r;
  asm volatile("ld.global.nc.v2.u32 {%0, %1}, [%2];" : "=r"(r.x), "=r"(r.y) : "l"(p));
  return r;
}

template <bool kC>
__device__ __forceinline__ int hw_slot(const HeavyArgs& H, int w) {
  if (!kC) return w;
  const uint2 e = ld_nc_u32x2(H.rank + (w >> 5));
  const unsigned bit = 1u << (w & 31);
  return (e.x & bit) ? (int)e.y + __popc(e.x & (bit - 1u)) : -1;
}

// Commit heavy row v (heavy index hr) with colour c (one lane).
template <bool kC>
__device__ __forceinline__ void hw_commit(const HeavyArgs& H, int* colors, int v, long long hr, int c) {
  if (kC) st_color(H.hcol + hr, c);  // what the waiting rows poll
  commit_color(colors, v, c);        // what the light pass, the rounds and the caller read
}

// A warp holds at most one ticket at a time, so at most kHwWarps tickets are
// between "drawn" and "record read": a record is overwritten kHwBufs batches later.
static_assert(kHwBufs * kHwBatch >= kHwWarps + 2 * kHwBatch, "batch records must outlive their readers");

// Wait (warp-collective) until no entry of row (b, deg) at a position >= pos
// and an id below v reads as pending; colours that became final are marked.
// Past `polls` polls without progress the remaining pending entries are
// logged (returns false).  pos == INT_MAX: nothing to wait for.
template <class PL, bool kC>
__device__ __forceinline__ bool hw_wait(const int* __restrict__ cols, const int* colors, const HeavyArgs& H,
                                        int v, long long b, int deg, int pos, int lim,
                                        unsigned long long& reg, unsigned* win, uint64_t pol, int polls,
                                        const PL& L, long long& n_polls) {
  const int lane = lane_id();
  const int* cbase = kC ? H.hcol : colors;
  int idle = 0, base = -1;
  int a[kHwWin];  // the window's colour slots (-1: nothing to read)
  bool end = false;
  while (pos != INT_MAX) {
    int c[kHwWin];
    if (base < 0) {  // (re)load the window: its ids stay in registers while pos moves inside it
      base = pos;
      end = false;
#pragma unroll
      int w[kHwWin];
#pragma unroll
      for (int u = 0; u < kHwWin; ++u) {
        const int i = base + u * 32 + lane;
        w[u] = i < deg ? ld_col(cols + b + i, pol) : INT_MAX;
        end |= w[u] > v;
      }
#pragma unroll
      for (int u = 0; u < kHwWin; ++u) a[u] = w[u] < v ? hw_slot<kC>(H, w[u]) : -1;
    }
    // entries before pos are final and marked already
#pragma unroll
    for (int u = 0; u < kHwWin; ++u)
      c[u] = (a[u] >= 0 && base + u * 32 + lane >= pos) ? ld_color(cbase + a[u]) : -3;
    int first = INT_MAX;
#pragma unroll
    for (int u = 0; u < kHwWin; ++u) {
      hv_mark(reg, win, c[u], lim);
      if (c[u] == kPending) first = min(first, base + u * 32 + lane);
    }
    first = __reduce_min_sync(kFull, first);
    ++n_polls;
    if (first == INT_MAX) {  // the window is final
      if (__any_sync(kFull, end)) break;
      pos = base + kHwWin * 32;
      base = -1;
      idle = 0;
      continue;
    }
    if (first != pos) {
      pos = first;
      idle = 0;
      continue;
    }
    if (++idle > polls) {  // guard: colour past what is still pending, as k1_heavy
      for (;; pos += kHwWin * 32) {
        bool e2 = false;
#pragma unroll
        for (int u = 0; u < kHwWin; ++u) {
          const int i = pos + u * 32 + lane;
          const int ww = i < deg ? ld_col(cols + b + i, pol) : INT_MAX;
          const int aa = ww < v ? hw_slot<kC>(H, ww) : -1;
          const int cc = aa >= 0 ? ld_color(cbase + aa) : -3;
          hv_mark(reg, win, cc, lim);
          log_pairs(L, cc == kPending, ww, v);
          e2 |= ww > v;
        }
        if (__any_sync(kFull, e2)) break;
      }
      return false;
    }
    if (idle > 4) __nanosleep(idle < 64 ? 32 : 256);
  }
  return true;
}

// One heavy row below the split threshold (warp-collective).
template <class PL, bool kC>
__device__ __forceinline__ void hw_row(const int* __restrict__ cols, int* colors, const HeavyArgs& H,
                                       const HeavyRow& e0, long long hr, unsigned* win, uint64_t pol, const PL& L,
                                       unsigned& gathers, long long& p_scan, long long& p_wait,
                                       long long& n_polls, long long& n_waited, long long& t_last) {
  const int lane = lane_id();
  const int v = e0.v, deg = e0.deg;
  const long long b = e0.b;
  win[lane] = 0u;
  __syncwarp();
  unsigned long long reg = 0ull;
  int pmin = INT_MAX;
  const int* cbase = kC ? H.hcol : colors;
  HvCols cb = hv_load_block(cols, b, deg, 0, pol);
  for (int base = 0;;) {
    int c[kHvU];
    bool past = false;
    if (kC) {  // the rank words first (eight independent loads), then the colours
      int a[kHvU];
#pragma unroll
      for (int u = 0; u < kHvU; ++u) {
        a[u] = cb.w[u] < v ? hw_slot<true>(H, cb.w[u]) : -1;
        past |= cb.w[u] > v;  // sorted row (INT_MAX past the end)
      }
#pragma unroll
      for (int u = 0; u < kHvU; ++u) c[u] = a[u] >= 0 ? hv_ld_color(cbase + a[u]) : -3;
    } else {
#pragma unroll
      for (int u = 0; u < kHvU; ++u) {
        c[u] = cb.w[u] < v ? hv_ld_color(cbase + cb.w[u]) : -3;
        past |= cb.w[u] > v;
      }
    }
    const bool more = base + kHvBlock < deg && !__any_sync(kFull, past);
    HvCols nb;
    if (more) nb = hv_load_block(cols, b, deg, base + kHvBlock, pol);  // in flight with the gathers
#pragma unroll
    for (int u = 0; u < kHvU; ++u) {
      gathers += cb.w[u] < v;
      hv_mark(reg, win, c[u], deg);
      if (c[u] == kPending) pmin = min(pmin, base + u * 32 + lane);
    }
    if (!more) break;
    cb = nb;
    base += kHvBlock;
  }
  pmin = __reduce_min_sync(kFull, pmin);
  hv_tick(H.prof, t_last, p_scan);
  if (pmin != INT_MAX) {
    ++n_waited;
    hw_wait<PL, kC>(cols, colors, H, v, b, deg, pmin, deg, reg, win, pol, H.polls, L, n_polls);
    hv_tick(H.prof, t_last, p_wait);
  }
  const unsigned lo = __reduce_or_sync(kFull, (unsigned)reg);
  const unsigned hi = __reduce_or_sync(kFull, (unsigned)(reg >> 32));
  __syncwarp();
  unsigned word = win[lane];
  if (lane == 0) word |= lo;
  if (lane == 1) word |= hi;
  const unsigned nf = __ballot_sync(kFull, word != kFull);
  const int j = __ffs(nf) - 1;
  const unsigned wj = __shfl_sync(kFull, word, j);
  if (lane == 0) hw_commit<kC>(H, colors, v, hr, j * 32 + __ffs(~wj) - 1);
  __syncwarp();
}

// First-Fit of a split row restricted to the colour window [wb, wb + 1024),
// over its lower heavy neighbours (all final by now); -1 when the window
// holds no free colour <= deg.  Only when the first 1024 colours are all taken.
template <bool kC>
__device__ __noinline__ int hw_ff_window(const int* __restrict__ cols, const int* colors, const HeavyArgs& H,
                                         int v, long long b, int deg, int wb, unsigned* win, uint64_t pol) {
  const int lane = lane_id();
  const int* cbase = kC ? H.hcol : colors;
  win[lane] = 0u;
  __syncwarp();
  for (int i0 = 0; i0 < deg; i0 += 32) {
    const int i = i0 + lane;
    const int w = i < deg ? ld_col(cols + b + i, pol) : INT_MAX;
    const int a = w < v ? hw_slot<kC>(H, w) : -1;
    const int c = a >= 0 ? ld_color(cbase + a) : -1;
    if (c >= wb && c < wb + 1024 && c <= deg) atomicOr(&win[(c - wb) >> 5], 1u << (c & 31));
    if (__any_sync(kFull, w > v)) break;
  }
  __syncwarp();
  const unsigned word = win[lane];
  const unsigned nf = __ballot_sync(kFull, word != kFull);
  if (!nf) return -1;
  const int j = __ffs(nf) - 1;
  const int c = wb + j * 32 + __ffs(~__shfl_sync(kFull, word, j)) - 1;
  return c <= deg ? c : -1;
}

// One split row (warp-collective; the owner): publish its pieces, wait for
// them, wait for what they read as pending, First-Fit, commit.
template <class PL, bool kC>
__device__ __forceinline__ void hw_hub(const long long* __restrict__ off, const int* __restrict__ cols,
                                       int* colors, const SplitArgs& S, const HeavyArgs& H,
                                       const HeavyRow& e0, long long hr, unsigned* win, uint64_t pol, const PL& L,
                                       long long& p_pieces, long long& p_wait, long long& n_polls,
                                       long long& n_waited, long long& t_last) {
  const int lane = lane_id();
  const int v = e0.v, deg = e0.deg;
  const long long b = e0.b;
  const int np = (deg + kPiece - 1) / kPiece;
  unsigned slot = 0, t = 0;
  if (lane == 0) {
    slot = atomicAdd(S.slot_ctr, 1u);
    t = atomicAdd(S.piece_ctr, (unsigned)np);
    S.slot_v[slot] = v;
    S.slot_deg[slot] = deg;
    atom_add_acq_rel(S.slot_left + slot, np);
  }
  slot = __shfl_sync(kFull, slot, 0);
  t = __shfl_sync(kFull, t, 0);
  for (int i = lane; i < np; i += 32) {
    const int len = min(kPiece, deg - i * kPiece);
    const long long a = b + (long long)i * kPiece;
    const unsigned slot_len = (slot << 10) | (unsigned)(len - 1);
    asm volatile("st.relaxed.gpu.global.v2.b64 [%0], {%1, %2};" ::"l"(H.q16 + t + i), "l"(a),
                 "l"(((unsigned long long)slot_len << 32) | (unsigned)v)
                 : "memory");
  }
  win[lane] = 0u;
  // the pieces: the slot's count returns to zero (its decrements and this
  // warp's add are acq_rel atomics on one word: the acquire load that reads
  // zero sees every piece's bitmap and position updates)
  if (lane == 0)
    while (ld_acquire_u32(reinterpret_cast<const unsigned*>(S.slot_left + slot)) != 0u) __nanosleep(64);
  __syncwarp();
  hv_tick(H.prof, t_last, p_pieces);
  unsigned long long reg = 0ull;
  const unsigned pw = ld_relaxed_u32(H.slot_pend + slot);
  // the pieces' bitmap is final here: read it before the wait, off the hop to the next row
  const unsigned slot_word = ld_relaxed_u32(S.slot_bm + (size_t)slot * 32 + lane);
  if (pw != 0u) {
    ++n_waited;
    hw_wait<PL, kC>(cols, colors, H, v, b, deg, INT_MAX - (int)pw, 1023, reg, win, pol, H.polls, L, n_polls);
    hv_tick(H.prof, t_last, p_wait);
  }
  const unsigned lo = __reduce_or_sync(kFull, (unsigned)reg);
  const unsigned hi = __reduce_or_sync(kFull, (unsigned)(reg >> 32));
  __syncwarp();
  unsigned word = win[lane] | slot_word;
  if (lane == 0) word |= lo;
  if (lane == 1) word |= hi;
  const unsigned nz = __ballot_sync(kFull, word != kFull);
  int color;
  if (nz) {
    const int j = __ffs(nz) - 1;
    color = j * 32 + __ffs(~__shfl_sync(kFull, word, j)) - 1;
  } else {  // 1024 distinct lower colours: the next windows, scanning the row (all final now)
    color = -1;
    for (int wb = 1024; color < 0 && wb <= deg; wb += 1024)
      color = hw_ff_window<kC>(cols, colors, H, v, b, deg, wb, win, pol);
  }
  if (lane == 0) hw_commit<kC>(H, colors, v, hr, color);
  __syncwarp();
}

// One piece of a split row (piece warps; never waits): as hv_piece, except
// that a pending neighbour is not logged -- the smallest position of one is
// left for the owner in H.slot_pend[slot] -- and the last piece does not
// commit.
template <bool kC>
__device__ __forceinline__ void hw_piece(const long long* __restrict__ off, const int* __restrict__ cols,
                                         const int* colors, const SplitArgs& S, const HeavyArgs& H,
                                         const HvPiece& r, int* buf, unsigned long long* bar,
                                         unsigned& phase, unsigned* win, uint64_t pol, unsigned& gathers,
                                         long long& t_last, long long* pp) {
  const int lane = lane_id();
  const int v = r.v;
  const int slot = (int)(r.slot_len >> 10);
  const int len = (int)(r.slot_len & 1023u) + 1;
  const long long A = r.a & ~3LL;
  const int o = (int)(r.a - A);
  long long end = A + ((o + len + 3) & ~3);
  if (end > H.m) end = H.m & ~3LL;
  const int nc = end > A ? (int)(end - A) : 0;  // staged entries; the rest from global
  __syncwarp();
  if (lane == 0) {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    mbar_arrive_expect_tx(bar, (unsigned)nc * 4u);
    if (nc) tma_load_1d_hint(buf, cols + A, (unsigned)nc * 4u, bar, pol);
  }
  win[lane] = 0u;
  mbar_wait(bar, phase);
  phase ^= 1u;
  hv_tick(H.prof, t_last, pp[0]);
  unsigned long long reg = 0ull;
  int pmin = INT_MAX;  // first pending entry of this piece (index within the piece)
  constexpr int B = kHvPieceBatch;
  for (int t0 = 0; t0 < 32; t0 += B) {
    int w[B], c[B];
    bool past = false;
#pragma unroll
    for (int u = 0; u < B; ++u) {
      const int i = (t0 + u) * 32 + lane;
      w[u] = i >= len ? INT_MAX : (o + i < nc ? buf[o + i] : ld_col(cols + r.a + i, pol));
      past |= w[u] > v;
    }
    if (kC) {
      int a[B];
#pragma unroll
      for (int u = 0; u < B; ++u) a[u] = w[u] < v ? hw_slot<true>(H, w[u]) : -1;
#pragma unroll
      for (int u = 0; u < B; ++u) c[u] = a[u] >= 0 ? hv_ld_color(H.hcol + a[u]) : -3;
    } else {
#pragma unroll
      for (int u = 0; u < B; ++u) c[u] = w[u] < v ? hv_ld_color(colors + w[u]) : -3;
    }
#pragma unroll
    for (int u = 0; u < B; ++u) {
      gathers += w[u] < v;
      hv_mark(reg, win, c[u], 1023);  // deg >= 1024 > every colour of this window
      if (c[u] == kPending) pmin = min(pmin, (t0 + u) * 32 + lane);
    }
    if (__any_sync(kFull, past)) break;  // sorted row: the rest is above v
  }
  hv_tick(H.prof, t_last, pp[1]);
  const unsigned lo = __reduce_or_sync(kFull, (unsigned)reg);
  const unsigned hi = __reduce_or_sync(kFull, (unsigned)(reg >> 32));
  pmin = __reduce_min_sync(kFull, pmin);
  __syncwarp();
  unsigned word = win[lane];
  if (lane == 0) word |= lo;
  if (lane == 1) word |= hi;
  if (word) atomicOr(S.slot_bm + (size_t)slot * 32 + lane, word);
  if (pmin != INT_MAX && lane == 0) {
    const long long b = ld_off(off + v, pol);
    atomicMax(H.slot_pend + slot, (unsigned)(INT_MAX - ((int)(r.a - b) + pmin)));
  }
  __syncwarp();
  // nobody needs the old value (the owner polls the count): a release reduction, so the
  // warp moves on to its next piece without waiting for the round trip
  if (lane == 0)
    asm volatile("red.release.gpu.global.add.s32 [%0], %1;" ::"l"(S.slot_left + slot), "r"(-1) : "memory");
  hv_tick(H.prof, t_last, pp[2]);
}

template <class PL, bool kC>
__global__ void __launch_bounds__(kHwThreads, 1)
    k1_heavy_wait(const long long* __restrict__ off, const int* __restrict__ cols, int* colors, Ctrl* ctrl,
                  PairLogArgs LA, SplitArgs S, HeavyArgs H) {
  extern __shared__ __align__(16) unsigned char k1hw_raw[];
  auto s_pbuf = reinterpret_cast<int(*)[kHvPieceBuf]>(k1hw_raw);
  __shared__ unsigned s_win[kHwWarps][32];
  __shared__ unsigned long long s_pbar[kHvPieceWarps];
  __shared__ __align__(16) int4 s_brec[kHwBufs][kHwBatch];  // the claimed batches' table records
  __shared__ int s_bgb[kHwBufs], s_btag[kHwBufs];
  __shared__ int s_ticket, s_npairs, s_mbhead;
  __shared__ unsigned s_gathers;
  const int RW = H.row_warps;
  if (threadIdx.x == 0) {
    s_ticket = 0;
    s_npairs = 0;
    s_mbhead = 0;
    s_gathers = 0;
  }
  if (threadIdx.x < kHvPieceWarps) mbar_init(&s_pbar[threadIdx.x], 1);
  if (threadIdx.x < kHwBufs) s_btag[threadIdx.x] = -1;
  if (threadIdx.x == 0) asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  init_peers(ctrl);
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = lane_id();
  const int G = gridDim.x;
  const uint64_t pol = policy_evict_first();
  const bool split = S.min_deg != INT_MAX;
  unsigned* win = s_win[warp];
  PL L;
  L.region = LA.pairs + (size_t)blockIdx.x * LA.region_cap;
  L.cap = LA.region_cap;
  L.s_count = &s_npairs;
  L.overflow = LA.overflow;
  unsigned gathers = 0;
  // GCOL_K1_PROFILE (cycles): row warps -- claiming a row, first scan, waiting
  // for pending neighbours, waiting for a split row's pieces, the rest; piece
  // warps as in k1_heavy; counts: rows, pieces, polls, rows that waited
  long long p_claim = 0, p_scan = 0, p_wait = 0, p_pieces = 0, p_idle = 0;
  long long n_rows = 0, n_pieces = 0, n_polls = 0, n_waited = 0;
  long long pp[4] = {0, 0, 0, 0};
  long long t_last = clock64();

  if (warp < RW) {
    // ------------------------------- row warps -------------------------------
    for (;;) {
      // ticket t = row t % B of the CTA's batch t / B; the warp that draws a
      // batch's first ticket claims the batch from the global cursor, in
      // ticket order (so a higher ticket is always a higher row).  One global
      // claim per row was measured and lost: the same-address atomics cost
      // 2.4k -> 4.8k cycles per row on R-MAT 27 (heavy pass 32 -> 39 ms).
      // Claiming each batch one ahead (records waiting in shared memory when
      // the tickets are drawn) was measured too and changed nothing (R-MAT 24
      // 4.62 -> 4.76 ms, R-MAT 27 32.3 -> 32.9 ms): the ~2k cycles between two
      // rows of a warp are the previous row's commit path, not the claim.
      int t = 0;
      if (lane == 0) t = atomicAdd(&s_ticket, 1);
      t = __shfl_sync(kFull, t, 0);
      const int lb = t / kHwBatch, p = t % kHwBatch, bb = lb % kHwBufs;
      if (p == 0) {
        // the claimer also brings the batch's table records (one 128-byte line)
        // into shared memory, so the other seven rows start without that miss
        int gb = 0;
        if (lane == 0) {
          if (lb > 0)
            while (ld_acquire_cta_s32(&s_btag[(lb - 1) % kHwBufs]) != lb - 1) {
            }
          gb = (int)atomicAdd(H.cursor, 1u);
          s_bgb[bb] = gb;
        }
        gb = __shfl_sync(kFull, gb, 0);
        const long long rr = (long long)gb * kHwBatch + lane;
        if (lane < kHwBatch && rr < H.nh)
          s_brec[bb][lane] = __ldg(reinterpret_cast<const int4*>(H.rows + rr));
        __syncwarp();
        if (lane == 0) st_release_cta_s32(&s_btag[bb], lb);
      } else {
        if (lane == 0)
          while (ld_acquire_cta_s32(&s_btag[bb]) != lb) {
          }
        __syncwarp();
      }
      const long long r = (long long)s_bgb[bb] * kHwBatch + p;
      if (r >= H.nh) break;
      const int4 q = s_brec[bb][p];
      HeavyRow e0;
      e0.b = ((long long)(unsigned)q.y << 32) | (unsigned)q.x;
      e0.v = q.z;
      e0.deg = q.w;
      // streamed upload: a row starts only once its whole adjacency is resident
      if (H.piece_ready && lane == 0)
        for (long long qq = e0.b >> H.piece_shift; qq <= (e0.b + e0.deg - 1) >> H.piece_shift; ++qq)
          while (ld_acquire_u32(H.piece_ready + qq) == 0u) __nanosleep(256);
      __syncwarp();
      hv_tick(H.prof, t_last, p_claim);
      if (e0.deg >= S.min_deg)
        hw_hub<PL, kC>(off, cols, colors, S, H, e0, r, win, pol, L, p_pieces, p_wait, n_polls, n_waited, t_last);
      else
        hw_row<PL, kC>(cols, colors, H, e0, r, win, pol, L, gathers, p_scan, p_wait, n_polls, n_waited, t_last);
      ++n_rows;
    }
    // retired: its piece allocations before the count drops
    if (lane == 0 && split) {
      __threadfence();
      atomicSub(S.alive, 1);
    }
  } else if (warp < RW + H.piece_warps) {
    // ------------------------------ piece warps ------------------------------
    const int pw = warp - RW;
    unsigned pphase = 0, pc_hint = 0;
    while (split) {
      const unsigned pc_new = ld_relaxed_u32(S.piece_ctr);
      HvPiece pr;
      if (hv_pop16(S, H.q16, &s_mbhead, pc_hint, pr)) {
        hv_tick(H.prof, t_last, pp[3]);
        hw_piece<kC>(off, cols, colors, S, H, pr, s_pbuf[pw], &s_pbar[pw], pphase, win, pol, gathers, t_last, pp);
        pc_hint = pc_new;
        ++n_pieces;
        continue;
      }
      const unsigned alive = ld_acquire_u32(reinterpret_cast<const unsigned*>(S.alive));
      const unsigned alloc = ld_acquire_u32(S.piece_ctr);
      int head = *reinterpret_cast<volatile int*>(&s_mbhead);
      head = __shfl_sync(kFull, head, 0);
      const bool empty = (unsigned)head * (unsigned)G + blockIdx.x >= alloc;
      if (__shfl_sync(kFull, (int)(alive == 0u && empty), 0)) break;
      pc_hint = __shfl_sync(kFull, alloc, 0);
      if (empty) __nanosleep(128);
      hv_tick(H.prof, t_last, p_idle);
    }
  }
  if (H.prof && lane == 0) {
    unsigned long long* P = ctrl->prof;
    const long long vals[13] = {p_claim, p_scan, p_wait, p_pieces, n_polls, p_idle, n_rows, n_pieces,
                                n_waited, pp[0],  pp[1],  pp[2],    pp[3]};
    for (int i = 0; i < 13; ++i)
      if (vals[i]) atomicAdd(P + i, (unsigned long long)vals[i]);
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
