// gcol_k1c.cuh -- the class-split initial pass for skewed-degree graphs
// (R-MAT): K1H over the heavy rows, then K1L (the waiting pass, kClass mode)
// over the light rows.
//
// Same contract as K1 (parallel.hpp:286-296): every vertex is
// coloured once with First-Fit over the neighbours it reads, colours never
// exceed the degree, and every read of a neighbour that was still in flight
// is logged, so round 1 (k_candidates) finds every monochromatic edge among
// the losers of logged pairs.  What changes is the ORDER of the pass:
//
//   K1H  rows of degree >= T (heavy; R-MAT 24: 1.18 M of 16.8 M rows, 88 %
//        of the adjacency) in ascending id order, each reading only its LOWER
//        heavy neighbours.  Heavy rows start as kPending (-2): a lower
//        neighbour read as -2 is in flight (re-read once, then logged); -1 is
//        a light row, which has not started and reads this row itself later.
//   K1L  rows of degree < T in ascending id order, each reading its WHOLE row
//        (all heavy neighbours are final) and waiting for uncoloured lower
//        light neighbours as K1W does (gcol_k1w.cuh), so the light rows are
//        First-Fit exact given the heavy colours.
//
// Why: in the single ascending sweep (k1_pipe) a warp holds 32 mostly-light
// rows for ~28 us, so keeping the in-flight window small (the colour count
// grows with it) starves the GPU: one 9-warp CTA per SM, 5 % of
// the HBM roofline.  Light rows barely affect the colour count (colours <=
// degree < T) and, waiting, never conflict; heavy rows are what must be kept
// few in flight, and with only heavy rows in the sweep every warp moves from
// one heavy row to the next with its data already staged.
//
// K1H schedule (k1_heavy below): rows are handed out in ascending order by
// CTA tickets over batches claimed from a global cursor (no static
// assignment, hence no drift bound: measured, a drift bound between statically
// scheduled warps cost 45 % of the pass in waits); a producer warp per CTA
// stages the next batch by TMA; split rows (degree >= 1024) are cut into
// kPiece-entry pieces served by dedicated piece warps from per-CTA mailboxes.
// The in-flight window -- ~2 x row_warps x G rows -- is the knob that trades
// colours for time.  The grid must be co-resident (ticket and
// mailbox waits): it is launched cooperatively.
#pragma once
#include "gcol_k1w.cuh"

namespace gcol {
namespace dev {

constexpr int kPending = -2;   // heavy row not coloured yet (K1H)

// K1H colour gathers.  Inside K1H a colour is -1 (light row: ignored), -2
// (pending heavy row) or final, and changes at most once (-2 -> final); a
// read that returns an older value returns -2, which is logged -- safe.  So
// the gathers may use the non-coherent read-only path without L1 allocation
// (LDG.E.NA.CONSTANT, served by L2) instead of ld.relaxed.gpu
// (LDG.E.STRONG.GPU).  Re-checks of a pending neighbour stay relaxed.
#ifndef GCOL_K1H_NC
#define GCOL_K1H_NC 1
#endif
__device__ __forceinline__ int hv_ld_color(const int* p) {
#if GCOL_K1H_NC
  int r;
  asm volatile("ld.global.nc.L1::no_allocate.b32 %0, [%1];" : "=r"(r) : "l"(p));
  return r;
#else
  return ld_color(p);
#endif
}
constexpr int kHvWarps = 8;    // row-warp slots per K1H CTA (row warps + the producer)
constexpr int kClassTDefault = kSmallMax + 1;  // heavy: degree >= 64

// One heavy row: where its adjacency starts, its id and degree (16 B, one
// load per row).  Built once per graph in ascending id order.
struct alignas(16) HeavyRow {
  long long b;
  int v;
  int deg;
};

// One piece of a split heavy row, as K1H publishes it: everything the piece
// needs in one 16-byte record, so popping it costs one load.  Initialised to
// all ones (0xff bytes) before the run; both halves change exactly once, so a
// reader that sees neither half at its initial value sees the whole record.
struct alignas(16) HvPiece {
  long long a;          // adjacency index of its first entry
  int v;                // the row
  unsigned slot_len;    // slot << 10 | (entries - 1)
};
constexpr int kHvSlotMax = 1 << 22;

// Heavy-rank table (per graph, built with the heavy-row table): per 32-id
// word, the heavy ids' bit mask and the number of heavy ids below the word,
// so rank(w) = base + popc(bits below w).  The compact variant of the waiting
// heavy pass (gcol_k1hw.cuh) keeps the heavy rows' colours in an array indexed
// by rank: 4 x heavy rows bytes (R-MAT 27: 32 MB, L2-resident) instead of
// gathers into a 537 MB colour array that miss L2 four times out of five.
struct alignas(8) HvRank {
  unsigned bits;
  int base;
};

struct HeavyArgs {
  HvPiece* q16;       // [npieces] piece records (split rows)
  const HeavyRow* rows;
  int nh;
  int row_warps;      // row warps per CTA (1 .. kHvWarps - 1; the batch size): the
                      //   in-flight window is ~2 row_warps rows per CTA
  int recheck;        // re-read a pending lower neighbour once before logging it
  unsigned* cursor;   // batches claimed (global, ascending)
  int prof;           // GCOL_K1_PROFILE: per-phase cycle counters into ctrl->prof
  long long m;        // adjacency length (bulk copies never read past it)
  int piece_warps;    // active piece warps per CTA (1 .. kHvPieceWarps)
  const unsigned* piece_ready;  // streamed upload: flag per 2^piece_shift adjacency
  int piece_shift;              //   entries resident (null: the whole CSR is resident)
  // k1_heavy_wait (gcol_k1hw.cuh): polls without progress before a row colours past what
  // is still pending; per split-row slot, INT_MAX - the position of the
  // first entry a piece read as pending (0: none); zeroed before every run
  int polls;
  unsigned* slot_pend;
  // compact variant of k1_heavy_wait: rank table and the heavy colours by rank
  // (-2 pending); every commit writes both this array and the colour array
  const HvRank* rank;
  int* hcol;
};

// K1H colour reads and writes.  (A compact heavy-colour array behind a rank
// table, as a run-time option of THIS pass, was measured and removed: two
// dependent loads per gather lost in a window-limited pass, and even switched
// off its branch in these helpers kept the compiler from batching the gathers
// -- R-MAT 24 K1H 4.4 -> 5.9 ms.  The waiting pass has it as a compile-time
// variant, gcol_k1hw.cuh.)
__device__ __forceinline__ int hv_gather(const HeavyArgs&, const int* colors, int w) {
  return hv_ld_color(colors + w);
}
__device__ __forceinline__ int hv_gather_relaxed(const HeavyArgs&, const int* colors, int w) {
  return ld_color(colors + w);
}
// Commit heavy row v with colour c (one lane).
__device__ __forceinline__ void hv_commit(const HeavyArgs&, int* colors, int v, int, int c) {
  commit_color(colors, v, c);
}

// --------------------------------------------------------------------------
// Heavy-row table (per graph): ordered compaction of {v : deg(v) >= T}.
// Blocks of kClassSpan ids: count, exclusive scan of the counts (one CTA),
// then write in order.
// --------------------------------------------------------------------------
constexpr int kClassSpan = 2048;

__global__ void __launch_bounds__(kBlock) k_class_count(const long long* __restrict__ off, int n,
                                                        int T, int* counts) {
  __shared__ int s_c;
  if (threadIdx.x == 0) s_c = 0;
  __syncthreads();
  const long long v0 = (long long)blockIdx.x * kClassSpan;
  int c = 0;
  for (int j = threadIdx.x; j < kClassSpan; j += kBlock) {
    const long long v = v0 + j;
    if (v < n && off[v + 1] - off[v] >= T) ++c;
  }
  c = (int)__reduce_add_sync(kFull, (unsigned)c);
  if (lane_id() == 0 && c) atomicAdd(&s_c, c);
  __syncthreads();
  if (threadIdx.x == 0) counts[blockIdx.x] = s_c;
}

// Exclusive scan of nb counts in place (one CTA; nb <= 2^20), total -> *total.
__global__ void __launch_bounds__(1024) k_class_scan(int* counts, int nb, int* total) {
  __shared__ int s_part[1024];
  const int per = (nb + 1023) / 1024;
  const int lo = threadIdx.x * per, hi = min(nb, lo + per);
  int sum = 0;
  for (int i = lo; i < hi; ++i) sum += counts[i];
  s_part[threadIdx.x] = sum;
  __syncthreads();
  for (int d = 1; d < 1024; d <<= 1) {
    const int y = threadIdx.x >= d ? s_part[threadIdx.x - d] : 0;
    __syncthreads();
    s_part[threadIdx.x] += y;
    __syncthreads();
  }
  int run = s_part[threadIdx.x] - sum;
  for (int i = lo; i < hi; ++i) {
    const int c = counts[i];
    counts[i] = run;
    run += c;
  }
  if (threadIdx.x == 1023) *total = s_part[1023];
}

__global__ void __launch_bounds__(kBlock) k_class_write(const long long* __restrict__ off, int n,
                                                        int T, const int* pre, HeavyRow* rows,
                                                        HvRank* rank) {
  __shared__ int s_w[kWarps];
  __shared__ int s_base;
  if (threadIdx.x == 0) s_base = pre[blockIdx.x];
  const int warp = threadIdx.x >> 5, lane = lane_id();
  const long long v0 = (long long)blockIdx.x * kClassSpan;
  for (int j0 = 0; j0 < kClassSpan; j0 += kBlock) {
    const long long v = v0 + j0 + threadIdx.x;
    long long b = 0;
    int d = 0;
    if (v < n) {
      b = off[v];
      d = (int)(off[v + 1] - b);
    }
    const bool h = v < n && d >= T;
    const unsigned m = __ballot_sync(kFull, h);
    __syncthreads();  // s_base of the previous step is final
    if (lane == 0) s_w[warp] = __popc(m);
    __syncthreads();
    int before = s_base;
    for (int k = 0; k < warp; ++k) before += s_w[k];
    if (h) rows[before + __popc(m & ((1u << lane) - 1u))] = HeavyRow{b, (int)v, d};
    if (rank && lane == 0 && v < n) rank[v >> 5] = HvRank{m, before};  // v = the word's first id
    __syncthreads();
    if (threadIdx.x == 0) {
      int t = 0;
      for (int k = 0; k < kWarps; ++k) t += s_w[k];
      s_base += t;
    }
  }
}

// Heavy rows start pending: colors[v] := -2; compact variant: hcol[*] := -2
// (K1HW then reads heavy colours only through hcol).
__global__ void k_mark_pending(const HeavyRow* __restrict__ rows, int nh, int* colors, int* hcol) {
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < nh;
       i += (long long)gridDim.x * blockDim.x) {
    if (hcol) hcol[i] = kPending;
    else colors[rows[i].v] = kPending;
  }
}

// --------------------------------------------------------------------------
// K1H
// --------------------------------------------------------------------------
constexpr int kHvU = 8;                         // adjacency entries per lane per block
constexpr int kHvBlock = 32 * kHvU;             // 256 per warp
constexpr int kHvStageCols = kHvBlock + 4;      // a row's staged first block (+ alignment slack)

struct HvCols {
  int w[kHvU];
};

__device__ __forceinline__ HvCols hv_load_block(const int* __restrict__ cols, long long b, int deg,
                                                int base, uint64_t pol) {
  HvCols r;
  const int lane = lane_id();
#pragma unroll
  for (int u = 0; u < kHvU; ++u) {
    const int i = base + u * 32 + lane;
    r.w[u] = i < deg ? ld_col(cols + b + i, pol) : INT_MAX;
  }
  return r;
}

__device__ __forceinline__ unsigned ld_relaxed_u32(const unsigned* p) {
  unsigned r;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(r) : "l"(p) : "memory");
  return r;
}

__device__ __forceinline__ int ld_acquire_cta_s32(const int* p) {
  int r;
  asm volatile("ld.acquire.cta.shared::cta.b32 %0, [%1];" : "=r"(r) : "r"(smem_u32(p)) : "memory");
  return r;
}

__device__ __forceinline__ void st_release_cta_s32(int* p, int v) {
  asm volatile("st.release.cta.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(p)), "r"(v) : "memory");
}

// Entries of row e staged from its aligned base A = b & ~3: [A, A + n).
__device__ __forceinline__ int hv_staged(const HeavyRow& e, long long m, int min_deg) {
  if (e.v < 0 || e.deg <= 0 || e.deg >= min_deg) return 0;
  const long long A = e.b & ~3LL;
  const long long want = (e.b - A) + min(e.deg, kHvBlock);
  long long end = A + ((want + 3) & ~3LL);
  if (end > m) end = m & ~3LL;  // never past the adjacency: the tail is read from global
  return end > A ? (int)(end - A) : 0;
}

// The row of a split slot is complete: First-Fit over the slot's bitmap
// (colours 0..1023 OR-ed in by its pieces), commit.  Warp-collective.
__device__ __noinline__ void hv_finish_row(const long long* __restrict__ off,
                                           const int* __restrict__ cols, int* colors,
                                           const SplitArgs& S, const HeavyArgs& H, int slot, int v,
                                           unsigned* win, uint64_t pol) {
  const int lane = lane_id();
  const unsigned wd = ld_acquire_u32(S.slot_bm + (size_t)slot * 32 + lane);
  const unsigned fr = ~wd;
  const unsigned nz = __ballot_sync(kFull, fr != 0u);
  int color;
  if (nz) {
    const int j = __ffs(nz) - 1;
    color = j * 32 + __ffs(__shfl_sync(kFull, fr, j)) - 1;
  } else {  // 1024 distinct lower colours: the next windows, scanning the row
    const int deg = S.slot_deg[slot];
    const long long b = ld_off(off + v, pol);
    color = -1;
    for (int wb = 1024; color < 0 && wb <= deg; wb += 1024)
      color = warp_ff_window<false, true>(cols, colors, v, b, deg, wb, win, pol);
  }
  if (lane == 0) hv_commit(H, colors, v, -1, color);
  __syncwarp();
}

// Publish the pieces of heavy row v (warp-collective; the warp's own row).
// slot_left[slot] starts at 0 each run; the publisher adds np, every piece
// subtracts one (all acq_rel atomics on one word, so totally ordered), and
// whichever of them brings it to zero commits the row: normally the last
// piece, or the publisher itself if every piece finished before its add was
// performed.  No fence is needed on either side, and the records are stored
// without waiting for the add.
__device__ __forceinline__ void hv_push_long(const long long* __restrict__ off,
                                             const int* __restrict__ cols, int* colors,
                                             const SplitArgs& S, const HeavyArgs& H, int v, int deg,
                                             long long b, unsigned* win, uint64_t pol) {
  HvPiece* q16 = H.q16;
  const int lane = lane_id();
  const int np = (deg + kPiece - 1) / kPiece;
  unsigned slot = 0, t = 0;
  int before = 0;
  if (lane == 0) {
    slot = atomicAdd(S.slot_ctr, 1u);
    t = atomicAdd(S.piece_ctr, (unsigned)np);
  }
  slot = __shfl_sync(kFull, slot, 0);
  t = __shfl_sync(kFull, t, 0);
  if (lane == 0) {
    S.slot_v[slot] = v;
    S.slot_deg[slot] = deg;
    before = atom_add_acq_rel(S.slot_left + slot, np);  // its value is waited for below
  }
  for (int i = lane; i < np; i += 32) {
    const int len = min(kPiece, deg - i * kPiece);
    HvPiece r;
    r.a = b + (long long)i * kPiece;
    r.v = v;
    r.slot_len = (slot << 10) | (unsigned)(len - 1);
    asm volatile("st.relaxed.gpu.global.v2.b64 [%0], {%1, %2};" ::"l"(q16 + t + i), "l"(r.a),
                 "l"(((unsigned long long)r.slot_len << 32) | (unsigned)r.v)
                 : "memory");
  }
  // the count may be added after every piece finished (the records can be
  // seen first): then the publisher is the one that brings it to zero
  if (__shfl_sync(kFull, (int)(before == -np), 0)) hv_finish_row(off, cols, colors, S, H, (int)slot, v, win, pol);
}

// Claim the next piece of this CTA's mailbox below `alloc` and read its
// record.  Warp-uniform control flow throughout (the mailbox head is read by
// lane 0 and broadcast; only the claiming CAS is single-lane): a lane-0 loop
// here left the warp diverged at every step, and the reconvergence
// (WARPSYNC.COLLECTIVE + shuffles) was the top stall of K1H.
__device__ __forceinline__ bool hv_pop16(const SplitArgs& S, HvPiece* q16, int* s_mbhead,
                                         unsigned alloc, HvPiece& r) {
  const int lane = lane_id();
  for (;;) {
    int j = *reinterpret_cast<volatile int*>(s_mbhead);
    j = __shfl_sync(kFull, j, 0);
    const unsigned p = (unsigned)j * (unsigned)S.G + blockIdx.x;
    if (p >= alloc) return false;
    int won = 0;
    if (lane == 0) won = atomicCAS(s_mbhead, j, j + 1) == j;
    if (!__shfl_sync(kFull, won, 0)) continue;
    long long a;
    unsigned long long hi;
    for (;;) {  // the same address in every lane: one request, one value
      asm volatile("ld.relaxed.gpu.global.v2.b64 {%0, %1}, [%2];"
                   : "=l"(a), "=l"(hi) : "l"(q16 + p) : "memory");
      if (a != -1LL && hi != ~0ull) break;
      __nanosleep(32);
    }
    r.a = a;
    r.v = (int)(unsigned)hi;
    r.slot_len = (unsigned)(hi >> 32);
    return true;
  }
}

// Mark colour c (if 0 <= c <= lim) in the 64-bit register mask or the warp's
// 1024-colour window; branch-light (predicated shared atomic).
__device__ __forceinline__ void hv_mark(unsigned long long& reg, unsigned* win, int c, int lim) {
  const bool ok = static_cast<unsigned>(c) <= static_cast<unsigned>(lim);
  reg |= (ok && c < 64) ? (1ull << (c & 63)) : 0ull;
  if (ok && c >= 64) atomicOr(&win[c >> 5], 1u << (c & 31));
}

__device__ __forceinline__ void hv_tick(int on, long long& t_last, long long& acc) {
  if (on) {
    const long long t = clock64();
    acc += t - t_last;
    t_last = t;
  }
}

constexpr int kHvPieceBuf = kPiece + 4;
#ifndef GCOL_K1H_PB
#define GCOL_K1H_PB 8
#endif
constexpr int kHvPieceBatch = GCOL_K1H_PB;  // colour gathers per lane in flight (piece warps)

// One piece: staged by TMA into the warp's buffer, its lower neighbours'
// colours gathered 16 per lane at a time, OR-ed into the row's bitmap; the
// last piece commits the row.
template <class PL>
__device__ __forceinline__ void hv_piece(const long long* __restrict__ off,
                                         const int* __restrict__ cols, int* colors,
                                         const SplitArgs& S, const HeavyArgs& H, const HvPiece& r, int* buf,
                                         unsigned long long* bar, unsigned& phase, long long m,
                                         unsigned* win, uint64_t pol, const PL& L,
                                         unsigned& gathers, int prof, long long& t_last,
                                         long long* pp) {
  const int lane = lane_id();
  const int v = r.v;
  const int slot = (int)(r.slot_len >> 10);
  const int len = (int)(r.slot_len & 1023u) + 1;
  const long long A = r.a & ~3LL;
  const int o = (int)(r.a - A);
  long long end = A + ((o + len + 3) & ~3);
  if (end > m) end = m & ~3LL;
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
  hv_tick(prof, t_last, pp[0]);
  unsigned long long reg = 0ull;
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
#pragma unroll
    for (int u = 0; u < B; ++u) c[u] = w[u] < v ? hv_gather(H, colors, w[u]) : -3;
#pragma unroll
    for (int u = 0; u < B; ++u) {
      gathers += w[u] < v;
      hv_mark(reg, win, c[u], 1023);  // deg >= 1024 > every colour of this window
    }
    unsigned stale = 0;
#pragma unroll
    for (int u = 0; u < B; ++u) stale |= (c[u] == kPending ? 1u : 0u) << u;
    if (__any_sync(kFull, stale != 0u)) {
#pragma unroll
      for (int u = 0; u < B; ++u) log_pairs(L, (stale >> u) & 1u, w[u], v);
    }
    if (__any_sync(kFull, past)) break;  // sorted row: the rest is above v
  }
  hv_tick(prof, t_last, pp[1]);
  const unsigned lo = __reduce_or_sync(kFull, (unsigned)reg);
  const unsigned hi = __reduce_or_sync(kFull, (unsigned)(reg >> 32));
  __syncwarp();
  unsigned word = win[lane];
  if (lane == 0) word |= lo;
  if (lane == 1) word |= hi;
  if (word) atomicOr(S.slot_bm + (size_t)slot * 32 + lane, word);
  __syncwarp();
  int last = 0;
  if (lane == 0) last = atom_add_acq_rel(S.slot_left + slot, -1) == 1;
  last = __shfl_sync(kFull, last, 0);
  if (last) hv_finish_row(off, cols, colors, S, H, slot, v, win, pol);
  hv_tick(prof, t_last, pp[2]);
}

// One heavy row of degree < the split threshold (warp-collective): First-Fit
// over its LOWER heavy neighbours (colours <= deg < 1024), pending ones
// (kPending) re-read once and then logged, commit.  `staged`: the first
// nc entries from the row's aligned base (shared memory), the rest global.
template <class PL>
__device__ __forceinline__ void hv_row(const int* __restrict__ cols, int* colors,
                                       const HeavyArgs& H, const HeavyRow& e0, int hr, const int* staged,
                                       int nc, unsigned* win, uint64_t pol, const PL& L,
                                       unsigned& gathers, long long& p_g0, long long& p_gx,
                                       long long& p_rc, long long& n_xb, long long& t_last) {
  const int lane = lane_id();
  const int v = e0.v, deg = e0.deg;
  const long long b = e0.b;
  // First-Fit over the lower heavy neighbours (colours <= deg < 1024)
  win[lane] = 0u;
  __syncwarp();
  unsigned long long reg = 0ull;
  int sw = -1;  // one pending neighbour per lane, re-read before logging
  HvCols cb;
  {
    const int o = (int)(b - (b & ~3LL));
#pragma unroll
    for (int u = 0; u < kHvU; ++u) {
      const int i = u * 32 + lane;
      cb.w[u] = i >= deg ? INT_MAX : (o + i < nc ? staged[o + i] : ld_col(cols + b + i, pol));
    }
  }
  for (int base = 0;;) {
    int c[kHvU];
#pragma unroll
    for (int u = 0; u < kHvU; ++u) c[u] = cb.w[u] < v ? hv_gather(H, colors, cb.w[u]) : -3;
    bool past = false;
    unsigned stale = 0;
#pragma unroll
    for (int u = 0; u < kHvU; ++u) {
      gathers += cb.w[u] < v;
      past |= cb.w[u] > v;  // sorted row (INT_MAX past the end)
      hv_mark(reg, win, c[u], deg);
      stale |= (c[u] == kPending ? 1u : 0u) << u;
    }
    if (__any_sync(kFull, stale != 0u)) {  // rare: keep one per lane, log the rest
#pragma unroll
      for (int u = 0; u < kHvU; ++u) {
        const bool pend = (stale >> u) & 1u;
        const bool keep = pend && H.recheck && sw < 0;
        if (keep) sw = cb.w[u];
        log_pairs(L, pend && !keep, cb.w[u], v);
      }
    }
    base += kHvBlock;
    hv_tick(H.prof, t_last, base == kHvBlock ? p_g0 : p_gx);
    if (__any_sync(kFull, past) || base >= deg) break;
    cb = hv_load_block(cols, b, deg, base, pol);
    ++n_xb;
  }
  if (__any_sync(kFull, sw >= 0)) {
    const int c = sw >= 0 ? hv_gather_relaxed(H, colors, sw) : -3;
    hv_mark(reg, win, c, deg);
    log_pairs(L, c == kPending, sw, v);
    hv_tick(H.prof, t_last, p_rc);
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
  if (lane == 0) hv_commit(H, colors, v, hr, j * 32 + __ffs(~wj) - 1);
  __syncwarp();
}

constexpr int kHvPieceWarps = 8;                       // piece-warp slots per CTA
constexpr int kHvBufs = 3;                             // staged batches per CTA
constexpr int kHvThreads = (kHvWarps + kHvPieceWarps) * 32;
// dynamic shared memory: piece buffers, then the staged rows' first blocks
constexpr size_t kHvPieceBytes = sizeof(int) * kHvPieceWarps * kHvPieceBuf;
constexpr size_t kHvSmem = kHvPieceBytes + sizeof(int) * kHvBufs * (kHvWarps - 1) * kHvStageCols;

// K1H.  Warp-specialised CTAs:
//   - row warps (H.row_warps of them) colour heavy rows handed out by CTA
//     tickets: ticket t = row t % RW of the CTA's batch t / RW, a batch being
//     RW consecutive heavy rows claimed from the global cursor in ascending
//     order -- rows go out in ascending order as warps become free, so no
//     warp ever waits for another (no drift bound, no imbalance stalls) and
//     the rows claimed but not committed stay ~2 RW per CTA;
//   - one producer warp keeps the next batch claimed and staged (table
//     entries, then each row's first 256 adjacency entries, by TMA) one batch
//     ahead of the row warps, so a row starts with its data in shared memory;
//   - kHvPieceWarps piece warps serve the CTA's mailbox of pieces of split
//     rows (degree >= 1024), which therefore neither slow the row warps nor
//     wait behind them: a split row is in flight for about one piece's latency.
template <class PL>
__global__ void __launch_bounds__(kHvThreads, 1)
    k1_heavy(const long long* __restrict__ off, const int* __restrict__ cols, int* colors,
             Ctrl* ctrl, PairLogArgs LA, SplitArgs S, HeavyArgs H) {
  extern __shared__ __align__(16) unsigned char k1h_raw[];
  auto s_pbuf = reinterpret_cast<int(*)[kHvPieceBuf]>(k1h_raw);
  auto s_pcols = reinterpret_cast<int(*)[kHvWarps - 1][kHvStageCols]>(k1h_raw + kHvPieceBytes);
  __shared__ unsigned s_win[kHvWarps + kHvPieceWarps][32];
  __shared__ unsigned long long s_pbar[kHvPieceWarps];
  __shared__ __align__(16) HeavyRow s_pool[kHvBufs][kHvWarps];
  __shared__ unsigned long long s_poolbar[kHvBufs], s_colbar[kHvBufs];
  __shared__ int s_ticket, s_tag[kHvBufs], s_gb[kHvBufs], s_read[kHvBufs];
  __shared__ int s_npairs, s_mbhead;
  __shared__ unsigned s_gathers;
  const int RW = H.row_warps;
  if (threadIdx.x == 0) {
    s_npairs = 0;
    s_mbhead = 0;
    s_gathers = 0;
    s_ticket = 0;
  }
  if (threadIdx.x < kHvPieceWarps) mbar_init(&s_pbar[threadIdx.x], 1);
  if (threadIdx.x < kHvBufs) {
    mbar_init(&s_poolbar[threadIdx.x], 1);
    mbar_init(&s_colbar[threadIdx.x], 1);
    s_tag[threadIdx.x] = -1;
    s_read[threadIdx.x] = RW;  // free
  }
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
  // GCOL_K1_PROFILE (cycles): row warps -- taking the staged row, block 0,
  // later blocks, re-check, the rest; piece warps -- pieces (pop, TMA wait,
  // gathers, finish), idle; counts: rows, pieces, later blocks
  long long p_pre = 0, p_g0 = 0, p_gx = 0, p_rc = 0, p_row = 0;
  long long p_idle = 0, n_rows = 0, n_pieces = 0, n_xb = 0;
  long long pp[4] = {0, 0, 0, 0};
  long long t_last = clock64();

  if (warp >= kHvWarps + H.piece_warps) {
    // idle piece slot
  } else if (warp >= kHvWarps) {
    // ------------------------------ piece warps ------------------------------
    const int pw = warp - kHvWarps;
    unsigned pphase = 0, pc_hint = 0;
    while (split) {
      const unsigned pc_new = ld_relaxed_u32(S.piece_ctr);
      HvPiece pr;
      if (hv_pop16(S, H.q16, &s_mbhead, pc_hint, pr)) {
        hv_tick(H.prof, t_last, pp[3]);
        hv_piece<PL>(off, cols, colors, S, H, pr, s_pbuf[pw], &s_pbar[pw], pphase, H.m, win, pol, L,
                     gathers, H.prof, t_last, pp);
        pc_hint = pc_new;
        ++n_pieces;
        continue;
      }
      // nothing below the hint: fresh counts; done once every row warp has
      // retired (no more pieces can appear) and the mailbox is drained
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
  } else if (warp == RW) {
    // -------------------------------- producer -------------------------------
    for (int lb = 0;; ++lb) {
      const int buf = lb % kHvBufs;
      const unsigned par = (unsigned)((lb / kHvBufs) & 1);
      int avail = 0;
      if (lane == 0) {
        // one batch ahead: batch lb - 1 has started; buffer free: batch lb - 3 done
        while (lb >= 1 && *reinterpret_cast<volatile int*>(&s_ticket) <= (lb - 1) * RW) __nanosleep(32);
        while (*reinterpret_cast<volatile int*>(&s_read[buf]) < RW) __nanosleep(32);
        s_read[buf] = 0;
        const unsigned gb = atomicAdd(H.cursor, 1u);
        const long long r0 = (long long)gb * RW;
        avail = (int)max(0LL, min((long long)RW, (long long)H.nh - r0));
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        mbar_arrive_expect_tx(&s_poolbar[buf], (unsigned)avail * 16u);
        if (avail) tma_load_1d_hint(s_pool[buf], H.rows + r0, (unsigned)avail * 16u, &s_poolbar[buf], pol);
        s_gb[buf] = (int)gb;
      }
      avail = __shfl_sync(kFull, avail, 0);
      mbar_wait(&s_poolbar[buf], par);
      // the batch rows' first blocks (lane p copies row p's)
      int nc = 0;
      HeavyRow e{0, -1, 0};
      if (lane < avail) {
        e = s_pool[buf][lane];
        nc = hv_staged(e, H.m, S.min_deg);
        // streamed upload: rows go out in ascending id = ascending adjacency
        // order, following the upload front; a row is handed out only once
        // its whole adjacency is resident
        if (H.piece_ready && e.deg > 0)
          for (long long q = e.b >> H.piece_shift; q <= (e.b + e.deg - 1) >> H.piece_shift; ++q)
            while (ld_acquire_u32(H.piece_ready + q) == 0u) __nanosleep(256);
      }
      __syncwarp();
      const unsigned bytes = __reduce_add_sync(kFull, (unsigned)nc * 4u);
      if (lane == 0) mbar_arrive_expect_tx(&s_colbar[buf], bytes);
      __syncwarp();
      if (nc) tma_load_1d_hint(s_pcols[buf][lane], cols + (e.b & ~3LL), (unsigned)nc * 4u, &s_colbar[buf], pol);
      __syncwarp();
      if (lane == 0) st_release_cta_s32(&s_tag[buf], lb);
      if (avail == 0) break;  // the empty batch retires every row warp
    }
  } else if (warp < RW) {
    // ------------------------------- row warps -------------------------------
    const HeavyRow none{0, -1, 0};
    for (;;) {
      int t = 0;
      if (lane == 0) t = atomicAdd(&s_ticket, 1);
      t = __shfl_sync(kFull, t, 0);
      const int lb = t / RW, p = t % RW, buf = lb % kHvBufs;
      const unsigned par = (unsigned)((lb / kHvBufs) & 1);
      if (lane == 0)
        while (ld_acquire_cta_s32(&s_tag[buf]) != lb) {
        }
      __syncwarp();
      mbar_wait(&s_poolbar[buf], par);
      mbar_wait(&s_colbar[buf], par);
      const long long r = (long long)s_gb[buf] * RW + p;
      const HeavyRow e0 = r < H.nh ? s_pool[buf][p] : none;
      hv_tick(H.prof, t_last, p_pre);
      if (e0.v >= 0) {
        if (e0.deg >= S.min_deg)
          hv_push_long(off, cols, colors, S, H, e0.v, e0.deg, e0.b, win, pol);
        else
          hv_row<PL>(cols, colors, H, e0, (int)r, s_pcols[buf][p], hv_staged(e0, H.m, S.min_deg), win, pol,
                     L, gathers, p_g0, p_gx, p_rc, n_xb, t_last);
      }
      __syncwarp();
      if (lane == 0) atomicAdd(&s_read[buf], 1);  // its staged entry and block are free
      if (e0.v < 0) break;
      ++n_rows;
      hv_tick(H.prof, t_last, p_row);
    }
    // retired: its piece allocations before the count drops
    if (lane == 0 && split) {
      __threadfence();
      atomicSub(S.alive, 1);
    }
  }
  if (H.prof && lane == 0) {
    unsigned long long* P = ctrl->prof;
    const long long vals[13] = {p_pre, p_g0, p_gx, p_rc, p_row, p_idle, n_rows, n_pieces, n_xb,
                                pp[0], pp[1], pp[2], pp[3]};
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
