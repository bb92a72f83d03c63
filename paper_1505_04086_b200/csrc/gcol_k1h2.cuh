// gcol_k1h2.cuh -- K1H with the gathers decoupled from the commit order
// (an experiment, GCOL_K1H_V=2; gcol_k1c.cuh holds the default heavy pass,
// k1_heavy, and everything the two share).
//
// Same contract as k1_heavy: heavy rows (degree >= T) in ascending id order,
// each First-Fit over its LOWER heavy neighbours, a lower neighbour still
// pending (-2) at the row's LAST look logged for round 1.  What k1_heavy
// could not do is hide latency: the colour count grows with the rows that
// are claimed but not committed, so it kept ~8 rows per SM in
// flight and each of them paid the whole chain -- staged row, one round trip
// of colour gathers, re-check, First-Fit, commit (~4.2k cycles; 25 % of the
// warp slots busy, 0.2 eligible warps per cycle).
//
// Here a row is handled twice:
//   build   (many warps, far ahead of the commit front, in ticket order):
//           stream the row's lower prefix, gather the colours, OR the final
//           ones into the row's forbidden bitmap in shared memory, and keep
//           the ids of the neighbours read as pending (<= kH2Pend per row;
//           more are logged at once, which only adds round-1 candidates).
//   commit  (few warps, strictly in ticket order): re-read the kept pending
//           neighbours (they are few, and by now nearly all final), mark,
//           log the ones still pending, First-Fit over the bitmap, commit.
// What decides the colour count is now the time between a row's last look
// and its commit -- one short round trip for the few rows that kept a
// pending neighbour, nothing for the others -- and the number of commit
// warps; the memory latency is paid by the build warps, whose number and
// lead (the ring of kH2Ring slots per CTA) are free to fill the SM.
//
// Split rows (degree >= 1024) go through the commit warps only: the commit
// warp publishes the row's pieces at the row's turn (hv_push_long) and the
// piece warps of the whole grid serve them as in k1_heavy, so a hub is still
// in flight for one piece latency in its ascending position.
//
// Ring protocol (per CTA; ticket t -> slot t % R, generation t / R):
//   builder t waits for s_gen[slot] == t / R (the slot's previous row is
//   committed), builds, then releases s_ready[slot] = t / R + 1;
//   committer t waits for that value, commits, releases s_gen[slot] + 1.
// Rows come from the global cursor in batches of kH2Batch consecutive heavy
// rows, claimed two batches ahead by the builder that takes a batch's first
// ticket; the first ticket past the last heavy row sets s_end, which retires
// every builder and committer that draws a later ticket.
#pragma once
#include "gcol_k1c.cuh"

namespace gcol {
namespace dev {

constexpr int kH2Warps = 24;                 // warps per CTA: commit + build + piece
constexpr int kH2Threads = kH2Warps * 32;
constexpr int kH2Ring = 64;                  // slots per CTA (H.ring <= this)
constexpr int kH2Batch = 16;                 // heavy rows per cursor claim
constexpr int kH2Bufs = 8;                   // batch record buffers (>= ring / batch + 3)
constexpr int kH2Pend = 32;                  // pending lower neighbours kept per row
constexpr size_t kH2Smem = sizeof(int) * kHvPieceWarps * kHvPieceBuf;  // dynamic: piece buffers

static_assert(kH2Bufs >= kH2Ring / kH2Batch + 3, "batch buffers must outlive the ring");

// Claim the next batch of heavy rows for local batch index lbn (warp-collective).
__device__ __forceinline__ void h2_claim(const HeavyArgs& H, int lbn, HeavyRow (*s_brec)[kH2Batch],
                                         int* s_bgb, int* s_btag) {
  const int lane = lane_id();
  const int buf = lbn % kH2Bufs;
  unsigned gb = 0;
  if (lane == 0) gb = atomicAdd(H.cursor, 1u);
  gb = __shfl_sync(kFull, gb, 0);
  if (lane < kH2Batch) {
    const long long r = (long long)gb * kH2Batch + lane;
    HeavyRow e{r, -1, 0};  // past the table: v < 0
    if (r < H.nh) {
      const int4 q = __ldg(reinterpret_cast<const int4*>(H.rows + r));
      e.b = ((long long)(unsigned)q.y << 32) | (unsigned)q.x;
      e.v = q.z;
      e.deg = q.w;
    }
    s_brec[buf][lane] = e;
  }
  if (lane == 0) s_bgb[buf] = (int)gb;
  __syncwarp();
  if (lane == 0) st_release_cta_s32(&s_btag[buf], lbn);
}

// Build one non-split heavy row into its ring slot: forbidden bitmap (colours
// 0..1023 >= every colour of a row of degree < 1024) and the pending list.
// Returns the number of pending neighbours kept (warp-uniform).
template <class PL>
__device__ __forceinline__ int h2_build(const int* __restrict__ cols, const int* colors,
                                        const HeavyArgs& H, const HeavyRow& e0, unsigned* bm, int* pend,
                                        uint64_t pol, const PL& L, unsigned& gathers) {
  const int lane = lane_id();
  const int v = e0.v, deg = e0.deg;
  const long long b = e0.b;
  bm[lane] = 0u;
  __syncwarp();
  unsigned long long reg = 0ull;
  int np = 0;
  HvCols cb = hv_load_block(cols, b, deg, 0, pol);
  for (int base = 0;;) {
    int c[kHvU];
    bool past = false;
#pragma unroll
    for (int u = 0; u < kHvU; ++u) {
      c[u] = cb.w[u] < v ? hv_gather(H, colors, cb.w[u]) : -3;
      past |= cb.w[u] > v;  // sorted row (INT_MAX past the end)
    }
    const bool more = base + kHvBlock < deg && !__any_sync(kFull, past);
    HvCols nb;
    if (more) nb = hv_load_block(cols, b, deg, base + kHvBlock, pol);  // in flight with the gathers
    unsigned stale = 0;
#pragma unroll
    for (int u = 0; u < kHvU; ++u) {
      gathers += cb.w[u] < v;
      hv_mark(reg, bm, c[u], deg);
      stale |= (c[u] == kPending ? 1u : 0u) << u;
    }
    if (__any_sync(kFull, stale != 0u)) {
#pragma unroll
      for (int u = 0; u < kHvU; ++u) {
        const bool p = (stale >> u) & 1u;
        const unsigned m = __ballot_sync(kFull, p);
        const int pos = np + __popc(m & ((1u << lane) - 1u));
        if (p && pos < kH2Pend) pend[pos] = cb.w[u];
        np += __popc(m);
        if (np > kH2Pend) log_pairs(L, p && pos >= kH2Pend, cb.w[u], v);
      }
    }
    if (!more) break;
    cb = nb;
    base += kHvBlock;
  }
  const unsigned lo = __reduce_or_sync(kFull, (unsigned)reg);
  const unsigned hi = __reduce_or_sync(kFull, (unsigned)(reg >> 32));
  if (lane == 0 && lo) atomicOr(&bm[0], lo);
  if (lane == 1 && hi) atomicOr(&bm[1], hi);
  return min(np, kH2Pend);
}

// Commit one built row (warp-collective): last look at its pending
// neighbours (polls extra re-reads while any is still pending), First-Fit
// over the bitmap, commit.
template <class PL>
__device__ __forceinline__ void h2_commit(int* colors, const HeavyArgs& H, const HeavyRow& e0, int hr,
                                          unsigned* bm, const int* pend, int np, int polls,
                                          const PL& L, long long& n_pend, long long& n_left) {
  const int lane = lane_id();
  if (np > 0) {
    const int w = lane < np ? pend[lane] : -1;
    int c = w >= 0 ? hv_gather_relaxed(H, colors, w) : -3;
    for (int k = 0; k < polls && __any_sync(kFull, c == kPending); ++k) {
      __nanosleep(64);
      if (c == kPending) c = hv_gather_relaxed(H, colors, w);
    }
    if (static_cast<unsigned>(c) <= static_cast<unsigned>(e0.deg)) atomicOr(&bm[c >> 5], 1u << (c & 31));
    log_pairs(L, c == kPending, w, e0.v);
    if (H.prof) {
      n_pend += np;
      n_left += __popc(__ballot_sync(kFull, c == kPending));
    }
    __syncwarp();
  }
  const unsigned word = bm[lane];
  const unsigned nf = __ballot_sync(kFull, word != kFull);
  const int j = __ffs(nf) - 1;
  const unsigned wj = __shfl_sync(kFull, word, j);
  if (lane == 0) hv_commit(H, colors, e0.v, hr, j * 32 + __ffs(~wj) - 1);
  __syncwarp();
}

template <class PL>
__global__ void __launch_bounds__(kH2Threads, 1)
    k1_heavy2(const long long* __restrict__ off, const int* __restrict__ cols, int* colors, Ctrl* ctrl,
              PairLogArgs LA, SplitArgs S, HeavyArgs H) {
  extern __shared__ __align__(16) unsigned char k1h2_raw[];
  auto s_pbuf = reinterpret_cast<int(*)[kHvPieceBuf]>(k1h2_raw);
  __shared__ unsigned s_bm[kH2Ring][32];
  __shared__ int s_pend[kH2Ring][kH2Pend];
  __shared__ __align__(16) HeavyRow s_rec[kH2Ring];
  __shared__ int s_np[kH2Ring], s_hr[kH2Ring], s_ready[kH2Ring], s_gen[kH2Ring];
  __shared__ __align__(16) HeavyRow s_brec[kH2Bufs][kH2Batch];
  __shared__ int s_bgb[kH2Bufs], s_btag[kH2Bufs];
  __shared__ unsigned s_win[kH2Warps][32];
  __shared__ unsigned long long s_pbar[kHvPieceWarps];
  __shared__ int s_bt, s_ct, s_end, s_npairs, s_mbhead;
  __shared__ unsigned s_gathers;
  const int NC = H.commit_warps, NB = H.build_warps, R = H.ring;
  if (threadIdx.x == 0) {
    s_bt = 0;
    s_ct = 0;
    s_end = INT_MAX;
    s_npairs = 0;
    s_mbhead = 0;
    s_gathers = 0;
  }
  if (threadIdx.x < kHvPieceWarps) mbar_init(&s_pbar[threadIdx.x], 1);
  if (threadIdx.x < kH2Ring) {
    s_ready[threadIdx.x] = 0;
    s_gen[threadIdx.x] = 0;
  }
  if (threadIdx.x < kH2Bufs) s_btag[threadIdx.x] = -1;
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
  // GCOL_K1_PROFILE: cycles -- commit warps waiting for a built row / at the
  // last look and commit; build warps waiting (batch, slot) / building; piece
  // warps as in k1_heavy; counts: rows, pieces, pending kept, pending left
  long long p_cwait = 0, p_commit = 0, p_bwait = 0, p_build = 0, p_idle = 0;
  long long n_rows = 0, n_pieces = 0, n_pend = 0, n_left = 0;
  long long pp[4] = {0, 0, 0, 0};
  long long t_last = clock64();

  if (warp < NC) {
    // ------------------------------ commit warps -----------------------------
    for (;;) {
      int t = 0;
      if (lane == 0) t = atomicAdd(&s_ct, 1);
      t = __shfl_sync(kFull, t, 0);
      const int slot = t % R, gen = t / R;
      int ok = 0;
      if (lane == 0) {
        for (;;) {
          if (ld_acquire_cta_s32(&s_ready[slot]) == gen + 1) {
            ok = 1;
            break;
          }
          if (t >= *reinterpret_cast<volatile int*>(&s_end)) break;
        }
      }
      ok = __shfl_sync(kFull, ok, 0);
      if (!ok) break;
      const HeavyRow e0 = s_rec[slot];
      hv_tick(H.prof, t_last, p_cwait);
      if (e0.deg >= S.min_deg)
        hv_push_long(off, cols, colors, S, H, e0.v, e0.deg, e0.b, win, pol);
      else
        h2_commit<PL>(colors, H, e0, s_hr[slot], s_bm[slot], s_pend[slot], s_np[slot], H.polls, L, n_pend,
                      n_left);
      __syncwarp();
      if (lane == 0) st_release_cta_s32(&s_gen[slot], gen + 1);
      ++n_rows;
      hv_tick(H.prof, t_last, p_commit);
    }
    // retired: its piece allocations before the count drops
    if (lane == 0 && split) {
      __threadfence();
      atomicSub(S.alive, 1);
    }
  } else if (warp < NC + NB) {
    // ------------------------------- build warps -----------------------------
    if (warp == NC) {
      h2_claim(H, 0, s_brec, s_bgb, s_btag);
      h2_claim(H, 1, s_brec, s_bgb, s_btag);
    }
    for (;;) {
      int t = 0;
      if (lane == 0) t = atomicAdd(&s_bt, 1);
      t = __shfl_sync(kFull, t, 0);
      const int lb = t / kH2Batch, p = t % kH2Batch, bb = lb % kH2Bufs;
      const int slot = t % R, gen = t / R;
      int ok = 0;
      if (lane == 0) {
        for (;;) {
          if (ld_acquire_cta_s32(&s_btag[bb]) == lb) {
            ok = 1;
            break;
          }
          if (t >= *reinterpret_cast<volatile int*>(&s_end)) break;
        }
      }
      ok = __shfl_sync(kFull, ok, 0);
      if (!ok) break;
      const HeavyRow e0 = s_brec[bb][p];
      const int hr = s_bgb[bb] * kH2Batch + p;
      if (e0.v < 0) {  // past the last heavy row: so is every later ticket
        if (lane == 0) atomicMin(&s_end, t);
        break;
      }
      if (lane == 0)
        while (ld_acquire_cta_s32(&s_gen[slot]) != gen) __nanosleep(32);
      __syncwarp();
      // two batches ahead; after the slot wait, so every reader of the buffer
      // it overwrites (batch lb + 2 - kH2Bufs) has committed
      if (p == 0) h2_claim(H, lb + 2, s_brec, s_bgb, s_btag);
      // streamed upload: a row is built only once its whole adjacency is resident
      if (H.piece_ready && lane == 0)
        for (long long q = e0.b >> H.piece_shift; q <= (e0.b + e0.deg - 1) >> H.piece_shift; ++q)
          while (ld_acquire_u32(H.piece_ready + q) == 0u) __nanosleep(256);
      __syncwarp();
      hv_tick(H.prof, t_last, p_bwait);
      int np = 0;
      if (e0.deg < S.min_deg)
        np = h2_build<PL>(cols, colors, H, e0, s_bm[slot], s_pend[slot], pol, L, gathers);
      if (lane == 0) {
        s_rec[slot] = e0;
        s_np[slot] = np;
        s_hr[slot] = hr;
      }
      __syncwarp();
      if (lane == 0) st_release_cta_s32(&s_ready[slot], gen + 1);
      hv_tick(H.prof, t_last, p_build);
    }
  } else if (warp < NC + NB + H.piece_warps) {
    // ------------------------------ piece warps ------------------------------
    const int pw = warp - NC - NB;
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
    const long long vals[13] = {p_cwait, p_commit, p_bwait, p_build, n_pend, p_idle, n_rows, n_pieces,
                                n_left,  pp[0],    pp[1],   pp[2],   pp[3]};
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
