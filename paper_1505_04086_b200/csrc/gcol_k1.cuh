// gcol_k1.cuh -- K1, the tentative-colour pass (parallel.hpp:286-296), v3.
//
// Every warp is an independent worker: it pulls 32-vertex sub-tiles in
// ascending id order (CTAs claim 256-vertex chunks from a global cursor;
// the warps of a CTA split a chunk through one 64-bit shared-memory word
// holding {chunk, next sub-tile}), so no CTA-wide barrier ever sits on the
// critical path.  Per sub-tile:
//   deg == 0          colour 0 (coloring.hpp:98-105)
//   1 <= deg <= 63    thread per row over the adjacency staged in shared
//                     memory with coalesced loads, 64-bit register mask;
//                     rows that read an in-flight (uncoloured) lower
//                     neighbour are parked and re-checked one sub-tile later
//   64 <= deg < split edge-parallel across all such rows of the sub-tile,
//                     per-row forbidden bitmaps in shared memory
//   deg >= split      split into kPiece-entry pieces pushed on a global
//                     queue; every warp pops pieces before it takes a new
//                     sub-tile, ORs its piece's forbidden colours into the
//                     row's global bitmap, and the last piece commits the
//                     colour -- so a hub is spread over the whole GPU and is
//                     in flight only briefly, in its ascending-id position
// In the initial pass a row gathers only its LOWER neighbours' colours:
// rows are sorted, every edge is examined by its higher endpoint, and each
// stale read that survives the re-check is logged for round 1.
#pragma once
#include "gcol_device.cuh"

namespace gcol {
namespace dev {

constexpr int kK1Warps = 8;
constexpr int kK1Block = kK1Warps * 32;
constexpr int kSubTiles = kK1Block / 32;  // sub-tiles per claimed chunk
constexpr int kBmWords = 512;             // per-warp medium-row bitmap pool
constexpr int kStaleMax = 4;              // stale neighbours remembered per parked row
constexpr int kSplitDefault = 1024;       // rows >= this are split into pieces
constexpr int kPiece = 1024;              // entries per piece

struct K1Warp {
  int stage[kStage];                   // staged small-row adjacency (4 KB)
  unsigned bm[kBmWords];               // medium-row bitmaps (2 KB)
  unsigned win[32];                    // window for the rare overflow path
  int dv[2][32];                       // parked row per lane (ping-pong tables)
  unsigned dmask[2][32][2];
  unsigned char ddeg[2][32];
  unsigned char dns[2][32];
  int dst[2][32][kStaleMax];           // in-flight neighbours to re-check
  int cv[32];                          // second-chance slot per lane (carry)
  unsigned cmask[32][2];
  unsigned char cdeg[32];
  unsigned char cns[32];
  int cst[32][kStaleMax];
  int redo[2][32];                     // medium rows parked for recomputation
  int nredo[2];
};

// Long-row pieces.  Piece p (global allocation order) is delivered to the
// mailbox of CTA p % G; each CTA drains its own mailbox with a shared-memory
// head, so no global atomic is contended by consumers.  Sized per graph so
// the arrays never wrap.
struct SplitArgs {
  int min_deg;          // rows with deg >= min_deg are split (INT_MAX: never)
  int* slot_v;          // [nslots] row of each slot
  int* slot_deg;
  int* slot_left;       // pieces still to finish
  unsigned* slot_bm;    // [nslots][32] forbidden colours 0..1023
  int2* q;              // [npieces] (slot, first entry)
  unsigned* q_seq;      // [npieces] = 1 once entry p is published
  unsigned* piece_ctr;  // pieces allocated so far
  unsigned* slot_ctr;
  int* alive;           // warps that may still publish pieces
  int G;                // mailboxes (= K1 grid)
};

// First-Fit restricted to the colour window [wb, wb + 1024) (warp-wide);
// returns -1 when the window holds no free colour <= deg.  Only used for
// rows whose first 1024 colours are all forbidden (needs deg >= 1024).
template <bool kSnap, bool kLower>
__device__ __noinline__ int warp_ff_window(const int* __restrict__ cols, const int* csrc, int v, long long b,
                              int deg, int wb, unsigned* win, uint64_t pol) {
  const int lane = lane_id();
  win[lane] = 0u;
  __syncwarp();
  for (int i = lane; i < deg; i += 32) {
    const int w = ld_col(cols + b + i, pol);
    if (kLower && w > v) break;
    const int c = read_color<kSnap>(csrc, w);
    if (c >= wb && c < wb + 1024 && c <= deg) atomicOr(&win[(c - wb) >> 5], 1u << ((c - wb) & 31));
  }
  __syncwarp();
  const int lim = deg - wb;  // candidates wb..deg
  const int bits_here = lim >= 1023 ? 32 : (lim < 0 ? 0 : ((lim >> 5) == lane ? (lim & 31) + 1 : (lane < (lim >> 5) ? 32 : 0)));
  const unsigned vm = bits_here == 32 ? kFull : ((1u << bits_here) - 1u);
  const unsigned fr = ~win[lane] & vm;
  const unsigned nz = __ballot_sync(kFull, fr != 0u);
  __syncwarp();
  if (!nz) return -1;
  const int j = __ffs(nz) - 1;
  const unsigned fj = __shfl_sync(kFull, fr, j);
  return wb + j * 32 + __ffs(fj) - 1;
}

// ---------------------------------------------------------------------------
// Staging.  Rows of consecutive ids are adjacent in memory, so a sub-tile's
// whole adjacency segment is usually one contiguous run: when it fits in
// the stage it is copied once with coalesced loads and every row (small and
// medium) reads shared memory.  Otherwise only small rows are staged, with
// a compact parallel copy (all loads of a batch issued together).
// ---------------------------------------------------------------------------
struct StageInfo {
  bool all;        // stage holds [base, base + kStage) of the segment
  long long base;
};

__device__ __forceinline__ StageInfo k1_stage(const int* __restrict__ cols, long long b, int deg,
                                              K1Warp& W, uint64_t pol) {
  const int lane = lane_id();
  const long long nb = __shfl_down_sync(kFull, b, 1);
  const bool contig = __all_sync(kFull, lane == 31 || nb == b + deg);
  const long long b0 = __shfl_sync(kFull, b, 0);
  const long long bend = __shfl_sync(kFull, b + deg, 31);
  StageInfo si{contig && bend - b0 <= kStage, b0};
  if (si.all) {
    const int len = (int)(bend - b0);
    for (int i = lane; i < len; i += 32 * 4) {
      int x[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int j = i + u * 32;
        x[u] = j < len ? ld_col(cols + b0 + j, pol) : 0;
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int j = i + u * 32;
        if (j < len) W.stage[j] = x[u];
      }
    }
    __syncwarp();
  }
  return si;
}

// Row of compact entry j: largest lane r with excl_r <= j.
__device__ __forceinline__ int row_of(int excl, int j) {
  int lo = 0;
#pragma unroll
  for (int s = 16; s >= 1; s >>= 1) {
    const int e = __shfl_sync(kFull, excl, lo + s);
    if (lo + s < 32 && e <= j) lo += s;
  }
  return lo;
}

// ---------------------------------------------------------------------------
// small rows: thread per row over staged adjacency, 64-bit register mask
// ---------------------------------------------------------------------------
template <bool kSnap, bool kLower, bool kLog>
__device__ __noinline__ void k1_small(const int* __restrict__ cols, const int* csrc, int* cdst,
                                      int v, long long b, int deg, bool small, K1Warp& W,
                                      int table, uint64_t pol, const PairLog& L,
                                      unsigned& gathers, StageInfo si) {
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
  const int nbatch = si.all ? 1 : (total + kStageStep - 1) / kStageStep;
  for (int bt = 0; bt < nbatch; ++bt) {
    const int lo = bt * kStageStep;
    const bool mine = small && (si.all || (excl >= lo && excl < lo + kStageStep));
    if (!si.all) {  // compact parallel copy of this batch's small rows
      const int hi = min(total, lo + kStage);
      for (int j0 = lo; j0 < hi; j0 += 32 * 4) {
        int x[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int j = j0 + u * 32 + lane;
          const int r = row_of(excl, j);
          const long long br = __shfl_sync(kFull, b, r);
          const int er = __shfl_sync(kFull, excl, r);
          x[u] = j < hi ? ld_col(cols + br + (j - er), pol) : 0;
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int j = j0 + u * 32 + lane;
          if (j < hi) W.stage[j - lo] = x[u];
        }
      }
    }
    __syncwarp();
    const int* row = si.all ? W.stage + (b - si.base) : W.stage + (excl - lo);
    const int maxk = __reduce_max_sync(kFull, (unsigned)(mine ? len : 0));
    bool active = mine;
    int ns = 0;
    unsigned long long mask = 0ull;
    for (int k = 0; k < maxk; k += 4) {
      int w[4];
      bool take[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const bool in = active && (k + u) < len;
        w[u] = in ? row[k + u] : 0;
        take[u] = in && (!kLower || w[u] < v);
        if (kLower && in && w[u] > v) active = false;  // sorted row: the rest is > v
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
          const bool keep = st && ns < kStaleMax;
          if (keep) W.dst[table][lane][ns] = w[u];
          ns += st ? 1 : 0;
          log_pairs(L, st && !keep, w[u], v);
        }
      }
      if (kLower && !__any_sync(kFull, active)) break;
    }
    if (mine) {
      if (kLog && ns > 0) {  // park; committed after the re-check one sub-tile later
        W.dv[table][lane] = v;
        W.dmask[table][lane][0] = (unsigned)mask;
        W.dmask[table][lane][1] = (unsigned)(mask >> 32);
        W.ddeg[table][lane] = (unsigned char)deg;
        W.dns[table][lane] = (unsigned char)min(ns, kStaleMax);
      } else {
        st_color(cdst + v, __ffsll((long long)~mask) - 1);
      }
    }
    __syncwarp();
  }
}

// Re-check the rows parked in `table` (warp-collective).  A row whose
// in-flight neighbours have all committed is committed now; otherwise it
// gets one more sub-tile in the lane's carry slot, and whatever is still
// uncoloured at that second check is logged for round 1.
__device__ __noinline__ void k1_drain(K1Warp& W, int table, int* cdst, const PairLog& L) {
  const int lane = lane_id();
  // (1) carry slot: final check
  {
    const int v = W.cv[lane];
    const int ns = v >= 0 ? (int)W.cns[lane] : 0;
    int c[kStaleMax], u[kStaleMax];
#pragma unroll
    for (int k = 0; k < kStaleMax; ++k) {
      u[k] = k < ns ? W.cst[lane][k] : 0;
      c[k] = k < ns ? ld_color(cdst + u[k]) : -2;
    }
    unsigned long long mask = 0ull;
    int deg = 0;
    if (v >= 0) {
      mask = (unsigned long long)W.cmask[lane][0] | ((unsigned long long)W.cmask[lane][1] << 32);
      deg = W.cdeg[lane];
    }
#pragma unroll
    for (int k = 0; k < kStaleMax; ++k) {
      if (c[k] >= 0 && c[k] <= deg) mask |= 1ull << c[k];
      log_pairs(L, k < ns && c[k] == -1, u[k], v);  // still in flight: round 1 checks it
    }
    if (v >= 0) {
      st_color(cdst + v, __ffsll((long long)~mask) - 1);
      W.cv[lane] = -1;
    }
  }
  // (2) rows parked one sub-tile ago
  const int v = W.dv[table][lane];
  const int ns = v >= 0 ? (int)W.dns[table][lane] : 0;
  int c[kStaleMax], u[kStaleMax];
#pragma unroll
  for (int k = 0; k < kStaleMax; ++k) {
    u[k] = k < ns ? W.dst[table][lane][k] : 0;
    c[k] = k < ns ? ld_color(cdst + u[k]) : -2;
  }
  if (v >= 0) {
    unsigned long long mask = (unsigned long long)W.dmask[table][lane][0] |
                              ((unsigned long long)W.dmask[table][lane][1] << 32);
    const int deg = W.ddeg[table][lane];
    int left = 0;
#pragma unroll
    for (int k = 0; k < kStaleMax; ++k) {
      if (c[k] >= 0 && c[k] <= deg) mask |= 1ull << c[k];
      if (k < ns && c[k] == -1) W.cst[lane][left++] = u[k];
    }
    if (left == 0) {
      st_color(cdst + v, __ffsll((long long)~mask) - 1);
    } else {  // second chance
      W.cv[lane] = v;
      W.cmask[lane][0] = (unsigned)mask;
      W.cmask[lane][1] = (unsigned)(mask >> 32);
      W.cdeg[lane] = (unsigned char)deg;
      W.cns[lane] = (unsigned char)left;
    }
    W.dv[table][lane] = -1;
  }
  __syncwarp();
}

// ---------------------------------------------------------------------------
// medium rows (64 <= deg < split): edge-parallel over all such rows of the
// sub-tile; per-row bitmaps of min(deg/32 + 1, 32) words in shared memory
// plus one flag word.  In park mode (first pass, in-place K1) a row that read
// an in-flight lower neighbour is not committed: its id goes to `redo`, and
// one sub-tile later the whole row is recomputed in log mode.
// ---------------------------------------------------------------------------
template <bool kSnap, bool kLower, bool kLog>
__device__ __noinline__ void k1_medium(const int* __restrict__ cols, const int* csrc, int* cdst,
                                       int v, long long b, int deg, bool med, K1Warp& W,
                                       uint64_t pol, const PairLog& L, unsigned& gathers,
                                       int* redo, int* nredo, StageInfo si) {
  const int lane = lane_id();
  const bool park_mode = kLog && redo != nullptr;
  unsigned medmask = __ballot_sync(kFull, med);
  while (medmask) {
    // rows of this batch: medium rows in lane order while their words fit
    const int words = med ? min((deg >> 5) + 1, 32) : 0;
    const int need = words + 1;  // + stale flag
    int wincl = (medmask >> lane) & 1u ? need : 0;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const int y = __shfl_up_sync(kFull, wincl, d);
      if (lane >= d) wincl += y;
    }
    const bool inb = ((medmask >> lane) & 1u) && wincl <= kBmWords;
    const unsigned batch = __ballot_sync(kFull, inb);
    medmask &= ~batch;
    const int woff = wincl - need;
    // rows of the batch that may park (room reserved in the redo list)
    const int rank = __popc(batch & ((1u << lane) - 1u));
    const bool parkable = park_mode && inb && (*nredo + rank) < 32;
    const int len = inb ? deg : 0;
    int eincl = len;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const int y = __shfl_up_sync(kFull, eincl, d);
      if (lane >= d) eincl += y;
    }
    const int eoff = eincl - len;
    const int E = __shfl_sync(kFull, eincl, 31);
    const int Wt = __shfl_sync(kFull, inb ? wincl : 0, 31 - __clz(batch));
    for (int i = lane; i < Wt; i += 32) W.bm[i] = 0u;
    __syncwarp();
    for (int i0 = 0; i0 < E; i0 += 32 * 4) {
      int w[4], r[4], vr[4], dr[4];
      bool take[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int idx = i0 + u * 32 + lane;
        const bool in = idx < E;
        const int lo = row_of(eoff, idx);
        r[u] = lo;
        const long long br = __shfl_sync(kFull, b, lo);
        const int er = __shfl_sync(kFull, eoff, lo);
        vr[u] = __shfl_sync(kFull, v, lo);
        dr[u] = __shfl_sync(kFull, deg, lo);
        w[u] = !in ? 0 : (si.all ? W.stage[br - si.base + (idx - er)]
                                 : ld_col(cols + br + (idx - er), pol));
        take[u] = in && (!kLower || w[u] < vr[u]);
      }
      int c[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) c[u] = take[u] ? read_color<kSnap>(csrc, w[u]) : -2;
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        gathers += take[u];
        const int wo = __shfl_sync(kFull, woff, r[u]);
        const int nw = __shfl_sync(kFull, words, r[u]);
        const bool pk = __shfl_sync(kFull, parkable, r[u]);
        const bool ok = c[u] >= 0 && c[u] <= dr[u] && c[u] < 1024;
        if (ok) atomicOr(&W.bm[wo + (c[u] >> 5)], 1u << (c[u] & 31));
        if (kLog) {
          const bool st = take[u] && c[u] == -1;
          if (st && pk) W.bm[wo + nw] = 1u;      // defer: recompute the row later
          log_pairs(L, st && !pk, w[u], vr[u]);
        }
      }
    }
    __syncwarp();
    // first free colour per row
    int color = -1;
    bool park = false;
    if (inb) {
      park = parkable && W.bm[woff + words] != 0u;
      for (int k = 0; k < words; ++k) {
        const unsigned fr = ~W.bm[woff + k];
        if (fr) {
          color = k * 32 + __ffs(fr) - 1;
          break;
        }
      }
      if (color > deg) color = -1;  // cannot happen: <= deg marks among deg+1 slots
    }
    // rows whose first 1024 colours are all taken (deg >= 1024 only)
    unsigned over = __ballot_sync(kFull, inb && !park && color < 0);
    while (over) {
      const int rr = __ffs(over) - 1;
      over &= over - 1;
      const int vv = __shfl_sync(kFull, v, rr);
      const long long bb = __shfl_sync(kFull, b, rr);
      const int dd = __shfl_sync(kFull, deg, rr);
      int c = -1;
      for (int wb = 1024; c < 0 && wb <= dd; wb += 1024)
        c = warp_ff_window<kSnap, kLower>(cols, csrc, vv, bb, dd, wb, W.win, pol);
      if (lane == rr) color = c;
    }
    if (park_mode) {
      const unsigned pm = __ballot_sync(kFull, park);
      if (park) redo[*nredo + __popc(pm & ((1u << lane) - 1u))] = v;
      __syncwarp();
      if (lane == 0) *nredo += __popc(pm);
    }
    if (inb && !park) st_color(cdst + v, color);
    __syncwarp();
  }
}

// Recompute the rows parked by k1_medium one sub-tile ago (log mode).
template <bool kLower>
__device__ __noinline__ void k1_redo(const long long* __restrict__ off, const int* __restrict__ cols,
                        int* cdst, K1Warp& W, int table, uint64_t pol, const PairLog& L,
                        unsigned& gathers) {
  const int lane = lane_id();
  const int nr = W.nredo[table];
  if (nr == 0) return;
  const bool in = lane < nr;
  const int v = in ? W.redo[table][lane] : 0;
  const long long b = in ? ld_off(off + v, pol) : 0;
  const int deg = in ? (int)(ld_off(off + v + 1, pol) - b) : 0;
  k1_medium<false, kLower, true>(cols, cdst, cdst, v, b, deg, in, W, pol, L, gathers, nullptr,
                                 nullptr, StageInfo{false, 0});
  if (lane == 0) W.nredo[table] = 0;
  __syncwarp();
}

// ---------------------------------------------------------------------------
// long rows: producer side (warp that meets the row) and piece processing
// ---------------------------------------------------------------------------
__device__ __forceinline__ unsigned ld_acquire_u32(const unsigned* p) {
  unsigned r;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(r) : "l"(p) : "memory");
  return r;
}

__device__ __forceinline__ int atom_add_acq_rel(int* p, int v) {
  int r;
  asm volatile("atom.acq_rel.gpu.global.add.s32 %0, [%1], %2;" : "=r"(r) : "l"(p), "r"(v) : "memory");
  return r;
}

__device__ __forceinline__ void st_release_u32(unsigned* p, unsigned v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" :: "l"(p), "r"(v) : "memory");
}

// Publish the pieces of every long row of this sub-tile (warp-collective).
__device__ __noinline__ void k1_push_long(const SplitArgs& S, int v, int deg, bool islong) {
  const int lane = lane_id();
  unsigned rows = __ballot_sync(kFull, islong);
  while (rows) {
    const int r = __ffs(rows) - 1;
    rows &= rows - 1;
    const int vr = __shfl_sync(kFull, v, r);
    const int dr = __shfl_sync(kFull, deg, r);
    const int np = (dr + kPiece - 1) / kPiece;
    unsigned slot = 0, t = 0;
    if (lane == 0) {
      slot = atomicAdd(S.slot_ctr, 1u);
      S.slot_v[slot] = vr;
      S.slot_deg[slot] = dr;
      S.slot_left[slot] = np;
      t = atomicAdd(S.piece_ctr, (unsigned)np);
    }
    slot = __shfl_sync(kFull, slot, 0);
    t = __shfl_sync(kFull, t, 0);
    for (int i = lane; i < np; i += 32) S.q[t + i] = make_int2((int)slot, i * kPiece);
    __syncwarp();  // slot fields (lane 0) before every lane's release store
    for (int i = lane; i < np; i += 32) st_release_u32(S.q_seq + t + i, 1u);
  }
}

// Pop one piece from this CTA's mailbox (lane 0 decides, result broadcast).
// *exhausted is set when every allocated piece of the mailbox is taken.
__device__ bool k1_pop(const SplitArgs& S, int* s_mbhead, int& slot, int& start,
                       bool* exhausted) {
  int ok = 0, sl = 0, st = 0, ex = 1;
  if (S.min_deg == INT_MAX) {  // no long rows in this graph
    *exhausted = true;
    return false;
  }
  ex = 0;
  if (lane_id() == 0) {
    const unsigned alloc = *reinterpret_cast<volatile const unsigned*>(S.piece_ctr);
    for (;;) {
      const int j = *reinterpret_cast<volatile int*>(s_mbhead);
      const unsigned p = (unsigned)j * (unsigned)S.G + blockIdx.x;
      if (p >= alloc) {
        ex = 1;
        break;
      }
      if (atomicCAS(s_mbhead, j, j + 1) == j) {
        while (ld_acquire_u32(S.q_seq + p) == 0u) __nanosleep(32);
        const int2 e = S.q[p];
        sl = e.x;
        st = e.y;
        ok = 1;
        break;
      }
    }
  }
  ok = __shfl_sync(kFull, ok, 0);
  slot = __shfl_sync(kFull, sl, 0);
  start = __shfl_sync(kFull, st, 0);
  *exhausted = __shfl_sync(kFull, ex, 0) != 0;
  return ok != 0;
}

template <bool kSnap, bool kLower, bool kLog>
__device__ __noinline__ void k1_piece(const long long* __restrict__ off, const int* __restrict__ cols,
                         const int* csrc, int* cdst, const SplitArgs& S, int slot, int start,
                         K1Warp& W, uint64_t pol, const PairLog& L, unsigned& gathers) {
  constexpr int U = 8;
  const int lane = lane_id();
  const int v = S.slot_v[slot];
  const int deg = S.slot_deg[slot];
  const long long b = ld_off(off + v, pol);
  const int end = min(deg, start + kPiece);
  W.win[lane] = 0u;
  __syncwarp();
  unsigned long long reg = 0ull;
  // a piece that starts above v holds no lower neighbour (sorted row)
  const bool skip = kLower && ld_col(cols + b + start, pol) > v;
  if (!skip) {
    for (int i0 = start; i0 < end; i0 += 32 * U) {
      int w[U], c[U];
      bool take[U];
      bool past = false;
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int i = i0 + u * 32 + lane;
        const bool in = i < end;
        w[u] = in ? ld_col(cols + b + i, pol) : 0;
        take[u] = in && (!kLower || w[u] < v);
        past |= kLower && in && w[u] > v;
      }
#pragma unroll
      for (int u = 0; u < U; ++u) c[u] = take[u] ? read_color<kSnap>(csrc, w[u]) : -2;
#pragma unroll
      for (int u = 0; u < U; ++u) {
        gathers += take[u];
        if (c[u] >= 0 && c[u] <= deg) {
          if (c[u] < 64) reg |= 1ull << c[u];
          else if (c[u] < 1024) atomicOr(&W.win[c[u] >> 5], 1u << (c[u] & 31));
        }
        if (kLog) log_pairs(L, take[u] && c[u] == -1, w[u], v);
      }
      if (kLower && __any_sync(kFull, past)) break;
    }
  }
  const unsigned lo = __reduce_or_sync(kFull, (unsigned)reg);
  const unsigned hi = __reduce_or_sync(kFull, (unsigned)(reg >> 32));
  __syncwarp();
  unsigned word = W.win[lane];
  if (lane == 0) word |= lo;
  if (lane == 1) word |= hi;
  if (word) atomicOr(S.slot_bm + (size_t)slot * 32 + lane, word);
  __syncwarp();
  int last = 0;
  if (lane == 0) last = atom_add_acq_rel(S.slot_left + slot, -1) == 1;
  last = __shfl_sync(kFull, last, 0);
  if (last) {
    const unsigned wd = ld_acquire_u32(S.slot_bm + (size_t)slot * 32 + lane);
    const unsigned fr = ~wd;  // deg >= 1024: every bit of window 0 is a candidate
    const unsigned nz = __ballot_sync(kFull, fr != 0u);
    int color;
    if (nz) {
      const int j = __ffs(nz) - 1;
      color = j * 32 + __ffs(__shfl_sync(kFull, fr, j)) - 1;
    } else {  // 1024 distinct lower colours: scan the next windows
      color = -1;
      for (int wb = 1024; color < 0 && wb <= deg; wb += 1024)
        color = warp_ff_window<kSnap, kLower>(cols, csrc, v, b, deg, wb, W.win, pol);
    }
    if (lane == 0) st_color(cdst + v, color);
  }
  __syncwarp();
}

// ---------------------------------------------------------------------------
// K1 kernel
// ---------------------------------------------------------------------------
template <bool kSnap, bool kLower, bool kLog>
__global__ void __launch_bounds__(kK1Block) k1_light(const long long* __restrict__ off,
                                                     const int* __restrict__ cols, int n,
                                                     int nitems, const int* worklist,
                                                     const int* csrc, int* cdst, Ctrl* ctrl,
                                                     PairLogArgs LA, SplitArgs S) {
  extern __shared__ __align__(16) unsigned char k1_smem[];
  __shared__ unsigned long long s_claim;  // {chunk << 32 | next sub-tile}
  __shared__ int s_npairs, s_mbhead;
  __shared__ unsigned s_gathers;
  const int warp = threadIdx.x >> 5, lane = lane_id();
  K1Warp& W = reinterpret_cast<K1Warp*>(k1_smem)[warp];
  const uint64_t pol = policy_evict_first();
  const int nchunks = (nitems + kK1Block - 1) / kK1Block;
  if (threadIdx.x == 0) {
    const int c0 = (int)atomicAdd(&ctrl->tile_cursor, 1ull);
    s_claim = ((unsigned long long)(unsigned)c0 << 32);
    s_npairs = 0;
    s_gathers = 0;
    s_mbhead = 0;
  }
  W.dv[0][lane] = -1;
  W.dv[1][lane] = -1;
  W.cv[lane] = -1;
  if (lane < 2) W.nredo[lane] = 0;
  __syncthreads();
  PairLog L{LA.pairs + (size_t)blockIdx.x * LA.region_cap, LA.region_cap, &s_npairs, LA.overflow};
  unsigned gathers = 0;
  int it = 0;
  for (;; ++it) {
    int pslot, pstart;
    bool ex;
    while (k1_pop(S, &s_mbhead, pslot, pstart, &ex))  // long-row pieces first
      k1_piece<kSnap, kLower, kLog>(off, cols, csrc, cdst, S, pslot, pstart, W, pol, L, gathers);
    int sub = -1;
    if (lane == 0) {
      for (;;) {
        const unsigned long long x = atomicAdd(&s_claim, 1ull);
        const int k = (int)(x & 0xffffffffu);
        const int c = (int)(x >> 32);
        if (c >= nchunks) break;
        if (k < kSubTiles) {
          sub = c * kSubTiles + k;
          break;
        }
        if (k == kSubTiles) {  // first to overflow claims the next chunk for the CTA
          const int nc = (int)atomicAdd(&ctrl->tile_cursor, 1ull);
          atomicExch(&s_claim, ((unsigned long long)(unsigned)nc << 32) | 1ull);
          if (nc < nchunks) sub = nc * kSubTiles;
          break;
        }
        __nanosleep(20);
      }
    }
    sub = __shfl_sync(kFull, sub, 0);
    if (sub < 0) break;
    const int table = it & 1;
    const int item = sub * 32 + lane;
    const bool valid = item < nitems;
    const int v = valid ? (worklist ? worklist[item] : item) : n;
    const long long b = ld_off(off + v, pol);
    const long long e = valid ? ld_off(off + v + 1, pol) : b;
    const int deg = (int)(e - b);
    if (valid && deg == 0) st_color(cdst + v, 0);  // limit 0: only colour 0
    const bool small = valid && deg >= 1 && deg <= kSmallMax;
    const bool med = valid && deg > kSmallMax && deg < S.min_deg;
    k1_push_long(S, v, deg, valid && deg >= S.min_deg);
    const StageInfo si = k1_stage(cols, b, deg, W, pol);
    k1_small<kSnap, kLower, kLog>(cols, csrc, cdst, v, b, deg, small, W, table, pol, L, gathers,
                                  si);
    k1_medium<kSnap, kLower, kLog>(cols, csrc, cdst, v, b, deg, med, W, pol, L, gathers,
                                   kLog ? W.redo[table] : nullptr, &W.nredo[table], si);
    if (kLog && it > 0) {  // rows parked one sub-tile ago
      k1_drain(W, table ^ 1, cdst, L);
      k1_redo<kLower>(off, cols, cdst, W, table ^ 1, pol, L, gathers);
    }
  }
  if (kLog && it > 0) {
    k1_drain(W, (it - 1) & 1, cdst, L);
    k1_redo<kLower>(off, cols, cdst, W, (it - 1) & 1, pol, L, gathers);
    k1_drain(W, it & 1, cdst, L);  // table it&1 is empty: this flushes the carry slots
  }
  // This warp publishes nothing more; keep serving the CTA's mailbox until
  // every warp is done publishing and the mailbox is empty.
  if (lane == 0) atomicSub(S.alive, 1);
  for (; S.min_deg != INT_MAX;) {
    int pslot, pstart;
    bool ex;
    if (k1_pop(S, &s_mbhead, pslot, pstart, &ex)) {
      k1_piece<kSnap, kLower, kLog>(off, cols, csrc, cdst, S, pslot, pstart, W, pol, L, gathers);
      continue;
    }
    int done = 0;
    if (lane == 0) done = ex && ld_acquire_u32(reinterpret_cast<const unsigned*>(S.alive)) == 0u;
    if (__shfl_sync(kFull, done, 0)) {
      // alive == 0 was read after the mailbox looked exhausted; re-check once
      // against the now-final allocation count
      if (!k1_pop(S, &s_mbhead, pslot, pstart, &ex)) break;
      k1_piece<kSnap, kLower, kLog>(off, cols, csrc, cdst, S, pslot, pstart, W, pol, L, gathers);
      continue;
    }
    __nanosleep(200);
  }
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

}  // namespace dev
}  // namespace gcol
