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
#include <type_traits>

#include "gcol_device.cuh"

namespace gcol {
namespace dev {

constexpr int kCW = 8;                    // consumer warps per CTA (narrow variant)
constexpr int kCWWide = 16;               // consumer warps per CTA (wide variant)
// producer warps (TMA bulk copies)
template <int CW>
constexpr int k1_producers() {
  return 1;
}
constexpr int kChunk = kCW * 32;          // vertices per chunk (narrow); ranges align to it
constexpr int kSlotsMax = 5;              // staged chunks in flight per CTA (multiple of producers)
// narrow K1 has the shared memory for a fifth slot (~217 of 227 KB), wide not;
// measured (A/B on one box): five make R-MAT 27 6 % slower, R-MAT 24 0.6 % faster
#ifndef GCOL_K1_SLOTS
#define GCOL_K1_SLOTS 4
#endif
template <int CW>
constexpr int k1_slots() {
  return CW <= 8 ? GCOL_K1_SLOTS : 4;
}
constexpr int kSlotStage = 6144;          // adjacency entries staged per chunk (24 KB)
constexpr int kBmWords = 512;             // per-warp medium-row bitmap pool
constexpr int kStaleMax = 4;              // stale neighbours remembered per parked row
constexpr int kSplitDefault = 1024;       // rows >= this are split into pieces
constexpr int kPiece = 1024;              // entries per piece
constexpr int kDriftDefault = 2;          // max rounds a CTA may run ahead

// Per consumer warp: forbidden-colour scratch and the deferral state.
struct K1Warp {
  unsigned bm[kBmWords];               // medium-row bitmaps
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

// Staged adjacency entries per slot: 32 KB (narrow) / 24 KB (wide, whose
// per-warp scratch takes the rest of the 227 KB).
template <int CW>
constexpr int stage_cap() {
  return CW <= kCW ? 8192 : kSlotStage;
}

// One staged chunk: its rows and their adjacency, packed.  The adjacency of
// the chunk's rows is contiguous in `cols` except where a long row (served
// by pieces from global memory) sits in between, so the producer stages the
// runs between long rows back to back (each run 16-byte aligned for TMA)
// and records per row where its entries landed.
template <int CW>
struct alignas(16) K1Slot {
  alignas(16) long long offs[CW * 32 + 2];  // contiguous mode: off[c0 .. c0 + rows]; worklist: b[]
  int wv[CW * 32];                     // worklist mode: vertex ids
  int aux[CW * 32];                    // worklist: degrees; contiguous: stage offset (-1: global)
  unsigned lm[CW];                     // producer scratch: long-row bitmap
  long long wbase;                     // window mode (wlen >= 0): stage = cols[wbase, +wlen)
  int wlen;
  alignas(16) int stage[stage_cap<CW>()];
  int chunk;                           // chunk index, -1: no more chunks
  int rows;
  unsigned long long full;             // mbarrier: slot staged (TMA tx + producer arrive)
  unsigned long long offb;             // mbarrier: offsets staged (producer only)
};

template <int CW>
struct alignas(16) K1Smem {
  K1Slot<CW> slot[k1_slots<CW>()];
  K1Warp cw[CW];
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
  int* alive;           // consumer warps that may still publish pieces
  int G;                // mailboxes (= K1 grid)
  unsigned* done_chunks;  // chunks fully consumed (drift bound)
  const unsigned* piece_ready;  // streamed upload: flag per 2^piece_shift adjacency entries
  int piece_shift;              //   resident (null: the whole CSR is resident)
  int dyn_tiles;        // 1: consumer warps take sub-tiles from a CTA counter
  int cstride, coffset; // this launch owns the chunks coffset + cstride * i (interleaved
                        // multi-GPU partition; 1, 0: all)
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
// small rows: thread per row over the staged adjacency, 64-bit register mask
// ---------------------------------------------------------------------------
template <bool kSnap, bool kLower, bool kLog, class PL>
__device__ __forceinline__ void k1_small(const int* __restrict__ cols, const int* csrc,
                                         int* cdst, int v, long long b, int deg, bool small,
                                         K1Warp& W, int table, uint64_t pol, const PL& L,
                                         unsigned& gathers, const int* rs) {
  // rs: the row's entries in shared memory, nullptr when not staged
  const int lane = lane_id();
  const bool inwin = rs != nullptr;
  const int maxk = __reduce_max_sync(kFull, (unsigned)(small ? deg : 0));
  bool active = small;
  int ns = 0;
  unsigned long long mask = 0ull;
  for (int k = 0; k < maxk; k += 4) {
    int w[4];
    bool take[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const bool in = active && (k + u) < deg;
      w[u] = in ? (inwin ? rs[k + u] : ld_col(cols + b + k + u, pol)) : 0;
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
  if (small) {
    if (kLog && ns > 0) {  // park; committed after the re-check one chunk later
      W.dv[table][lane] = v;
      W.dmask[table][lane][0] = (unsigned)mask;
      W.dmask[table][lane][1] = (unsigned)(mask >> 32);
      W.ddeg[table][lane] = (unsigned char)deg;
      W.dns[table][lane] = (unsigned char)min(ns, kStaleMax);
    } else {
      commit_color(cdst, v, __ffsll((long long)~mask) - 1);
    }
  }
  __syncwarp();
}

// Re-check the rows parked in `table` (warp-collective).  A row whose
// in-flight neighbours have all committed is committed now; otherwise it
// gets one more sub-tile in the lane's carry slot, and whatever is still
// uncoloured at that second check is logged for round 1.
template <class PL>
__device__ __forceinline__ void k1_drain(K1Warp& W, int table, int* cdst, const PL& L) {
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
      commit_color(cdst, v, __ffsll((long long)~mask) - 1);
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
      commit_color(cdst, v, __ffsll((long long)~mask) - 1);
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
template <bool kSnap, bool kLower, bool kLog, class PL>
__device__ __forceinline__ void k1_medium(const int* __restrict__ cols, const int* csrc,
                                          int* cdst, int v, long long b, int deg, bool med,
                                          K1Warp& W, uint64_t pol, const PL& L,
                                          unsigned& gathers, int* redo, int* nredo,
                                          const int* stage, int so) {
  // so: offset of the row's entries in `stage`, -1 when not staged
  const int lane = lane_id();
  const bool park_mode = kLog && redo != nullptr;
  // entries to visit: in a sorted staged row, only the lower-id prefix
  // (binary search in shared memory); elsewhere the whole row
  int lcnt = deg;
  if (kLower && med && so >= 0) {
    int lo = 0, hi = deg;
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if (stage[so + mid] < v) lo = mid + 1;
      else hi = mid;
    }
    lcnt = lo;
  }
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
    const int len = inb ? lcnt : 0;
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
        const int sr = __shfl_sync(kFull, so, lo);
        vr[u] = __shfl_sync(kFull, v, lo);
        dr[u] = __shfl_sync(kFull, deg, lo);
        w[u] = !in ? 0 : (sr >= 0 ? stage[sr + (idx - er)] : ld_col(cols + br + (idx - er), pol));
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
    if (inb && !park) commit_color(cdst, v, color);
    __syncwarp();
  }
}

// ---------------------------------------------------------------------------
// long rows: producer side (warp that meets the row) and piece processing
// ---------------------------------------------------------------------------
__device__ __forceinline__ unsigned ld_acquire_u32(const unsigned* p) {
  unsigned r;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(r) : "l"(p) : "memory");
  return r;
}

__device__ __forceinline__ unsigned long long ld_acquire_u64(const unsigned long long* p) {
  unsigned long long r;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(r) : "l"(p) : "memory");
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
__device__ __forceinline__ void k1_push_long(const SplitArgs& S, int v, int deg, bool islong) {
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

// win: 32 shared-memory words owned by the warp.  kPend: the colour value
// of a lower neighbour that is still in flight (-1 in K1; -2, "pending
// heavy row", in the class-split heavy pass, where -1 is a light row that
// has not started and reads this row itself later).
template <bool kSnap, bool kLower, bool kLog, class PL, int kPend = -1>
__device__ __forceinline__ void k1_piece(const long long* __restrict__ off, const int* __restrict__ cols,
                         const int* csrc, int* cdst, const SplitArgs& S, int slot, int start,
                         unsigned* win, uint64_t pol, const PL& L, unsigned& gathers) {
  constexpr int U = 8;
  const int lane = lane_id();
  const int v = S.slot_v[slot];
  const int deg = S.slot_deg[slot];
  const long long b = ld_off(off + v, pol);
  const int end = min(deg, start + kPiece);
  win[lane] = 0u;
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
          else if (c[u] < 1024) atomicOr(&win[c[u] >> 5], 1u << (c[u] & 31));
        }
        if (kLog) log_pairs(L, take[u] && c[u] == kPend, w[u], v);
      }
      if (kLower && __any_sync(kFull, past)) break;
    }
  }
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
        color = warp_ff_window<kSnap, kLower>(cols, csrc, v, b, deg, wb, win, pol);
    }
    if (lane == 0) commit_color(cdst, v, color);
  }
  __syncwarp();
}

__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void mbar_arrive_expect_tx(unsigned long long* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}

__device__ __forceinline__ bool mbar_try_wait(unsigned long long* bar, unsigned parity) {
  unsigned ok;
  asm volatile(
      "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
      " selp.u32 %0, 1, 0, p;\n}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}

__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned parity) {
  while (!mbar_try_wait(bar, parity)) {
  }
}

// Raise the barrier's expected transaction bytes without arriving.
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* bar, unsigned bytes) {
  asm volatile("mbarrier.expect_tx.relaxed.cta.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void mbar_arrive(unsigned long long* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

// 1-D TMA bulk copy global -> shared with an L2 cache policy (streamed CSR:
// evict_first, so the colour array stays L2-resident).
__device__ __forceinline__ void tma_load_1d_hint(void* dst, const void* src, unsigned bytes,
                                                 unsigned long long* bar, uint64_t pol) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1], %2, [%3], %4;" ::"r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(pol)
      : "memory");
}

// 1-D TMA bulk copy global -> shared, completion counted on `bar`.
__device__ __forceinline__ void tma_load_1d(void* dst, const void* src, unsigned bytes,
                                            unsigned long long* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
          "r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

// Request the offsets of chunk c (contiguous mode, one thread) into `sl`.
template <int CW>
__device__ __forceinline__ void k1_request_offsets(K1Slot<CW>& sl, const long long* off, int c,
                                                   int nitems, int item0, int n, uint64_t pol) {
  constexpr int kChunk = CW * 32;
  const int c0 = c * kChunk;
  if (c0 >= nitems) return;
  const int rows = min(kChunk, nitems - c0);
  const int cnt = rows + 1;           // off[item0 + c0 .. + rows]
  // whole 16-byte pairs (item0 is even); an odd count reads one offset more
  // unless that would pass off[n], where the last one is loaded here
  const bool pad = (cnt & 1) && item0 + c0 + cnt + 1 <= n + 1;
  const int bulk = pad ? cnt + 1 : (cnt & ~1);
  if (bulk < cnt) sl.offs[cnt - 1] = ld_off(off + item0 + c0 + cnt - 1, pol);
  mbar_arrive_expect_tx(&sl.offb, (unsigned)(bulk * 8));
  tma_load_1d(sl.offs, off + item0 + c0, (unsigned)(bulk * 8), &sl.offb);
}

// Stage the adjacency of one contiguous chunk (producer warp, all lanes;
// sl.offs must hold off[c0 .. c0 + rows]).  Run j (lane j) is the span of
// rows between the (j-1)-th and j-th long row; runs are packed back to back
// from stage[0], each starting at a 16-byte aligned source so one TMA bulk
// copy moves it (+ <= 3 scalar tail entries), as far as the capacity goes.
// Every row gets aux[i] = its first entry's stage offset, or -1.  Each
// copying lane registers its bytes on `full` (expect_tx) before issuing, so
// the copies overlap the aux[] computation; the caller's single arrive
// (after a __syncwarp) then publishes aux[] and the tails.
template <int CW>
__device__ __forceinline__ void stage_chunk(K1Slot<CW>& sl, int rows, int min_deg,
                                            const int* __restrict__ cols, long long m,
                                            uint64_t pol) {
  // Loops are kept rolled (long-row bitmap in shared memory): this runs once
  // per chunk on one warp, and unrolled it would crowd the instruction cache.
  constexpr int R = CW;                  // rows per lane (kChunk / 32)
  constexpr int CAP = stage_cap<CW>();
  const int lane = lane_id();
  int nl = 0;
#pragma unroll 1
  for (int t = 0; t < R; ++t) {          // lm[t]: long rows among rows t*32 ..
    const int i = t * 32 + lane;
    const bool lg = min_deg != INT_MAX && i < rows && sl.offs[i + 1] - sl.offs[i] >= min_deg;
    const unsigned w = __ballot_sync(kFull, lg);
    if (lane == 0) sl.lm[t] = w;
    nl += __popc(w);
  }
  __syncwarp();
  // run j = rows [s_j, e_j): after the (j-1)-th long row, up to the j-th
  // (the last run, j == min(nl, 31), extends to `rows`)
  const int nr = min(nl, 31) + 1;
  auto nth_long = [&](int q) {           // row index of the q-th long row
#pragma unroll 1
    for (int t = 0; t < R; ++t) {
      const unsigned w = sl.lm[t];
      const int p = __popc(w);
      if (q < p) return t * 32 + (int)__fns(w, 0, q + 1);
      q -= p;
    }
    return rows;
  };
  int s = 0, e = 0;
  if (lane < nr) {
    s = lane == 0 ? 0 : nth_long(lane - 1) + 1;
    e = lane == nr - 1 ? rows : nth_long(lane);
  }
  long long A = 0, span = 0;
  int sz = 0;
  if (lane < nr && s < e) {
    const long long bs = sl.offs[s], be = sl.offs[e];
    A = bs & ~3LL;
    span = be - A;
    sz = (int)min((span + 3) & ~3LL, (long long)CAP + 4);
  }
  int incl = sz;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const int y = __shfl_up_sync(kFull, incl, d);
    if (lane >= d) incl += y;            // <= 32 * (CAP + 4): no overflow
  }
  const int dst = incl - sz;
  const int room = max(0, min(CAP - dst, sz));     // multiple of 4
  const int avail = (int)min((long long)room, span);
  // the copy rounds up to whole 16-byte units (entries past the run are
  // harmless) except at the very end of `cols`, where <= 3 are loaded here
  const int bulk = A + room <= m ? room : (avail & ~3);
  if (bulk) {
    mbar_expect_tx(&sl.full, (unsigned)bulk * 4u);
    tma_load_1d_hint(sl.stage + dst, cols + A, (unsigned)bulk * 4u, &sl.full, pol);
  }
  for (int j = bulk; j < avail; ++j) sl.stage[dst + j] = ld_col(cols + A + j, pol);
  // per-row stage offsets: row i lies in run (long rows before i), capped at 31
  int before = 0;                        // long rows before word t
#pragma unroll 1
  for (int t = 0; t < R; ++t) {
    const unsigned w = sl.lm[t];
    const int i = t * 32 + lane;
    const int run = min(before + __popc(w & ((1u << lane) - 1u)), 31);
    const long long Ar = __shfl_sync(kFull, A, run);
    const int dr = __shfl_sync(kFull, dst, run);
    const int rr = __shfl_sync(kFull, avail, run);
    if (i < rows) {
      const long long b = sl.offs[i], bend = sl.offs[i + 1];
      const bool staged = !((w >> lane) & 1u) && bend - Ar <= rr;
      sl.aux[i] = staged ? dr + (int)(b - Ar) : -1;
    }
    before += __popc(w);
  }
}

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(
                   static_cast<unsigned>(__cvta_generic_to_shared(smem))),
               "l"(gmem)
               : "memory");
}

__device__ __forceinline__ void cp_async4(void* smem, const void* gmem) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(
                   static_cast<unsigned>(__cvta_generic_to_shared(smem))),
               "l"(gmem)
               : "memory");
}

__device__ __forceinline__ void cp_async_wait_all() {
  asm volatile("cp.async.wait_all;" ::: "memory");
}

// ---------------------------------------------------------------------------
// K1 kernel.  One CTA per SM: a producer warp stages chunks (256 rows:
// offsets + a window of their adjacency) into a ring of shared-memory slots
// with cp.async, up to k1_slots<CW>() chunks ahead; eight consumer warps colour them.
// Chunks are assigned round-robin (chunk c -> CTA c % G), so the producer
// can prefetch without claiming anything: the vertices in flight are only
// those being coloured (about G x 256), which is what governs the stale
// reads and hence the colour count.  A CTA may not run more than `drift`
// rounds ahead of the slowest one.
// ---------------------------------------------------------------------------
template <bool kSnap, bool kLower, bool kLog, int CW>
__global__ void __launch_bounds__((CW + k1_producers<CW>()) * 32, 1) k1_pipe(const long long* __restrict__ off,
                                                      const int* __restrict__ cols, int n,
                                                      int nitems, const int* worklist,
                                                      const int* csrc, int* cdst, Ctrl* ctrl,
                                                      PairLogArgs LA, SplitArgs S, int drift,
                                                      int item0) {
  extern __shared__ __align__(16) unsigned char k1_raw[];
  constexpr int kCW = CW;
  constexpr int kChunk = CW * 32;
  K1Smem<CW>& sm = *reinterpret_cast<K1Smem<CW>*>(k1_raw);
  __shared__ int s_ready[kSlotsMax];
  __shared__ int s_consumed[kSlotsMax];
  __shared__ int s_npairs, s_mbhead, s_next;
  __shared__ unsigned s_gathers;
  const int warp = threadIdx.x >> 5, lane = lane_id();
  const uint64_t pol = policy_evict_first();
  const int G = gridDim.x;
  const int nchunks_all = (nitems + kChunk - 1) / kChunk;
  // chunks of this launch: global chunk coffset + cstride * local index
  const int nchunks = nchunks_all > S.coffset ? (nchunks_all - S.coffset + S.cstride - 1) / S.cstride : 0;
  if (threadIdx.x < k1_slots<CW>()) {
    s_ready[threadIdx.x] = -1;
    s_consumed[threadIdx.x] = 0;
    mbar_init(&sm.slot[threadIdx.x].full, 1);
    mbar_init(&sm.slot[threadIdx.x].offb, 1);
  }
  if (threadIdx.x == 0) asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  if (threadIdx.x == 0) {
    s_npairs = 0;
    s_gathers = 0;
    s_mbhead = 0;
    s_next = 0;
  }
  init_peers(ctrl);
  if (warp < kCW) {
    K1Warp& W = sm.cw[warp];
    W.dv[0][lane] = -1;
    W.dv[1][lane] = -1;
    W.cv[lane] = -1;
    if (lane < 2) W.nredo[lane] = 0;
  }
  __syncthreads();

  if (warp >= kCW) {
    // ------------------------------ producer ------------------------------
    // Lane 0 drives TMA: per chunk one bulk copy of its offsets (waited for
    // here) and one of its adjacency window (waited for by the consumers on
    // the slot's `full` barrier).  Offsets of chunk k+1 are requested before
    // the adjacency of chunk k is published, so both stay in flight.
    long long pt_slot = 0, pt_drift = 0, pt_load = 0, pchunks = 0;
    const bool contig = worklist == nullptr;
    const long long m = ld_off(off + n, pol);  // adjacency length
    // offsets of the first chunk; each later chunk's go out one chunk ahead,
    // as soon as its slot is free
    if (lane == 0 && contig)
      k1_request_offsets<CW>(sm.slot[0], off, blockIdx.x * S.cstride + S.coffset, nitems, item0,
                             n, pol);
    for (int k = 0;; ++k) {
      const int cl = blockIdx.x + k * G;                // local chunk index
      const int c = cl * S.cstride + S.coffset;         // global chunk index
      const int si = k % k1_slots<CW>();
      K1Slot<CW>& sl = sm.slot[si];
      const unsigned par = (unsigned)((k / k1_slots<CW>()) & 1);
      long long t0 = clock64();
      if (cl >= nchunks) {
        if (lane == 0) {
          if (k >= k1_slots<CW>())
            while (*reinterpret_cast<volatile int*>(&s_consumed[si]) < kCW * (k / k1_slots<CW>()))
              __nanosleep(64);
          sl.chunk = -1;
          mbar_arrive_expect_tx(&sl.full, 0u);
        }
        break;
      }
      if (drift > 0 && k > drift && lane == 0)
        while (ld_acquire_u32(S.done_chunks) < (unsigned)((k - drift) * G)) __nanosleep(128);
      long long t1 = clock64();
      pt_drift += t1 - t0;
      const int c0 = c * kChunk;
      const int rows = min(kChunk, nitems - c0);
      if (contig) {
        mbar_wait(&sl.offb, par);              // offsets of chunk k (every lane)
        if (lane == 0) {  // chunk k+1's offsets go out as soon as its slot is free
          const int kn = k + 1;
          if (kn >= k1_slots<CW>())
            while (*reinterpret_cast<volatile int*>(&s_consumed[kn % k1_slots<CW>()]) < kCW * (kn / k1_slots<CW>()))
              __nanosleep(64);
          k1_request_offsets<CW>(sm.slot[kn % k1_slots<CW>()], off,
                                 (blockIdx.x + kn * G) * S.cstride + S.coffset, nitems, item0, n,
                                 pol);
        }
        if (S.piece_ready) {  // streamed upload: the chunk's adjacency must be resident
          const long long lo = sl.offs[0], hi = sl.offs[rows];
          if (lane == 0 && hi > lo)
            for (long long p = lo >> S.piece_shift; p <= (hi - 1) >> S.piece_shift; ++p)
              while (ld_acquire_u32(S.piece_ready + p) == 0u) __nanosleep(256);
          __syncwarp();
        }
        if (S.min_deg == INT_MAX) {
          // no long rows in the graph: the chunk's adjacency is one run, staged
          // as one window [wbase, wbase + wlen); rows inside it read shared memory
          if (lane == 0) {
            constexpr int CAP = stage_cap<CW>();
            const long long A = sl.offs[0] & ~3LL;
            const int len = (int)min(sl.offs[rows] - A, (long long)CAP);
            const int bulk = A + ((len + 3) & ~3) <= m ? ((len + 3) & ~3) : (len & ~3);
            for (int x = bulk; x < len; ++x) sl.stage[x] = ld_col(cols + A + x, pol);
            sl.wbase = A;
            sl.wlen = len;
            sl.rows = rows;
            sl.chunk = c;
            mbar_arrive_expect_tx(&sl.full, (unsigned)bulk * 4u);
            if (bulk) tma_load_1d_hint(sl.stage, cols + A, (unsigned)bulk * 4u, &sl.full, pol);
          }
        } else {
          stage_chunk<CW>(sl, rows, S.min_deg, cols, m, pol);
          if (lane == 0) {
            sl.wlen = -1;  // per-row offsets in aux[]
            sl.rows = rows;
            sl.chunk = c;
          }
          __syncwarp();  // every lane's expect_tx, tails and aux[] before the arrive
          if (lane == 0) mbar_arrive(&sl.full);
        }
      } else {  // worklist mode: per-row loads, nothing staged
        if (k >= k1_slots<CW>())
          while (*reinterpret_cast<volatile int*>(&s_consumed[si]) < kCW * (k / k1_slots<CW>()))
            __nanosleep(64);
        for (int i = lane; i < kChunk; i += 32) {
          const bool valid = i < rows;
          const int v = valid ? worklist[c0 + i] : -1;
          const long long bb = valid ? ld_off(off + v, pol) : 0;
          sl.wv[i] = v;
          sl.offs[i] = bb;
          sl.aux[i] = valid ? (int)(ld_off(off + v + 1, pol) - bb) : 0;
        }
        __syncwarp();
        if (lane == 0) {
          sl.rows = rows;
          sl.chunk = c;
          mbar_arrive_expect_tx(&sl.full, 0u);
        }
      }
      __syncwarp();
      pt_load += clock64() - t1;
      ++pchunks;
    }
    if (lane == 0) {
      atomicAdd(&ctrl->prof[8], (unsigned long long)pt_slot);
      atomicAdd(&ctrl->prof[9], (unsigned long long)pt_drift);
      atomicAdd(&ctrl->prof[10], (unsigned long long)pt_load);
      atomicAdd(&ctrl->prof[11], (unsigned long long)pchunks);
    }
    return;
  }

  // ------------------------------- consumers ---------------------------------
  K1Warp& W = sm.cw[warp];
  // the wide variant inlines the rare log append (register budget), the
  // narrow one keeps it out of line (instruction-cache footprint)
  using PL = typename std::conditional<(CW > dev::kCW), PairLogInl, PairLog>::type;
  PL L;
  L.region = LA.pairs + (size_t)blockIdx.x * LA.region_cap;
  L.cap = LA.region_cap;
  L.s_count = &s_npairs;
  L.overflow = LA.overflow;
  unsigned gathers = 0;
  bool finished = false;  // no more chunks for this warp
  bool retired = false;   // decremented S.alive
  long long ct_wait = 0, ct_piece = 0, ct_small = 0, ct_med = 0, ct_drain = 0, cchunks = 0;
  long long ct_redo = 0, n_med = 0, n_redo = 0;
  long long tw = clock64();
  // Sub-tile t is rows [32 (t mod CW), +32) of chunk k = t / CW.  Statically,
  // warp w takes t = w, w + CW, ...; with dyn_tiles (skewed degrees, where
  // sub-tile costs vary widely) warps take them in ascending order from a CTA
  // counter, so a slow sub-tile holds up only itself and the warps' current
  // rows always lie within two consecutive chunks.
  int t = -1;    // sub-tile taken and not finished (-1: none)
  int cnt = 0;   // sub-tiles finished by this warp: parity picks the park tables
  int k = 0, si = 0;
  for (;;) {
    // long-row pieces first (one call site)
    {
      int pslot = 0, pstart = 0;
      bool ex;
      bool got = k1_pop(S, &s_mbhead, pslot, pstart, &ex);
      if (!got && retired) {
        int stop = 1;
        if (S.min_deg != INT_MAX && lane == 0)
          stop = ex && ld_acquire_u32(reinterpret_cast<const unsigned*>(S.alive)) == 0u;
        if (!__shfl_sync(kFull, stop, 0)) {
          __nanosleep(200);
          continue;
        }
        if (S.min_deg == INT_MAX) break;
        // alive hit 0 after the mailbox looked empty: one last look
        got = k1_pop(S, &s_mbhead, pslot, pstart, &ex);
        if (!got) break;
      }
      if (got) {
        const long long tp = clock64();
        k1_piece<kSnap, kLower, kLog>(off, cols, csrc, cdst, S, pslot, pstart, W.win, pol, L,
                                      gathers);
        ct_piece += clock64() - tp;
        continue;
      }
    }
    int j = 0;
    if (!finished) {
      if (t < 0) {
        if (S.dyn_tiles) {
          if (lane == 0) t = atomicAdd(&s_next, 1);
          t = __shfl_sync(kFull, t, 0);
        } else {
          t = cnt * kCW + warp;
        }
      }
      k = t / kCW;
      j = t - k * kCW;
      si = k % k1_slots<CW>();
      int ok = 0;
      if (lane == 0) ok = mbar_try_wait(&sm.slot[si].full, (unsigned)((k / k1_slots<CW>()) & 1));
      if (!__shfl_sync(kFull, ok, 0)) {
        __nanosleep(32);
        continue;
      }
      if (sm.slot[si].chunk < 0) finished = true;
    }
    long long ta = clock64();
    ct_wait += ta - tw;
    const K1Slot<CW>& sl = sm.slot[si];
    const int i = j * 32 + lane;
    const bool valid = !finished && i < sl.rows;
    int v = -1, deg = 0;
    long long b = 0;
    if (valid) {
      if (worklist) {
        v = sl.wv[i];
        b = sl.offs[i];
        deg = sl.aux[i];
      } else {
        v = item0 + sl.chunk * kChunk + i;
        b = sl.offs[i];
        deg = (int)(sl.offs[i + 1] - b);
      }
    }
    int so = -1;  // stage offset of the row's entries, -1: global memory
    if (valid && !worklist) {
      if (sl.wlen >= 0) so = b >= sl.wbase && b + deg <= sl.wbase + sl.wlen ? (int)(b - sl.wbase) : -1;
      else so = sl.aux[i];
    }
    const int table = cnt & 1;
    if (valid && deg == 0) commit_color(cdst, v, 0);  // limit 0: only colour 0
    k1_push_long(S, v, deg, valid && deg >= S.min_deg);
    k1_small<kSnap, kLower, kLog>(cols, csrc, cdst, v, b, deg,
                                  valid && deg >= 1 && deg <= kSmallMax, W, table, pol, L,
                                  gathers, so >= 0 ? sl.stage + so : nullptr);
    long long tb = clock64();
    ct_small += tb - ta;
    // medium rows of this chunk (park mode), then the rows parked one chunk ago
    const bool any_med = __any_sync(kFull, valid && deg > kSmallMax && deg < S.min_deg) ||
                         (kLog && W.nredo[table ^ 1] > 0);
    for (int pass = 0; any_med && pass < (kLog ? 2 : 1); ++pass) {
      const long long tpass = clock64();
      int pv = v, pdeg = deg;
      long long pb = b;
      bool pm = valid && deg > kSmallMax && deg < S.min_deg;
      int pso = so;
      if (pass == 1) {
        const int nr = W.nredo[table ^ 1];
        pm = lane < nr;
        pv = pm ? W.redo[table ^ 1][lane] : 0;
        pb = pm ? ld_off(off + pv, pol) : 0;
        pdeg = pm ? (int)(ld_off(off + pv + 1, pol) - pb) : 0;
        pso = -1;
        if (__ballot_sync(kFull, pm) == 0u) break;
        n_redo += nr;
      } else {
        n_med += __popc(__ballot_sync(kFull, pm));
      }
      k1_medium<kSnap, kLower, kLog>(cols, csrc, cdst, pv, pb, pdeg, pm, W, pol, L, gathers,
                                     (kLog && pass == 0) ? W.redo[table] : nullptr,
                                     &W.nredo[table], sl.stage, pso);
      if (pass == 1 && lane == 0) W.nredo[table ^ 1] = 0;
      __syncwarp();
      if (pass == 1) ct_redo += clock64() - tpass;
    }
    long long tc = clock64();
    ct_med += tc - tb;
    if (kLog)  // small rows parked one chunk ago (twice on exit: flushes the carry)
      for (int rep = 0; rep < (finished ? 2 : 1); ++rep)
        k1_drain(W, rep == 0 ? table ^ 1 : table, cdst, L);
    tw = clock64();
    ct_drain += tw - tc;
    ++cchunks;
    if (!finished) {
      __syncwarp();
      if (lane == 0) {
        const int old = atomicAdd(&s_consumed[si], 1);
        if (old % kCW == kCW - 1 && S.done_chunks) atomicAdd(S.done_chunks, 1u);
      }
      t = -1;
      ++cnt;
    } else {
      retired = true;
      if (lane == 0 && S.min_deg != INT_MAX) atomicSub(S.alive, 1);
    }
  }
  if (lane == 0) {
    atomicAdd(&ctrl->prof[0], (unsigned long long)ct_wait);
    atomicAdd(&ctrl->prof[1], (unsigned long long)ct_piece);
    atomicAdd(&ctrl->prof[2], (unsigned long long)ct_small);
    atomicAdd(&ctrl->prof[3], (unsigned long long)ct_med);
    atomicAdd(&ctrl->prof[4], (unsigned long long)ct_drain);
    atomicAdd(&ctrl->prof[5], (unsigned long long)cchunks);
    atomicAdd(&ctrl->prof[6], (unsigned long long)ct_redo);
    atomicAdd(&ctrl->prof[7], (unsigned long long)n_med);
    atomicAdd(&ctrl->prof[12], (unsigned long long)n_redo);
  }
  peers_fence();
  const unsigned g = __reduce_add_sync(kFull, gathers);
  if (lane == 0 && g) atomicAdd(&s_gathers, g);
  // the producer warps have returned: count only consumer warps from here on
  asm volatile("bar.sync 1, %0;" ::"n"(CW * 32));
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
