// libagatha — B200-native (sm_100a) guided extension alignment behind the C ABI of
// include/agatha.h.
//
// The path:
//   a1 pack      ASCII -> 4-bit codes (§2.2 l.279-285), R forward, Q reversed
//   a2 plan      nominal in-band cells per pair, longest-first order (cf. §4.4 l.532-555)
//   a3 init      boundary row/column values (reading R2)
//   a4 sweep     Eq. 1-3 (l.207-221) over anti-diagonals (l.229), k-band (l.248-250)
//   a5 localmax  Eq. 5 (l.264) per anti-diagonal, ties -> smallest i
//   a6 zdrop     Eq. 4 & 6 (l.258-266), checked every anti-diagonal, early exit
//   a7 dispatch  persistent warps pulling pairs from a global queue in plan order
//   a8 result    24-byte record per pair
//
// Kernel design: one warp per pair.  The band's D = bl+br+1
// diagonals are split into 32 lanes x K consecutive diagonals ("slots"); a slot keeps
// the H / H-alpha / E / F of its diagonal in registers and walks along it, so the whole
// band front is register-resident.  Anti-diagonal c updates the slots whose diagonal
// has the parity of c (cells of one anti-diagonal are independent);
// the only cross-lane dependency per step is one neighbour slot, exchanged with two
// shuffles.  The local max of every anti-diagonal is one warp REDUX of a packed
// (score, rank) key; the Z-drop test consumes it one step later so the reduction
// latency hides behind the next anti-diagonal's cells.
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>
#include <atomic>
#include <climits>
#include <cmath>

#include <cub/device/device_radix_sort.cuh>

#include "agatha.h"

namespace {

constexpr int kNegE = -(1 << 22);       // "-infinity" for E/F (and H-alpha) outside the band
constexpr int kHLimit = 1 << 20;        // every computed in-band H satisfies |H| < kHLimit
constexpr int kCapStep = 1 << 21;       // per-slot step of the padding cap (see cap_top)
constexpr int kPadH = -(1 << 21);       // initial H of a padding slot
constexpr int kNegKey = -(1 << 30);     // key of a cell outside the table
constexpr int kEmptyH = -kHLimit;       // lane max H at or below this: no cell on the diagonal
constexpr unsigned kFull = 0xffffffffu;
constexpr int kMaxSlots = 1024;         // one warp: 32 lanes x 32 slots (the 16-bit kernel)
constexpr int kMaxWarpsWide = 4;        // wide-band tier: up to 4 warps per pair (NEXT #3)
constexpr int kMaxSlotsWide = kMaxWarpsWide * kMaxSlots;
constexpr int kMaxChunks = 255;         // input chunks of one call (chunk ids are uint8)
constexpr uint64_t kChunkBytes = 48ull << 20;  // target ASCII bytes per streamed chunk
constexpr int kRampChunks = 5;                  // the first chunks start at 1/32 of it
#ifndef AGATHA_CHUNK_RAMP
#define AGATHA_CHUNK_RAMP 1
#endif

// A federated batch (NEXT #1, agatha_align_federated): the global batch is the
// concatenation of up to kMaxOwners owners' device batches, each possibly in another
// GPU's or process's memory (peer-mapped); global pair g lies in owner o with
// start[o] <= g < start[o + 1], at local index g - start[o].  n_owners == 0: one batch.
constexpr int kMaxOwners = 8;
struct Owners {
  int n_owners;
  const uint8_t* ref[kMaxOwners];
  const uint8_t* qry[kMaxOwners];
  const uint64_t* roff[kMaxOwners];
  const uint64_t* qoff[kMaxOwners];
  uint32_t start[kMaxOwners + 1];
};

// Sequence offsets (and the owner's ASCII) of global pair p.
struct PairSrc {
  const uint8_t* ref;
  const uint8_t* qry;
  uint64_t r0, q0;
  int64_t m, n;
};
__device__ __forceinline__ PairSrc pair_src(const Owners& O, const uint8_t* ref, const uint8_t* qry,
                                            const uint64_t* roff, const uint64_t* qoff, uint64_t p) {
  uint64_t l = p;
  if (O.n_owners > 0) {
    int o = 0;
    while (o + 1 < O.n_owners && p >= O.start[o + 1]) ++o;
    l = p - O.start[o];
    ref = O.ref[o]; qry = O.qry[o]; roff = O.roff[o]; qoff = O.qoff[o];
  }
  PairSrc s;
  s.ref = ref; s.qry = qry;
  s.r0 = roff[l]; s.q0 = qoff[l];
  s.m = (int64_t)(roff[l + 1] - s.r0);
  s.n = (int64_t)(qoff[l + 1] - s.q0);
  return s;
}

struct AlignArgs {
  uint32_t* rw;              // packed R scratch: work unit u (a warp, or a wide-tier block) packs
                             // its current pair at rw + (unit_base + u) * rstride (guard word,
                             // data, guard word: see load_word_rw)
  uint32_t* qw;              // packed reversed-Q scratch, qstride words per unit
  uint64_t rstride, qstride; // words per unit: max over the batch of len / 8 + 4, rounded up
  int unit_base;             // first scratch unit of this launch (tier launches run together)
  Owners own;                // federated batch, or n_owners = 0
  const uint8_t* ref_ascii;  // ASCII inputs (device), packed by the align kernel (a1)
  const uint8_t* qry_ascii;
  const uint8_t* chunk_of;   // input chunk of each pair
  const int* ready;          // per-chunk arrival flags (host inputs stream in), or null
  int* err_flags;            // bit 0: non-ACGTN byte
  int nmap;                  // AGATHA_N_MAP
  const uint64_t* roff;
  const uint64_t* qoff;
  const uint32_t* order;     // dispatch order (a2)
  const uint8_t* bad;        // per-pair validation flag from the prep kernel
  agatha_result_t* out;
  agatha_ends_t* ends;       // NEXT #4: end scores per pair (device), or null
  int* queue;                // global work counter (a7)
  int sysq;                  // 1: the counter is shared across GPUs/processes (system scope)
  int static_assign;         // 1: no queue, unit u takes positions u + k * nunits (ablation)
  uint32_t n_pairs;
  int bl, br;                // band; negative = unbounded
  int alpha, beta, zdrop;
  int variant;               // AGATHA_VAR_* bits (0 = the DESIGN.md readings)
  uint32_t T0, T1;           // PRMT score table: byte x = S for code-combination x (0..7)
  long long trace_pair;      // -1: no tracing
  int* trace_score;
  int* trace_i;
  long long trace_cap;
  int sixteen;               // the constant 16, passed at run time (see make_key)
  uint32_t T16_0, T16_1;     // 16-bit kernel table: byte x = S + 2*alpha
  uint32_t k65536;           // the constant 65536, passed at run time (see shr16_fma)
  uint32_t one;              // the constant 1, passed at run time (see add16x2_fma)
  int rebase16;              // split 32-slot front: iterations between re-centrings
  int ref16;                 // 16-bit kernel: stored value of the anti-diagonal max after
                             // a re-centring (negative)
};

// a7: the next position of the dispatch order for work unit `unit` of `nunits` (a warp,
// or a block of the wide tier), whose k-th claim this is.  A shared counter (NEXT #1) lives
// in another GPU's or process's memory, so it is claimed with a system-scope atomic.  The
// static ablation (AGATHA_STATIC_ASSIGN, the analogue of the paper's no-refill baseline,
// P:754-761) gives unit u the positions u, u + nunits, u + 2 nunits, ... with no queue.
__device__ __forceinline__ int claim_next(const AlignArgs& A, int unit, int nunits, int& k) {
  if (A.static_assign) return unit + (k++) * nunits;
  return A.sysq ? atomicAdd_system(A.queue, 1) : atomicAdd(A.queue, 1);
}

// ---- NEXT #4: end scores (agatha_ends_t; reading R19) -------------------------
// A per-warp (per-block in the wide tier) record in shared memory: e[0..1] mqe, mqe_i,
// e[2..3] mte, mte_j, e[4] end score.  Each processed anti-diagonal c holds at most one
// cell with j = n and one with i = m, found by the lane that holds them; anti-diagonals
// are processed in order, so a strict '>' keeps the earliest (smallest i / j) on ties.
__device__ __forceinline__ void ends_init(int* e) {
  e[0] = AGATHA_NO_SCORE; e[1] = -1; e[2] = AGATHA_NO_SCORE; e[3] = -1; e[4] = AGATHA_NO_SCORE;
}
__device__ __forceinline__ void ends_cell(int* e, int i, int j, int h, int m, int n) {
  if (j == n && h > e[0]) { e[0] = h; e[1] = i; }
  if (i == m && h > e[2]) { e[2] = h; e[3] = j; }
  if (i == m && j == n) e[4] = h;
}
__device__ __forceinline__ void ends_store(agatha_ends_t* dst, const int* e) {
  agatha_ends_t r;
  r.mqe = e[0]; r.mqe_i = e[1]; r.mte = e[2]; r.mte_j = e[3]; r.end_score = e[4]; r.reserved = 0;
  *dst = r;
}
// The end cells of anti-diagonal c among this lane's cells t = 0..nc-1 at (ib + t, jb - t):
// cell t_q has j = n, t_t has i = m.  valid(t): the cell's slot lies in the band.
template <typename ValueOf, typename Valid>
__device__ __forceinline__ void ends_capture(int* e, int ib, int jb, int nc, int m, int n,
                                             ValueOf value_of, Valid valid) {
#pragma unroll
  for (int w = 0; w < 2; ++w) {
    const int t = w == 0 ? jb - n : m - ib;
    const int i = ib + t, j = jb - t;
    if (t >= 0 && t < nc && i >= 1 && i <= m && j >= 1 && j <= n && valid(t)) ends_cell(e, i, j, value_of(t), m, n);
  }
}

__device__ __forceinline__ uint32_t prmt(uint32_t a, uint32_t b, uint32_t sel) {
  uint32_t d;
  asm("prmt.b32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(sel));
  return d;
}

// Code combination of eight cells at once (4-bit codes A0 C1 G2 T3 N4 in both R and
// reversed Q, 8 for a position outside the sequence): x = (r ^ q) | (r & q & 0xC) per
// nibble.  x == 0 exactly on a match of two non-N bases, x in 1..3 on a mismatch of two
// non-N bases, x in 4..7 when either is N (N vs N gives 4), and bit 3 set when either
// position is outside its sequence (a PRMT selector nibble with bit 3 set returns the
// sign byte of a table entry: 0 for the 16-bit table, whose entries are all >= 0).
// One LOP3.
__device__ __forceinline__ uint32_t combine(uint32_t r, uint32_t q) {
  uint32_t x;  // LUT 0xBC = (a ^ b) | (a & b & c) with a = r, b = q, c = 0xCCCCCCCC
  asm("lop3.b32 %0, %1, %2, %3, 0xBC;" : "=r"(x) : "r"(r), "r"(q), "n"(0xCCCCCCCC));
  return x;
}


// Packed (score, rank) key for the local max (Eq. 5): max key = max H, and among equal
// H the smallest t (smallest diagonal inside a lane = smallest i on the anti-diagonal).
// Computed as an IMAD with a runtime multiplier (always 16) so that it issues on the
// FMA pipe: the kernel is ALU-pipe bound (profiles/r01_ncu_align_kernel_summary.csv).
__device__ __forceinline__ int make_key(int h, int t, int sixteen) {
  int k;
  asm("mad.lo.s32 %0, %1, %2, %3;" : "=r"(k) : "r"(h), "r"(sixteen), "r"(15 - t));
  return k;
}

__device__ __forceinline__ uint32_t base_code(uint8_t ch, bool nmap, int* err) {
  const uint8_t u = ch & 0xDF;  // upper case
  uint32_t c;
  if (u == 'A') c = 0;
  else if (u == 'C') c = 1;
  else if (u == 'G') c = 2;
  else if (u == 'T') c = 3;
  else if (u == 'N') c = 4;
  else {
    c = 4;
    if (!nmap) *err = 1;
  }
  return c;
}

// Word w of a packed sequence whose first base sits at nibble `pad` (0..7): nibble t
// holds base 8w + t - pad (forward) or base len-1-(8w + t - pad) (reversed), and `fill`
// for a position outside the sequence (0 in agatha_pack4's layout, the out-of-range
// code 8 in the align kernels' own buffers).
constexpr uint32_t kOutWord = 0x88888888u;
__device__ __forceinline__ uint32_t pack_word(const uint8_t* seq, int64_t len, int64_t w, bool rev,
                                              bool nmap, int* err, int pad = 0, uint32_t fill = 0) {
  uint32_t word = 0;
#pragma unroll
  for (int t = 0; t < 8; ++t) {
    const int64_t k = 8 * w + t - pad;
    uint32_t c = fill;
    if (k >= 0 && k < len) {
      const uint8_t ch = rev ? seq[len - 1 - k] : seq[k];
      c = base_code(ch, nmap, err);
    }
    word |= c << (4 * t);
  }
  return word;
}

// a1 fused into the align kernels: the warp that takes a pair packs its R (forward)
// and Q (reversed) from ASCII into the packed buffers, after its input chunk has
// arrived (host inputs stream in chunks that overlap the kernel).
__device__ __forceinline__ int ld_acquire(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ void pack_pair_fused(const uint8_t* __restrict__ ref, const uint8_t* __restrict__ qry,
                                                uint64_t r0, uint64_t q0, int m, int n, uint32_t* Rw,
                                                uint32_t* Qw, const int* ready, int chunk, bool nmap,
                                                int* err_flags, int lane, int padR = 0, int padQ = 0,
                                                int stride = 32) {
  if (ready) {
    while (ld_acquire(ready + chunk) == 0) __nanosleep(500);
  }
  int err = 0;
  const int nwR = (m + padR + 7) / 8, nwQ = (n + padQ + 7) / 8;
  for (int w = lane; w < nwR; w += stride) Rw[1 + w] = pack_word(ref + r0, m, w, false, nmap, &err, padR, 8u);
  for (int w = lane; w < nwQ; w += stride) Qw[1 + w] = pack_word(qry + q0, n, w, true, nmap, &err, padQ, 8u);
  if (lane == 0) {
    Rw[0] = kOutWord; Rw[nwR + 1] = kOutWord;
    Qw[0] = kOutWord; Qw[nwQ + 1] = kOutWord;
  }
  if (__any_sync(kFull, err) && (lane & 31) == 0) atomicOr(err_flags, 1);
  __syncwarp();
}

// Packed words are written by this kernel (pack_pair_fused), so they are read with
// plain loads, not through the read-only path.
// A packed sequence occupies nw + 2 words from `base`: a guard word (kOutWord), data
// words 0..nw-1 at base[1..nw], another guard.  Clamping w + 1 to [0, nw + 1] returns
// the out-of-range code for every position outside the sequence.
__device__ __forceinline__ uint32_t load_word_rw(const uint32_t* base, int w, int nw) {
  int i = w + 1;
  i = i < 0 ? 0 : (i > nw + 1 ? nw + 1 : i);
  return base[i];
}

struct TrueT { static constexpr bool value = true; };
struct FalseT { static constexpr bool value = false; };

struct PairState {
  int m, n, dlo, D;
  int G_H, G_i, G_j, G_d;
  bool haveG;
  int term;
};

// Eq. 4 / Eq. 6 bookkeeping for anti-diagonal c (whose cells had slot parity PARP),
// given the lane-local key maximum `lk` and the warp max H `rH`.  Returns true when
// Eq. 4 fires at c (the caller stops).
template <int K, int PARP, bool TRACE>
__device__ __forceinline__ bool process_antidiag(PairState& s, const AlignArgs& A, int c, int lk,
                                                 int rH, int lane, long long pid) {
  if (rH <= kEmptyH) return false;  // empty anti-diagonal: skipped (reading R11)
  const bool upd = !s.haveG || rH > s.G_H;
  const int c_end = (A.variant & AGATHA_VAR_CHECK_LAST) ? s.m + s.n + 1 : s.m + s.n;
  const bool chk = s.haveG && A.zdrop >= 0 && (s.G_H - rH > A.zdrop) && (c < c_end);
  if (!(upd || chk || TRACE)) return false;
  // argmax: smallest lane holding rH, then its smallest slot (encoded in the key)
  const unsigned bal = __ballot_sync(kFull, (lk >> 4) == rH);
  const int ls = __ffs(bal) - 1;
  const int kk = __shfl_sync(kFull, lk, ls);
  const int t = 15 - (kk & 15);
  const int d = s.dlo + ls * K + PARP + 2 * t;
  const int i = (c + d) >> 1;
  const int j = c - i;
  if (TRACE && pid == A.trace_pair && lane == 0 && c < A.trace_cap) {
    A.trace_score[c] = rH;
    A.trace_i[c] = i;
  }
  const bool gated = (A.variant & AGATHA_VAR_GATE_GE) ? (s.G_i <= i && s.G_j <= j)
                                                       : (s.G_i < i && s.G_j < j);
  if (chk && gated) {
    const int gap = d - s.G_d;
    if (s.G_H - rH > A.zdrop + A.beta * (gap < 0 ? -gap : gap)) {
      s.term = c;
      return true;
    }
  }
  if (upd) {
    s.G_H = rH;
    s.G_i = i;
    s.G_j = j;
    s.G_d = d;
    s.haveG = true;
  }
  return false;
}

// One anti-diagonal step: update the K/2 slots of parity PAR.  `S` holds the
// substitution scores of the step as sign-extendable bytes (4 cells per word).
//
// Storage per slot: H, and E and F shifted by +alpha (Eh = E + alpha, Fh = F + alpha),
// which turns Eq. 2-3 into one VIADDMNMX each without a stored H - alpha:
//   Eh(i,j) = max(Eh(i-1,j) - beta, H(i-1,j))      [= Eq. 2 + alpha]
//   Fh(i,j) = max(Fh(i,j-1) - beta, H(i,j-1))      [= Eq. 3 + alpha]
//   H(i,j)  = max(max(Eh, Fh) - alpha, H(i-1,j-1) + S)   [= Eq. 1]
// edgeH / edgeEF: the neighbour of the warp's edge lane (lane 0 for PAR = 0, lane 31 for
// PAR = 1): -infinity at the band's ends, the adjacent warp's slot in the wide tier.
template <int K, int PAR, bool MASKED>
__device__ __forceinline__ int step_cells(int (&H)[K], int (&Eh)[K], int (&Fh)[K],
                                          const uint32_t (&S)[K / 8], int lane, int nalpha,
                                          int nbeta, int capT, int tlo, int thi, int sixteen,
                                          int edgeH = kNegE, int edgeEF = kNegE) {
  // edge exchange: the one neighbour slot that lives in the adjacent lane
  int xH, xEF;
  if (PAR == 0) {
    xH = __shfl_up_sync(kFull, H[K - 1], 1);
    xEF = __shfl_up_sync(kFull, Eh[K - 1], 1);
    if (lane == 0) { xH = edgeH; xEF = edgeEF; }    // below the band (or the previous warp)
  } else {
    xH = __shfl_down_sync(kFull, H[0], 1);
    xEF = __shfl_down_sync(kFull, Fh[0], 1);
    if (lane == 31) { xH = edgeH; xEF = edgeEF; }   // above the band (or the next warp)
  }
  int lk = kNegKey, kprev = kNegKey;
#pragma unroll
  for (int t = 0; t < K / 2; ++t) {
    const int k = PAR + 2 * t;
    const int hu = (k == 0) ? xH : H[k - 1];
    const int eu = (k == 0) ? xEF : Eh[k - 1];
    const int hl = (k == K - 1) ? xH : H[k + 1];
    const int fl = (k == K - 1) ? xEF : Fh[k + 1];
    const int e = __viaddmax_s32(eu, nbeta, hu);           // Eq. 2 (+alpha)
    const int f = __viaddmax_s32(fl, nbeta, hl);           // Eq. 3 (+alpha)
    const uint32_t sel = (uint32_t)(t & 3) | ((uint32_t)((t & 3) | 8) * 0x1110u);
    const int sub = (int)prmt(S[t >> 2], 0u, sel);         // S(R[i],Q[j]), sign-extended
    int h = __viaddmax_s32(max(e, f), nalpha, H[k] + sub); // Eq. 1
    h = __viaddmin_s32(capT, -k * kCapStep, h);            // padding slots stay below -2^20
    int key = make_key(h, t, sixteen);
    if (MASKED) {
      const bool v = (t >= tlo) && (t <= thi);
      H[k] = v ? h : H[k];
      Eh[k] = v ? e : kNegE;
      Fh[k] = v ? f : kNegE;
      key = v ? key : kNegKey;
    } else {
      H[k] = h;
      Eh[k] = e;
      Fh[k] = f;
    }
    if (t & 1) lk = __vimax3_s32(lk, kprev, key); else kprev = key;  // Eq. 5, 2 cells per VIMNMX3
  }
  return (K / 2) & 1 ? max(lk, kprev) : lk;
}

template <int K, bool TRACE>
__device__ void align_pair(const AlignArgs& A, uint32_t pid, int lane, int unit, int* erec) {
  const PairSrc ps = pair_src(A.own, A.ref_ascii, A.qry_ascii, A.roff, A.qoff, pid);
  const uint64_t r0 = ps.r0, q0 = ps.q0;
  const int m = (int)ps.m;
  const int n = (int)ps.n;
  if (A.bad[pid]) {  // (the call fails; the rows are zero)
    if (lane == 0) {
      agatha_result_t z = {0, 0, 0, -1, 0};
      A.out[pid] = z;
    }
    return;
  }
  uint32_t* Rw = A.rw + (uint64_t)(A.unit_base + unit) * A.rstride;
  uint32_t* Qw = A.qw + (uint64_t)(A.unit_base + unit) * A.qstride;
  const int nwR = (m + 7) >> 3, nwQ = (n + 7) >> 3;
  pack_pair_fused(ps.ref, ps.qry, r0, q0, m, n, Rw, Qw, A.ready, A.chunk_of[pid],
                  A.nmap != 0, A.err_flags, lane);
  const int bl = (A.bl < 0 || A.bl > n) ? n : A.bl;   // diagonals beyond hold no cell
  const int br = (A.br < 0 || A.br > m) ? m : A.br;
  const int alpha = A.alpha, beta = A.beta, nbeta = -A.beta, nalpha = -A.alpha;

  PairState s;
  s.m = m; s.n = n; s.dlo = -bl; s.D = bl + br + 1;
  s.haveG = (A.variant & AGATHA_VAR_ORIGIN_MAX) != 0;  // G = H(0,0) = 0 at the origin
  s.G_H = 0; s.G_i = 0; s.G_j = 0; s.G_d = 0; s.term = -1;
  const int dlo = -bl, D = s.D;

  // padding cap: slot k of this lane is capped at capT - k*kCapStep
  const int gbase = lane * K;
  int capT;
  if (gbase + K <= D) capT = 1 << 30;
  else if (gbase >= D) capT = -kHLimit;
  else capT = (D - gbase - 1) * kCapStep + kHLimit;

  // a3: boundary values H(d,0) / H(0,-d) (reading R2); E = F = -infinity
  int H[K], Eh[K], Fh[K];
#pragma unroll
  for (int k = 0; k < K; ++k) {
    const int g = gbase + k, d = dlo + g;
    const int ad = d < 0 ? -d : d;
    H[k] = (g < D) ? (d == 0 ? 0 : -(alpha + (ad - 1) * beta)) : kPadH;
    Eh[k] = kNegE;
    Fh[k] = kNegE;
  }

  // phases: head (masked) / steady (every band slot in the table) / tail (masked)
  auto fdiag = [&](int d) { return 2 * min(m, n + d) - d; };  // last anti-diagonal of diagonal d
  const int dhi = br;
  const int cs = 2 + max(bl, br);
  const int ce = min(fdiag(dlo), fdiag(dhi));
  const int dmid = min(max(m - n, dlo), dhi);
  const int c_last = fdiag(dmid);

  // sequence windows (R forward, Q reversed), nibble-granular, uniform phase across lanes
  int cb = 2 - (dlo & 1);                     // first step parity 0: cb == dlo (mod 2)
  int u = (cb + dlo) >> 1;
  int rpos = u - 1 + lane * (K / 2);          // nibble index of R[i] at t = 0, PAR = 0
  int wR = rpos >> 3, oR = rpos & 7;
  uint32_t Wr0 = load_word_rw(Rw, wR, nwR), Wr1 = load_word_rw(Rw, wR + 1, nwR),
           Wr2 = load_word_rw(Rw, wR + 2, nwR);
  int qpos = n + dlo - u + lane * (K / 2);    // nibble index of Qrev[x] at t = 0
  int wQ = qpos >> 3, oQ = qpos & 7;
  uint32_t Wq0 = load_word_rw(Qw, wQ, nwQ), Wq1 = load_word_rw(Qw, wQ + 1, nwQ),
           Wq2 = load_word_rw(Qw, wQ + 2, nwQ);

  const uint32_t T0 = A.T0, T1 = A.T1;
  int lk_prev = kNegKey, rH_prev = kEmptyH - 1;  // nothing pending before the first step
  bool stop = false;
  if (A.ends) {
    if (lane == 0) ends_init(erec);
    __syncwarp();
  }
  // NEXT #4: the end cells of processed anti-diagonal c (slot parity P, still in H)
  auto capture = [&](int c, int P) {
    const int uc = (c - P + dlo) >> 1;
    const int ib = uc + P + lane * (K / 2), jb = uc - dlo - lane * (K / 2);
    ends_capture(erec, ib, jb, K / 2, m, n,
                 [&](int t) {
                   int v = 0;
#pragma unroll
                   for (int k = 0; k < K / 2; ++k)
                     if (k == t) v = P ? H[1 + 2 * k] : H[2 * k];
                   return v;
                 },
                 [&](int t) { return gbase + P + 2 * t < D; });
    __syncwarp();
  };

  auto iteration = [&](auto masked_tag) {
    constexpr bool MASKED = decltype(masked_tag)::value;
    constexpr int NG = (K >= 16) ? K / 16 : 1;
    uint32_t qg[NG], S[K / 8 > 0 ? K / 8 : 1];
    const uint32_t Wq[3] = {Wq0, Wq1, Wq2}, Wr[3] = {Wr0, Wr1, Wr2};
#pragma unroll
    for (int g = 0; g < NG; ++g) qg[g] = __funnelshift_rc(Wq[g], Wq[g + 1], 4 * oQ);
    // ---- step PAR = 0, anti-diagonal cb ----
    {
#pragma unroll
      for (int g = 0; g < NG; ++g) {
        const uint32_t x = combine(__funnelshift_rc(Wr[g], Wr[g + 1], 4 * oR), qg[g]);
        S[2 * g] = prmt(T0, T1, x);
        if (2 * g + 1 < K / 8) S[2 * g + 1] = prmt(T0, T1, x >> 16);
      }
      int tlo = 0, thi = K;
      if (MASKED) {
        const int ib = u + lane * (K / 2), jb = u - dlo - lane * (K / 2);
        tlo = max(1 - ib, jb - n);
        thi = min(m - ib, jb - 1);
      }
      const int lk = step_cells<K, 0, MASKED>(H, Eh, Fh, S, lane, nalpha, nbeta, capT, tlo, thi, A.sixteen);
      const int rH = __reduce_max_sync(kFull, lk >> 4);
      if (MASKED && A.ends) capture(cb - 1, 1);
      if (process_antidiag<K, 1, TRACE>(s, A, cb - 1, lk_prev, rH_prev, lane, pid)) { stop = true; return; }
      lk_prev = lk;
      rH_prev = rH;
    }
    // ---- step PAR = 1, anti-diagonal cb + 1 ----
    {
#pragma unroll
      for (int g = 0; g < NG; ++g) {
        const uint32_t x = combine(__funnelshift_rc(Wr[g], Wr[g + 1], 4 * oR + 4), qg[g]);
        S[2 * g] = prmt(T0, T1, x);
        if (2 * g + 1 < K / 8) S[2 * g + 1] = prmt(T0, T1, x >> 16);
      }
      int tlo = 0, thi = K;
      if (MASKED) {
        const int ib = u + 1 + lane * (K / 2), jb = u - dlo - lane * (K / 2);
        tlo = max(1 - ib, jb - n);
        thi = min(m - ib, jb - 1);
      }
      const int lk = step_cells<K, 1, MASKED>(H, Eh, Fh, S, lane, nalpha, nbeta, capT, tlo, thi, A.sixteen);
      const int rH = __reduce_max_sync(kFull, lk >> 4);
      if (MASKED && A.ends) capture(cb, 0);
      if (process_antidiag<K, 0, TRACE>(s, A, cb, lk_prev, rH_prev, lane, pid)) { stop = true; return; }
      lk_prev = lk;
      rH_prev = rH;
    }
    // ---- advance the windows by one base each: R forward, reversed Q backward ----
    cb += 2;
    ++u;
    if (++oR == 8) {
      oR = 0;
      ++wR;
      Wr0 = Wr1; Wr1 = Wr2; Wr2 = load_word_rw(Rw, wR + 2, nwR);
    }
    if (--oQ < 0) {
      oQ = 7;
      --wQ;
      Wq2 = Wq1; Wq1 = Wq0; Wq0 = load_word_rw(Qw, wQ, nwQ);
    }
  };

  // with end scores, the steady phase stops before anti-diagonal ce (the first that can
  // hold an end cell), so that every end cell is processed by a masked step
  const int ce_steady = A.ends ? ce - 1 : ce;
  while (!stop && cb <= c_last && cb < cs) iteration(TrueT{});
  while (!stop && cb + 1 <= ce_steady) iteration(FalseT{});
  while (!stop && cb <= c_last) iteration(TrueT{});
  if (!stop) {
    // the last computed step (cb - 1, slot parity 1) is still pending
    if (A.ends) capture(cb - 1, 1);
    process_antidiag<K, 1, TRACE>(s, A, cb - 1, lk_prev, rH_prev, lane, pid);
  }
  if (A.ends && lane == 0) ends_store(A.ends + pid, erec);

  // a8: cells = in-band in-table cells on anti-diagonals 2 .. c_end (closed form per slot)
  const int c_end = s.term >= 0 ? s.term : m + n;
  int cnt = 0;
#pragma unroll
  for (int k = 0; k < K; ++k) {
    const int g = gbase + k;
    if (g < D) {
      const int d = dlo + g;
      const int clo = (d < 0 ? -d : d) + 2;
      const int hi = min(fdiag(d), c_end);
      if (hi >= clo) cnt += ((hi - clo) >> 1) + 1;
    }
  }
  cnt = (int)__reduce_add_sync(kFull, (unsigned)cnt);
  if (lane == 0) {
    agatha_result_t r;
    r.score = s.G_H;
    r.ref_end = s.G_i;
    r.query_end = s.G_j;
    r.zdrop_antidiag = s.term;
    r.cells = cnt;
    A.out[pid] = r;
  }
}

// Register budget: the band front (H for all K slots, E/F/H-alpha for the last parity)
// plus the per-pair state needs ~150 registers at K = 32, so 3 blocks of 4 warps
// (12 warps, 3 per scheduler) per SM; K = 16 fits 4 blocks.
template <int K>
struct MinBlocks { static constexpr int value = K >= 32 ? 3 : 4; };

template <int K, bool TRACE>
__global__ void __launch_bounds__(128, MinBlocks<K>::value) align_kernel(AlignArgs A) {
  __shared__ int erec_all[4][8];  // NEXT #4 end-score records, one per warp
  const int lane = threadIdx.x & 31;
  const int unit = blockIdx.x * 4 + (threadIdx.x >> 5), nunits = gridDim.x * 4;
  int k = 0;
  for (;;) {
    int q = 0;
    if (lane == 0) q = claim_next(A, unit, nunits, k);
    q = __shfl_sync(kFull, q, 0);
    if ((uint32_t)q >= A.n_pairs) break;
    align_pair<K, TRACE>(A, A.order[q], lane, unit, erec_all[threadIdx.x >> 5]);
  }
}


// ---- NEXT #3: the wide-band tier (32-bit, W warps per pair) --------------------------
// Bands wider than one warp's 1024 slots (w > 511) split the D <= 1024*W diagonals over
// the 32*W lanes of a W-warp block in order (global lane gl = 32*warp + lane; K = 32
// slots each).  Per step, the two warp-edge slots cross warps through shared memory and
// each warp publishes its anti-diagonal max with the diagonal of its first maximal cell;
// one __syncthreads orders both (two per iteration).  Every Eq. 4-6 decision is taken
// from the block-wide values, identically in all warps, so control flow stays
// block-uniform.  Same cells, same arithmetic, same results as align_kernel.
struct WideShared {
  int ends[8];                                     // NEXT #4 end-score record of the pair
  int up_H[kMaxWarpsWide], up_E[kMaxWarpsWide];   // lane 31's slot K-1 after a PAR = 1 step
  int dn_H[kMaxWarpsWide], dn_F[kMaxWarpsWide];   // lane 0's slot 0 after a PAR = 0 step
  int rH[2][kMaxWarpsWide], d[2][kMaxWarpsWide];  // per step parity: warp max, its diagonal
  int cnt[kMaxWarpsWide];
  int q;
};

// Eq. 4 / Eq. 6 for anti-diagonal c given the block-wide max rH and the diagonal d of its
// first (smallest i) maximal cell; true when Eq. 4 fires.
template <bool TRACE>
__device__ __forceinline__ bool process_wide(PairState& s, const AlignArgs& A, int c, int rH, int d,
                                             bool leader, long long pid) {
  if (rH <= kEmptyH) return false;  // empty anti-diagonal: skipped (reading R11)
  const bool upd = !s.haveG || rH > s.G_H;
  const int c_end = (A.variant & AGATHA_VAR_CHECK_LAST) ? s.m + s.n + 1 : s.m + s.n;
  const bool chk = s.haveG && A.zdrop >= 0 && (s.G_H - rH > A.zdrop) && (c < c_end);
  if (!(upd || chk || TRACE)) return false;
  const int i = (c + d) >> 1;
  const int j = c - i;
  if (TRACE && leader && pid == A.trace_pair && c < A.trace_cap) {
    A.trace_score[c] = rH;
    A.trace_i[c] = i;
  }
  const bool gated = (A.variant & AGATHA_VAR_GATE_GE) ? (s.G_i <= i && s.G_j <= j)
                                                       : (s.G_i < i && s.G_j < j);
  if (chk && gated) {
    const int gap = d - s.G_d;
    if (s.G_H - rH > A.zdrop + A.beta * (gap < 0 ? -gap : gap)) {
      s.term = c;
      return true;
    }
  }
  if (upd) {
    s.G_H = rH;
    s.G_i = i;
    s.G_j = j;
    s.G_d = d;
    s.haveG = true;
  }
  return false;
}

template <int W, bool TRACE>
__device__ void align_pair_wide(const AlignArgs& A, uint32_t pid, int lane, int wid, WideShared& sh) {
  constexpr int K = 32;
  const int gl = wid * 32 + lane;
  const PairSrc ps = pair_src(A.own, A.ref_ascii, A.qry_ascii, A.roff, A.qoff, pid);
  const uint64_t r0 = ps.r0, q0 = ps.q0;
  const int m = (int)ps.m;
  const int n = (int)ps.n;
  if (A.bad[pid]) {  // block-uniform
    if (gl == 0) {
      agatha_result_t z = {0, 0, 0, -1, 0};
      A.out[pid] = z;
    }
    return;
  }
  uint32_t* Rw = A.rw + (uint64_t)(A.unit_base + (int)blockIdx.x) * A.rstride;  // one pair per block
  uint32_t* Qw = A.qw + (uint64_t)(A.unit_base + (int)blockIdx.x) * A.qstride;
  const int nwR = (m + 7) >> 3, nwQ = (n + 7) >> 3;
  pack_pair_fused(ps.ref, ps.qry, r0, q0, m, n, Rw, Qw, A.ready, A.chunk_of[pid],
                  A.nmap != 0, A.err_flags, gl, 0, 0, 32 * W);
  const int bl = (A.bl < 0 || A.bl > n) ? n : A.bl;
  const int br = (A.br < 0 || A.br > m) ? m : A.br;
  const int alpha = A.alpha, beta = A.beta, nbeta = -A.beta, nalpha = -A.alpha;

  PairState s;
  s.m = m; s.n = n; s.dlo = -bl; s.D = bl + br + 1;
  s.haveG = (A.variant & AGATHA_VAR_ORIGIN_MAX) != 0;  // G = H(0,0) = 0 at the origin
  s.G_H = 0; s.G_i = 0; s.G_j = 0; s.G_d = 0; s.term = -1;
  const int dlo = -bl, D = s.D;

  // padding cap: slot k of this lane is capped at capT - k*kCapStep
  const int gbase = gl * K;
  int capT;
  if (gbase + K <= D) capT = 1 << 30;
  else if (gbase >= D) capT = -kHLimit;
  else capT = (D - gbase - 1) * kCapStep + kHLimit;

  int H[K], Eh[K], Fh[K];
#pragma unroll
  for (int k = 0; k < K; ++k) {
    const int g = gbase + k, d = dlo + g;
    const int ad = d < 0 ? -d : d;
    H[k] = (g < D) ? (d == 0 ? 0 : -(alpha + (ad - 1) * beta)) : kPadH;
    Eh[k] = kNegE;
    Fh[k] = kNegE;
  }
  if (lane == 31) { sh.up_H[wid] = H[K - 1]; sh.up_E[wid] = Eh[K - 1]; }
  __syncthreads();  // the packed words and the first edge values are visible block-wide

  auto fdiag = [&](int d) { return 2 * min(m, n + d) - d; };
  const int dhi = br;
  const int cs = 2 + max(bl, br);
  const int ce = min(fdiag(dlo), fdiag(dhi));
  const int dmid = min(max(m - n, dlo), dhi);
  const int c_last = fdiag(dmid);

  int cb = 2 - (dlo & 1);
  int u = (cb + dlo) >> 1;
  int rpos = u - 1 + gl * (K / 2);
  int wR = rpos >> 3, oR = rpos & 7;
  uint32_t Wr0 = load_word_rw(Rw, wR, nwR), Wr1 = load_word_rw(Rw, wR + 1, nwR),
           Wr2 = load_word_rw(Rw, wR + 2, nwR);
  int qpos = n + dlo - u + gl * (K / 2);
  int wQ = qpos >> 3, oQ = qpos & 7;
  uint32_t Wq0 = load_word_rw(Qw, wQ, nwQ), Wq1 = load_word_rw(Qw, wQ + 1, nwQ),
           Wq2 = load_word_rw(Qw, wQ + 2, nwQ);
  const uint32_t T0 = A.T0, T1 = A.T1;
  bool stop = false;
  if (A.ends) {
    if (gl == 0) ends_init(sh.ends);
    __syncthreads();
  }
  // NEXT #4: the end cells of anti-diagonal c (slot parity P, just computed)
  auto capture = [&](int c, int P) {
    const int uc = (c - P + dlo) >> 1;
    const int ib = uc + P + gl * (K / 2), jb = uc - dlo - gl * (K / 2);
    ends_capture(sh.ends, ib, jb, K / 2, m, n,
                 [&](int t) {
                   int v = 0;
#pragma unroll
                   for (int k = 0; k < K / 2; ++k)
                     if (k == t) v = P ? H[1 + 2 * k] : H[2 * k];
                   return v;
                 },
                 [&](int t) { return gbase + P + 2 * t < D; });
  };

  // warp max and the diagonal of its first maximal cell (smallest lane, then slot)
  auto publish = [&](int lk, int par) {
    const int wmax = __reduce_max_sync(kFull, lk >> 4);
    const unsigned bal = __ballot_sync(kFull, (lk >> 4) == wmax);
    const int ls = __ffs(bal) - 1;
    const int kk = __shfl_sync(kFull, lk, ls);
    const int t = 15 - (kk & 15);
    if (lane == 0) {
      sh.rH[par][wid] = wmax;
      sh.d[par][wid] = dlo + (wid * 32 + ls) * K + par + 2 * t;
    }
  };
  // block max (warps in diagonal order: the first warp holding it has the smallest d)
  auto combine_warps = [&](int par, int& rH, int& d) {
    rH = sh.rH[par][0];
    d = sh.d[par][0];
#pragma unroll
    for (int w = 1; w < W; ++w) {
      const int v = sh.rH[par][w];
      if (v > rH) { rH = v; d = sh.d[par][w]; }
    }
  };

  auto iteration = [&](auto masked_tag) {
    constexpr bool MASKED = decltype(masked_tag)::value;
    uint32_t qg[2], S[4];
    const uint32_t Wq[3] = {Wq0, Wq1, Wq2}, Wr[3] = {Wr0, Wr1, Wr2};
#pragma unroll
    for (int g = 0; g < 2; ++g) qg[g] = __funnelshift_rc(Wq[g], Wq[g + 1], 4 * oQ);
    // ---- step PAR = 0, anti-diagonal cb ----
    {
#pragma unroll
      for (int g = 0; g < 2; ++g) {
        const uint32_t x = combine(__funnelshift_rc(Wr[g], Wr[g + 1], 4 * oR), qg[g]);
        S[2 * g] = prmt(T0, T1, x);
        S[2 * g + 1] = prmt(T0, T1, x >> 16);
      }
      int tlo = 0, thi = K;
      if (MASKED) {
        const int ib = u + gl * (K / 2), jb = u - dlo - gl * (K / 2);
        tlo = max(1 - ib, jb - n);
        thi = min(m - ib, jb - 1);
      }
      const int eH = wid > 0 ? sh.up_H[wid > 0 ? wid - 1 : 0] : kNegE;
      const int eE = wid > 0 ? sh.up_E[wid > 0 ? wid - 1 : 0] : kNegE;
      const int lk = step_cells<K, 0, MASKED>(H, Eh, Fh, S, lane, nalpha, nbeta, capT, tlo, thi,
                                              A.sixteen, eH, eE);
      publish(lk, 0);
      if (lane == 0) { sh.dn_H[wid] = H[0]; sh.dn_F[wid] = Fh[0]; }
      __syncthreads();
      int rH, d;
      combine_warps(0, rH, d);
      if (MASKED && A.ends) {
        capture(cb, 0);
        __syncthreads();
      }
      if (process_wide<TRACE>(s, A, cb, rH, d, gl == 0, pid)) { stop = true; return; }
    }
    // ---- step PAR = 1, anti-diagonal cb + 1 ----
    {
#pragma unroll
      for (int g = 0; g < 2; ++g) {
        const uint32_t x = combine(__funnelshift_rc(Wr[g], Wr[g + 1], 4 * oR + 4), qg[g]);
        S[2 * g] = prmt(T0, T1, x);
        S[2 * g + 1] = prmt(T0, T1, x >> 16);
      }
      int tlo = 0, thi = K;
      if (MASKED) {
        const int ib = u + 1 + gl * (K / 2), jb = u - dlo - gl * (K / 2);
        tlo = max(1 - ib, jb - n);
        thi = min(m - ib, jb - 1);
      }
      const int eH = wid < W - 1 ? sh.dn_H[wid < W - 1 ? wid + 1 : 0] : kNegE;
      const int eF = wid < W - 1 ? sh.dn_F[wid < W - 1 ? wid + 1 : 0] : kNegE;
      const int lk = step_cells<K, 1, MASKED>(H, Eh, Fh, S, lane, nalpha, nbeta, capT, tlo, thi,
                                              A.sixteen, eH, eF);
      publish(lk, 1);
      if (lane == 31) { sh.up_H[wid] = H[K - 1]; sh.up_E[wid] = Eh[K - 1]; }
      __syncthreads();
      int rH, d;
      combine_warps(1, rH, d);
      if (MASKED && A.ends) {
        capture(cb + 1, 1);
        __syncthreads();
      }
      if (process_wide<TRACE>(s, A, cb + 1, rH, d, gl == 0, pid)) { stop = true; return; }
    }
    cb += 2;
    ++u;
    if (++oR == 8) {
      oR = 0;
      ++wR;
      Wr0 = Wr1; Wr1 = Wr2; Wr2 = load_word_rw(Rw, wR + 2, nwR);
    }
    if (--oQ < 0) {
      oQ = 7;
      --wQ;
      Wq2 = Wq1; Wq1 = Wq0; Wq0 = load_word_rw(Qw, wQ, nwQ);
    }
  };

  const int ce_steady = A.ends ? ce - 1 : ce;  // every end cell in a masked step (NEXT #4)
  while (!stop && cb <= c_last && cb < cs) iteration(TrueT{});
  while (!stop && cb + 1 <= ce_steady) iteration(FalseT{});
  while (!stop && cb <= c_last) iteration(TrueT{});
  if (A.ends) {
    __syncthreads();
    if (gl == 0) ends_store(A.ends + pid, sh.ends);
  }

  // a8: cells on anti-diagonals 2 .. c_end (closed form per slot), summed over the block
  const int c_end = s.term >= 0 ? s.term : m + n;
  int cnt = 0;
#pragma unroll
  for (int k = 0; k < K; ++k) {
    const int g = gbase + k;
    if (g < D) {
      const int d = dlo + g;
      const int clo = (d < 0 ? -d : d) + 2;
      const int hi = min(fdiag(d), c_end);
      if (hi >= clo) cnt += ((hi - clo) >> 1) + 1;
    }
  }
  cnt = (int)__reduce_add_sync(kFull, (unsigned)cnt);
  if (lane == 0) sh.cnt[wid] = cnt;
  __syncthreads();
  if (gl == 0) {
    long long tot = 0;
#pragma unroll
    for (int w = 0; w < W; ++w) tot += sh.cnt[w];
    agatha_result_t r;
    r.score = s.G_H;
    r.ref_end = s.G_i;
    r.query_end = s.G_j;
    r.zdrop_antidiag = s.term;
    r.cells = tot;
    A.out[pid] = r;
  }
}

// 12 warps per SM as for align_kernel<32> (~168 registers).
template <int W, bool TRACE>
__global__ void __launch_bounds__(32 * W, 12 / W) align_wide_kernel(AlignArgs A) {
  __shared__ WideShared sh;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  int k = 0;
  for (;;) {
    if (threadIdx.x == 0) sh.q = claim_next(A, blockIdx.x, gridDim.x, k);
    __syncthreads();
    const int q = sh.q;
    __syncthreads();  // every thread has read q before thread 0 takes the next one
    if ((uint32_t)q >= A.n_pairs) break;
    align_pair_wide<W, TRACE>(A, A.order[q], lane, wid, sh);
  }
}

// ===================================================================================
// 16-bit packed variant (DPX .S16x2): two cells per instruction.
//
// Same wavefront, same per-lane slot ranges, same windows as align_kernel<K>, with
// K = 2*NREG slots per lane held in NREG 32-bit registers as (slot j | slot j+NREG)
// half-word pairs, so that a slot's two diagonal neighbours j-1 and j+1 live in the
// same halves of registers j-1 and j+1 (only registers 0 and NREG-1 need a lane
// exchange, one PRMT each).  Values are stored relative and shifted:
//     stored = X + alpha*c - B        (X in {H, E, F}, c the anti-diagonal)
// The alpha*c shift turns Eq. 1-3 into 4 DPX ops per register (2 cells):
//     Eh = max(Eh_up + (alpha-beta), H_up)          VIADDMNMX.S16x2
//     Fh = max(Fh_left + (alpha-beta), H_left)      VIADDMNMX.S16x2
//     H  = max(H_diag + (S + 2alpha), max(Eh, Fh))  VIMNMX.S16x2 + VIADDMNMX.S16x2
// B is a per-pair base re-centred on the anti-diagonal max every kRebase16 steps.
// Exactness: all in-band H of one anti-diagonal lie
// within alpha + D*(beta + a + max(b,n)) below its max, so with the host-side guard
// every live value stays in (-16000, 12000) and no half-word add wraps.
// ===================================================================================

#ifndef AGATHA_FMA_ADD
#define AGATHA_FMA_ADD 1
#endif
// A/B switches (DESIGN.md §6.5 "Tried and reverted"); the defaults are the measured best
#ifndef AGATHA_RREUSE
#define AGATHA_RREUSE 0  // 1: carry the PAR = 1 R shift into the next PAR = 0 step (-1.6%)
#endif
#ifndef AGATHA_RREUSE_NARROW
#define AGATHA_RREUSE_NARROW 1  // the same for the 16- and 8-slot fronts (+0.5-0.8%)
#endif
#ifndef AGATHA_LMSHL
#define AGATHA_LMSHL 1  // lane max of the two halves via lm << 16 (IMAD) instead of hi16_fma
#endif
#if AGATHA_LMSHL
#define LANEMAX16(x) ((x) >> 16)
#else
#define LANEMAX16(x) (x)
#endif
#ifndef AGATHA_S2EARLY
#define AGATHA_S2EARLY 0  // 1: both steps' substitution scores at the top of the iteration
#endif
#ifndef AGATHA_VOTE
#define AGATHA_VOTE 1    // 0: plain uniform branch instead of the vote in process16 (-0.2%)
#endif
#ifndef AGATHA_VOTE_NARROW
#define AGATHA_VOTE_NARROW 0  // the same for the 16- and 8-slot fronts: no vote (+0.3-2.3%)
#endif
// Issue-slot trims of the steady loop (A/B switches):
//   LMTREE   the 32-slot front's lane max over its eight registers as a depth-2 tree
//   SNAP128  the deferred-argmax snapshot as 128-bit shared stores
//   STEADYC  the steady phase keeps the previous anti-diagonal's cell range and base
//            instead of re-setting them every step (re-centring adjusts rH_prev)
#ifndef AGATHA_LMTREE
#define AGATHA_LMTREE 0  // the split front: the serial lane max schedules better (4345 vs 4246 GCUPS)
#endif
#ifndef AGATHA_SNAP128
#define AGATHA_SNAP128 0
#endif
#ifndef AGATHA_STEADYC
#define AGATHA_STEADYC 1
#endif
//   SNAPSLIM the snapshot stores only the registers, the base and G: the parity and cell
//            range of the snapshot's anti-diagonal are recomputed from G_c when resolved,
//            validity is G_c == posC, and a disabled Z-drop uses a huge threshold
//   LOOPSLIM the iteration carries one window offset (oQ = 7 - oR) and no u (masked
//            steps derive it from cb)
#ifndef AGATHA_SNAPSLIM
#define AGATHA_SNAPSLIM 1
#endif
#ifndef AGATHA_LOOPSLIM
#define AGATHA_LOOPSLIM 0
#endif

// Stored half-words live in [kW16, kTop16 + 127].  With AGATHA_POS16 (default) the domain
// is shifted up by kShift16 into [2495, 31743]: every live half-word is then a positive
// int16 whose bit pattern is also a finite, normal, positive fp16, and positive fp16 bit
// patterns order exactly like the integers, so pure min/max steps may run as fp16x2
// HMNMX2; the IMAD diagonal add stays carry-free (low half + 127 <= 31743).
#ifndef AGATHA_POS16
#define AGATHA_POS16 1
#endif
constexpr int kShift16 = AGATHA_POS16 ? 31745 : 0;
constexpr int kW16 = -29250 + kShift16;       // "-infinity" (walls, E/F of boundary cells)
constexpr int kCapNeg16 = -21250 + kShift16;  // padding cap
constexpr int kEmpty16 = -17250 + kShift16;   // lane max at or below: no valid cell on the anti-diagonal
constexpr int kTop16 = -129 + kShift16;       // every stored H is at most this
#ifndef AGATHA_REBASE16
#define AGATHA_REBASE16 32
#endif
constexpr int kRebase16 = AGATHA_REBASE16;  // iterations (2x anti-diagonals) between re-centrings

__device__ __forceinline__ uint32_t pack2(int lo, int hi) {
  return ((uint32_t)lo & 0xFFFFu) | ((uint32_t)hi << 16);
}
__device__ __forceinline__ int lo16(uint32_t x) { return (int)(int16_t)(x & 0xFFFFu); }
__device__ __forceinline__ int hi16(uint32_t x) { return ((int)x) >> 16; }
__device__ __forceinline__ uint32_t vmax2(uint32_t a, uint32_t b) { return __vmaxs2(a, b); }
// x >> 16 (logical / arithmetic) as the high word of x * 65536 on the FMA pipe: the
// kernel is ALU-pipe bound and the FMA pipe is ~85% idle.  k65536 is passed at run time
// so that ptxas cannot strength-reduce the multiply back into an ALU shift.
#ifndef AGATHA_SHR_WIDE
#define AGATHA_SHR_WIDE 0  // 1: x >> 16 as the high word of a 64-bit IMAD.WIDE
#endif
__device__ __forceinline__ uint32_t shr16_fma(uint32_t x, uint32_t k65536) {
  uint32_t d;
#if AGATHA_SHR_WIDE
  asm("{\n\t.reg .u64 w;\n\tmul.wide.u32 w, %1, %2;\n\tmov.b64 {_, %0}, w;\n\t}" : "=r"(d) : "r"(x), "r"(k65536));
#else
  asm("mad.hi.u32 %0, %1, %2, 0;" : "=r"(d) : "r"(x), "r"(k65536));
#endif
  return d;
}
[[maybe_unused]] __device__ __forceinline__ int hi16_fma(uint32_t x, uint32_t k65536) {
  int d;
  asm("mad.hi.s32 %0, %1, %2, 0;" : "=r"(d) : "r"((int)x), "r"((int)k65536));
  return d;
}
[[maybe_unused]] __device__ __forceinline__ uint32_t vmin2(uint32_t a, uint32_t b) { return __vmins2(a, b); }
// Pure max / min of two half-word pairs as fp16x2 HMNMX2 (AGATHA_POS16 domain: every
// operand that matters is a positive int16 <= 31743 = 0x7BFF, i.e. a finite positive fp16
// whose order is the integer order; exact on all pairs in [0, 0x7BFF],
// profiles/r02_hmnmx.jsonl).  It issues on the ALU pipe (same file), so AGATHA_HMAX is off.
[[maybe_unused]] __device__ __forceinline__ uint32_t hmax2(uint32_t a, uint32_t b) {
  uint32_t d;
  asm("max.f16x2 %0, %1, %2;" : "=r"(d) : "r"(a), "r"(b));
  return d;
}
[[maybe_unused]] __device__ __forceinline__ uint32_t hmin2(uint32_t a, uint32_t b) {
  uint32_t d;
  asm("min.f16x2 %0, %1, %2;" : "=r"(d) : "r"(a), "r"(b));
  return d;
}
// Half-word pair add h + s on the FMA pipe (IMAD h * one + s).  Exact with no carry
// between the halves because every stored H half is in [kW16, kTop16] and every s half in
// [0, 127]: a low-half sum stays below 0xFFFF (negative halves, AGATHA_POS16 = 0) or
// below 0x7BFF (positive halves, AGATHA_POS16 = 1), so it never carries.
__device__ __forceinline__ uint32_t add16x2_fma(uint32_t h, uint32_t s, uint32_t one) {
  uint32_t d;
  asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(d) : "r"(h), "r"(one), "r"(s));
  return d;
}
__device__ __forceinline__ uint32_t vaddmax2(uint32_t a, uint32_t b, uint32_t c) {
  return __viaddmax_s16x2(a, b, c);
}

struct State16 {
  int m, n, mn, dlo, D, alpha, beta, zdrop;
  int B;                      // stored = X + alpha*c - B
  int G_H, G_c, G_i, G_j, G_d;  // G_H = INT_MIN/2 until the first cell (no global max yet)
  int zthr;                   // G_H - Z (INT_MIN when Z is off or there is no G yet)
  bool posValid;
  int snapB, snapPar, snapTlo, snapThi;
  int posC;                   // SNAPSLIM: G_i, G_j, G_d hold the position of G at anti-diagonal posC
  int zeff;                   // SNAPSLIM: Z, or 2^30 when Z-drop is off
  int term;
};

// First slot of this lane (in slot order: low halves, then high halves) whose value
// equals v, among the NREG/2 registers r[] of parity P; 99 if none.
// Only cells t in [tlo, thi] (in the table) are candidates: held boundary values and
// out-of-table cells of a masked step must never be taken for the argmax.
template <int NREG>
__device__ __forceinline__ int first_slot16(const uint32_t (&r)[NREG / 2], int v, int tlo, int thi) {
  int first = 99;
#pragma unroll
  for (int s = NREG / 2 - 1; s >= 0; --s)
    if (hi16(r[s]) == v && NREG / 2 + s >= tlo && NREG / 2 + s <= thi) first = NREG / 2 + s;
#pragma unroll
  for (int s = NREG / 2 - 1; s >= 0; --s)
    if (lo16(r[s]) == v && s >= tlo && s <= thi) first = s;
  return first;
}

// Warp argmax over first_slot16 results -> diagonal d of the smallest (lane, slot).
template <int NREG>
__device__ __forceinline__ int argmax_diag16(int first, int P, int dlo) {
  const unsigned bal = __ballot_sync(kFull, first < 99);
  const int ls = __ffs(bal) - 1;
  const int tt = __shfl_sync(kFull, first, ls);
  const int slot = (tt < NREG / 2) ? P + 2 * tt : NREG + P + 2 * (tt - NREG / 2);
  return dlo + ls * (2 * NREG) + slot;
}

// Split layout (align_pair16s): low halves hold slots lane*NREG + j of
// the first 32*NREG slots, high halves the same of the next 32*NREG, so the cell of a
// high half lies HV = 16*NREG positions further along the anti-diagonal than its low
// half.  Cells are numbered t = k (low) and t = HV + k (high) for the [tlo, thi] range.
// The smallest d (smallest i) holding v: the lowest lane with a low-half candidate, else
// the lowest lane with a high-half candidate.
template <int NREG>
__device__ __forceinline__ int argmax_diag16s(const uint32_t (&r)[NREG / 2], int v, int tlo, int thi, int P,
                                              int dls) {
  constexpr int HS = 32 * NREG, HV = HS / 2;
  int flo = 99, fhi = 99;
#pragma unroll
  for (int k = NREG / 2 - 1; k >= 0; --k) {
    if (lo16(r[k]) == v && k >= tlo && k <= thi) flo = k;
    if (hi16(r[k]) == v && HV + k >= tlo && HV + k <= thi) fhi = k;
  }
  unsigned bal = __ballot_sync(kFull, flo < 99);
  int half = 0, first = flo;
  if (bal == 0u) {
    bal = __ballot_sync(kFull, fhi < 99);
    half = 1;
    first = fhi;
  }
  const int ls = __ffs(bal) - 1;
  const int tt = __shfl_sync(kFull, first, ls);
  return dls + half * HS + ls * NREG + P + 2 * tt;
}
template <int NREG, bool SPLIT>
__device__ __forceinline__ int argmax16(const uint32_t (&r)[NREG / 2], int v, int tlo, int thi, int P, int dls) {
  if (SPLIT) return argmax_diag16s<NREG>(r, v, tlo, thi, P, dls);
  return argmax_diag16<NREG>(first_slot16<NREG>(r, v, tlo, thi), P, dls);
}

// Word of the deferred-argmax snapshot holding register k (of one parity) of `lane`.
template <int NREG>
__device__ __forceinline__ int snap_word(int k, int lane) {
  if (AGATHA_SNAP128 && NREG >= 8) return (k >> 2) * 128 + lane * 4 + (k & 3);
  if (AGATHA_SNAP128 && NREG == 4) return lane * 2 + k;
  return k * 32 + lane;
}

template <int NREG, int PARC>
__device__ __forceinline__ void store_snapshot(uint32_t* snap, const uint32_t (&H)[NREG], int lane) {
  if (AGATHA_SNAP128 && NREG >= 8) {
#pragma unroll
    for (int q = 0; q < NREG / 8; ++q)
      reinterpret_cast<uint4*>(snap)[q * 32 + lane] =
          make_uint4(H[PARC + 8 * q], H[PARC + 8 * q + 2], H[PARC + 8 * q + 4], H[PARC + 8 * q + 6]);
  } else if (AGATHA_SNAP128 && NREG == 4) {
    reinterpret_cast<uint2*>(snap)[lane] = make_uint2(H[PARC], H[PARC + 2]);
  } else {
#pragma unroll
    for (int k = 0; k < NREG / 2; ++k) snap[k * 32 + lane] = H[PARC + 2 * k];
  }
}

template <int NREG, bool SPLIT = false>
__device__ __forceinline__ void resolve_G16(State16& s, const uint32_t* snap, int lane) {
  int par, tlo, thi;
  if (AGATHA_SNAPSLIM) {
    if (s.posC == s.G_c) return;
    // the snapshot's anti-diagonal c = G_c: register parity and in-table cell range of this
    // lane, as the masked steps compute them (step PAR = 0 holds c = 2u - dlo)
    const int c = s.G_c;
    par = (c - s.dlo) & 1;
    const int u = (c - par + s.dlo) >> 1;
    constexpr int LC = SPLIT ? NREG / 2 : NREG;  // positions per lane along the anti-diagonal
    const int ib = u + par + lane * LC, jb = u - s.dlo - lane * LC;
    tlo = max(1 - ib, jb - s.n);
    thi = min(s.m - ib, jb - 1);
    s.posC = c;
  } else {
    if (s.posValid) return;
    par = s.snapPar;
    tlo = s.snapTlo;
    thi = s.snapThi;
  }
  uint32_t r[NREG / 2];
#pragma unroll
  for (int k = 0; k < NREG / 2; ++k) r[k] = snap[snap_word<NREG>(k, lane)];
  const int v = s.G_H + s.alpha * s.G_c - s.snapB;
  const int d = argmax16<NREG, SPLIT>(r, v, tlo, thi, par, s.dlo);
  s.G_d = d;
  s.G_i = (s.G_c + d) >> 1;
  s.G_j = s.G_c - s.G_i;
  s.posValid = true;
}

// Eq. 4 / Eq. 6 for anti-diagonal c (slot parity PARC), whose registers H[PARC+2k] are
// still intact (relative to the current base s.B); rH is the warp max relative to Bc.
// Fast path: three compares and one vote; the argmax work runs only when the global max
// moves (deferred snapshot) or when Eq. 4 could fire.
template <int NREG, int PARC, bool TRACE, bool STEADY, bool SPLIT = false>
__device__ __forceinline__ bool process16(State16& s, const AlignArgs& A, int c, int rH, int Bc,
                                          int tlo, int thi, const uint32_t (&H)[NREG], int lane,
                                          uint32_t* snap, long long pid) {
  // Empty anti-diagonals are skipped (R11).  Inside the steady phase (STEADY: the
  // anti-diagonal and the one before it lie inside the table, D >= 2) no anti-diagonal
  // is empty and c < m + n, so the fast path is two compares.
  const bool nonempty = (STEADY && !TRACE) || rH > kEmpty16;
  const int Hs = rH + Bc - s.alpha * c;
  const bool upd = nonempty && Hs > s.G_H;
  const bool chk = nonempty && Hs < s.zthr && ((STEADY && !TRACE) || c < s.mn);
  // upd and chk are warp-uniform (rH is a warp reduction, the rest is per-pair state):
  // a plain uniform branch, no vote
  if ((NREG >= 16) ? AGATHA_VOTE : AGATHA_VOTE_NARROW) {
    if (!__any_sync(kFull, upd || chk || (TRACE && nonempty))) return false;
  } else if (!(upd || chk || (TRACE && nonempty))) {
    return false;
  }
  if (TRACE || chk) {
    uint32_t r[NREG / 2];
#pragma unroll
    for (int k = 0; k < NREG / 2; ++k) r[k] = H[PARC + 2 * k];
    const int d = argmax16<NREG, SPLIT>(r, Hs + s.alpha * c - s.B, tlo, thi, PARC, s.dlo);
    const int i = (c + d) >> 1, j = c - i;
    if (TRACE && pid == A.trace_pair && lane == 0 && c < A.trace_cap) {
      A.trace_score[c] = Hs;
      A.trace_i[c] = i;
    }
    if (chk) {
      resolve_G16<NREG, SPLIT>(s, snap, lane);
      const bool gated = (A.variant & AGATHA_VAR_GATE_GE) ? (s.G_i <= i && s.G_j <= j)
                                                           : (s.G_i < i && s.G_j < j);
      if (gated) {
        const int gap = d - s.G_d;
        if (s.G_H - Hs > s.zdrop + s.beta * (gap < 0 ? -gap : gap)) {
          s.term = c;
          return true;
        }
      }
    }
  }
  if (upd) {
    // defer the argmax: keep the anti-diagonal's registers (one per lane) in shared memory
    store_snapshot<NREG, PARC>(snap, H, lane);
    s.snapB = s.B;
    s.G_H = Hs;
    s.G_c = c;
    if (AGATHA_SNAPSLIM) {
      s.zthr = Hs - s.zeff;
    } else {
      s.snapPar = PARC;
      s.snapTlo = tlo;
      s.snapThi = thi;
      s.zthr = s.zdrop >= 0 ? Hs - s.zdrop : INT_MIN;
      s.posValid = false;
    }
  }
  return false;
}

// One anti-diagonal step on the NREG/2 registers of parity PAR.  S2[k] holds the
// shifted substitution scores (S + 2alpha) of register PAR+2k as a half-word pair.
// MASKED (head and tail anti-diagonals): cells outside the table are computed like the
// others and only excluded from the max (Eq. 5).  Their substitution score is 0 (the
// out-of-range nibble code, see combine), which makes every cell before the table hold
// exactly the boundary value of reading R2 with E/F at most H - (alpha - beta), so the
// cells a valid cell reads are exact without any select ("Masking").
//
// Band walls (DESIGN.md §6.1 "Layout"): the band's low end sits at lane 0 slot `off`;
// the `off` slots under it are padding that the caps of registers < NCAP hold at
// kCapNeg16.  Its high end is NREG-aligned, so the wall there is a half-word of the
// PAR = 1 exchange (KEEPX clears it to -inf in the one lane that needs it), and the slots
// above it are never read by a band cell; LMK removes them from the lane max.
// Pure min/max steps as fp16x2 HMNMX2 (AGATHA_POS16 only): bit 0 the padding caps, bit 1
// the lane max of the two halves.  Measured: HMNMX2 issues on the ALU pipe like
// VIMNMX.S16x2 (profiles/r02_hmnmx.jsonl), and with both bits ptxas allots 164 registers
// and C2 falls 3592 -> 3400 GCUPS, so the default is 0.
#ifndef AGATHA_HMAX
#define AGATHA_HMAX 0
#endif
#ifndef AGATHA_PIN_CONSTS
#define AGATHA_PIN_CONSTS 0
#endif
#if AGATHA_POS16 && (AGATHA_HMAX & 1)
#define HCAP(a, b) hmin2(a, b)
#else
#define HCAP(a, b) vmin2(a, b)
#endif
#if AGATHA_POS16 && (AGATHA_HMAX & 2)
#define HLMAX(a, b) hmax2(a, b)
#else
#define HLMAX(a, b) vmax2(a, b)
#endif

// Hout: the registers of parity PAR written by this step; Hd: the same registers two
// anti-diagonals back (the diagonal term); Hn: the other parity, one anti-diagonal back
// (the neighbours).  The loop passes one array three times (each step updates its parity
// in place); a double-buffered front was measured 32% slower.
// Padding below the band (DESIGN.md §6.1 "Layout"): NCAP < 100 caps registers 0..NCAP-1
// every step (any off <= NCAP); NCAP = 100 + off ("pinned", every pair of the launch has
// this off) caps only slot off-1, the one padding slot a band cell reads: its H, E and F
// every step, and the dead slots under it only at each re-centring (their growth between
// re-centrings is bounded on the host, pin16_ok), so they stay below kEmpty16.
template <int NCAP> struct CapMode {
  static constexpr bool pin = NCAP >= 100;
  static constexpr int off = pin ? NCAP - 100 : 0;
  static constexpr int ncap = pin ? 1 : NCAP;  // cap words held
};
#ifndef AGATHA_REDUX2
#define AGATHA_REDUX2 0  // 1: warp max of both halves as two REDUX (no VIMNMX half merge)
#endif

template <int NREG, int NCAP, int PAR, bool MASKED, bool SPLIT = false>
__device__ __forceinline__ uint32_t step16(uint32_t (&Hout)[NREG], const uint32_t (&Hd)[NREG], const uint32_t (&Hn)[NREG],
                                      uint32_t (&E)[NREG], uint32_t (&F)[NREG],
                                      const uint32_t (&CAP)[CapMode<NCAP>::ncap], const uint32_t (&S2)[NREG / 2],
                                      uint32_t AmB2, int lane, uint32_t V2, uint32_t k65536,
                                      uint32_t one, uint32_t KEEPX, uint32_t LMK, uint32_t SEL0 = 0u) {
  const uint32_t W2 = pack2(kW16, kW16);
  uint32_t xH, xEF;
  if (SPLIT) {
    // split layout: register 0's up neighbours are lane-1's register NREG-1 (both halves;
    // lane 0: the wall and lane 31's low half), register NREG-1's left neighbours are
    // lane+1's register 0 (lane 31: lane 0's high half and the wall); the walls of the
    // band come in through the per-lane byte selectors SEL0 / KEEPX (= SEL1)
    if (PAR == 0) {
      const uint32_t vh = __shfl_sync(kFull, Hn[NREG - 1], (lane + 31) & 31);
      const uint32_t ve = __shfl_sync(kFull, E[NREG - 1], (lane + 31) & 31);
      xH = prmt(vh, W2, SEL0);
      xEF = prmt(ve, W2, SEL0);
    } else {
      const uint32_t vh = __shfl_sync(kFull, Hn[0], (lane + 1) & 31);
      const uint32_t vf = __shfl_sync(kFull, F[0], (lane + 1) & 31);
      xH = prmt(vh, W2, KEEPX);
      xEF = prmt(vf, W2, KEEPX);
    }
  } else if (PAR == 0) {  // register 0: (lane-1's slot K-1, own slot NREG-1) from register NREG-1
    uint32_t sh = __shfl_up_sync(kFull, Hn[NREG - 1], 1);
    uint32_t se = __shfl_up_sync(kFull, E[NREG - 1], 1);
    if (lane == 0) { sh = W2; se = W2; }
    xH = prmt(sh, Hn[NREG - 1], 0x5432);
    xEF = prmt(se, E[NREG - 1], 0x5432);
  } else {         // register NREG-1: (own slot NREG, lane+1's slot 0) from register 0
    const uint32_t sh = __shfl_down_sync(kFull, Hn[0], 1);
    const uint32_t sf = __shfl_down_sync(kFull, F[0], 1);
    xH = (prmt(Hn[0], sh, 0x5432) & KEEPX) | (W2 & ~KEEPX);
    xEF = (prmt(F[0], sf, 0x5432) & KEEPX) | (W2 & ~KEEPX);
  }
  uint32_t lm = W2, prev = W2;
  uint32_t hv[NREG / 2];
#pragma unroll
  for (int k = 0; k < NREG / 2; ++k) {
    const int j = PAR + 2 * k;
    const uint32_t hu = (j == 0) ? xH : Hn[j - 1];
    const uint32_t eu = (j == 0) ? xEF : E[j - 1];
    const uint32_t hl = (j == NREG - 1) ? xH : Hn[j + 1];
    const uint32_t fl = (j == NREG - 1) ? xEF : F[j + 1];
    uint32_t e = vaddmax2(eu, AmB2, hu);                       // Eq. 2 (shifted)
    uint32_t f = vaddmax2(fl, AmB2, hl);                       // Eq. 3 (shifted)
#if AGATHA_FMA_ADD
    uint32_t h = __vimax3_s16x2(add16x2_fma(Hd[j], S2[k], one), e, f);  // Eq. 1 (shifted)
#else
    uint32_t h = vaddmax2(Hd[j], S2[k], vmax2(e, f));                    // Eq. 1 (shifted)
#endif
    if (CapMode<NCAP>::pin) {
      if (j == CapMode<NCAP>::off - 1) {  // slot off-1 (lane 0): the only padding a band cell reads
        h = vmin2(h, CAP[0]);
        e = vmin2(e, CAP[0]);
        f = vmin2(f, CAP[0]);
      }
    } else if (j < NCAP) {
      h = HCAP(h, CAP[j < NCAP ? j : 0]);                      // padding slots stay <= kCapNeg16
    }
    Hout[j] = h;
    E[j] = e;
    F[j] = f;
    if (MASKED) {
      // V2 bit k: cell t = k in the table; bit 16+k: cell t = k + NREG/2 in the table
      const uint32_t M = ((V2 >> k) & 0x00010001u) * 0xFFFFu;
      h = (h & M) | (W2 & ~M);
    }
    if (AGATHA_LMTREE && NREG == 16) {
      hv[k] = h;
    } else {
      if (k & 1) lm = __vimax3_s16x2(lm, prev, h); else prev = h;  // Eq. 5, per half
    }
  }
  if (AGATHA_LMTREE && NREG == 16) {  // depth 2: max3(max3(h0..h2), max3(h3..h5), max(h6, h7))
    lm = __vimax3_s16x2(__vimax3_s16x2(hv[0], hv[1], hv[2]), __vimax3_s16x2(hv[3], hv[4], hv[5]),
                        vmax2(hv[6], hv[7 % (NREG / 2)]));
  }
  if ((NREG / 2) & 1) lm = vmax2(lm, prev);
  lm = (lm & LMK) | (W2 & ~LMK);  // slots above the band's high wall
  // max of the two halves as an int32: hi16_fma gives (sign(hi) = -1 : hi), and every
  // H half is negative (<= kTop16), so the pair max is (-1 : max(lo, hi)), which read as
  // an int32 is exactly max(lo, hi)
  if (AGATHA_REDUX2) return lm;  // warp_max16 reduces both halves
#if AGATHA_LMSHL
  // (lm << 16 as a full-rate IMAD): the high half becomes max(hi, lo) and the low half
  // max(lo, 0) (= 0 for negative halves, lo for AGATHA_POS16), so the high half of the
  // lane value is max(lo, hi) and the warp max is recovered by one uniform arithmetic
  // shift after the REDUX (LANEMAX16); the low half only breaks ties between lanes
  return HLMAX(lm, lm * k65536);
#else
  return vmax2(lm, (uint32_t)hi16_fma(lm, k65536));
#endif
}

// Warp max (Eq. 5) of one step's lane value (step16's return)
__device__ __forceinline__ int warp_max16(uint32_t lv, uint32_t k65536) {
  if (AGATHA_REDUX2) {  // lv = the masked lane max pair: one REDUX per half
    const int a = __reduce_max_sync(kFull, (int)lv);              // max hi (ties by lo)
    const int b = __reduce_max_sync(kFull, (int)(lv * k65536));   // max lo
    return (a > b ? a : b) >> 16;
  }
  return LANEMAX16(__reduce_max_sync(kFull, (int)lv));
}

template <int NREG, bool TRACE, int NCAP, bool ENDS = false>
__device__ void align_pair16(const AlignArgs& A, uint32_t pid, int lane, uint32_t* snap, uint32_t* pref,
                             int unit, int* erec) {
  constexpr int K = 2 * NREG;        // slots per lane
  constexpr int NC = NREG;           // cells per step per lane (K/2)
  const PairSrc ps = pair_src(A.own, A.ref_ascii, A.qry_ascii, A.roff, A.qoff, pid);
  const uint64_t r0 = ps.r0, q0 = ps.q0;
  const int m = (int)ps.m;
  const int n = (int)ps.n;
  if (A.bad[pid]) {
    if (lane == 0) {
      agatha_result_t z = {0, 0, 0, -1, 0};
      A.out[pid] = z;
    }
    return;
  }
  const int bl = (A.bl < 0 || A.bl > n) ? n : A.bl;
  const int br = (A.br < 0 || A.br > m) ? m : A.br;
  const int alpha = A.alpha, beta = A.beta;
  // Slot layout: slot g (lane g / K, slot g % K) holds diagonal dls + g.  The band
  // [dlo, dhi] occupies slots [off, off + D) with off = (-D) mod NREG, so its high end
  // off + D falls on a half-word boundary (a cheap wall) and the low padding fits in the
  // first `off` <= NCAP registers of lane 0 (the capped ones).
  const int Dband = bl + br + 1;
  const int off = (int)__reduce_max_sync(kFull, (unsigned)((-Dband) & (NREG - 1)));
  const int dls = -bl - off;
  // Phase-aligned packing: R starts at nibble padR and Q (reversed) at nibble padQ so
  // that every lane's R window offset starts at 0 and its Q offset at 7; both windows
  // then advance one word together every 8 iterations (one refill point, not two).
  const int u0 = ((dls & 1) + dls) >> 1;  // u of the first step (cb = dls mod 2, below)
  const int padR = (1 - u0) & 7;
  const int padQ = (7 - (n + dls - u0)) & 7;
  uint32_t* Rw = A.rw + (uint64_t)(A.unit_base + unit) * A.rstride;
  uint32_t* Qw = A.qw + (uint64_t)(A.unit_base + unit) * A.qstride;
  const int nwR = (m + padR + 7) >> 3, nwQ = (n + padQ + 7) >> 3;
  pack_pair_fused(ps.ref, ps.qry, r0, q0, m, n, Rw, Qw, A.ready, A.chunk_of[pid],
                  A.nmap != 0, A.err_flags, lane, padR, padQ);

  State16 s;
  s.m = m; s.n = n; s.dlo = dls; s.D = Dband; s.alpha = alpha; s.beta = beta;
  s.mn = (A.variant & AGATHA_VAR_CHECK_LAST) ? m + n + 1 : m + n;  // Eq. 4 tested for c < mn
  s.zdrop = A.zdrop; s.B = -A.ref16; s.posValid = true;  // stored = X + alpha*c + ref16
  s.G_H = INT_MIN / 2; s.G_c = 0; s.G_i = 0; s.G_j = 0; s.G_d = 0; s.zthr = INT_MIN;
  if (A.variant & AGATHA_VAR_ORIGIN_MAX) {  // G = H(0,0) = 0 at the origin
    s.G_H = 0;
    s.zthr = A.zdrop >= 0 ? -A.zdrop : INT_MIN;
  }
  s.snapB = 0; s.snapPar = 0; s.snapTlo = 0; s.snapThi = 0; s.term = -1;
  s.posC = 0;  // = G_c: the initial position (none, or the origin) is resolved
  s.zeff = A.zdrop >= 0 ? A.zdrop : (1 << 30);
  const int dlo = -bl, D = Dband;
  const uint32_t AmB2 = pack2(alpha - beta, alpha - beta);
  const int gend = off + D;  // first slot above the band (a multiple of NREG)
  const bool wall_lo = (gend & (K - 1)) == NREG && lane == gend / K;
  const bool wall_hi = lane == 31 || ((gend & (K - 1)) == 0 && lane == gend / K - 1);
  const uint32_t KEEPX = (wall_lo ? 0u : 0xFFFFu) | (wall_hi ? 0u : 0xFFFF0000u);
  const uint32_t LMK = (K * lane + K <= gend) ? 0xFFFFFFFFu : (K * lane + NREG <= gend ? 0xFFFFu : 0u);

  auto fdiag = [&](int d) { return 2 * min(m, n + d) - d; };
  const int dhi = br;
  const int cs = 2 + max(bl, br);
  const int ce = min(fdiag(dlo), fdiag(dhi));
  const int dmid = min(max(m - n, dlo), dhi);
  const int c_last = fdiag(dmid);

  // The first step computes anti-diagonal cb = 0 (even dlo) or 1 (odd dlo): the origin
  // and the first boundary cells come out of the DP itself, which starts the two gap
  // chains along the boundary (E of (i,0), F of (0,j)) that the masked steps carry.
  int cb = dls & 1;
  int u = (cb + dls) >> 1;
  // boundary value of diagonal d (reading R2); slots beyond the band hold the cap
  auto bnd = [&](int d) { const int ad = d < 0 ? -d : d; return d == 0 ? 0 : -(alpha + (ad - 1) * beta); };

  // a3: slot k of register j (j or j+NREG) on diagonal dls + K*lane + k; a slot of
  // parity(cb) holds anti-diagonal cb-2, the other parity cb-1 (both <= 0).  Slots start
  // at bnd(d) + alpha*c (stored units), diagonal 0 at the origin value 0, E/F at -inf;
  // DESIGN.md §6.2 "Masking" shows these reproduce the boundary exactly.
  uint32_t H[NREG], E[NREG], F[NREG], CAP[CapMode<NCAP>::ncap];
  const uint32_t W2 = pack2(kW16, kW16);
#pragma unroll
  for (int j = 0; j < NREG; ++j) {
    int v2[2], c2[2];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int k = j + h * NREG, g = K * lane + k, d = dls + g;
      const bool valid = g >= off && g < gend;
      c2[h] = valid ? kTop16 + 127 : kCapNeg16;  // no cap: the largest live value
      const int ci = ((k & 1) == 0) ? cb - 2 : cb - 1;  // (dls + K*lane) has parity of cb
      v2[h] = valid ? (d == 0 ? 0 : bnd(d) + alpha * ci) - s.B : kCapNeg16;
    }
    H[j] = pack2(v2[0], v2[1]);
    if (!CapMode<NCAP>::pin && j < NCAP) CAP[j < NCAP ? j : 0] = pack2(c2[0], c2[1]);
    E[j] = W2;
    F[j] = W2;
  }
  if (CapMode<NCAP>::pin) CAP[0] = pack2(lane == 0 ? kCapNeg16 : 0x7FFF, 0x7FFF);

  int rpos = u - 1 + padR + lane * NC;
  int wR = rpos >> 3, oR = rpos & 7;  // oR = 0
  uint32_t Wr0 = load_word_rw(Rw, wR, nwR), Wr1 = load_word_rw(Rw, wR + 1, nwR),
           Wr2 = load_word_rw(Rw, wR + 2, nwR);
  int qpos = n + dls - u + padQ + lane * NC;
  int wQ = qpos >> 3, oQ = qpos & 7;  // oQ = 7 = 7 - oR from here on
  uint32_t Wq0 = load_word_rw(Qw, wQ, nwQ), Wq1 = load_word_rw(Qw, wQ + 1, nwQ),
           Wq2 = load_word_rw(Qw, wQ + 2, nwQ);
  // the words the next refill needs are copied global -> shared asynchronously (no
  // registers held, the load latency hides behind 8 iterations)
  auto prefetch = [&]() {
    const uint32_t* gr = Rw + min(max(wR + 3 + 1, 0), nwR + 1);
    const uint32_t* gq = Qw + min(max(wQ - 1 + 1, 0), nwQ + 1);
    const unsigned sr = (unsigned)__cvta_generic_to_shared(pref + lane);
    const unsigned sq = (unsigned)__cvta_generic_to_shared(pref + 32 + lane);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" :: "r"(sr), "l"(gr) : "memory");
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" :: "r"(sq), "l"(gq) : "memory");
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  prefetch();

#if AGATHA_PIN_CONSTS
  // pinned in vector registers: a volatile copy cannot be rematerialised, so ptxas keeps
  // the table words instead of re-copying them from uniform registers before every lookup
  uint32_t T0, T1, k65536, one;
  asm volatile("mov.b32 %0, %1;" : "=r"(T0) : "r"(A.T16_0));
  asm volatile("mov.b32 %0, %1;" : "=r"(T1) : "r"(A.T16_1));
  asm volatile("mov.b32 %0, %1;" : "=r"(k65536) : "r"(A.k65536));
  asm volatile("mov.b32 %0, %1;" : "=r"(one) : "r"(A.one));
#else
  const uint32_t T0 = A.T16_0, T1 = A.T16_1, k65536 = A.k65536, one = A.one;
#endif
  const int ref16 = -s.B;
  int rH_prev = kEmpty16 - 1, B_prev = s.B, tlo_prev = 0, thi_prev = NC - 1;
  bool stop = false;
  int iters = 0;

  // substitution pairs (cells t, t+NC/2) of one step, from the nibble windows
  // rs: the R window shifted to the step's first cell (rshift)
  auto scores = [&](uint32_t (&S2)[NREG / 2], const uint32_t (&rs)[2], const uint32_t (&qg)[2]) {
    if (NREG == 16) {
      const uint32_t x0 = combine(rs[0], qg[0]);
      const uint32_t x1 = combine(rs[1], qg[1]);
      const uint32_t a0 = prmt(T0, T1, x0), a1 = prmt(T0, T1, shr16_fma(x0, k65536));
      const uint32_t b0 = prmt(T0, T1, x1), b1 = prmt(T0, T1, shr16_fma(x1, k65536));
#pragma unroll
      for (int k = 0; k < NREG / 2; ++k) {
        const uint32_t b = (uint32_t)(k & 3);
        S2[k] = prmt(k < 4 ? a0 : a1, k < 4 ? b0 : b1, b | ((b | 8) << 4) | ((4 + b) << 8) | (((4 + b) | 8) << 12));
      }
    } else if (NREG == 8) {  // cells 0..7 in one word, pairs (t, t+4)
      const uint32_t x0 = combine(rs[0], qg[0]);
      const uint32_t a0 = prmt(T0, T1, x0), a1 = prmt(T0, T1, shr16_fma(x0, k65536));
#pragma unroll
      for (int k = 0; k < NREG / 2; ++k) {
        const uint32_t b = (uint32_t)k;
        S2[k] = prmt(a0, a1, b | ((b | 8) << 4) | ((4 + b) << 8) | (((4 + b) | 8) << 12));
      }
    } else {  // NREG == 4 (narrow tier): cells 0..3 from the low half-word, pairs (t, t+2)
      const uint32_t x0 = combine(rs[0], qg[0]);
      const uint32_t a0 = prmt(T0, T1, x0);
#pragma unroll
      for (int k = 0; k < NREG / 2; ++k) {
        const uint32_t b = (uint32_t)k;
        S2[k] = prmt(a0, 0u, b | ((b | 8) << 4) | ((2 + b) << 8) | (((2 + b) | 8) << 12));
      }
    }
  };
  // bit t (t < NC/2) and bit 16 + t - NC/2 (t >= NC/2) set for the cells t in [tlo, thi]
  auto valid_bits = [&](int tlo, int thi) {
    const int lo = max(tlo, 0), hi = min(thi, NC - 1);
    if (hi < lo) return 0u;
    const uint32_t v = ((hi >= 31) ? 0xFFFFFFFFu : ((1u << (hi + 1)) - 1u)) & ~((1u << lo) - 1u);
    return (v & ((1u << (NC / 2)) - 1u)) | ((v >> (NC / 2)) << 16);
  };

  auto rshift = [&](uint32_t (&rs)[2], int sh) {
    rs[0] = __funnelshift_rc(Wr0, Wr1, sh);
    if (NREG == 16) rs[1] = __funnelshift_rc(Wr1, Wr2, sh);
  };
  // The R window shifted for the PAR = 1 step (4*oR + 4) is the next iteration's PAR = 0
  // shift (oR advances by one), also across a refill: the clamped shift by 32 returns
  // the second word, which the refill makes the first.
  // NEXT #4: the end cells of processed anti-diagonal c (slot parity P, registers still
  // intact, relative to the base Bc of their step)
  if (ENDS) {
    if (lane == 0) ends_init(erec);
    __syncwarp();
  }
  auto capture = [&](const uint32_t (&H)[NREG], int c, int P, int Bc) {
    const int uc = (c - P + dls) >> 1;
    const int ib = uc + P + lane * NC, jb = uc - dls - lane * NC;
    ends_capture(erec, ib, jb, NC, m, n,
                 [&](int t) {
                   const int tk = t % (NC / 2);
                   uint32_t v = 0;
#pragma unroll
                   for (int k = 0; k < NREG / 2; ++k)
                     if (k == tk) v = P ? H[1 + 2 * k] : H[2 * k];
                   const int st = t >= NC / 2 ? hi16(v) : lo16(v);
                   return st - alpha * c + Bc;  // stored = X + alpha*c - B
                 },
                 [&](int t) {
                   const int g = K * lane + (t >= NC / 2 ? NREG : 0) + P + 2 * (t % (NC / 2));
                   return g >= off && g < gend;
                 });
    __syncwarp();
  };
  constexpr bool kRReuse = NREG >= 16 ? AGATHA_RREUSE : AGATHA_RREUSE_NARROW;
  uint32_t rsc[2] = {0u, 0u};
  rshift(rsc, 4 * oR);
  auto iteration = [&](auto masked_tag) {
    constexpr bool MASKED = decltype(masked_tag)::value;
    uint32_t qg[2], S2[NREG / 2], V2 = 0u, rs[2];
    const int oq4 = AGATHA_LOOPSLIM ? 28 - 4 * oR : 4 * oQ;
    qg[0] = __funnelshift_rc(Wq0, Wq1, oq4);
    qg[1] = __funnelshift_rc(Wq1, Wq2, oq4);
#if AGATHA_S2EARLY
    // both steps' scores up front: the PAR = 1 lookups (with their long-latency IMAD.HI)
    // then issue under the PAR = 0 cells instead of stalling in front of PAR = 1
    uint32_t S2b[NREG / 2];
    rshift(rs, 4 * oR + 4);
    scores(S2b, rs, qg);
#endif
    // ---- step PAR = 0, anti-diagonal cb ----
    {
      if (kRReuse) {
        scores(S2, rsc, qg);
      } else {
        rshift(rs, 4 * oR);
        scores(S2, rs, qg);
      }
      int tlo = 0, thi = NC;
      if (MASKED) {
        const int uu = AGATHA_LOOPSLIM ? (cb + dls) >> 1 : u;
        const int ib = uu + lane * NC, jb = uu - dls - lane * NC;
        tlo = max(1 - ib, jb - n);
        thi = min(m - ib, jb - 1);
        V2 = valid_bits(tlo, thi);
      }
      const uint32_t lmax = step16<NREG, NCAP, 0, MASKED>(H, H, H, E, F, CAP, S2, AmB2, lane, V2, k65536, one, KEEPX, LMK);
      const int rH = warp_max16(lmax, k65536);
      if (MASKED && ENDS) capture(H, cb - 1, 1, B_prev);
      if (process16<NREG, 1, TRACE, !MASKED>(s, A, cb - 1, rH_prev, B_prev, tlo_prev, thi_prev, H, lane, snap, pid)) { stop = true; return; }
      rH_prev = rH;
      if (!AGATHA_STEADYC || MASKED) {
        B_prev = s.B;
        tlo_prev = MASKED ? tlo : 0;
        thi_prev = MASKED ? thi : NC - 1;
      }
    }
    // ---- step PAR = 1, anti-diagonal cb + 1 ----
    {
#if AGATHA_S2EARLY
#pragma unroll
      for (int k = 0; k < NREG / 2; ++k) S2[k] = S2b[k];
#else
      rshift(rs, 4 * oR + 4);
      scores(S2, rs, qg);
#endif
      if (kRReuse) {
        rsc[0] = rs[0];
        rsc[1] = rs[1];
      }
      int tlo = 0, thi = NC;
      if (MASKED) {
        const int uu = AGATHA_LOOPSLIM ? (cb + dls) >> 1 : u;
        const int ib = uu + 1 + lane * NC, jb = uu - dls - lane * NC;
        tlo = max(1 - ib, jb - n);
        thi = min(m - ib, jb - 1);
        V2 = valid_bits(tlo, thi);
      }
      const uint32_t lmax = step16<NREG, NCAP, 1, MASKED>(H, H, H, E, F, CAP, S2, AmB2, lane, V2, k65536, one, KEEPX, LMK);
      const int rH = warp_max16(lmax, k65536);
      if (MASKED && ENDS) capture(H, cb, 0, B_prev);
      if (process16<NREG, 0, TRACE, !MASKED>(s, A, cb, rH_prev, B_prev, tlo_prev, thi_prev, H, lane, snap, pid)) { stop = true; return; }
      rH_prev = rH;
      if (!AGATHA_STEADYC || MASKED) {
        B_prev = s.B;
        tlo_prev = MASKED ? tlo : 0;
        thi_prev = MASKED ? thi : NC - 1;
      }
    }
    cb += 2;
    if (!AGATHA_LOOPSLIM) {
      ++u;
      --oQ;
    }
    ++oR;
  };

  // Window refills (every 8 iterations for each sequence) and base re-centring happen
  // between runs of iterations whose count is computed up front, so the hot inner loop
  // carries no per-iteration refill predicates.
  auto housekeeping = [&]() {
    if (oR == 8) {  // oQ == -1 at the same time (phase-aligned packing)
      oR = 0;
      ++wR;
      oQ = 7;
      --wQ;
      asm volatile("cp.async.wait_all;" ::: "memory");
      Wr0 = Wr1; Wr1 = Wr2; Wr2 = pref[lane];
      Wq2 = Wq1; Wq1 = Wq0; Wq0 = pref[32 + lane];
      prefetch();
    }
    if (iters >= kRebase16) {  // re-centre: the last anti-diagonal max moves to ref16
      iters = 0;
      // (only the last 1-2 anti-diagonals of a pair can be empty with D >= 2; a
      // one-diagonal band, where every other one is empty, runs the 32-bit kernel)
      if (rH_prev > kEmpty16) {
        const int delta = rH_prev + B_prev - s.B - ref16;
        if (AGATHA_STEADYC) {  // the steady steps do not refresh B_prev: keep rH_prev in s.B units
          rH_prev -= delta - (B_prev - s.B);
          B_prev = s.B + delta;
        }
        const uint32_t nd2 = pack2(-delta, -delta);
#pragma unroll
        for (int j = 0; j < NREG; ++j) {
          H[j] = vaddmax2(H[j], nd2, W2);
          if (j & 1) {  // E/F of the last step's parity are the live ones
            E[j] = vaddmax2(E[j], nd2, W2);
            F[j] = vaddmax2(F[j], nd2, W2);
          }
        }
        s.B += delta;
      }
      if (CapMode<NCAP>::pin) {  // (after the shift) re-pin the dead padding slots under slot off-1
#pragma unroll
        for (int j = 0; j < CapMode<NCAP>::off - 1; ++j) {
          H[j] = vmin2(H[j], CAP[0]);
          if (j & 1) {  // E/F of the last step's parity are the live ones
            E[j] = vmin2(E[j], CAP[0]);
            F[j] = vmin2(F[j], CAP[0]);
          }
        }
      }
    }
  };
  // run `total` iterations of one phase
  int ph = 0;  // iterations so far (mod 8): lane-uniform, unlike oR when NC = 4
  auto run_phase = [&](auto masked_tag, int total) {
    while (!stop && total > 0) {
      // iters == oR (mod 8): runs end at refill / re-centring points together.  With
      // NC = 4 cells per lane, odd lanes sit half a word (oR = 4) ahead of even lanes, so
      // runs end every 4 iterations and each lane refills when its own oR reaches 8; the
      // run length must be lane-uniform (the iterations hold warp shuffles).
      int k = NC >= 8 ? 8 - oR : 4 - (ph & 3);
      k = min(k, kRebase16 - iters);
      k = min(k, total);
      ph += k;
      total -= k;
      iters += k;
#pragma unroll 1
      for (int t = 0; t < k; ++t) {
        iteration(masked_tag);
        if (stop) break;
      }
      housekeeping();
    }
  };

  {
    const int head_end = min(cs, c_last + 1);                 // head: cb < cs (and cb <= c_last)
    run_phase(TrueT{}, cb < head_end ? (head_end - cb + 1) >> 1 : 0);
    // steady: cb + 1 <= ce; with end scores it stops before ce, the first anti-diagonal
    // that can hold an end cell, so every end cell is processed by a masked step
    const int ce_s = ENDS ? ce - 1 : ce;
    run_phase(FalseT{}, cb + 1 <= ce_s ? ((ce_s - cb + 1) >> 1) : 0);
    run_phase(TrueT{}, cb <= c_last ? ((c_last - cb) >> 1) + 1 : 0);  // tail: cb <= c_last
  }
  if (!stop) {
    if (ENDS) capture(H, cb - 1, 1, B_prev);
    process16<NREG, 1, TRACE, false>(s, A, cb - 1, rH_prev, B_prev, tlo_prev, thi_prev, H, lane, snap, pid);
  }
  if (ENDS && lane == 0) ends_store(A.ends + pid, erec);
  resolve_G16<NREG>(s, snap, lane);

  const int c_end = s.term >= 0 ? s.term : m + n;
  int cnt = 0;
#pragma unroll
  for (int k = 0; k < K; ++k) {
    const int g = K * lane + k;
    if (g >= off && g < gend) {
      const int d = dls + g;
      const int clo = (d < 0 ? -d : d) + 2;
      const int hi = min(fdiag(d), c_end);
      if (hi >= clo) cnt += ((hi - clo) >> 1) + 1;
    }
  }
  cnt = (int)__reduce_add_sync(kFull, (unsigned)cnt);
  if (lane == 0) {
    agatha_result_t r;
    r.score = s.G_H;
    r.ref_end = s.G_i;
    r.query_end = s.G_j;
    r.zdrop_antidiag = s.term;
    r.cells = cnt;
    A.out[pid] = r;
  }
}

#ifndef AGATHA_SPLIT16
#define AGATHA_SPLIT16 1  // 0: the 32-slot front keeps the paired (j, j + NREG) layout
#endif
#ifndef AGATHA_SPLITLATE
#define AGATHA_SPLITLATE 0  // split front: the window shift at the end of the iteration
#endif
#ifndef AGATHA_SPLITS2E
#define AGATHA_SPLITS2E 0   // split front: both steps' score lookups at the top of the iteration
#endif
#ifndef AGATHA_STREAM_PF
#define AGATHA_STREAM_PF 256  // split front: L2 prefetch distance of the stream loads (words), 0 = none
#endif
#ifndef AGATHA_SPLITU2
#define AGATHA_SPLITU2 0  // split front: steady loop trips of two iterations
#endif
// ---- The split-layout 32-slot front (AGATHA_SPLIT16, DESIGN.md §6.1 "Split layout") ----
// Slot g of the band front lives in lane (g mod HS) / NREG, register g mod NREG, half
// g / HS (HS = 32 * NREG): the low halves of the warp hold the first HS diagonals, the
// high halves the next HS.  A lane's low and high cells of one register then sit HV =
// HS / 2 positions apart along the anti-diagonal, so each register's substitution-score
// pair (S_t, S_{t+HV}) is one table lookup of a selector pair precomputed per position:
//   P(x) = c(R_x) | 0x80 | (c(R_{x+HV}) | 0x80) << 8     (c = 4-bit code, 8 outside R)
//   W_R(x) = P(x) | P(x+1) << 16   (low: the PAR = 0 step, high: the PAR = 1 step)
//   V_Q(y) = Pq(y) | Pq(y) << 16   (Pq likewise on the reversed Q)
// combine(W_R, V_Q) holds both steps' selectors (nibbles 1 and 3 of each are 8: a zero
// byte), so a register costs one LOP3 (both steps) and one PRMT per step, with no
// funnel shifts or pair assembly.  The streams are written per pair into the work unit's
// scratch (rw / qw); each lane keeps its eight R and eight Q words of an iteration in
// registers and loads one new word of each per iteration.  Both cross-lane exchanges
// become one shuffle and one PRMT whose per-lane byte selector also inserts the walls.
constexpr int kStreamPad = 256;    // >= AGATHA_STREAM_PF
static_assert(kStreamPad >= AGATHA_STREAM_PF, "stream prefetches must stay inside a unit");
__host__ __device__ inline long long s16_len(long long mn) {  // stream words for m + n
  const long long nit = mn / 2 + 2, np = (nit + 7) / 8 + 2;
  return 8 * np + 8 * 32 + 24;
}
__host__ __device__ inline long long s16_unit_words(long long mn) {  // words + bytes, per sequence
  const long long L = s16_len(mn);
  // + kStreamPad: the Q stream starts kStreamPad words into its unit and both streams end
  // at least that far before the unit's end, so the L2 prefetches (AGATHA_STREAM_PF words
  // ahead of a read) stay inside the unit's own scratch
  return L + (L + 264 + 3) / 4 + 8 + 2 * kStreamPad;
}

// The high half of a selector word in its low half, on the FMA pipe at full rate: an
// fp16x2 add of -0.0 to the high half broadcast (HADD2 R, R.H1_H1, -RZ).  Exact: every
// selector half is 0x8?8? (nibbles 1 and 3 are 8), a finite fp16 (exponent <= 3; small
// ones are subnormal, which f16 arithmetic keeps without .ftz), and x + (-0) = x.  The
// PRMT that consumes it reads only the low 16 bits.  (IMAD.HI, the alternative on the FMA
// pipe, issues at a quarter rate.)
#ifndef AGATHA_HSWAP
#define AGATHA_HSWAP 1
#endif
__device__ __forceinline__ uint32_t hi_to_lo(uint32_t x, uint32_t k65536) {
  if (!AGATHA_HSWAP) return shr16_fma(x, k65536);
  uint32_t d;
  asm("{\n\t.reg .b16 lo, hi;\n\t.reg .b32 t, z;\n\tmov.b32 {lo, hi}, %1;\n\tmov.b32 t, {hi, hi};\n\t"
      "mov.b32 z, 0x80008000;\n\tadd.rn.f16x2 %0, t, z;\n\t}" : "=r"(d) : "r"(x));
  return d;
}
template <int NREG, bool TRACE, int NCAP, bool ENDS = false>
__device__ void align_pair16s(const AlignArgs& A, uint32_t pid, int lane, uint32_t* snap, int unit, int* erec) {
  constexpr int HS = 32 * NREG, HV = HS / 2, LC = NREG / 2;  // LC: cells per lane per half
  constexpr int K = 2 * NREG;
  const PairSrc ps = pair_src(A.own, A.ref_ascii, A.qry_ascii, A.roff, A.qoff, pid);
  const uint64_t r0 = ps.r0, q0 = ps.q0;
  const int m = (int)ps.m;
  const int n = (int)ps.n;
  if (A.bad[pid]) {
    if (lane == 0) {
      agatha_result_t z = {0, 0, 0, -1, 0};
      A.out[pid] = z;
    }
    return;
  }
  const int bl = (A.bl < 0 || A.bl > n) ? n : A.bl;
  const int br = (A.br < 0 || A.br > m) ? m : A.br;
  const int alpha = A.alpha, beta = A.beta;
  const int Dband = bl + br + 1;
  const int off = (int)__reduce_max_sync(kFull, (unsigned)((-Dband) & (NREG - 1)));
  const int dls = -bl - off;
  const int gend = off + Dband;  // first slot above the band (a multiple of NREG)

  // ---- a1: the selector streams of this pair ----
  const int cb0 = dls & 1, u0 = (cb0 + dls) >> 1;
  const int L = (int)s16_len((long long)m + n);
  const int NP = (L - 8 * 32 - 24) / 8;  // periods the streams cover
  const int ylo = n - u0 - 8 * NP - 7 + dls;
  uint32_t* WR = A.rw + (uint64_t)(A.unit_base + unit) * A.rstride;
  uint32_t* VQ = A.qw + (uint64_t)(A.unit_base + unit) * A.qstride + kStreamPad;
  {
    if (A.ready) {
      while (ld_acquire(A.ready + A.chunk_of[pid]) == 0) __nanosleep(500);
    }
    const bool nmap = A.nmap != 0;
    int err = 0;
    // every base of both sequences is validated (the streams below cover only the
    // positions the band can reach, which for very unequal lengths is not all of them)
    for (int x = lane; x < m; x += 32) base_code(ps.ref[r0 + x], nmap, &err);
    for (int x = lane; x < n; x += 32) base_code(ps.qry[q0 + x], nmap, &err);
    int err_unused = 0;
    uint32_t* BR = WR + L;  // byte codes | 0x80: BR[ix] for x = u0 + ix, BQ[iy] for y = ylo + iy
    uint32_t* BQ = VQ + L;
    const int NBW = (L + 264) / 4;
    const uint8_t* ref = ps.ref + r0;
    const uint8_t* qry = ps.qry + q0;
    for (int w = lane; w < NBW; w += 32) {
      uint32_t br4 = 0, bq4 = 0;
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        const int x = u0 + 4 * w + t;  // R position (1-based)
        uint32_t c = 8;
        if (x >= 1 && x <= m) c = base_code(ref[x - 1], nmap, &err_unused);
        br4 |= (c | 0x80u) << (8 * t);
        const int y = ylo + 4 * w + t;  // reversed-Q position: Q_{n - y}
        c = 8;
        if (y >= 0 && y < n) c = base_code(qry[n - 1 - y], nmap, &err_unused);
        bq4 |= (c | 0x80u) << (8 * t);
      }
      BR[w] = br4;
      BQ[w] = bq4;
    }
    if (__any_sync(kFull, err) && lane == 0) atomicOr(A.err_flags, 1);
    __syncwarp();
    for (int a = lane; a < L / 4; a += 32) {
      const uint32_t a0 = BR[a], a1 = BR[a + 1], c0 = BR[a + HV / 4], c1 = BR[a + HV / 4 + 1];
      const uint32_t e0 = BQ[a], e1 = BQ[a + 1], f0 = BQ[a + HV / 4], f1 = BQ[a + HV / 4 + 1];
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        const uint32_t u = __funnelshift_r(a0, a1, 8 * t), v = __funnelshift_r(c0, c1, 8 * t);
        WR[4 * a + t] = prmt(u, v, 0x5140);
        const uint32_t uq = __funnelshift_r(e0, e1, 8 * t), vq = __funnelshift_r(f0, f1, 8 * t);
        VQ[4 * a + t] = prmt(uq, vq, 0x4040);
      }
    }
    __syncwarp();
  }
  State16 s;
  s.m = m; s.n = n; s.dlo = dls; s.D = Dband; s.alpha = alpha; s.beta = beta;
  s.mn = (A.variant & AGATHA_VAR_CHECK_LAST) ? m + n + 1 : m + n;
  s.zdrop = A.zdrop; s.B = -A.ref16; s.posValid = true;
  s.G_H = INT_MIN / 2; s.G_c = 0; s.G_i = 0; s.G_j = 0; s.G_d = 0; s.zthr = INT_MIN;
  if (A.variant & AGATHA_VAR_ORIGIN_MAX) {
    s.G_H = 0;
    s.zthr = A.zdrop >= 0 ? -A.zdrop : INT_MIN;
  }
  s.snapB = 0; s.snapPar = 0; s.snapTlo = 0; s.snapThi = 0; s.term = -1;
  s.posC = 0;
  s.zeff = A.zdrop >= 0 ? A.zdrop : (1 << 30);
  const int dlo = -bl, D = Dband;
  const uint32_t AmB2 = pack2(alpha - beta, alpha - beta);
  // exchange byte selectors (prmt(v, W2, sel): bytes 0-3 of v, 4-7 of the wall W2)
  uint32_t sel0 = lane == 0 ? (0x54u | (0x10u << 8)) : 0x3210u;
  uint32_t s1lo = lane == 31 ? 0x32u : 0x10u, s1hi = lane == 31 ? 0x76u : 0x32u;
  if (gend < 2 * HS) {  // the band top's left neighbour (slot gend) is the wall
    const int gt = gend - 1;
    if (lane == (gt % HS) / NREG) {
      if (gt < HS) s1lo = 0x54u; else s1hi = 0x76u;
    }
  }
  const uint32_t sel1 = s1lo | (s1hi << 8);
  const uint32_t LMK = ((lane + 1) * NREG <= gend ? 0xFFFFu : 0u) | (HS + (lane + 1) * NREG <= gend ? 0xFFFF0000u : 0u);

  auto fdiag = [&](int d) { return 2 * min(m, n + d) - d; };
  const int dhi = br;
  const int cs = 2 + max(bl, br);
  const int ce = min(fdiag(dlo), fdiag(dhi));
  const int dmid = min(max(m - n, dlo), dhi);
  const int c_last = fdiag(dmid);
  int cb = cb0;
  auto bnd = [&](int d) { const int ad = d < 0 ? -d : d; return d == 0 ? 0 : -(alpha + (ad - 1) * beta); };

  uint32_t H[NREG], E[NREG], F[NREG], CAP[CapMode<NCAP>::ncap];
  const uint32_t W2 = pack2(kW16, kW16);
#pragma unroll
  for (int j = 0; j < NREG; ++j) {
    int v2[2], c2[2];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int g = h * HS + lane * NREG + j, d = dls + g;
      const bool valid = g >= off && g < gend;
      c2[h] = valid ? kTop16 + 127 : kCapNeg16;
      const int ci = ((g & 1) == 0) ? cb - 2 : cb - 1;
      v2[h] = valid ? (d == 0 ? 0 : bnd(d) + alpha * ci) - s.B : kCapNeg16;
    }
    H[j] = pack2(v2[0], v2[1]);
    if (!CapMode<NCAP>::pin && j < NCAP) CAP[j < NCAP ? j : 0] = pack2(c2[0], c2[1]);
    E[j] = W2;
    F[j] = W2;
  }
  if (CapMode<NCAP>::pin) CAP[0] = pack2(lane == 0 ? kCapNeg16 : 0x7FFF, 0x7FFF);

#ifndef AGATHA_SPLITPIN
#define AGATHA_SPLITPIN 1
#endif
  // the table words pinned in vector registers (a volatile copy cannot be rematerialised
  // from the uniform registers before every PRMT)
  uint32_t T0, T1;
  if (AGATHA_SPLITPIN) {
    // T0 + lane * 0 (A.one - 1 is a run-time zero): a per-lane value lives in a vector
    // register, which PRMT reads as its table operand with no copy from a uniform one
    T0 = A.T16_0 + (uint32_t)lane * (A.one - 1u);
    T1 = A.T16_1;
  } else {
    T0 = A.T16_0;
    T1 = A.T16_1;
  }
  const uint32_t k65536 = A.k65536, one = A.one;
  const int ref16 = -s.B;
  int rH_prev = kEmpty16 - 1, B_prev = s.B, tlo_prev = 0, thi_prev = HV + LC - 1;
  bool stop = false;
  int iters = 0, it = 0, itc = 0;  // itc: index of the running iteration
  const int rebase = A.rebase16;  // iterations between re-centrings (<= 128)
  uint32_t xs[NREG / 2];
  // the words of iteration `it` sit in registers, wr[k] = W_R(u + 8 lane + k)
  // and wq[k] = V_Q(n - u + dls + 8 lane + k); each iteration shifts them by one word
  // (register moves on the FMA pipe) and loads the one new word of each from the
  // stream (L1), one iteration ahead
  uint32_t wr[NREG / 2], wq[NREG / 2], nr = 0, nq = 0;
  const int iq0 = 8 * NP + 7 + 8 * lane;  // V_Q index of y(u0, k = 0)
  // the new words of the next iteration (R ascending, Q descending); advanced with a
  // 64-bit IMAD (mad.wide) on the FMA pipe
  unsigned long long nextR = (unsigned long long)(WR + 8 * lane + 8), nextQ = (unsigned long long)(VQ + iq0 - 1);
  const int oneV = (int)(one + (uint32_t)lane * (one - 1u));  // 1, per lane (not uniform)
  auto adv = [&](unsigned long long p, int by) {
    unsigned long long d;
    asm("mad.wide.s32 %0, %1, %2, %3;" : "=l"(d) : "r"(oneV), "r"(by), "l"(p));
    return d;
  };
  nr = __ldca(reinterpret_cast<const uint32_t*>(nextR));
  nq = __ldca(reinterpret_cast<const uint32_t*>(nextQ));
  nextR = adv(nextR, 4);
  nextQ = adv(nextQ, -4);
#pragma unroll
  for (int k = 0; k < NREG / 2; ++k) {
    wr[k] = WR[8 * lane + k];
    wq[k] = VQ[iq0 + k];
  }
  auto load_xs = [&]() {
#pragma unroll
    for (int k = 0; k < NREG / 2; ++k) xs[k] = combine(wr[k], wq[k]);
  };
  auto shift_win = [&](int itn) {  // -> the words of iteration itn; load those of itn + 1
    (void)itn;  // (kept: the counter shapes ptxas's loop code)
    {
#pragma unroll
      for (int k = 0; k < NREG / 2 - 1; ++k) wr[k] = wr[k + 1];
      wr[NREG / 2 - 1] = nr;
#pragma unroll
      for (int k = NREG / 2 - 1; k > 0; --k) wq[k] = wq[k - 1];
      wq[0] = nq;
      nr = __ldca(reinterpret_cast<const uint32_t*>(nextR));
      nq = __ldca(reinterpret_cast<const uint32_t*>(nextQ));
      if (AGATHA_STREAM_PF) {  // the streams' lines a few hundred iterations ahead into L2
        asm volatile("prefetch.global.L2 [%0];" :: "l"(nextR + 4 * AGATHA_STREAM_PF));
        asm volatile("prefetch.global.L2 [%0];" :: "l"(nextQ - 4 * AGATHA_STREAM_PF));
      }
      nextR = adv(nextR, 4);
      nextQ = adv(nextQ, -4);
    }
  };
  load_xs();

  // cells t in [tlo, thi] (t = k low, HV + k high) -> V2 bits k and 16 + k
  auto valid_bits = [&](int tlo, int thi) {
    auto run = [](int lo, int hi) -> uint32_t {
      lo = max(lo, 0);
      hi = min(hi, LC - 1);
      if (hi < lo) return 0u;
      return ((1u << (hi + 1)) - 1u) & ~((1u << lo) - 1u);
    };
    return run(tlo, thi) | (run(tlo - HV, thi - HV) << 16);
  };
  if (ENDS) {
    if (lane == 0) ends_init(erec);
    __syncwarp();
  }
  auto capture = [&](const uint32_t (&H)[NREG], int c, int P, int Bc) {
    const int uc = (c - P + dls) >> 1;
    const int ib = uc + P + lane * LC, jb = uc - dls - lane * LC;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      ends_capture(erec, ib + h * HV, jb - h * HV, LC, m, n,
                   [&](int t) {
                     uint32_t v = 0;
#pragma unroll
                     for (int k = 0; k < NREG / 2; ++k)
                       if (k == t) v = P ? H[1 + 2 * k] : H[2 * k];
                     const int st = h ? hi16(v) : lo16(v);
                     return st - alpha * c + Bc;
                   },
                   [&](int t) {
                     const int g = h * HS + lane * NREG + P + 2 * t;
                     return g >= off && g < gend;
                   });
    }
    __syncwarp();
  };
  auto iteration = [&](auto masked_tag) {
    constexpr bool MASKED = decltype(masked_tag)::value;
    uint32_t S2[NREG / 2], S2b[AGATHA_SPLITS2E ? NREG / 2 : 1], V2 = 0u;
    const int u = (cb + dls) >> 1;
    // ---- step PAR = 0, anti-diagonal cb ----
    {
#pragma unroll
      for (int k = 0; k < NREG / 2; ++k) S2[k] = prmt(T0, T1, xs[k]);
      if (AGATHA_SPLITS2E) {  // both steps' lookups up front; the next words right after
#pragma unroll
        for (int k = 0; k < NREG / 2; ++k) S2b[k] = prmt(T0, T1, hi_to_lo(xs[k], k65536));
        shift_win(itc + 1);
        load_xs();
      }
      int tlo = 0, thi = HV + LC - 1;
      if (MASKED) {
        const int ib = u + lane * LC, jb = u - dls - lane * LC;
        tlo = max(1 - ib, jb - n);
        thi = min(m - ib, jb - 1);
        V2 = valid_bits(tlo, thi);
      }
      const uint32_t lmax = step16<NREG, NCAP, 0, MASKED, true>(H, H, H, E, F, CAP, S2, AmB2, lane, V2, k65536, one,
                                                                sel1, LMK, sel0);
      const int rH = warp_max16(lmax, k65536);
      if (MASKED && ENDS) capture(H, cb - 1, 1, B_prev);
      if (process16<NREG, 1, TRACE, !MASKED, true>(s, A, cb - 1, rH_prev, B_prev, tlo_prev, thi_prev, H, lane, snap, pid)) { stop = true; return; }
      rH_prev = rH;
      if (!AGATHA_STEADYC || MASKED) {
        B_prev = s.B;
        tlo_prev = MASKED ? tlo : 0;
        thi_prev = MASKED ? thi : HV + LC - 1;
      }
    }
    // ---- step PAR = 1, anti-diagonal cb + 1 ----
    {
      if (AGATHA_SPLITS2E) {
#pragma unroll
        for (int k = 0; k < NREG / 2; ++k) S2[k] = S2b[k];
      } else {
#pragma unroll
        for (int k = 0; k < NREG / 2; ++k) S2[k] = prmt(T0, T1, hi_to_lo(xs[k], k65536));
      }
      if (!AGATHA_SPLITLATE && !AGATHA_SPLITS2E) {
        shift_win(itc + 1);
        load_xs();
      }
      int tlo = 0, thi = HV + LC - 1;
      if (MASKED) {
        const int ib = u + 1 + lane * LC, jb = u - dls - lane * LC;
        tlo = max(1 - ib, jb - n);
        thi = min(m - ib, jb - 1);
        V2 = valid_bits(tlo, thi);
      }
      const uint32_t lmax = step16<NREG, NCAP, 1, MASKED, true>(H, H, H, E, F, CAP, S2, AmB2, lane, V2, k65536, one,
                                                                sel1, LMK, sel0);
      const int rH = warp_max16(lmax, k65536);
      if (MASKED && ENDS) capture(H, cb, 0, B_prev);
      if (process16<NREG, 0, TRACE, !MASKED, true>(s, A, cb, rH_prev, B_prev, tlo_prev, thi_prev, H, lane, snap, pid)) { stop = true; return; }
      rH_prev = rH;
      if (!AGATHA_STEADYC || MASKED) {
        B_prev = s.B;
        tlo_prev = MASKED ? tlo : 0;
        thi_prev = MASKED ? thi : HV + LC - 1;
      }
      if (AGATHA_SPLITLATE && !AGATHA_SPLITS2E) {
        shift_win(itc + 1);
        load_xs();
      }
    }
    cb += 2;
    ++itc;
  };

  auto housekeeping = [&]() {
    if (iters >= rebase) {
      iters = 0;
      if (rH_prev > kEmpty16) {
        const int delta = rH_prev + B_prev - s.B - ref16;
        if (AGATHA_STEADYC) {
          rH_prev -= delta - (B_prev - s.B);
          B_prev = s.B + delta;
        }
        const uint32_t nd2 = pack2(-delta, -delta);
#pragma unroll
        for (int j = 0; j < NREG; ++j) {
          H[j] = vaddmax2(H[j], nd2, W2);
          if (j & 1) {
            E[j] = vaddmax2(E[j], nd2, W2);
            F[j] = vaddmax2(F[j], nd2, W2);
          }
        }
        s.B += delta;
      }
      if (CapMode<NCAP>::pin) {
#pragma unroll
        for (int j = 0; j < CapMode<NCAP>::off - 1; ++j) {
          H[j] = vmin2(H[j], CAP[0]);
          if (j & 1) {
            E[j] = vmin2(E[j], CAP[0]);
            F[j] = vmin2(F[j], CAP[0]);
          }
        }
      }
    }
  };
  auto run_phase = [&](auto masked_tag, int total) {
    while (!stop && total > 0) {
      // (register windows need no period boundary: runs end at re-centrings only)
      int k = rebase - iters;
      k = min(k, total);
      total -= k;
      iters += k;
      it += k;
      if (AGATHA_SPLITU2 && !decltype(masked_tag)::value) {
        // steady runs two iterations per trip: the window shift by two words renames
        // registers in the copies instead of moving them
#pragma unroll 1
        for (int t = 0; t + 1 < k; t += 2) {
          iteration(masked_tag);
          if (stop) break;
          iteration(masked_tag);
          if (stop) break;
        }
        if (!stop && (k & 1)) iteration(masked_tag);
      } else {
#pragma unroll 1
        for (int t = 0; t < k; ++t) {
          iteration(masked_tag);
          if (stop) break;
        }
      }
      housekeeping();
    }
  };
  {
    const int head_end = min(cs, c_last + 1);
    run_phase(TrueT{}, cb < head_end ? (head_end - cb + 1) >> 1 : 0);
    const int ce_s = ENDS ? ce - 1 : ce;
    run_phase(FalseT{}, cb + 1 <= ce_s ? ((ce_s - cb + 1) >> 1) : 0);
    run_phase(TrueT{}, cb <= c_last ? ((c_last - cb) >> 1) + 1 : 0);
  }
  if (!stop) {
    if (ENDS) capture(H, cb - 1, 1, B_prev);
    process16<NREG, 1, TRACE, false, true>(s, A, cb - 1, rH_prev, B_prev, tlo_prev, thi_prev, H, lane, snap, pid);
  }
  if (ENDS && lane == 0) ends_store(A.ends + pid, erec);
  resolve_G16<NREG, true>(s, snap, lane);

  const int c_end = s.term >= 0 ? s.term : m + n;
  int cnt = 0;
#pragma unroll
  for (int k = 0; k < K; ++k) {
    const int g = (k / NREG) * HS + lane * NREG + (k % NREG);
    if (g >= off && g < gend) {
      const int d = dls + g;
      const int clo = (d < 0 ? -d : d) + 2;
      const int hi = min(fdiag(d), c_end);
      if (hi >= clo) cnt += ((hi - clo) >> 1) + 1;
    }
  }
  cnt = (int)__reduce_add_sync(kFull, (unsigned)cnt);
  if (lane == 0) {
    agatha_result_t r;
    r.score = s.G_H;
    r.ref_end = s.G_i;
    r.query_end = s.G_j;
    r.zdrop_antidiag = s.term;
    r.cells = cnt;
    A.out[pid] = r;
  }
  (void)dlo; (void)D;
}

// Warps per block and blocks per SM of each front (A/B: AGATHA_WPB16 / AGATHA_MINB16)
#ifndef AGATHA_WPB16
#define AGATHA_WPB16 4
#endif
#ifndef AGATHA_MINB16
#define AGATHA_MINB16 3
#endif
// NREG = 8: off = (-D) mod 8 <= 7, so seven capped registers always cover the padding
#ifndef NCAP8
#define NCAP8 7
#endif
#ifndef AGATHA_MINB8
#define AGATHA_MINB8 4
#endif
#ifndef AGATHA_MINB4
#define AGATHA_MINB4 4
#endif
template <int NREG> struct Front16 {
  static constexpr int wpb = NREG >= 16 ? AGATHA_WPB16 : 4;
  static constexpr int minb = NREG >= 16 ? AGATHA_MINB16 : (NREG >= 8 ? AGATHA_MINB8 : AGATHA_MINB4);
};

// The 32-slot front may instead be built with an exact register cap (__maxnreg__) and no
// minimum-blocks bound, to run more warps per SM at the register count ptxas chose for
// 12 (A/B switch: AGATHA_MAXNREG16 = the cap, with AGATHA_WPB16 / AGATHA_MINB16 giving
// the block shape and the blocks per SM the launch assumes).
#ifndef AGATHA_MAXNREG16
#define AGATHA_MAXNREG16 0
#endif
template <int NREG, bool TRACE, int NCAP, bool ENDS = false>
__device__ __forceinline__ void align16_body(const AlignArgs& A) {
  __shared__ uint32_t snap_all[Front16<NREG>::wpb][NREG / 2 * 32];
  __shared__ uint32_t pref_all[Front16<NREG>::wpb][64];
  __shared__ int erec_all[Front16<NREG>::wpb][8];  // NEXT #4 end-score records
  constexpr bool kSplit = AGATHA_SPLIT16 && NREG == 16;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int unit = blockIdx.x * Front16<NREG>::wpb + warp, nunits = gridDim.x * Front16<NREG>::wpb;
  int k = 0;
  for (;;) {
    int q = 0;
    if (lane == 0) q = claim_next(A, unit, nunits, k);
    q = __shfl_sync(kFull, q, 0);
    if ((uint32_t)q >= A.n_pairs) break;
    if constexpr (kSplit)
      align_pair16s<NREG, TRACE, NCAP, ENDS>(A, A.order[q], lane, snap_all[warp], unit, erec_all[warp]);
    else
      align_pair16<NREG, TRACE, NCAP, ENDS>(A, A.order[q], lane, snap_all[warp], pref_all[warp], unit, erec_all[warp]);
  }
}

template <int NREG, bool TRACE, int NCAP, bool ENDS = false>
__global__ void __launch_bounds__(32 * Front16<NREG>::wpb, Front16<NREG>::minb) align16_kernel(AlignArgs A) {
  align16_body<NREG, TRACE, NCAP, ENDS>(A);
}

#if AGATHA_MAXNREG16
template <int NREG, bool TRACE, int NCAP, bool ENDS = false>
__global__ void __maxnreg__(AGATHA_MAXNREG16) align16w_kernel(AlignArgs A) {
  align16_body<NREG, TRACE, NCAP, ENDS>(A);
}
#endif

// ---- a1: pack (one warp per pair; R forward, Q reversed) ---------------------------

__global__ void pack_seq_kernel(const uint8_t* __restrict__ seq, uint64_t len, uint32_t* __restrict__ words,
                                bool rev, bool nmap, int* __restrict__ err_flags) {
  int err = 0;
  const uint64_t nw = (len + 7) / 8;
  for (uint64_t w = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; w < nw;
       w += (uint64_t)gridDim.x * blockDim.x)
    words[w] = pack_word(seq, (int64_t)len, (int64_t)w, rev, nmap, &err);
  if (err) atomicOr(err_flags, 1);
}

// ---- NEXT #1: shared-queue fingerprint check ------------------------------------------
// queue[8] holds the fingerprint of the first participant of this batch (0 = none yet);
// *err = 1 when this participant's differs.
__global__ void queue_fp_kernel(int* queue, uint32_t fp, const unsigned long long* len_hash, int* err) {
  const unsigned long long h = *len_hash;
  fp ^= (uint32_t)h ^ (uint32_t)(h >> 32);
  if (fp == 0u) fp = 1u;
  const uint32_t old = atomicCAS_system((unsigned int*)queue + 8, 0u, fp);
  *err = (old != 0u && old != fp) ? 1 : 0;
}

// ---- a2: validation + nominal work (one warp per pair) ------------------------------

struct PrepArgs {
  const uint64_t* roff;
  const uint64_t* qoff;
  Owners own;       // federated batch, or n_owners = 0
  int* max_len;     // [2] max m, max n over the batch (the packing scratch per unit), or null
  uint64_t n_pairs;
  int bl, br, alpha, beta, maxs;  // maxs = max(a, b, n)
  uint32_t* nominal;
  uint32_t* iota;
  uint8_t* bad;
  int* err_flags;   // bit 1: empty sequence, bit 2: out of range
  int* max_slots;   // max D over the batch
  int* max_off16;   // max (-D) mod 16 over the batch (align16_kernel's low padding)
  const uint64_t* chunk_first;  // nchunks + 1 pair boundaries of the input chunks
  int nchunks;
  uint8_t* chunk_of;            // out: chunk of each pair
  uint64_t* key64;              // out: dispatch key (tier << tier_shift) | (chunk << 32) | ~nominal,
                                // ascending: tier-major, chunk-major, longest first
  int tier_shift;               // 32 + chunk-id bits
  int lpt_from;                 // chunks >= lpt_from share one key group (one longest-first
                                // range): the queue reaches them after they have arrived
  int* tier_count;              // [3] pairs per slot tier (tier_of)
  int* max_off16_t0;            // max (-D) mod 16 over the pairs of tier 0
  int* off_mask16;              // OR of 1 << ((-D) mod 16) over: [0] the batch, [1] its tier 0, [8] its tier 1
  unsigned long long* len_hash; // shared queue (NEXT #1): sum over pairs of a hash of
                                // (p, m, n), the batch part of the queue fingerprint
};

__device__ __forceinline__ unsigned long long splitmix(unsigned long long z) {
  z += 0x9e3779b97f4a7c15ull;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}

// Slot tier of a pair of the 16-bit kernel (DESIGN.md §6.1 "Slot tiers"): the narrowest
// of 32 / 16 / 8 slots per lane (NREG 16 / 8 / 4) whose 32-lane front holds its D
// diagonals.  Tier 0 first in the dispatch key, so the widest pairs start first.
#ifndef AGATHA_NARROW_TIER
#define AGATHA_NARROW_TIER 1
#endif
__host__ __device__ __forceinline__ int tier_of(int64_t D) {
  return D > 512 ? 0 : ((D > 256 || !AGATHA_NARROW_TIER) ? 1 : 2);
}

__global__ void prep_kernel(PrepArgs P) {
  const int lane = threadIdx.x & 31;
  const uint64_t warp = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
  const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  for (uint64_t p = warp; p < P.n_pairs; p += nwarps) {
    const PairSrc ps = pair_src(P.own, nullptr, nullptr, P.roff, P.qoff, p);
    const int64_t m = ps.m;
    const int64_t n = ps.n;
    int flag = 0;
    int64_t bl = (P.bl < 0 || P.bl > n) ? n : P.bl;
    int64_t br = (P.br < 0 || P.br > m) ? m : P.br;
    if (m <= 0 || n <= 0) flag = 2;
    const int64_t D = bl + br + 1;
    // |H| bound: alpha + max(bl,br)*beta + max(a,b,n)*min(m,n)
    const int64_t hb = (int64_t)P.alpha + (bl > br ? bl : br) * (int64_t)P.beta +
                       (int64_t)P.maxs * (m < n ? m : n);
    // Range: every kernel keeps alpha*c + |H| and a pair's cell count in
    // int32 (flag 4: ERANGE); only the 32-bit kernels pack H into a 16*H key with per-slot
    // caps, which needs |H| < 2^20 (flag 8: ERANGE unless the 16-bit kernel runs)
    if (!flag && (D > kMaxSlotsWide || m + n >= (1LL << 30) ||
                  (int64_t)P.alpha * (m + n + 2) + hb >= (1LL << 30)))
      flag = 4;
    // nominal in-band in-table cells: sum over diagonals d of |{i : 1<=i<=m, 1<=i-d<=n}|
    uint64_t cnt = 0;
    if (!flag) {
      for (int64_t d = -bl + lane; d <= br; d += 32) {
        const int64_t lo = d + 1 > 1 ? d + 1 : 1;
        const int64_t hi = n + d < m ? n + d : m;
        if (hi >= lo) cnt += (uint64_t)(hi - lo + 1);
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) cnt += __shfl_xor_sync(kFull, cnt, o);
    if (!flag && cnt >= (1ull << 31)) flag = 4;
    const bool long32 = !flag && hb >= kHLimit - 16;
    if (lane == 0) {
      const uint32_t nom = (uint32_t)(cnt > 0xffffffffull ? 0xffffffffull : cnt);
      P.nominal[p] = nom;
      P.iota[p] = (uint32_t)p;
      if (P.chunk_of) {
        int lo = 0, hi = P.nchunks - 1;  // last chunk c with chunk_first[c] <= p
        while (lo < hi) {
          const int mid = (lo + hi + 1) >> 1;
          if (P.chunk_first[mid] <= p) lo = mid; else hi = mid - 1;
        }
        P.chunk_of[p] = (uint8_t)lo;
        const uint64_t tier = flag ? 0 : (uint64_t)tier_of(D);
        const uint64_t grp = (uint64_t)(lo < P.lpt_from ? lo : P.lpt_from);
        P.key64[p] = (tier << P.tier_shift) | (grp << 32) | (uint64_t)(0xffffffffu - nom);
      }
      P.bad[p] = (uint8_t)(flag != 0);
      if (P.len_hash)
        atomicAdd(P.len_hash, splitmix(splitmix(splitmix(p) ^ (unsigned long long)m) ^ (unsigned long long)n));
      if (flag) {
        atomicOr(P.err_flags, flag);
        if (P.tier_count) atomicAdd(P.tier_count, 1);  // (the call then fails anyway)
      } else {
        if (long32) atomicOr(P.err_flags, 8);
        if (P.max_len) {
          atomicMax(P.max_len, (int)m);
          atomicMax(P.max_len + 1, (int)n);
        }
        atomicMax(P.max_slots, (int)D);
        atomicMax(P.max_off16, (int)((-D) & 15));
        if (P.off_mask16) atomicOr(P.off_mask16, 1 << ((-D) & 15));
        if (P.tier_count) {
          atomicAdd(P.tier_count + tier_of(D), 1);
          if (tier_of(D) == 0) {
            atomicMax(P.max_off16_t0, (int)((-D) & 15));
            if (P.off_mask16) atomicOr(P.off_mask16 + 1, 1 << ((-D) & 15));
          } else if (tier_of(D) == 1 && P.off_mask16) {
            atomicOr(P.off_mask16 + 8, 1 << ((-D) & 15));
          }
        }
      }
    }
  }
}

}  // namespace

// ===================================================================================
// Host runtime
// ===================================================================================

struct DevBuf {
  void* p = nullptr;
  size_t cap = 0;
};

struct agatha_ctx {
  int device = 0;
  int num_sms = 0;
  DevBuf ref_ascii, qry_ascii, ref_off, qry_off;     // staging for host inputs
  DevBuf rw, qw;                                      // packed sequences
  DevBuf nominal, nominal_sorted, iota, order, bad;   // plan
  DevBuf sort_tmp;
  DevBuf results;                                     // staging for host outputs
  DevBuf scalars;                                     // err_flags, max_slots, queue
  DevBuf trace;                                       // trace buffers
  DevBuf chunk_first, chunk_of, key64, key64_sorted, ready;  // chunked input streaming
  int* h_scalars = nullptr;                           // pinned mirror of scalars
  int* h_ones = nullptr;                              // pinned 1s (chunk-arrival flags)
  uint64_t* h_chunk_first = nullptr;                  // pinned chunk boundaries
  cudaStream_t copy_stream = nullptr;                 // H2D of input chunks
  uint64_t chunk_bytes = kChunkBytes;                 // target ASCII bytes per chunk
                                                      // (env AGATHA_CHUNK_BYTES, for tests)
  cudaEvent_t ev[6];
  cudaEvent_t cev[2];
  cudaStream_t tier_stream[2] = {nullptr, nullptr};  // slot tiers 1 and 2
  cudaEvent_t tev[3];                                 // fork (0) / joins (1, 2) of the tiers
  agatha_stats_t stats;
};

namespace {

int grow(DevBuf& b, size_t bytes) {
  if (bytes == 0) bytes = 16;
  if (b.cap >= bytes) return AGATHA_OK;
  if (b.p) cudaFree(b.p);
  b.p = nullptr;
  b.cap = 0;
  size_t want = bytes + bytes / 8;
  if (cudaMalloc(&b.p, want) != cudaSuccess) {
    cudaGetLastError();
    return AGATHA_ENOMEM;
  }
  b.cap = want;
  return AGATHA_OK;
}

int check_params(const agatha_params_t* p) {
  if (!p) return AGATHA_EINVAL;
  if (p->match <= 0 || p->mismatch <= 0 || p->ambig < 0) return AGATHA_EINVAL;
  if (p->gap_extend < 0 || p->gap_open < p->gap_extend) return AGATHA_EINVAL;
  if (p->match > 127 || p->mismatch > 127 || p->ambig > 127) return AGATHA_ERANGE;
  if (p->gap_open > 65535 || p->zdrop > (1 << 24)) return AGATHA_ERANGE;
  if (p->band_left > 4096 || p->band_right > 4096) return AGATHA_ERANGE;
  if (p->variant & ~7) return AGATHA_EINVAL;
  return AGATHA_OK;
}

// Score table for prmt: byte x (0..7) = S for code combination x (see combine()).
void score_table(const agatha_params_t* p, uint32_t* T0, uint32_t* T1) {
  uint8_t t[8];
  t[0] = (uint8_t)(int8_t)p->match;
  for (int x = 1; x < 4; ++x) t[x] = (uint8_t)(int8_t)(-p->mismatch);
  for (int x = 4; x < 8; ++x) t[x] = (uint8_t)(int8_t)(-p->ambig);
  *T0 = t[0] | (t[1] << 8) | (t[2] << 16) | ((uint32_t)t[3] << 24);
  *T1 = t[4] | (t[5] << 8) | (t[6] << 16) | ((uint32_t)t[7] << 24);
}

#define CUDA_TRY(x)                          \
  do {                                       \
    cudaError_t e_ = (x);                    \
    if (e_ != cudaSuccess) {                 \
      fprintf(stderr, "libagatha: %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__); \
      return AGATHA_ECUDA;                   \
    }                                        \
  } while (0)

// 16-bit packed kernel eligibility: the within-anti-
// diagonal spread of H plus the drift between re-centrings must stay inside the
// half-word range with margin, and S + 2*alpha must fit the int8 score table.
// the anti-diagonal max sits at ref16 after a re-centring; every stored H
// stays in (kEmpty16, kTop16] and every wall/cap value above -32768.
static long long drift16(const agatha_params_t* p, int iv = kRebase16) {
  const long long mx = std::max<long long>(p->match, std::max<long long>(p->mismatch, p->ambig));
  return (2 * (long long)iv + 6) * (2 * (long long)p->gap_open + mx);  // 70 at 32 iterations
}
// Cells outside the table may rise above the anti-diagonal max of the valid cells by at
// most (alpha - beta) per anti-diagonal for as long as they stay outside (at most
// maxD + 2 anti-diagonals); the ref16 margin covers that, the drift between
// re-centrings and the largest table entry, so every stored H stays <= kTop16.
static int ref16_of(const agatha_params_t* p, int maxD, int iv = kRebase16) {
  const long long a = p->match, al = p->gap_open, be = p->gap_extend;
  const long long mx = std::max<long long>(a, std::max<long long>(p->mismatch, p->ambig));
  return (int)(kTop16 - 127 - (drift16(p, iv) + 3 * al + 2 * a + mx + (al - be) * ((long long)maxD + 2)));
}
// Pinned fronts (CapMode): between two re-centrings (kRebase16 iterations) the dead
// padding slots, pinned at kCapNeg16 at the last one, rise by at most kRebase16 times
// max(S + 2 alpha, 2 (alpha - beta)) in stored units (a diagonal move every two
// anti-diagonals, or a gap extension every one); they must stay below kEmpty16.
static bool pin16_ok(const agatha_params_t* p, int iv) {
  const long long al = p->gap_open, be = p->gap_extend;
  const long long mx = std::max<long long>(p->match, std::max<long long>(-p->mismatch, -p->ambig)) + 2 * al;
  const long long g = std::max<long long>(mx, 2 * (al - be));
  return ((long long)iv + 1) * g + 2 * g < kEmpty16 - kCapNeg16;
}
// the common off = (-D) mod 16 of a launch's pairs, or -1 when they differ
static int pin_off(int mask) { return (mask != 0 && (mask & (mask - 1)) == 0) ? __builtin_ctz(mask) : -1; }
bool use16(const agatha_params_t* p, int maxD, int iv = kRebase16) {
  const long long a = p->match, al = p->gap_open, be = p->gap_extend;
  const long long mx = std::max<long long>(a, std::max<long long>(p->mismatch, p->ambig));
  const long long spread = al + (long long)maxD * (be + a + mx) + 4 * mx;
  const long long drift = drift16(p, iv);
  // int8 table entries S + 2*alpha must lie in [0, 127] (add16x2_fma); alpha >= beta
  // (the boundary chains of the masked steps)
  if (a + 2 * al > 127 || 2 * al - p->mismatch < 0 || 2 * al - p->ambig < 0 || al < be) return false;
  // a one-diagonal band (bl = br = 0) leaves every other anti-diagonal empty, so the
  // re-centring (on the last anti-diagonal's max) would never run
  if (p->band_left == 0 && p->band_right == 0) return false;
  const long long ref = ref16_of(p, maxD, iv);
  return ref - (spread + drift) > kEmpty16 && kW16 - drift > -32768 && maxD <= kMaxSlots;
}

// The 16-bit kernels' re-centring interval (iterations): the split 32-slot front takes the
// longest of AGATHA_REBASE_MAX, ..., 64, 32 for which the 16-bit guard holds (a longer
// interval means fewer loop runs but a larger drift term); the other
// fronts re-centre every kRebase16 = 32, which the same ref16 covers (drift16 grows with
// the interval).  0: the 16-bit kernels do not apply.
#ifndef AGATHA_REBASE_MAX
#define AGATHA_REBASE_MAX 128
#endif
static int rebase16_for(const agatha_params_t* p, int maxD) {
  for (int iv = AGATHA_REBASE_MAX; iv >= kRebase16; iv /= 2)
    if (use16(p, maxD, iv)) return iv;
  return 0;
}

void score_table16(const agatha_params_t* p, uint32_t* T0, uint32_t* T1) {
  uint8_t t[8];
  const int a2 = 2 * p->gap_open;
  t[0] = (uint8_t)(int8_t)(p->match + a2);
  for (int x = 1; x < 4; ++x) t[x] = (uint8_t)(int8_t)(a2 - p->mismatch);
  for (int x = 4; x < 8; ++x) t[x] = (uint8_t)(int8_t)(a2 - p->ambig);
  *T0 = t[0] | (t[1] << 8) | (t[2] << 16) | ((uint32_t)t[3] << 24);
  *T1 = t[4] | (t[5] << 8) | (t[6] << 16) | ((uint32_t)t[7] << 24);
}

template <int NREG, bool TRACE, int NCAP, bool ENDS = false>
int occupancy16() {  // resident blocks per SM
  // cached per instantiation; contexts on several host threads may race to fill it
  // (they compute the same value), so the cache is an atomic
  static std::atomic<int> cache{-1};
  int occ = cache.load(std::memory_order_relaxed);
  if (occ < 0) {
#if AGATHA_MAXNREG16
    const auto kfn = NREG == 16 ? align16w_kernel<NREG, TRACE, NCAP, ENDS> : align16_kernel<NREG, TRACE, NCAP, ENDS>;
#else
    const auto kfn = align16_kernel<NREG, TRACE, NCAP, ENDS>;
#endif
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kfn, 32 * Front16<NREG>::wpb, 0) != cudaSuccess) {
      cudaGetLastError();
      occ = 1;
    }
    if (occ < 1) occ = 1;
    cache.store(occ, std::memory_order_relaxed);
  }
  return occ;
}

// warps (pairs in flight) of the persistent grid of slot tier t
long long warp_slots16(const agatha_ctx* ctx, int t) {
  const int occ = t == 0 ? occupancy16<16, false, 8>() * Front16<16>::wpb
                : (t == 1 ? occupancy16<8, false, NCAP8>() * Front16<8>::wpb : occupancy16<4, false, 3>() * Front16<4>::wpb);
  return (long long)ctx->num_sms * occ;
}

// Launch helpers: grid = the persistent grid; *units_out = packing-scratch units the
// launch uses (warps, or blocks of the wide tier).  dry: size only, launch nothing.
template <int NREG, bool TRACE, int NCAP, bool ENDS = false>
int launch_align16(agatha_ctx* ctx, const AlignArgs& A, cudaStream_t st, int* grid_out, int* units_out = nullptr,
                   bool dry = false) {
  const int occ = occupancy16<NREG, TRACE, NCAP, ENDS>();
  const long long want = (long long)ctx->num_sms * occ;
  constexpr int wpb = Front16<NREG>::wpb;
  const long long need = ((long long)A.n_pairs + wpb - 1) / wpb;
  int grid = (int)(want < need ? want : need);
  if (grid < 1) grid = 1;
  *grid_out = grid;
  if (units_out) *units_out = grid * wpb;
  if (dry) return AGATHA_OK;
#if AGATHA_MAXNREG16
  if (NREG == 16) align16w_kernel<NREG, TRACE, NCAP, ENDS><<<grid, 32 * wpb, 0, st>>>(A);
  else
#endif
  align16_kernel<NREG, TRACE, NCAP, ENDS><<<grid, 32 * wpb, 0, st>>>(A);
  CUDA_TRY(cudaGetLastError());
  return AGATHA_OK;
}

// NREG = 16: the capped registers must cover every pair's low padding off = (-D) mod 16
#ifndef AGATHA_NCAP7
#define AGATHA_NCAP7 0  // 1: seven capped registers when every off <= 7 (-0.1%)
#endif
#ifndef AGATHA_PIN
#define AGATHA_PIN 1  // 0: always the capped fronts
#endif
template <int OFF>
int launch_pin16(agatha_ctx* ctx, const AlignArgs& A, cudaStream_t st, int* grid_out, int* units_out, bool dry,
                 int off) {
  if constexpr (OFF < 16) {
    if (off == OFF) return launch_align16<16, false, 100 + OFF>(ctx, A, st, grid_out, units_out, dry);
    return launch_pin16<OFF + 1>(ctx, A, st, grid_out, units_out, dry, off);
  }
  return AGATHA_EINVAL;
}
template <int OFF>
int launch_pin8(agatha_ctx* ctx, const AlignArgs& A, cudaStream_t st, int* grid_out, int* units_out, bool dry,
                int off) {
  if constexpr (OFF < 8) {
    if (off == OFF) return launch_align16<8, false, 100 + OFF>(ctx, A, st, grid_out, units_out, dry);
    return launch_pin8<OFF + 1>(ctx, A, st, grid_out, units_out, dry, off);
  }
  return AGATHA_EINVAL;
}
// the 16-slot front: pinned (one capped slot) when the launch's pairs share their off
inline int launch_align16_mid(agatha_ctx* ctx, const AlignArgs& A, cudaStream_t st, int* grid_out,
                              int* units_out, bool dry, int pin) {
  if (AGATHA_PIN && pin >= 0) return launch_pin8<0>(ctx, A, st, grid_out, units_out, dry, pin);
  return launch_align16<8, false, NCAP8>(ctx, A, st, grid_out, units_out, dry);
}
template <bool ENDS>
int launch_align16_wide(agatha_ctx* ctx, const AlignArgs& A, cudaStream_t st, int* grid_out, int maxoff,
                        int* units_out = nullptr, bool dry = false, int pin = -1) {
  if (AGATHA_PIN && !ENDS && pin >= 0) return launch_pin16<0>(ctx, A, st, grid_out, units_out, dry, pin);
#if AGATHA_NCAP7
  if (maxoff <= 7) return launch_align16<16, false, 7, ENDS>(ctx, A, st, grid_out, units_out, dry);
#endif
  if (maxoff <= 8) return launch_align16<16, false, 8, ENDS>(ctx, A, st, grid_out, units_out, dry);
  return launch_align16<16, false, 16, ENDS>(ctx, A, st, grid_out, units_out, dry);
}

template <int W, bool TRACE>
int launch_align_wide(agatha_ctx* ctx, const AlignArgs& A, cudaStream_t st, int* grid_out, int* units_out = nullptr,
                      bool dry = false) {
  static std::atomic<int> cache{-1};  // see occupancy16
  int occ = cache.load(std::memory_order_relaxed);
  if (occ < 0) {
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, align_wide_kernel<W, TRACE>, 32 * W, 0) != cudaSuccess) {
      cudaGetLastError();
      occ = 1;
    }
    if (occ < 1) occ = 1;
    cache.store(occ, std::memory_order_relaxed);
  }
  const long long want = (long long)ctx->num_sms * occ;  // persistent: one pair per block
  const long long need = (long long)A.n_pairs;
  int grid = (int)(want < need ? want : need);
  if (grid < 1) grid = 1;
  *grid_out = grid;
  if (units_out) *units_out = grid;
  if (dry) return AGATHA_OK;
  align_wide_kernel<W, TRACE><<<grid, 32 * W, 0, st>>>(A);
  CUDA_TRY(cudaGetLastError());
  return AGATHA_OK;
}

template <int K, bool TRACE>
int launch_align(agatha_ctx* ctx, const AlignArgs& A, cudaStream_t st, int* grid_out, int* units_out = nullptr,
                 bool dry = false) {
  static std::atomic<int> cache{-1};  // see occupancy16
  int occ = cache.load(std::memory_order_relaxed);
  if (occ < 0) {
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, align_kernel<K, TRACE>, 128, 0) != cudaSuccess) {
      cudaGetLastError();
      occ = 1;
    }
    if (occ < 1) occ = 1;
    cache.store(occ, std::memory_order_relaxed);
  }
  const long long want = (long long)ctx->num_sms * occ;      // persistent: fill every SM once
  const long long need = ((long long)A.n_pairs + 3) / 4;    // 4 warps (pairs in flight) per block
  int grid = (int)(want < need ? want : need);
  if (grid < 1) grid = 1;
  *grid_out = grid;
  if (units_out) *units_out = grid * 4;
  if (dry) return AGATHA_OK;
  align_kernel<K, TRACE><<<grid, 128, 0, st>>>(A);
  CUDA_TRY(cudaGetLastError());
  return AGATHA_OK;
}

// Shared body of agatha_align_batch / agatha_localmax_trace.
int run_batch(agatha_ctx* ctx, const agatha_batch_t* b, const agatha_params_t* p,
              agatha_result_t* out, cudaStream_t st, long long trace_pair, int* trace_score,
              int* trace_i, long long trace_cap, const Owners* fed = nullptr) {
  if (!ctx || !b || !out) return AGATHA_EINVAL;
  if (fed && !(b->flags & AGATHA_MEM_DEVICE)) return AGATHA_EINVAL;
  int rc = check_params(p);
  if (rc) return rc;
  if (b->n_pairs == 0) return AGATHA_EEMPTY;
  if (b->n_pairs >= (1ull << 31)) return AGATHA_ERANGE;
  if (b->queue && (b->flags & AGATHA_STATIC_ASSIGN)) return AGATHA_EINVAL;  // no queue to share
  CUDA_TRY(cudaSetDevice(ctx->device));
  memset(&ctx->stats, 0, sizeof(ctx->stats));
  const uint64_t P = b->n_pairs;
  const bool dev_in = (b->flags & AGATHA_MEM_DEVICE) != 0;
  const bool dev_out = (b->flags & AGATHA_OUT_DEVICE) != 0;
  const bool nmap = (b->flags & AGATHA_N_MAP) != 0;

  CUDA_TRY(cudaEventRecord(ctx->ev[0], st));
  uint64_t tot_r, tot_q;
  const uint8_t *d_ref, *d_qry;
  const uint64_t *d_roff, *d_qoff;
  // Input chunks: host inputs stream in as contiguous ranges of pairs (~48 MB of ASCII
  // each) on the copy stream while the align kernel runs; a pair waits for its chunk's
  // flag.  Device inputs are one chunk that is ready from the start.
  int nchunks = 1;
  double est_cells = 0.0;  // host inputs: sum of min(m,n) * D, the kernel-time estimate
  ctx->h_chunk_first[0] = 0;
  // pinned mirror: ints [0..17] the scalars below, u64 [12] [13] the device inputs' total
  // lengths (read with the plan's scalars: one host round trip), int [14] the final flags
  uint64_t* h_tot = (uint64_t*)ctx->h_scalars + 12;  // ints 24..27
  if (fed) {  // federated: every owner's inputs are device-resident (maybe peer-mapped)
    h_tot[0] = h_tot[1] = 0;
    tot_r = tot_q = 0;
    d_ref = d_qry = nullptr; d_roff = d_qoff = nullptr;
  } else if (dev_in) {
    CUDA_TRY(cudaMemcpyAsync(h_tot, b->ref_off + P, 8, cudaMemcpyDeviceToHost, st));
    CUDA_TRY(cudaMemcpyAsync(h_tot + 1, b->qry_off + P, 8, cudaMemcpyDeviceToHost, st));
    tot_r = tot_q = 0;  // known after the plan's synchronisation
    d_ref = b->ref; d_qry = b->qry; d_roff = b->ref_off; d_qoff = b->qry_off;
  } else {
    tot_r = b->ref_off[P];
    tot_q = b->qry_off[P];
    if ((rc = grow(ctx->ref_ascii, tot_r)) || (rc = grow(ctx->qry_ascii, tot_q)) ||
        (rc = grow(ctx->ref_off, 8 * (P + 1))) || (rc = grow(ctx->qry_off, 8 * (P + 1))))
      return rc;
    CUDA_TRY(cudaMemcpyAsync(ctx->ref_off.p, b->ref_off, 8 * (P + 1), cudaMemcpyHostToDevice, st));
    CUDA_TRY(cudaMemcpyAsync(ctx->qry_off.p, b->qry_off, 8 * (P + 1), cudaMemcpyHostToDevice, st));
    d_ref = (const uint8_t*)ctx->ref_ascii.p;
    d_qry = (const uint8_t*)ctx->qry_ascii.p;
    d_roff = (const uint64_t*)ctx->ref_off.p;
    d_qoff = (const uint64_t*)ctx->qry_off.p;
    uint64_t target = ctx->chunk_bytes;
    const uint64_t total = tot_r + tot_q;
    if (total / target + 2 + kRampChunks > (uint64_t)kMaxChunks)
      target = total / (kMaxChunks - 2 - kRampChunks) + 1;
    // the first chunks ramp up from target / 2^kRampChunks, doubling: the kernel starts
    // on the first pairs after a short copy instead of a full chunk's
    // (a batch under one chunk stays one chunk: small copies cost more in API calls
    // than they save in latency, measured on C1)
#if AGATHA_CHUNK_RAMP
    uint64_t cur = total <= target ? target
                                   : std::max<uint64_t>(target >> kRampChunks, std::min<uint64_t>(target, 64u << 10));
#else
    uint64_t cur = target;
#endif
    uint64_t acc = 0;
    const int64_t pbl = p->band_left, pbr = p->band_right;
    for (uint64_t k = 0; k < P; ++k) {
      const int64_t m = (int64_t)(b->ref_off[k + 1] - b->ref_off[k]), n = (int64_t)(b->qry_off[k + 1] - b->qry_off[k]);
      acc += (uint64_t)(m + n);
      const int64_t bl = (pbl < 0 || pbl > n) ? n : pbl, br = (pbr < 0 || pbr > m) ? m : pbr;
      est_cells += (double)(m < n ? m : n) * (double)(bl + br + 1);  // for lpt_from below
      if (acc >= cur && k + 1 < P) {
        ctx->h_chunk_first[nchunks++] = k + 1;
        acc = 0;
        cur = std::min(2 * cur, target);
      }
    }
  }
  ctx->h_chunk_first[nchunks] = P;
  // Streamed inputs: the order is chunk-major so that no warp waits on a
  // chunk still in flight, but then a long pair of a late chunk starts late and ends
  // after everything else (the tail).  The queue reaches chunk c after about c/nchunks
  // of the kernel time, while every chunk has arrived after the copy time; from the
  // first chunk the queue reaches after the copies end, all later chunks form one
  // longest-first group.  Estimates (conservative: a fast kernel, a slow link):
  // kernel = sum min(m,n)*D / 4 TCUPS, copy = bytes / 20 GB/s, margin 1.25.
  int lpt_from = nchunks;
  if (b->queue) {
    // a shared queue (NEXT #1): every participant must derive the same order, so the
    // chunk grouping (which depends on the input memory and AGATHA_CHUNK_BYTES) is off:
    // one longest-first group per tier
    lpt_from = 0;
  } else if (!dev_in && nchunks > 2) {
    const double t_kernel = est_cells / 4e12, t_copy = (double)(tot_r + tot_q) / 20e9;
    const double f = t_kernel > 0 ? 1.25 * t_copy / t_kernel : 1.0;
    if (f < 1.0) lpt_from = std::max(1, (int)std::ceil(f * nchunks));
  }
  CUDA_TRY(cudaEventRecord(ctx->ev[1], st));

  // device scratch
  size_t sort_bytes = 0, sort_bytes64 = 0;
  cub::DeviceRadixSort::SortPairsDescending(nullptr, sort_bytes, (const uint32_t*)nullptr,
                                            (uint32_t*)nullptr, (const uint32_t*)nullptr,
                                            (uint32_t*)nullptr, (int)P, 0, 32, st);
  cub::DeviceRadixSort::SortPairs(nullptr, sort_bytes64, (const uint64_t*)nullptr, (uint64_t*)nullptr,
                                  (const uint32_t*)nullptr, (uint32_t*)nullptr, (int)P, 0, 40, st);
  if (sort_bytes64 > sort_bytes) sort_bytes = sort_bytes64;
  if ((rc = grow(ctx->nominal, 4 * P)) || (rc = grow(ctx->nominal_sorted, 4 * P)) ||
      (rc = grow(ctx->iota, 4 * P)) || (rc = grow(ctx->order, 4 * P)) || (rc = grow(ctx->bad, P)) ||
      (rc = grow(ctx->sort_tmp, sort_bytes)) || (rc = grow(ctx->scalars, 128)) ||
      (rc = grow(ctx->chunk_first, 8 * (kMaxChunks + 1))) || (rc = grow(ctx->chunk_of, P)) ||
      (rc = grow(ctx->key64, 8 * P)) || (rc = grow(ctx->key64_sorted, 8 * P)) ||
      (rc = grow(ctx->ready, 4 * kMaxChunks)))
    return rc;
  agatha_result_t* d_out = out;
  agatha_ends_t* d_ends = b->ends;
  if (!dev_out) {
    if ((rc = grow(ctx->results, (sizeof(agatha_result_t) + (b->ends ? sizeof(agatha_ends_t) : 0)) * P)))
      return rc;
    d_out = (agatha_result_t*)ctx->results.p;
    if (b->ends) d_ends = (agatha_ends_t*)(d_out + P);
  }
  // scalars: [0] err_flags [1] max_slots [2] queue (tier 0 / one launch) [3] max (-D) mod 16
  // [4..6] pairs per slot tier [7] max (-D) mod 16 of tier 0 [8] [9] queues of tiers 1, 2
  // [12..13] len_hash (shared queue) [15] fingerprint mismatch [16] [17] max m, max n
  int* d_sc = (int*)ctx->scalars.p;
  int* d_ready = (int*)ctx->ready.p;
  CUDA_TRY(cudaMemsetAsync(d_sc, 0, 128, st));
  CUDA_TRY(cudaMemcpyAsync(ctx->chunk_first.p, ctx->h_chunk_first, 8 * (nchunks + 1),
                           cudaMemcpyHostToDevice, st));
  if (dev_in) CUDA_TRY(cudaMemcpyAsync(d_ready, ctx->h_ones, 4, cudaMemcpyHostToDevice, st));
  else CUDA_TRY(cudaMemsetAsync(d_ready, 0, 4 * nchunks, st));

  const int maxs = p->match > p->mismatch ? (p->match > p->ambig ? p->match : p->ambig)
                                          : (p->mismatch > p->ambig ? p->mismatch : p->ambig);
  PrepArgs pa;
  pa.roff = d_roff; pa.qoff = d_qoff; pa.n_pairs = P;
  if (fed) pa.own = *fed; else pa.own.n_owners = 0;
  pa.max_len = d_sc + 16;
  pa.bl = p->band_left; pa.br = p->band_right; pa.alpha = p->gap_open; pa.beta = p->gap_extend;
  pa.maxs = maxs;
  pa.nominal = (uint32_t*)ctx->nominal.p; pa.iota = (uint32_t*)ctx->iota.p;
  pa.bad = (uint8_t*)ctx->bad.p; pa.err_flags = d_sc; pa.max_slots = d_sc + 1; pa.max_off16 = d_sc + 3;
  pa.chunk_first = (const uint64_t*)ctx->chunk_first.p; pa.nchunks = nchunks;
  pa.chunk_of = (uint8_t*)ctx->chunk_of.p; pa.key64 = (uint64_t*)ctx->key64.p;
  int chunk_bits = 0;
  while ((1 << chunk_bits) < nchunks) ++chunk_bits;
  pa.tier_shift = 32 + chunk_bits; pa.tier_count = d_sc + 4; pa.max_off16_t0 = d_sc + 7;
  pa.off_mask16 = d_sc + 10;
  pa.lpt_from = lpt_from;
  pa.len_hash = b->queue ? (unsigned long long*)(d_sc + 12) : nullptr;  // zeroed with d_sc
  const int prep_blocks = (int)(((P + 7) / 8) < 4096 ? ((P + 7) / 8) : 4096);
  prep_kernel<<<prep_blocks, 256, 0, st>>>(pa);
  CUDA_TRY(cudaGetLastError());
  int launches = 1, lib_launches = 0;
  const uint32_t* d_order = (const uint32_t*)ctx->iota.p;
  // K (slots per lane) from the widest band in the batch
  CUDA_TRY(cudaMemcpyAsync(ctx->h_scalars, d_sc, 76, cudaMemcpyDeviceToHost, st));
  CUDA_TRY(cudaStreamSynchronize(st));
  const int err0 = ctx->h_scalars[0], maxD = ctx->h_scalars[1], maxoff16 = ctx->h_scalars[3];
  const int tier_n[3] = {ctx->h_scalars[4], ctx->h_scalars[5], ctx->h_scalars[6]};
  const int maxoff16_t0 = ctx->h_scalars[7];
  // the pinned 32-slot front (CapMode) when every pair of the launch has one off
  const int iv16 = rebase16_for(p, maxD);
  const int pin_all = pin16_ok(p, iv16) ? pin_off(ctx->h_scalars[10]) : -1;
  ctx->stats.pin_off = -1;
  ctx->stats.rebase_iters = iv16;
  const int pin_t0 = pin16_ok(p, iv16) ? pin_off(ctx->h_scalars[11]) : -1;
  // the 16-slot front (paired layout, re-centring every kRebase16): its low padding is
  // off = (-D) mod 8, common to a launch's pairs when their (-D) mod 16 agree mod 8
  auto fold8 = [](int m16) { return (m16 | (m16 >> 8)) & 0xFF; };
  const int pin8_all = (iv16 > 0 && pin16_ok(p, kRebase16)) ? pin_off(fold8(ctx->h_scalars[10])) : -1;
  const int pin8_t1 = (iv16 > 0 && pin16_ok(p, kRebase16)) ? pin_off(fold8(ctx->h_scalars[18])) : -1;
  ctx->stats.pin_off8 = -1;
  const int max_m = ctx->h_scalars[16], max_n = ctx->h_scalars[17];
  if (dev_in) {
    tot_r = h_tot[0];
    tot_q = h_tot[1];
  }
  // packing scratch per work unit: guard word + up to len/8 + 2 data words + guard word
  // (load_word_rw), rounded up to 32 B; the unit count is sized at the launches below
  uint64_t rstride = ((uint64_t)max_m / 8 + 4 + 7) & ~7ull, qstride = ((uint64_t)max_n / 8 + 4 + 7) & ~7ull;
  if (AGATHA_SPLIT16) {  // the split 32-slot front's selector streams (align_pair16s)
    const uint64_t w = ((uint64_t)s16_unit_words((long long)max_m + max_n) + 7) & ~7ull;
    rstride = std::max(rstride, w);
    qstride = std::max(qstride, w);
  }
  if (err0 & 2) return AGATHA_EEMPTY;
  if (err0 & 4) return AGATHA_ERANGE;

  const int K = maxD <= 512 ? 16 : 32;
  const bool k16 = iv16 > 0 && !(b->flags & AGATHA_FORCE_32BIT);
  if ((err0 & 8) && !k16) return AGATHA_ERANGE;  // a pair the 32-bit kernels cannot hold
  if (b->queue) {
    // Participants of a shared queue claim positions of ONE order with one counter per
    // launch: they must agree on the batch, the parameters and every choice that shapes
    // the order or the launches.  The fingerprint covers the pair count, every pair's
    // (index, m, n) (hashed by the prep kernel), the parameters and the flags; not the
    // bases themselves.  The first participant stores a fingerprint of those in
    // the queue (queue[8]); a participant whose fingerprint differs is refused before it
    // claims anything (agatha.h, agatha_queue_create).
    uint32_t fp = 2166136261u;
    auto mix = [&fp](uint64_t v) {
      for (int i = 0; i < 8; ++i) { fp ^= (uint32_t)(v & 0xff); fp *= 16777619u; v >>= 8; }
    };
    mix(P); mix((uint64_t)tier_n[0]); mix((uint64_t)tier_n[1]); mix((uint64_t)tier_n[2]);
    mix((uint64_t)maxD); mix((uint64_t)k16);
    mix(b->flags & (AGATHA_ORDER_INPUT | AGATHA_SINGLE_TIER | AGATHA_FORCE_32BIT));
    mix((uint64_t)(uint32_t)p->match | ((uint64_t)(uint32_t)p->mismatch << 32));
    mix((uint64_t)(uint32_t)p->ambig | ((uint64_t)(uint32_t)p->gap_open << 32));
    mix((uint64_t)(uint32_t)p->gap_extend | ((uint64_t)(uint32_t)p->band_left << 32));
    mix((uint64_t)(uint32_t)p->band_right | ((uint64_t)(uint32_t)p->zdrop << 32));
    mix((uint64_t)(uint32_t)p->variant);
    mix(tot_r); mix(tot_q); mix(fed ? (uint64_t)fed->n_owners : 0);
    if (fp == 0) fp = 1;
    queue_fp_kernel<<<1, 1, 0, st>>>(b->queue, fp, (const unsigned long long*)(d_sc + 12), d_sc + 15);
    CUDA_TRY(cudaGetLastError());
    CUDA_TRY(cudaMemcpyAsync(ctx->h_scalars + 15, d_sc + 15, 4, cudaMemcpyDeviceToHost, st));
    CUDA_TRY(cudaStreamSynchronize(st));
    if (ctx->h_scalars[15]) return AGATHA_EINVAL;
  }
  const bool tr = trace_pair >= 0;
  // Slot tiers: each pair runs at the narrowest front that holds its
  // band, one persistent launch per non-empty tier on its own stream, so the narrow
  // tiers fill the SMs as the wide tier's blocks retire.  The order is tier-major, so
  // tier t's pairs are a contiguous range of it.  One launch (the widest front the batch
  // needs) in input order or when tracing.
  const bool split = k16 && !tr && !(b->flags & (AGATHA_ORDER_INPUT | AGATHA_SINGLE_TIER));
  bool sort = !(b->flags & AGATHA_ORDER_INPUT);
  if (sort && k16 && !b->queue) {
    // one launch whose persistent warps take every pair at once: the order is moot
    const int t = tier_of(maxD);
    const bool one = !split || (tier_n[0] > 0) + (tier_n[1] > 0) + (tier_n[2] > 0) == 1;
    if (one && (long long)P <= warp_slots16(ctx, t)) sort = false;
  }
  if (sort) {
    // a2: longest first within each input chunk group (chunk-major) within
    // each slot tier (tier-major): key = (tier << (32 + chunk_bits)) | (group << 32) | ~nominal
    const int end_bit = 32 + chunk_bits + 2;
    size_t tb = ctx->sort_tmp.cap;
    CUDA_TRY(cub::DeviceRadixSort::SortPairs(
        ctx->sort_tmp.p, tb, (const uint64_t*)ctx->key64.p, (uint64_t*)ctx->key64_sorted.p,
        (const uint32_t*)ctx->iota.p, (uint32_t*)ctx->order.p, (int)P, 0, end_bit, st));
    d_order = (const uint32_t*)ctx->order.p;
    lib_launches = 4;
  }
  CUDA_TRY(cudaEventRecord(ctx->ev[2], st));

  AlignArgs A;
  A.rstride = rstride; A.qstride = qstride; A.unit_base = 0;
  if (fed) A.own = *fed; else A.own.n_owners = 0;
  A.rw = (uint32_t*)ctx->rw.p; A.qw = (uint32_t*)ctx->qw.p;
  A.ref_ascii = d_ref; A.qry_ascii = d_qry; A.chunk_of = (const uint8_t*)ctx->chunk_of.p;
  A.ready = d_ready; A.err_flags = d_sc; A.nmap = nmap ? 1 : 0;
  A.roff = d_roff; A.qoff = d_qoff; A.order = d_order; A.bad = (const uint8_t*)ctx->bad.p;
  A.out = d_out; A.n_pairs = (uint32_t)P;
  A.ends = d_ends;
  A.queue = b->queue ? b->queue : d_sc + 2;  // NEXT #1: a counter shared with other GPUs
  A.sysq = b->queue ? 1 : 0;
  A.static_assign = (b->flags & AGATHA_STATIC_ASSIGN) ? 1 : 0;
  if (b->queue)  // rows this participant does not claim stay zero (merged by the caller)
    CUDA_TRY(cudaMemsetAsync(d_out, 0, sizeof(agatha_result_t) * P, st));
  A.bl = p->band_left; A.br = p->band_right;
  A.alpha = p->gap_open; A.beta = p->gap_extend; A.zdrop = p->zdrop; A.sixteen = 16;
  A.variant = p->variant;
  A.k65536 = 65536u;
  A.one = 1u;
  A.ref16 = ref16_of(p, maxD, iv16 > 0 ? iv16 : kRebase16);
  A.rebase16 = iv16 > 0 ? iv16 : kRebase16;
  score_table(p, &A.T0, &A.T1);
  score_table16(p, &A.T16_0, &A.T16_1);
  A.trace_pair = trace_pair; A.trace_score = trace_score; A.trace_i = trace_i; A.trace_cap = trace_cap;
  if (!dev_in) {
    // stream the ASCII in chunk by chunk while the kernel runs; each chunk's flag is
    // written after its bytes (same stream), and the kernel reads it with acquire.
    // The copies are enqueued before the kernel so that a launch that blocks the host
    // (CUDA_LAUNCH_BLOCKING, a serialising profiler) cannot wait on flags not yet issued.
    CUDA_TRY(cudaEventRecord(ctx->cev[0], ctx->copy_stream));
    for (int c = 0; c < nchunks; ++c) {
      const uint64_t k0 = ctx->h_chunk_first[c], k1 = ctx->h_chunk_first[c + 1];
      const uint64_t rb = b->ref_off[k0], re = b->ref_off[k1], qb = b->qry_off[k0], qe = b->qry_off[k1];
      if (re > rb)
        CUDA_TRY(cudaMemcpyAsync((uint8_t*)ctx->ref_ascii.p + rb, b->ref + rb, re - rb,
                                 cudaMemcpyHostToDevice, ctx->copy_stream));
      if (qe > qb)
        CUDA_TRY(cudaMemcpyAsync((uint8_t*)ctx->qry_ascii.p + qb, b->qry + qb, qe - qb,
                                 cudaMemcpyHostToDevice, ctx->copy_stream));
      CUDA_TRY(cudaMemcpyAsync(d_ready + c, ctx->h_ones, 4, cudaMemcpyHostToDevice, ctx->copy_stream));
    }
    CUDA_TRY(cudaEventRecord(ctx->cev[1], ctx->copy_stream));
  }
  int grid = 0, units_total = 0;
  const bool ends = d_ends != nullptr;
  int tiers_launched = 0, slots = 0;
  memset(ctx->stats.tier_pairs, 0, sizeof(ctx->stats.tier_pairs));
  // two passes over the launch selection: the dry one sizes the packing scratch (units of
  // every launch of this call; the tier launches run together, so theirs are disjoint),
  // the second launches
  for (int pass = 0; pass < 2 && !rc; ++pass) {
  const bool dry = pass == 0;
  int units = 0;
  grid = 0; tiers_launched = 0; slots = 0;
  if (!dry) {
    if ((rc = grow(ctx->rw, 4 * rstride * (uint64_t)(units_total > 0 ? units_total : 1))) ||
        (rc = grow(ctx->qw, 4 * qstride * (uint64_t)(units_total > 0 ? units_total : 1))))
      break;
    A.rw = (uint32_t*)ctx->rw.p; A.qw = (uint32_t*)ctx->qw.p;
  }
  if (split) {
    if (!dry) CUDA_TRY(cudaEventRecord(ctx->tev[0], st));
    uint32_t start = 0;
    int unit_base = 0;
    for (int t = 0; t < 3 && !rc; ++t) {
      if (tier_n[t] == 0) continue;
      AlignArgs At = A;
      At.order = d_order + start;
      At.n_pairs = (uint32_t)tier_n[t];
      // a shared queue (NEXT #1) holds one counter per tier, claimed in the same
      // tier-major order by every participant
      At.queue = b->queue ? b->queue + t : (t == 0 ? d_sc + 2 : d_sc + 7 + t);
      At.unit_base = unit_base;  // the tiers run together: disjoint packing scratch
      start += (uint32_t)tier_n[t];
      cudaStream_t ts = st;
      if (t > 0 && !dry) {
        ts = ctx->tier_stream[t - 1];
        if (cudaStreamWaitEvent(ts, ctx->tev[0], 0) != cudaSuccess) { rc = AGATHA_ECUDA; break; }
      }
      int g = 0, u = 0;
      if (ends) {  // NEXT #4: the end-score instantiations
        if (t == 0) rc = launch_align16_wide<true>(ctx, At, ts, &g, maxoff16_t0, &u, dry);
        else if (t == 1) rc = launch_align16<8, false, NCAP8, true>(ctx, At, ts, &g, &u, dry);
        else rc = launch_align16<4, false, 3, true>(ctx, At, ts, &g, &u, dry);
      } else {
        if (t == 0) {
          rc = launch_align16_wide<false>(ctx, At, ts, &g, maxoff16_t0, &u, dry, pin_t0);
          ctx->stats.pin_off = AGATHA_PIN ? pin_t0 : -1;
        }
        else if (t == 1) {
          rc = launch_align16_mid(ctx, At, ts, &g, &u, dry, pin8_t1);
          ctx->stats.pin_off8 = AGATHA_PIN ? pin8_t1 : -1;
        }
        else rc = launch_align16<4, false, 3>(ctx, At, ts, &g, &u, dry);
      }
      unit_base += u;
      units += u;
      if (t > 0 && !rc && !dry && cudaEventRecord(ctx->tev[t], ts) != cudaSuccess) rc = AGATHA_ECUDA;
      grid += g;
      ++tiers_launched;
      ctx->stats.tier_pairs[t] = tier_n[t];
      if (!slots) slots = 32 >> t;
    }
    for (int t = 1; t < 3 && !rc && !dry; ++t)
      if (tier_n[t] && cudaStreamWaitEvent(st, ctx->tev[t], 0) != cudaSuccess) rc = AGATHA_ECUDA;
  } else if (k16) {
    // (NREG = 16) eight capped registers suffice when every pair's low padding
    // off = (-D) mod 16 is at most 8 (prep_kernel's max); else all sixteen
    const int t = tier_of(maxD);
    int* u = &units;
    if (ends) {  // (tracing never asks for end scores)
      if (t == 2) rc = launch_align16<4, false, 3, true>(ctx, A, st, &grid, u, dry);
      else if (t == 1) rc = launch_align16<8, false, NCAP8, true>(ctx, A, st, &grid, u, dry);
      else rc = launch_align16_wide<true>(ctx, A, st, &grid, maxoff16, u, dry);
    } else if (t == 2) rc = tr ? launch_align16<4, true, 3>(ctx, A, st, &grid, u, dry) : launch_align16<4, false, 3>(ctx, A, st, &grid, u, dry);
    else if (t == 1 && tr) rc = launch_align16<8, true, NCAP8>(ctx, A, st, &grid, u, dry);
    else if (t == 1) {
      rc = launch_align16_mid(ctx, A, st, &grid, u, dry, pin8_all);
      ctx->stats.pin_off8 = AGATHA_PIN ? pin8_all : -1;
    }
    else if (tr) rc = launch_align16<16, true, 16>(ctx, A, st, &grid, u, dry);
    else {
      rc = launch_align16_wide<false>(ctx, A, st, &grid, maxoff16, u, dry, pin_all);
      ctx->stats.pin_off = AGATHA_PIN ? pin_all : -1;
    }
    tiers_launched = 1;
    ctx->stats.tier_pairs[t] = (int)P;
    slots = 32 >> t;
  } else {
    int* u = &units;
    if (K == 16) rc = tr ? launch_align<16, true>(ctx, A, st, &grid, u, dry) : launch_align<16, false>(ctx, A, st, &grid, u, dry);
    else if (maxD <= kMaxSlots) rc = tr ? launch_align<32, true>(ctx, A, st, &grid, u, dry) : launch_align<32, false>(ctx, A, st, &grid, u, dry);
    else if (maxD <= 2 * kMaxSlots)  // NEXT #3: wide bands, two or four warps per pair
      rc = tr ? launch_align_wide<2, true>(ctx, A, st, &grid, u, dry) : launch_align_wide<2, false>(ctx, A, st, &grid, u, dry);
    else rc = tr ? launch_align_wide<4, true>(ctx, A, st, &grid, u, dry) : launch_align_wide<4, false>(ctx, A, st, &grid, u, dry);
    tiers_launched = 1;
    slots = K;
  }
  if (dry) units_total = units;
  }
  ctx->stats.packed16 = k16 ? 1 : 0;
  if (rc) {  // nothing launched may still be using the caller's buffers on return
    cudaStreamSynchronize(st);
    for (int i = 0; i < 2; ++i) cudaStreamSynchronize(ctx->tier_stream[i]);
    if (!dev_in) cudaStreamSynchronize(ctx->copy_stream);
    return rc;
  }
  launches += tiers_launched;
  CUDA_TRY(cudaEventRecord(ctx->ev[3], st));
  if (!dev_out) {
    CUDA_TRY(cudaMemcpyAsync(out, d_out, sizeof(agatha_result_t) * P, cudaMemcpyDeviceToHost, st));
    if (b->ends)
      CUDA_TRY(cudaMemcpyAsync(b->ends, d_ends, sizeof(agatha_ends_t) * P, cudaMemcpyDeviceToHost, st));
  }
  CUDA_TRY(cudaEventRecord(ctx->ev[4], st));
  CUDA_TRY(cudaMemcpyAsync(ctx->h_scalars + 14, d_sc, 4, cudaMemcpyDeviceToHost, st));
  CUDA_TRY(cudaStreamSynchronize(st));
  if (!dev_in) CUDA_TRY(cudaStreamSynchronize(ctx->copy_stream));
  if (ctx->h_scalars[14] & 1) return AGATHA_ECHAR;  // set by the fused pack (a1)
  if (dev_in) cudaEventElapsedTime(&ctx->stats.h2d_ms, ctx->ev[0], ctx->ev[1]);
  else cudaEventElapsedTime(&ctx->stats.h2d_ms, ctx->cev[0], ctx->cev[1]);
  cudaEventElapsedTime(&ctx->stats.prep_ms, ctx->ev[1], ctx->ev[2]);
  cudaEventElapsedTime(&ctx->stats.align_ms, ctx->ev[2], ctx->ev[3]);
  cudaEventElapsedTime(&ctx->stats.d2h_ms, ctx->ev[3], ctx->ev[4]);
  ctx->stats.slots_per_lane = slots;
  ctx->stats.warps_per_pair = k16 || maxD <= kMaxSlots ? 1 : (maxD <= 2 * kMaxSlots ? 2 : 4);
  ctx->stats.grid_blocks = grid;
  ctx->stats.input_chunks = nchunks;
  ctx->stats.lpt_from_chunk = lpt_from;
  ctx->stats.kernel_launches = launches;
  ctx->stats.library_launches = lib_launches;
  return AGATHA_OK;
}

}  // namespace

extern "C" {

int agatha_version(void) { return 1; }

const char* agatha_strerror(int code) {
  switch (code) {
    case AGATHA_OK: return "ok";
    case AGATHA_EINVAL: return "invalid argument or scoring parameters";
    case AGATHA_EEMPTY: return "empty sequence or empty batch";
    case AGATHA_ECHAR: return "non-ACGTN byte in a sequence";
    case AGATHA_ERANGE: return "band, penalty or sequence length beyond the supported range";
    case AGATHA_ECUDA: return "CUDA error or no sm_100 device";
    case AGATHA_ENOMEM: return "device allocation failed";
    default: return "unknown error";
  }
}

int agatha_ctx_create(agatha_ctx_t** out, int device) {
  if (!out) return AGATHA_EINVAL;
  *out = nullptr;
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || device < 0 || device >= ndev) {
    cudaGetLastError();
    return AGATHA_ECUDA;
  }
  cudaDeviceProp prop;
  if (cudaGetDeviceProperties(&prop, device) != cudaSuccess) return AGATHA_ECUDA;
  if (prop.major != 10) return AGATHA_ECUDA;  // built for sm_100a only
  if (cudaSetDevice(device) != cudaSuccess) return AGATHA_ECUDA;
  agatha_ctx* ctx = new agatha_ctx();
  ctx->device = device;
  ctx->num_sms = prop.multiProcessorCount;
  if (const char* e = getenv("AGATHA_CHUNK_BYTES")) {
    const unsigned long long v = strtoull(e, nullptr, 10);
    if (v >= 256) ctx->chunk_bytes = v;
  }
  for (int i = 0; i < 6; ++i) cudaEventCreate(&ctx->ev[i]);
  for (int i = 0; i < 2; ++i) cudaEventCreate(&ctx->cev[i]);
  for (int i = 0; i < 3; ++i) cudaEventCreateWithFlags(&ctx->tev[i], cudaEventDisableTiming);
  cudaStreamCreateWithFlags(&ctx->copy_stream, cudaStreamNonBlocking);
  for (int i = 0; i < 2; ++i) cudaStreamCreateWithFlags(&ctx->tier_stream[i], cudaStreamNonBlocking);
  if (cudaMallocHost(&ctx->h_scalars, 256) != cudaSuccess ||
      cudaMallocHost(&ctx->h_ones, 4 * kMaxChunks) != cudaSuccess ||
      cudaMallocHost(&ctx->h_chunk_first, 8 * (kMaxChunks + 1)) != cudaSuccess) {
    cudaGetLastError();
    agatha_ctx_destroy(ctx);  // releases the events, streams and any pinned buffer made
    return AGATHA_ENOMEM;
  }
  for (int i = 0; i < kMaxChunks; ++i) ctx->h_ones[i] = 1;
  *out = ctx;
  return AGATHA_OK;
}

void agatha_ctx_destroy(agatha_ctx_t* ctx) {
  if (!ctx) return;
  cudaSetDevice(ctx->device);
  DevBuf* bufs[] = {&ctx->ref_ascii, &ctx->qry_ascii, &ctx->ref_off, &ctx->qry_off, &ctx->rw,
                    &ctx->qw, &ctx->nominal, &ctx->nominal_sorted, &ctx->iota, &ctx->order,
                    &ctx->bad, &ctx->sort_tmp, &ctx->results, &ctx->scalars, &ctx->trace,
                    &ctx->chunk_first, &ctx->chunk_of, &ctx->key64, &ctx->key64_sorted, &ctx->ready};
  for (DevBuf* b : bufs)
    if (b->p) cudaFree(b->p);
  for (int i = 0; i < 6; ++i) cudaEventDestroy(ctx->ev[i]);
  for (int i = 0; i < 2; ++i) cudaEventDestroy(ctx->cev[i]);
  for (int i = 0; i < 3; ++i) cudaEventDestroy(ctx->tev[i]);
  if (ctx->copy_stream) cudaStreamDestroy(ctx->copy_stream);
  for (int i = 0; i < 2; ++i)
    if (ctx->tier_stream[i]) cudaStreamDestroy(ctx->tier_stream[i]);
  if (ctx->h_scalars) cudaFreeHost(ctx->h_scalars);
  if (ctx->h_ones) cudaFreeHost(ctx->h_ones);
  if (ctx->h_chunk_first) cudaFreeHost(ctx->h_chunk_first);
  delete ctx;
}

int agatha_align_batch(agatha_ctx_t* ctx, const agatha_batch_t* batch, const agatha_params_t* params,
                       agatha_result_t* out, void* stream) {
  return run_batch(ctx, batch, params, out, (cudaStream_t)stream, -1, nullptr, nullptr, 0);
}

int agatha_align_federated(agatha_ctx_t* ctx, const agatha_batch_t* owners, int n_owners,
                           const agatha_params_t* params, agatha_result_t* out, int32_t* queue,
                           uint32_t flags, void* stream) {
  if (!ctx || !owners || !out || n_owners < 1 || n_owners > kMaxOwners) return AGATHA_EINVAL;
  Owners O;
  memset(&O, 0, sizeof(O));
  O.n_owners = n_owners;
  uint64_t total = 0;
  for (int o = 0; o < n_owners; ++o) {
    const agatha_batch_t& b = owners[o];
    if (!(b.flags & AGATHA_MEM_DEVICE) || !b.ref || !b.qry || !b.ref_off || !b.qry_off) return AGATHA_EINVAL;
    if (b.n_pairs == 0) return AGATHA_EEMPTY;
    O.ref[o] = b.ref; O.qry[o] = b.qry; O.roff[o] = b.ref_off; O.qoff[o] = b.qry_off;
    O.start[o] = (uint32_t)total;
    total += b.n_pairs;
    if (total >= (1ull << 31)) return AGATHA_ERANGE;
  }
  O.start[n_owners] = (uint32_t)total;
  agatha_batch_t g;
  memset(&g, 0, sizeof(g));
  g.n_pairs = total;
  g.flags = (flags & ~(AGATHA_MEM_DEVICE | AGATHA_OUT_DEVICE)) | AGATHA_MEM_DEVICE | AGATHA_OUT_DEVICE;
  g.queue = queue;
  return run_batch(ctx, &g, params, out, (cudaStream_t)stream, -1, nullptr, nullptr, 0, &O);
}

// Device buffers other processes can map (CUDA IPC; over NVLink when on another GPU).
int agatha_ipc_alloc(agatha_ctx_t* ctx, uint64_t bytes, void** ptr, uint8_t handle[64]) {
  if (!ctx || !ptr || !handle || bytes == 0) return AGATHA_EINVAL;
  CUDA_TRY(cudaSetDevice(ctx->device));
  void* q = nullptr;
  if (cudaMalloc(&q, bytes) != cudaSuccess) {
    cudaGetLastError();
    return AGATHA_ENOMEM;
  }
  cudaIpcMemHandle_t h;
  if (cudaIpcGetMemHandle(&h, q) != cudaSuccess) {
    cudaGetLastError();
    cudaFree(q);
    return AGATHA_ECUDA;
  }
  memcpy(handle, &h, 64);
  *ptr = q;
  return AGATHA_OK;
}

int agatha_ipc_open(agatha_ctx_t* ctx, const uint8_t handle[64], void** ptr) {
  if (!ctx || !ptr || !handle) return AGATHA_EINVAL;
  CUDA_TRY(cudaSetDevice(ctx->device));
  cudaIpcMemHandle_t h;
  memcpy(&h, handle, 64);
  CUDA_TRY(cudaIpcOpenMemHandle(ptr, h, cudaIpcMemLazyEnablePeerAccess));
  return AGATHA_OK;
}

int agatha_ipc_close(agatha_ctx_t* ctx, void* ptr, int opened) {
  if (!ctx || !ptr) return AGATHA_EINVAL;
  CUDA_TRY(cudaSetDevice(ctx->device));
  CUDA_TRY(opened ? cudaIpcCloseMemHandle(ptr) : cudaFree(ptr));
  return AGATHA_OK;
}

int agatha_localmax_trace(agatha_ctx_t* ctx, const agatha_batch_t* batch, const agatha_params_t* params,
                          uint64_t pair, int32_t* score, int32_t* ref_i, int64_t cap, void* stream) {
  if (!ctx || !batch || !score || !ref_i || cap <= 0 || pair >= batch->n_pairs) return AGATHA_EINVAL;
  cudaStream_t st = (cudaStream_t)stream;
  CUDA_TRY(cudaSetDevice(ctx->device));
  int rc = grow(ctx->trace, 8 * (size_t)cap + sizeof(agatha_result_t) * batch->n_pairs);
  if (rc) return rc;
  int* ts = (int*)ctx->trace.p;
  int* ti = ts + cap;
  agatha_result_t* tout = (agatha_result_t*)(ti + cap);
  CUDA_TRY(cudaMemsetAsync(ts, 0, 4 * (size_t)cap, st));
  CUDA_TRY(cudaMemsetAsync(ti, 0xff, 4 * (size_t)cap, st));
  agatha_batch_t b2 = *batch;
  b2.flags |= AGATHA_OUT_DEVICE;
  b2.queue = nullptr;  // the traced pair must run on this context
  b2.ends = nullptr;
  rc = run_batch(ctx, &b2, params, tout, st, (long long)pair, ts, ti, cap);
  if (rc) return rc;
  CUDA_TRY(cudaMemcpyAsync(score, ts, 4 * (size_t)cap, cudaMemcpyDeviceToHost, st));
  CUDA_TRY(cudaMemcpyAsync(ref_i, ti, 4 * (size_t)cap, cudaMemcpyDeviceToHost, st));
  CUDA_TRY(cudaStreamSynchronize(st));
  return AGATHA_OK;
}

int agatha_pack4(agatha_ctx_t* ctx, const uint8_t* ascii, uint64_t len, uint32_t* words, uint32_t flags,
                 void* stream) {
  if (!ctx || !ascii || !words) return AGATHA_EINVAL;
  if (len == 0) return AGATHA_EEMPTY;
  cudaStream_t st = (cudaStream_t)stream;
  CUDA_TRY(cudaSetDevice(ctx->device));
  int rc = grow(ctx->scalars, 64);
  if (rc) return rc;
  int* d_sc = (int*)ctx->scalars.p;
  CUDA_TRY(cudaMemsetAsync(d_sc, 0, 4, st));
  const uint64_t nw = (len + 7) / 8;
  int blocks = (int)((nw + 255) / 256 < 8192 ? (nw + 255) / 256 : 8192);
  pack_seq_kernel<<<blocks, 256, 0, st>>>(ascii, len, words, (flags & AGATHA_PACK_REVERSE) != 0,
                                          (flags & AGATHA_N_MAP) != 0, d_sc);
  CUDA_TRY(cudaGetLastError());
  CUDA_TRY(cudaMemcpyAsync(ctx->h_scalars, d_sc, 4, cudaMemcpyDeviceToHost, st));
  CUDA_TRY(cudaStreamSynchronize(st));
  return ctx->h_scalars[0] ? AGATHA_ECHAR : AGATHA_OK;
}

int agatha_plan(agatha_ctx_t* ctx, const agatha_batch_t* b, const agatha_params_t* p, uint32_t* order,
                uint32_t* nominal, void* stream) {
  if (!ctx || !b || !order || !nominal) return AGATHA_EINVAL;
  int rc = check_params(p);
  if (rc) return rc;
  if (b->n_pairs == 0) return AGATHA_EEMPTY;
  if (!(b->flags & AGATHA_MEM_DEVICE)) return AGATHA_EINVAL;
  cudaStream_t st = (cudaStream_t)stream;
  CUDA_TRY(cudaSetDevice(ctx->device));
  const uint64_t P = b->n_pairs;
  size_t sort_bytes = 0;
  cub::DeviceRadixSort::SortPairsDescending(nullptr, sort_bytes, (const uint32_t*)nullptr,
                                            (uint32_t*)nullptr, (const uint32_t*)nullptr,
                                            (uint32_t*)nullptr, (int)P, 0, 32, st);
  if ((rc = grow(ctx->iota, 4 * P)) || (rc = grow(ctx->bad, P)) || (rc = grow(ctx->sort_tmp, sort_bytes)) ||
      (rc = grow(ctx->scalars, 64)))
    return rc;
  int* d_sc = (int*)ctx->scalars.p;
  CUDA_TRY(cudaMemsetAsync(d_sc, 0, 16, st));
  const int maxs = p->match > p->mismatch ? (p->match > p->ambig ? p->match : p->ambig)
                                          : (p->mismatch > p->ambig ? p->mismatch : p->ambig);
  PrepArgs pa;
  pa.roff = b->ref_off; pa.qoff = b->qry_off; pa.n_pairs = P;
  pa.bl = p->band_left; pa.br = p->band_right; pa.alpha = p->gap_open; pa.beta = p->gap_extend;
  pa.maxs = maxs;
  pa.nominal = nominal; pa.iota = (uint32_t*)ctx->iota.p;
  pa.bad = (uint8_t*)ctx->bad.p; pa.err_flags = d_sc; pa.max_slots = d_sc + 1; pa.max_off16 = d_sc + 3;
  pa.chunk_first = nullptr; pa.nchunks = 1; pa.chunk_of = nullptr; pa.key64 = nullptr;
  pa.tier_shift = 32; pa.tier_count = nullptr; pa.max_off16_t0 = nullptr; pa.lpt_from = 1;
  pa.off_mask16 = nullptr;
  pa.len_hash = nullptr; pa.own.n_owners = 0; pa.max_len = nullptr;
  const int prep_blocks = (int)(((P + 7) / 8) < 4096 ? ((P + 7) / 8) : 4096);
  prep_kernel<<<prep_blocks, 256, 0, st>>>(pa);
  CUDA_TRY(cudaGetLastError());
  if ((rc = grow(ctx->nominal_sorted, 4 * P))) return rc;
  size_t tb = ctx->sort_tmp.cap;
  CUDA_TRY(cub::DeviceRadixSort::SortPairsDescending(ctx->sort_tmp.p, tb, (const uint32_t*)nominal,
                                                     (uint32_t*)ctx->nominal_sorted.p,
                                                     (const uint32_t*)ctx->iota.p, order, (int)P, 0, 32, st));
  CUDA_TRY(cudaMemcpyAsync(ctx->h_scalars, d_sc, 4, cudaMemcpyDeviceToHost, st));
  CUDA_TRY(cudaStreamSynchronize(st));
  if (ctx->h_scalars[0] & 2) return AGATHA_EEMPTY;
  if (ctx->h_scalars[0] & 4) return AGATHA_ERANGE;
  return AGATHA_OK;
}

int agatha_get_stats(const agatha_ctx_t* ctx, agatha_stats_t* stats) {
  if (!ctx || !stats) return AGATHA_EINVAL;
  *stats = ctx->stats;
  return AGATHA_OK;
}

// NEXT #1: shared pair counters (cross-GPU / cross-process dynamic balancing).
int agatha_queue_create(agatha_ctx_t* ctx, int32_t** queue, uint8_t handle[64]) {
  if (!ctx || !queue || !handle) return AGATHA_EINVAL;
  CUDA_TRY(cudaSetDevice(ctx->device));
  int32_t* q = nullptr;
  if (cudaMalloc(&q, 256) != cudaSuccess) {
    cudaGetLastError();
    return AGATHA_ENOMEM;
  }
  CUDA_TRY(cudaMemset(q, 0, 256));
  cudaIpcMemHandle_t h;
  static_assert(sizeof(h) == 64, "CUDA IPC handles are 64 bytes");
  if (cudaIpcGetMemHandle(&h, q) != cudaSuccess) {
    cudaGetLastError();
    cudaFree(q);
    return AGATHA_ECUDA;
  }
  memcpy(handle, &h, 64);
  *queue = q;
  return AGATHA_OK;
}

int agatha_queue_open(agatha_ctx_t* ctx, const uint8_t handle[64], int32_t** queue) {
  if (!ctx || !queue || !handle) return AGATHA_EINVAL;
  CUDA_TRY(cudaSetDevice(ctx->device));
  cudaIpcMemHandle_t h;
  memcpy(&h, handle, 64);
  void* p = nullptr;
  CUDA_TRY(cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess));
  *queue = (int32_t*)p;
  return AGATHA_OK;
}

int agatha_queue_reset(agatha_ctx_t* ctx, int32_t* queue, void* stream) {
  if (!ctx || !queue) return AGATHA_EINVAL;
  CUDA_TRY(cudaSetDevice(ctx->device));
  // the tier counters [0..2] and the batch fingerprint [8]
  CUDA_TRY(cudaMemsetAsync(queue, 0, 16 * sizeof(int32_t), (cudaStream_t)stream));
  return AGATHA_OK;
}

int agatha_queue_close(agatha_ctx_t* ctx, int32_t* queue, int opened) {
  if (!ctx || !queue) return AGATHA_EINVAL;
  CUDA_TRY(cudaSetDevice(ctx->device));
  CUDA_TRY(opened ? cudaIpcCloseMemHandle(queue) : cudaFree(queue));
  return AGATHA_OK;
}

}  // extern "C"
