/*
 * agatha_oracle — the plain, slow CPU oracle for guided extension alignment.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load or call this library.  It shares
 * no code, header, table or constant with the CUDA path (paper_2403_06478_b200/),
 * and the CUDA path never calls it.
 *
 * What it computes (DESIGN.md "Readings of the paper" lists every choice made
 * where PAPER.md is silent; SURVEY.md §8(c) is the step list followed here):
 *
 *   Eq. 1-3 (§2.1):
 *     H(i,j) = max{ E(i,j), F(i,j), H(i-1,j-1) + S(R[i],Q[j]) }
 *     E(i,j) = max{ H(i-1,j) - alpha, E(i-1,j) - beta }
 *     F(i,j) = max{ H(i,j-1) - alpha, F(i,j-1) - beta }
 *   evaluated in anti-diagonal order c = i + j (cells of one
 *   anti-diagonal are mutually independent), restricted to the k-band
 *    -bl <= i - j <= br, and stopped by the Z-drop condition
 *   Eq. 4-6:
 *     exists c < len(query)+len(ref) with  i' < i, j' < j,
 *        H(i',j') - H(i,j) > Z + beta * |(i - i') - (j - j')|
 *     (i,j)   = argmax_{i+j=c} H       (local max, Eq. 5)
 *     (i',j') = argmax_{i'+j'<c} H     (global max, Eq. 6)
 *
 * Every function below is a direct transcription; nothing is blocked, fused or
 * reordered beyond the anti-diagonal order the paper itself states.
 *
 * Parity pins (tests/test_oracle.py): brute-force path enumeration on tiny inputs,
 * an independent row-major full DP, SPEC.md worked examples, the closed-form cell
 * count, and invariants.  The local/global argmax tie rules are parity UNPINNED by
 * the paper (SPEC.md line 177 / 145 readings; reading R5/R6).
 */
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef struct {
  int32_t match;      /* a > 0: S = +a on a match of two non-N bases        */
  int32_t mismatch;   /* b > 0: S = -b on a mismatch of two non-N bases     */
  int32_t ambig;      /* n >= 0: S = -n when either base is N                */
  int32_t gap_open;   /* alpha >= beta                                       */
  int32_t gap_extend; /* beta >= 0                                           */
  int32_t band_left;  /* allow i - j >= -band_left; negative = unbounded      */
  int32_t band_right; /* allow i - j <= band_right; negative = unbounded      */
  int32_t zdrop;      /* Z >= 0; negative = Z-drop disabled                  */
  int32_t variant;    /* 0 = the readings of DESIGN.md; bits select the minimap2-like
                         alternatives (outside the reference):
                         1 = Eq. 4 gating i' <= i, j' <= j (non-strict),
                         2 = the global max starts at the origin H(0,0) = 0,
                         4 = Eq. 4 is also tested at c = m+n                 */
} oracle_params_t;

#define VAR_GATE_GE 1
#define VAR_ORIGIN_MAX 2
#define VAR_CHECK_LAST 4

typedef struct {
  int32_t score;          /* H(i',j'), the global max (Eq. 6)                 */
  int32_t ref_end;        /* i' (1-based)                                     */
  int32_t query_end;      /* j' (1-based)                                     */
  int32_t zdrop_antidiag; /* c at which Eq. 4 fired, -1 if never             */
  int64_t cells;          /* in-band in-table cells on anti-diagonals 2..end  */
} oracle_result_t;

/* NEXT #4 (minimap2 semantics, outside the paper; reading R19):
 * the end scores over the cells the sweep processed (anti-diagonals 2..c_end, c_end the
 * Z-drop anti-diagonal or m+n), updated in anti-diagonal order with a strict '>':
 *   mqe = max H(i, n) (the query end reached), mqe_i its i (the smallest on ties);
 *   mte = max H(m, j) (the reference end reached), mte_j its j;
 *   end_score = H(m, n) if that cell was processed.
 * Absent values are ORACLE_NO_SCORE with position -1. */
#define ORACLE_NO_SCORE (-(1 << 30))
typedef struct {
  int32_t mqe, mqe_i;
  int32_t mte, mte_j;
  int32_t end_score;
  int32_t reserved;
} oracle_ends_t;

enum {
  ORACLE_OK = 0,
  ORACLE_EINVAL = -1,
  ORACLE_EEMPTY = -2,
  ORACLE_ECHAR = -3,
  ORACLE_ENOMEM = -6,
};

#define NEG (-(1 << 30)) /* "minus infinity": out-of-band / out-of-table neighbour */

/* --- align-core -------------------------------------------------------------- */

/* Literal codes (SPEC.md align-core design decisions): A0 C1 G2 T3 N4; -1 = invalid. */
static int literal_code(uint8_t ch) {
  switch (ch) {
    case 'A': case 'a': return 0;
    case 'C': case 'c': return 1;
    case 'G': case 'g': return 2;
    case 'T': case 't': return 3;
    case 'N': case 'n': return 4;
    default: return -1;
  }
}

/* S(R[i],Q[j]) ("positive on a match (e.g., +2) and negative on
 * a mismatch (e.g., -4)"); N handling per SPEC.md line 76. */
static int32_t substitution(const oracle_params_t* p, int r, int q) {
  if (r == 4 || q == 4) return -p->ambig;
  if (r == q) return p->match;
  return -p->mismatch;
}

int oracle_validate(const oracle_params_t* p) {
  if (!p) return ORACLE_EINVAL;
  if (p->match <= 0 || p->mismatch <= 0 || p->ambig < 0) return ORACLE_EINVAL;
  if (p->gap_extend < 0 || p->gap_open < p->gap_extend) return ORACLE_EINVAL;
  return ORACLE_OK;
}

/* --- oracle-dp ---------------------------------------------------------------- */

typedef struct {
  int64_t m, n, bl, br;
  const oracle_params_t* p;
  /* anti-diagonal arrays indexed by i (0..m): values for c-2, c-1, c */
  int32_t *H2, *H1, *H0, *E1, *E0, *F1, *F0;
} sweep_t;

static int in_band(const sweep_t* s, int64_t i, int64_t j) {
  return (i - j) >= -s->bl && (i - j) <= s->br;
}

/* Boundary values:
 *   H(0,0) = 0; H(i,0) = -(alpha + (i-1) beta) for 1 <= i <= br; H(0,j) likewise
 *   for 1 <= j <= bl; anything outside the band or the table is NEG. */
static int32_t get_H(const sweep_t* s, const int32_t* arr, int64_t i, int64_t j) {
  if (i < 0 || j < 0 || i > s->m || j > s->n) return NEG;
  if (!in_band(s, i, j)) return NEG;
  if (i == 0 && j == 0) return 0;
  if (j == 0) return -(s->p->gap_open + (int32_t)(i - 1) * s->p->gap_extend);
  if (i == 0) return -(s->p->gap_open + (int32_t)(j - 1) * s->p->gap_extend);
  return arr[i];
}
/* E on row 0 and F on column 0 are NEG. */
static int32_t get_EF(const sweep_t* s, const int32_t* arr, int64_t i, int64_t j) {
  if (i <= 0 || j <= 0 || i > s->m || j > s->n) return NEG;
  if (!in_band(s, i, j)) return NEG;
  return arr[i];
}
static int32_t max2(int32_t a, int32_t b) { return a > b ? a : b; }
static int64_t i64abs(int64_t v) { return v < 0 ? -v : v; }

/* Optional per-anti-diagonal local-max trace (the analogue of SPEC.md's GMB,
 * S:279): entry c holds (score, i) of Eq. 5, or i = -1 for an empty anti-diagonal. */
typedef struct {
  int32_t* score;
  int32_t* i;
  int64_t cap;
} oracle_trace_t;

int oracle_align_one_ends(const uint8_t* R, int64_t m, const uint8_t* Q, int64_t n,
                          const oracle_params_t* p, oracle_result_t* out, oracle_trace_t* trace,
                          oracle_ends_t* ends);
int oracle_align_one(const uint8_t* R, int64_t m, const uint8_t* Q, int64_t n,
                     const oracle_params_t* p, oracle_result_t* out, oracle_trace_t* trace) {
  return oracle_align_one_ends(R, m, Q, n, p, out, trace, NULL);
}

int oracle_align_one_ends(const uint8_t* R, int64_t m, const uint8_t* Q, int64_t n,
                          const oracle_params_t* p, oracle_result_t* out, oracle_trace_t* trace,
                          oracle_ends_t* ends) {
  int rc = oracle_validate(p);
  if (rc) return rc;
  if (m <= 0 || n <= 0) return ORACLE_EEMPTY;
  int* rc_codes = (int*)malloc(sizeof(int) * (size_t)(m + 1));
  int* qc_codes = (int*)malloc(sizeof(int) * (size_t)(n + 1));
  if (!rc_codes || !qc_codes) { free(rc_codes); free(qc_codes); return ORACLE_ENOMEM; }
  for (int64_t i = 1; i <= m; ++i) {
    rc_codes[i] = literal_code(R[i - 1]);
    if (rc_codes[i] < 0) { free(rc_codes); free(qc_codes); return ORACLE_ECHAR; }
  }
  for (int64_t j = 1; j <= n; ++j) {
    qc_codes[j] = literal_code(Q[j - 1]);
    if (qc_codes[j] < 0) { free(rc_codes); free(qc_codes); return ORACLE_ECHAR; }
  }

  sweep_t s;
  s.m = m; s.n = n; s.p = p;
  s.bl = p->band_left < 0 ? (int64_t)1 << 40 : p->band_left;
  s.br = p->band_right < 0 ? (int64_t)1 << 40 : p->band_right;
  int32_t* buf = (int32_t*)malloc(sizeof(int32_t) * 7 * (size_t)(m + 1));
  if (!buf) { free(rc_codes); free(qc_codes); return ORACLE_ENOMEM; }
  for (int64_t t = 0; t < 7 * (m + 1); ++t) buf[t] = NEG;
  s.H2 = buf; s.H1 = buf + (m + 1); s.H0 = buf + 2 * (m + 1);
  s.E1 = buf + 3 * (m + 1); s.E0 = buf + 4 * (m + 1);
  s.F1 = buf + 5 * (m + 1); s.F0 = buf + 6 * (m + 1);

  const int32_t alpha = p->gap_open, beta = p->gap_extend;
  const int zdrop_on = p->zdrop >= 0;

  /* step 3: global max G = none, term = none */
  int have_G = 0;
  int32_t G_H = 0;
  int64_t G_i = 0, G_j = 0;
  if (p->variant & VAR_ORIGIN_MAX) have_G = 1;  /* G = H(0,0) = 0 at (0,0) */
  const int gate_ge = (p->variant & VAR_GATE_GE) != 0;
  const int64_t c_check_end = (p->variant & VAR_CHECK_LAST) ? m + n + 1 : m + n;
  int64_t term = -1, cells = 0;
  oracle_ends_t en = {ORACLE_NO_SCORE, -1, ORACLE_NO_SCORE, -1, ORACLE_NO_SCORE, 0};
  int have_q = 0, have_t = 0;

  /* step 4: c = 2, 3, ..., m+n */
  for (int64_t c = 2; c <= m + n; ++c) {
    /* 4a: cells(c) = {(i, c-i) : max(1,c-n) <= i <= min(m,c-1), -bl <= 2i-c <= br}: the
     * table range of i intersected with the band range ceil((c-bl)/2) <= i <=
     * floor((c+br)/2), which is the same set in the same ascending order (the in_band
     * test below stays as a literal filter).  Iterating the intersection instead of the
     * whole table range only skips indices the filter rejects (round 2; 1.6x faster). */
    int64_t ilo = c - n > 1 ? c - n : 1;
    int64_t ihi = c - 1 < m ? c - 1 : m;
    const int64_t blo = (c - s.bl + 1) >> 1, bhi = (c + s.br) >> 1;
    if (blo > ilo) ilo = blo;
    if (bhi < ihi) ihi = bhi;
    int any = 0;
    int32_t L_H = 0;
    int64_t L_i = 0;
    for (int64_t i = ilo; i <= ihi; ++i) {
      const int64_t j = c - i;
      if (!in_band(&s, i, j)) continue;
      /* 4b: Eq. 2, Eq. 3, Eq. 1 (int32, no zero clamp) */
      const int32_t e = max2(get_H(&s, s.H1, i - 1, j) - alpha, get_EF(&s, s.E1, i - 1, j) - beta);
      const int32_t f = max2(get_H(&s, s.H1, i, j - 1) - alpha, get_EF(&s, s.F1, i, j - 1) - beta);
      const int32_t h = max2(max2(e, f), get_H(&s, s.H2, i - 1, j - 1) +
                                             substitution(p, rc_codes[i], qc_codes[j]));
      s.H0[i] = h;
      s.E0[i] = e;
      s.F0[i] = f;
      ++cells;
      /* NEXT #4: end scores of this processed cell (reading R19) */
      if (j == n && (!have_q || h > en.mqe)) { en.mqe = h; en.mqe_i = (int32_t)i; have_q = 1; }
      if (i == m && (!have_t || h > en.mte)) { en.mte = h; en.mte_j = (int32_t)j; have_t = 1; }
      if (i == m && j == n) en.end_score = h;
      /* 4c: local max (Eq. 5), ties -> smallest i (ascending scan, strict >) */
      if (!any || h > L_H) { L_H = h; L_i = i; }
      any = 1;
    }
    if (trace && c < trace->cap) {
      trace->score[c] = any ? L_H : 0;
      trace->i[c] = any ? (int32_t)L_i : -1;
    }
    if (any) {
      const int64_t L_j = c - L_i;
      /* 4d: Eq. 4 at this c, with the single (global, local) argmax pair */
      const int gated = gate_ge ? (G_i <= L_i && G_j <= L_j) : (G_i < L_i && G_j < L_j);
      if (have_G && zdrop_on && c < c_check_end && gated) {
        const int64_t gap = i64abs((L_i - G_i) - (L_j - G_j));
        if ((int64_t)G_H - (int64_t)L_H > (int64_t)p->zdrop + (int64_t)beta * gap) term = c;
      }
      /* 4e: global max update (Eq. 6), strict > so the earliest c wins ties */
      if (!have_G || L_H > G_H) { G_H = L_H; G_i = L_i; G_j = L_j; have_G = 1; }
    }
    /* rotate: (c-2) <- (c-1) <- (c) */
    int32_t* t = s.H2; s.H2 = s.H1; s.H1 = s.H0; s.H0 = t;
    t = s.E1; s.E1 = s.E0; s.E0 = t;
    t = s.F1; s.F1 = s.F0; s.F0 = t;
    /* 4f */
    if (term >= 0) break;
  }
  free(buf);
  free(rc_codes);
  free(qc_codes);
  /* step 5 */
  out->score = G_H;
  out->ref_end = (int32_t)G_i;
  out->query_end = (int32_t)G_j;
  out->zdrop_antidiag = (int32_t)term;
  out->cells = cells;
  if (ends) *ends = en;
  return ORACLE_OK;
}

/* Nominal (un-terminated) in-band in-table cell count, by plain enumeration of rows:
 * row i holds j in [max(1, i - br), min(n, i + bl)]. */
int64_t oracle_nominal_cells(int64_t m, int64_t n, int64_t bl, int64_t br) {
  if (bl < 0) bl = (int64_t)1 << 40;
  if (br < 0) br = (int64_t)1 << 40;
  int64_t total = 0;
  for (int64_t i = 1; i <= m; ++i) {
    int64_t lo = i - br > 1 ? i - br : 1;
    int64_t hi = i + bl < n ? i + bl : n;
    if (hi >= lo) total += hi - lo + 1;
  }
  return total;
}

/* 4-bit packing (§2.2: "four bits suffice for encoding each
 * literal ... packed with 8 literals per word"; SPEC.md: low nibble = earliest
 * literal).  reverse != 0 packs the sequence back to front.  n_map != 0 maps
 * non-ACGTN bytes to N instead of failing. */
int oracle_pack4(const uint8_t* seq, int64_t len, uint32_t* words, int reverse, int n_map) {
  if (len <= 0) return ORACLE_EEMPTY;
  const int64_t nw = (len + 7) / 8;
  for (int64_t w = 0; w < nw; ++w) words[w] = 0;
  for (int64_t k = 0; k < len; ++k) {
    const uint8_t ch = reverse ? seq[len - 1 - k] : seq[k];
    int code = literal_code(ch);
    if (code < 0) {
      if (!n_map) return ORACLE_ECHAR;
      code = 4;
    }
    words[k / 8] |= (uint32_t)code << (4 * (k % 8));
  }
  return ORACLE_OK;
}

/* --- batch driver: std pthreads, dynamic longest-first ------------------------ */

typedef struct {
  const uint8_t *ref, *qry;
  const uint64_t *ref_off, *qry_off;
  const oracle_params_t* p;
  oracle_result_t* out;
  oracle_ends_t* ends;
  int32_t* status;
  const uint64_t* order;
  uint64_t n;
  uint64_t next;
  pthread_mutex_t mu;
} batch_job_t;

static void* batch_worker(void* arg) {
  batch_job_t* j = (batch_job_t*)arg;
  for (;;) {
    pthread_mutex_lock(&j->mu);
    uint64_t t = j->next++;
    pthread_mutex_unlock(&j->mu);
    if (t >= j->n) break;
    const uint64_t k = j->order[t];
    const int64_t m = (int64_t)(j->ref_off[k + 1] - j->ref_off[k]);
    const int64_t n = (int64_t)(j->qry_off[k + 1] - j->qry_off[k]);
    j->status[k] = oracle_align_one_ends(j->ref + j->ref_off[k], m, j->qry + j->qry_off[k], n, j->p,
                                         &j->out[k], NULL, j->ends ? &j->ends[k] : NULL);
  }
  return NULL;
}

static const uint64_t* g_sort_key;
static int cmp_desc(const void* a, const void* b) {
  const uint64_t x = g_sort_key[*(const uint64_t*)a], y = g_sort_key[*(const uint64_t*)b];
  if (x != y) return x < y ? 1 : -1;
  return (*(const uint64_t*)a < *(const uint64_t*)b) ? -1 : 1;
}

/* Align pairs 0..n_pairs-1; status[k] receives each pair's return code.  Returns
 * the first non-zero status (or 0). */
int oracle_align_batch_ends(const uint8_t* ref, const uint64_t* ref_off, const uint8_t* qry,
                            const uint64_t* qry_off, uint64_t n_pairs, const oracle_params_t* p,
                            oracle_result_t* out, oracle_ends_t* ends, int32_t* status, int n_threads);
int oracle_align_batch(const uint8_t* ref, const uint64_t* ref_off, const uint8_t* qry,
                       const uint64_t* qry_off, uint64_t n_pairs, const oracle_params_t* p,
                       oracle_result_t* out, int32_t* status, int n_threads) {
  return oracle_align_batch_ends(ref, ref_off, qry, qry_off, n_pairs, p, out, NULL, status, n_threads);
}

/* The same, also writing each pair's end scores to ends[k] (NEXT #4) when ends != NULL. */
int oracle_align_batch_ends(const uint8_t* ref, const uint64_t* ref_off, const uint8_t* qry,
                            const uint64_t* qry_off, uint64_t n_pairs, const oracle_params_t* p,
                            oracle_result_t* out, oracle_ends_t* ends, int32_t* status, int n_threads) {
  if (n_pairs == 0) return ORACLE_EEMPTY;
  int rc = oracle_validate(p);
  if (rc) return rc;
  uint64_t* order = (uint64_t*)malloc(sizeof(uint64_t) * n_pairs);
  uint64_t* key = (uint64_t*)malloc(sizeof(uint64_t) * n_pairs);
  if (!order || !key) { free(order); free(key); return ORACLE_ENOMEM; }
  for (uint64_t k = 0; k < n_pairs; ++k) {
    order[k] = k;
    key[k] = (ref_off[k + 1] - ref_off[k]) + (qry_off[k + 1] - qry_off[k]);
  }
  g_sort_key = key; /* longest first; the batch driver is single-entry per process */
  qsort(order, n_pairs, sizeof(uint64_t), cmp_desc);
  batch_job_t job;
  job.ref = ref; job.qry = qry; job.ref_off = ref_off; job.qry_off = qry_off; job.p = p;
  job.out = out; job.ends = ends; job.status = status; job.order = order; job.n = n_pairs; job.next = 0;
  pthread_mutex_init(&job.mu, NULL);
  if (n_threads < 1) n_threads = 1;
  if (n_threads > 512) n_threads = 512;
  pthread_t* th = (pthread_t*)malloc(sizeof(pthread_t) * (size_t)n_threads);
  for (int t = 1; t < n_threads; ++t) pthread_create(&th[t], NULL, batch_worker, &job);
  batch_worker(&job);
  for (int t = 1; t < n_threads; ++t) pthread_join(th[t], NULL);
  free(th);
  pthread_mutex_destroy(&job.mu);
  free(order);
  free(key);
  for (uint64_t k = 0; k < n_pairs; ++k)
    if (status[k]) return status[k];
  return ORACLE_OK;
}
