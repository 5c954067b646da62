/*
 * agatha_synth — seeded synthetic (reference window R, read Q) pair generator.
 *
 * This module is shared INPUT infrastructure: the oracle (oracle/), the CUDA path
 * (paper_2403_06478_b200/), the tests and bench.py all consume the pairs it writes.
 * It contains none of the alignment method's arithmetic (no scoring, no DP, no
 * packing): it only draws bases.
 *
 * Recipe (SURVEY.md §8(d) "Synthetic inputs"):
 *   - every random number is a pure function of (seed, pair k, stream, counter)
 *     (counter-based: splitmix64 finaliser over a keyed counter), so any rank can
 *     generate any shard of pairs independently and identically;
 *   - template T0: i.i.d. uniform ACGT with N at probability n_rate per base;
 *   - read length Ls from the configured length distribution;
 *   - read Q: walk T0 emitting exactly Ls bases; per emitted base an error event
 *     with probability e (per-pair e ~ U[err_lo, err_hi]) split into
 *     substitution / insertion / deletion by (f_sub, f_ins, f_del);
 *   - chimeric pairs (probability p_chim): after a breakpoint b ~ U[0.05,0.95]*Ls the
 *     read continues with unrelated i.i.d. bases (the Z-drop trigger);
 *   - reference window R = T0[0 : Ls + ceil(ref_extra_frac*Ls) + ref_extra_abs].
 * Output is upper-case ASCII, concatenated, with uint64 offsets.
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef struct {
  uint32_t len_dist;      /* 0: uniform [lo,hi]; 1: log-uniform [lo,hi]; 2: mixture of
                             log-uniforms; 3: two-point mixture (lo2 w.p. p_long, else lo) */
  uint32_t ref_extra_abs; /* extra reference bases after the read end */
  double lo, hi;          /* length range (short component for the mixture) */
  double lo2, hi2;        /* long component of the mixture (log-uniform) */
  double p_long;          /* mixture weight of the long component */
  double err_lo, err_hi;  /* per-pair error rate ~ U[err_lo, err_hi] */
  double f_sub, f_ins, f_del;
  double p_chim;          /* probability a pair is chimeric */
  double n_rate;          /* probability a template base is N */
  double ref_extra_frac;  /* reference window extension, fraction of Ls */
} synth_cfg_t;

enum { ST_LEN = 1, ST_ERR = 2, ST_CHIM = 3, ST_BRK = 4, ST_T0 = 5, ST_WALK = 6, ST_JUNK = 7 };

static inline uint64_t mix64(uint64_t z) {
  z += 0x9e3779b97f4a7c15ULL;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}
static inline uint64_t key_of(uint64_t seed, uint64_t k, uint64_t stream) {
  return mix64(mix64(seed * 0x632be59bd9b4e019ULL + stream) ^ (k * 0xd6e8feb86659fd93ULL));
}
static inline uint64_t rnd(uint64_t key, uint64_t ctr) { return mix64(key + ctr * 0x9e3779b97f4a7c15ULL); }
static inline double unif(uint64_t r) { return (double)(r >> 11) * (1.0 / 9007199254740992.0); }

static const char kACGT[4] = {'A', 'C', 'G', 'T'};

static uint64_t draw_len(const synth_cfg_t* c, uint64_t seed, uint64_t k) {
  uint64_t key = key_of(seed, k, ST_LEN);
  double u = unif(rnd(key, 0)), v = unif(rnd(key, 1));
  double lo = c->lo, hi = c->hi;
  int logu = (c->len_dist == 1);
  if (c->len_dist == 2) {
    logu = 1;
    if (v < c->p_long) { lo = c->lo2; hi = c->hi2; }
  }
  double L;
  if (c->len_dist == 3) return (uint64_t)(v < c->p_long ? c->lo2 : c->lo);
  if (logu) L = exp(log(lo) + u * (log(hi) - log(lo)));
  else L = lo + u * (hi - lo + 1.0);
  uint64_t Li = (uint64_t)floor(L);
  if (Li < (uint64_t)lo) Li = (uint64_t)lo;
  if (Li > (uint64_t)hi) Li = (uint64_t)hi;
  if (Li < 1) Li = 1;
  return Li;
}

static inline uint64_t ref_len_of(const synth_cfg_t* c, uint64_t Ls) {
  return Ls + (uint64_t)ceil(c->ref_extra_frac * (double)Ls) + c->ref_extra_abs;
}

/* Template base x of pair k: a pure function of (seed, k, x). */
static inline char t0_base(uint64_t key_t0, double n_rate, uint64_t x) {
  uint64_t r = rnd(key_t0, x);
  if (n_rate > 0.0 && unif(r) < n_rate) return 'N';
  return kACGT[(r >> 3) & 3];
}

int synth_lengths(const synth_cfg_t* c, uint64_t seed, uint64_t k0, uint64_t k1, uint64_t* rlen,
                  uint64_t* qlen) {
  if (!c || k1 < k0) return -1;
  for (uint64_t k = k0; k < k1; ++k) {
    uint64_t Ls = draw_len(c, seed, k);
    qlen[k - k0] = Ls;
    rlen[k - k0] = ref_len_of(c, Ls);
  }
  return 0;
}

static void fill_one(const synth_cfg_t* c, uint64_t seed, uint64_t k, uint8_t* R, uint8_t* Q) {
  const uint64_t Ls = draw_len(c, seed, k), Lr = ref_len_of(c, Ls);
  const uint64_t kt = key_of(seed, k, ST_T0);
  for (uint64_t x = 0; x < Lr; ++x) R[x] = (uint8_t)t0_base(kt, c->n_rate, x);

  const uint64_t ke = key_of(seed, k, ST_ERR);
  const double e = c->err_lo + unif(rnd(ke, 0)) * (c->err_hi - c->err_lo);
  const double fs = c->f_sub + c->f_ins + c->f_del;
  const double p_sub = fs > 0 ? e * c->f_sub / fs : 0, p_ins = fs > 0 ? e * c->f_ins / fs : 0,
               p_del = fs > 0 ? e * c->f_del / fs : 0;
  const int chim = unif(rnd(key_of(seed, k, ST_CHIM), 0)) < c->p_chim;
  uint64_t brk = Ls;
  if (chim) brk = (uint64_t)floor((0.05 + 0.9 * unif(rnd(key_of(seed, k, ST_BRK), 0))) * (double)Ls);

  const uint64_t kw = key_of(seed, k, ST_WALK), kj = key_of(seed, k, ST_JUNK);
  uint64_t x = 0, q = 0, step = 0;
  while (q < Ls) {
    if (q >= brk) {
      Q[q] = (uint8_t)kACGT[rnd(kj, q) & 3];
      ++q;
      continue;
    }
    const uint64_t r = rnd(kw, step++);
    const double u = unif(r);
    const char tb = x < Lr ? (char)R[x] : t0_base(kt, c->n_rate, x);
    if (u < p_sub) {          /* substitution: a different base */
      int code = (tb == 'A') ? 0 : (tb == 'C') ? 1 : (tb == 'G') ? 2 : (tb == 'T') ? 3 : 0;
      Q[q++] = (uint8_t)kACGT[(code + 1 + (int)((r >> 7) % 3)) & 3];
      ++x;
    } else if (u < p_sub + p_ins) { /* insertion: a random base, template not consumed */
      Q[q++] = (uint8_t)kACGT[(r >> 7) & 3];
    } else if (u < p_sub + p_ins + p_del) { /* deletion: template consumed, nothing emitted */
      ++x;
    } else {
      Q[q++] = (uint8_t)tb;
      ++x;
    }
  }
}

typedef struct {
  const synth_cfg_t* c;
  uint64_t seed, k0, k1;
  const uint64_t *roff, *qoff;
  uint8_t *R, *Q;
  volatile uint64_t* next;
  pthread_mutex_t* mu;
  const uint64_t* idx; /* NULL: pairs k0..k1-1; else pairs idx[0..k1-k0-1] */
} fill_job_t;

static void* fill_worker(void* arg) {
  fill_job_t* j = (fill_job_t*)arg;
  for (;;) {
    uint64_t k;
    pthread_mutex_lock(j->mu);
    k = *j->next;
    *j->next = k + 64;
    pthread_mutex_unlock(j->mu);
    if (k >= j->k1) break;
    uint64_t kend = k + 64 < j->k1 ? k + 64 : j->k1;
    for (; k < kend; ++k) {
      const uint64_t t = k - j->k0;
      fill_one(j->c, j->seed, j->idx ? j->idx[t] : k, j->R + j->roff[t], j->Q + j->qoff[t]);
    }
  }
  return NULL;
}

/* roff/qoff: k1-k0+1 offsets (bytes) into R/Q for pairs k0..k1-1, as produced from
 * synth_lengths by an exclusive prefix sum. */
int synth_fill(const synth_cfg_t* c, uint64_t seed, uint64_t k0, uint64_t k1, const uint64_t* roff,
               const uint64_t* qoff, uint8_t* R, uint8_t* Q, int nthreads) {
  if (!c || k1 < k0) return -1;
  if (nthreads < 1) nthreads = 1;
  if (nthreads > 256) nthreads = 256;
  volatile uint64_t next = k0;
  pthread_mutex_t mu;
  pthread_mutex_init(&mu, NULL);
  fill_job_t job = {c, seed, k0, k1, roff, qoff, R, Q, &next, &mu, NULL};
  pthread_t th[256];
  for (int t = 1; t < nthreads; ++t) pthread_create(&th[t], NULL, fill_worker, &job);
  fill_worker(&job);
  for (int t = 1; t < nthreads; ++t) pthread_join(th[t], NULL);
  pthread_mutex_destroy(&mu);
  return 0;
}

/* The same pairs by index: pair idx[t] of the stream at position t (a rank's share of a
 * partition that is not a contiguous range, bench.py --gpus N).  Identical bytes to
 * synth_lengths / synth_fill for every pair. */
int synth_lengths_idx(const synth_cfg_t* c, uint64_t seed, const uint64_t* idx, uint64_t n,
                      uint64_t* rlen, uint64_t* qlen) {
  if (!c) return -1;
  for (uint64_t t = 0; t < n; ++t) {
    const uint64_t Ls = draw_len(c, seed, idx[t]);
    qlen[t] = Ls;
    rlen[t] = ref_len_of(c, Ls);
  }
  return 0;
}

int synth_fill_idx(const synth_cfg_t* c, uint64_t seed, const uint64_t* idx, uint64_t n,
                   const uint64_t* roff, const uint64_t* qoff, uint8_t* R, uint8_t* Q, int nthreads) {
  if (!c) return -1;
  if (nthreads < 1) nthreads = 1;
  if (nthreads > 256) nthreads = 256;
  volatile uint64_t next = 0;
  pthread_mutex_t mu;
  pthread_mutex_init(&mu, NULL);
  fill_job_t job = {c, seed, 0, n, roff, qoff, R, Q, &next, &mu, idx};
  pthread_t th[256];
  for (int t = 1; t < nthreads; ++t) pthread_create(&th[t], NULL, fill_worker, &job);
  fill_worker(&job);
  for (int t = 1; t < nthreads; ++t) pthread_join(th[t], NULL);
  pthread_mutex_destroy(&mu);
  return 0;
}
