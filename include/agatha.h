/*
 * agatha.h — C ABI of the B200-native guided extension aligner (libagatha.so).
 *
 * The operation (§2.1):
 *   for every (reference window R, read Q) pair of a batch, fill the banded affine-gap
 *   DP table of Eq. 1-3 anti-diagonal by anti-diagonal
 *   (l.229), restricted to the k-band (l.248-250), stop at the first anti-diagonal c
 *   where the Z-drop condition Eq. 4 holds between the global max Eq. 6 and the local
 *   max Eq. 5 (l.258-266), and report the global max score and its position.
 * Every reading of a point the paper leaves open (boundary values, tie rules, gating,
 * N scoring, ...) is listed in DESIGN.md "Readings of the paper" and followed exactly.
 *
 * Calling conventions
 *   - Every function returns 0 (AGATHA_OK) or a negative AGATHA_E* code; the text of a
 *     code is agatha_strerror(code).  On error the contents of `out` are unspecified.
 *   - The caller owns every input and output buffer.  A context owns its device scratch
 *     (packed sequences, plan arrays, queue counter), grows it on demand and frees it in
 *     agatha_ctx_destroy.  Nothing is retained after a call returns.
 *   - One context per host thread.  Work is issued on `cuda_stream` (a cudaStream_t, or
 *     NULL for the legacy default stream); the call returns after the work completes
 *     (it synchronises `cuda_stream` to collect the error flags).
 *   - No CPU fallback exists: without a usable sm_100a device every call that needs the
 *     GPU returns AGATHA_ECUDA.
 */
#ifndef AGATHA_H_
#define AGATHA_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- error codes ---------------------------------------------------------------- */
#define AGATHA_OK 0
#define AGATHA_EINVAL (-1) /* invalid scoring parameters or arguments  */
#define AGATHA_EEMPTY (-2) /* a sequence of length 0 or n_pairs == 0 */
#define AGATHA_ECHAR (-3)  /* a non-ACGTN byte under AGATHA_N_REJECT         */
#define AGATHA_ERANGE (-4) /* band wider than 4096 diagonals, penalties > 127, a pair with
                              alpha*(m+n) + |H| >= 2^30 or >= 2^31 cells, or (only when the
                              32-bit kernel must run: scoring outside the 16-bit guard,
                              bands over 1024 diagonals, AGATHA_FORCE_32BIT) a pair so long
                              that |H| could reach 2^20            */
#define AGATHA_ECUDA (-5)  /* CUDA runtime failure / no sm_100a device                    */
#define AGATHA_ENOMEM (-6) /* device allocation failed                                    */

/* ---- batch flags ---------------------------------------------------------------- */
#define AGATHA_MEM_HOST 0u        /* ref/qry/offsets are host pointers (default)          */
#define AGATHA_MEM_DEVICE 1u      /* ref/qry/offsets are device pointers                  */
#define AGATHA_OUT_DEVICE 2u      /* `out` is a device pointer                            */
#define AGATHA_N_REJECT 0u        /* non-ACGTN bytes are an error (default)               */
#define AGATHA_N_MAP 4u           /* non-ACGTN bytes are scored as N                      */
#define AGATHA_PACK_REVERSE 8u    /* agatha_pack4 only: pack back to front                */
#define AGATHA_ORDER_INPUT 16u    /* dispatch pairs in input order instead of longest-first
                                     (ordering ablation; results are identical)           */
#define AGATHA_FORCE_32BIT 32u    /* use the 32-bit kernel even when the 16-bit packed one is
                                     exact for these parameters (results are identical)   */
#define AGATHA_SINGLE_TIER 64u    /* run every pair of the 16-bit kernel at the front the
                                     batch's widest band needs, in one launch, instead of
                                     each pair at the narrowest slot tier that holds its
                                     band (tier ablation; results are identical)          */
#define AGATHA_STATIC_ASSIGN 128u /* no work queue: persistent warp u of a launch takes the
                                     order positions u, u + W, u + 2W, ... (W warps), so a
                                     warp that finishes early is not refilled (the analogue
                                     of the paper's no-rejoining baseline, P:754-761;
                                     results are identical; not with a shared queue)      */

/* Scoring (Eq. 1-4 symbols).  Penalties are POSITIVE numbers. */
typedef struct {
  int32_t match;      /* a, 1..127: S = +a when R[i] == Q[j] and neither is N          */
  int32_t mismatch;   /* b, 1..127: S = -b                                              */
  int32_t ambig;      /* n, 0..127: S = -n when either base is N (N vs N included)      */
  int32_t gap_open;   /* alpha >= beta: a gap run of length k costs alpha + (k-1)*beta  */
  int32_t gap_extend; /* beta >= 0; also Eq. 4's beta                                   */
  int32_t band_left;  /* cells with -band_left <= i - j are computed; < 0 = unbounded   */
  int32_t band_right; /* cells with i - j <= band_right are computed; < 0 = unbounded   */
  int32_t zdrop;      /* Z >= 0; < 0 disables the Z-drop test                           */
  int32_t variant;    /* 0: the readings of DESIGN.md §2 (default).  Bits select the
                         minimap2-like alternatives (outside the reference; DESIGN.md §2,
                         SURVEY.md §8(f) NEXT #4):                                       */
} agatha_params_t;

#define AGATHA_VAR_GATE_GE 1     /* Eq. 4 gating i' <= i and j' <= j instead of strict <       */
#define AGATHA_VAR_ORIGIN_MAX 2  /* the global max starts at H(0,0) = 0 at (0,0): a pair whose
                                    cells all score below 0 reports (0, 0, 0)                */
#define AGATHA_VAR_CHECK_LAST 4  /* Eq. 4 is also tested at the last anti-diagonal c = m+n  */

/* A batch of n_pairs independent pairs.  Pair k is R = ref[ref_off[k] .. ref_off[k+1])
 * and Q = qry[qry_off[k] .. qry_off[k+1]), ASCII A/C/G/T/N (either case).  The offset
 * arrays hold n_pairs + 1 entries and are non-decreasing. */
typedef struct {
  const uint8_t* ref;
  const uint8_t* qry;
  const uint64_t* ref_off;
  const uint64_t* qry_off;
  uint64_t n_pairs;
  uint32_t flags; /* AGATHA_MEM_* | AGATHA_OUT_DEVICE | AGATHA_N_* | AGATHA_ORDER_INPUT */
  int32_t* queue; /* NULL: the context's own pair counter.  Otherwise a shared counter
                     from agatha_queue_create/_open (cross-GPU dynamic balancing, SURVEY.md
                     §8(f) NEXT #1): every participant aligns the SAME batch with the same
                     params; its persistent kernels claim pairs (in the common tier-major,
                     longest-first order; one counter per slot tier at queue[0..2]) with
                     system-scope atomics, align only those,
                     and writes only their result rows; all other rows of `out` are
                     zero-filled.  The caller resets the counter (agatha_queue_reset)
                     before the participants start and merges their outputs (each row is
                     non-zero in exactly one, e.g. an all-reduce sum).
                     Constraint: all participants must pass the same batch, params and
                     AGATHA_ORDER_INPUT / _SINGLE_TIER / _FORCE_32BIT bits; under a queue
                     the order ignores input chunking, so host and device inputs (and
                     any AGATHA_CHUNK_BYTES) agree.  The first participant stores a
                     fingerprint of these (pair count, every pair's lengths, params,
                     flags; not the bases) in the queue; a participant whose fingerprint
                     differs returns AGATHA_EINVAL before claiming any pair.          */
  struct agatha_ends* ends; /* NULL, or n_pairs end-score records (NEXT #4, below) on the
                     same side as `out` (AGATHA_OUT_DEVICE), written in pair order  */
} agatha_batch_t;

/* NEXT #4 (minimap2's mqe / mte / end score, outside the paper; DESIGN.md
 * reading R19): over the cells the sweep processed (anti-diagonals 2 .. c_end, c_end the
 * Z-drop anti-diagonal or m + n), in anti-diagonal order with a strict '>':
 *   mqe = max H(i, n) (the query end reached) and its i (smallest on ties);
 *   mte = max H(m, j) (the reference end reached) and its j;
 *   end_score = H(m, n) when that cell was processed.
 * An absent value is AGATHA_NO_SCORE with position -1.  24 bytes. */
#define AGATHA_NO_SCORE (-(1 << 30))
typedef struct agatha_ends {
  int32_t mqe, mqe_i;
  int32_t mte, mte_j;
  int32_t end_score;
  int32_t reserved;
} agatha_ends_t;

/* Per-pair result: 24 bytes, written in pair order. */
typedef struct {
  int32_t score;          /* H(i',j'): the global max over computed cells (Eq. 6)       */
  int32_t ref_end;        /* i' (1-based; ties: earliest anti-diagonal, then smallest i) */
  int32_t query_end;      /* j' (1-based)                                               */
  int32_t zdrop_antidiag; /* c = i + j at which Eq. 4 fired; -1 if it never fired       */
  int64_t cells;          /* in-band in-table cells on anti-diagonals 2 .. c_end        */
} agatha_result_t;

typedef struct agatha_ctx agatha_ctx_t;

/* Timings and counters of the last agatha_align_batch on this context. */
typedef struct {
  float h2d_ms;        /* host->device copy of inputs (0 for device inputs)             */
  float prep_ms;       /* validation + nominal work (a2) + packing (a1) + LPT sort (a2) */
  float align_ms;      /* the wavefront align kernel (a3-a8)                             */
  float d2h_ms;        /* device->host copy of results (0 for device outputs)          */
  int32_t slots_per_lane; /* K: band diagonals held per lane                             */
  int32_t grid_blocks; /* persistent grid of the align kernel                            */
  int32_t kernel_launches; /* kernels of this library launched by the call              */
  int32_t library_launches; /* CUB radix-sort kernels launched by the call             */
  int32_t packed16;    /* 1 if the 16-bit packed (DPX .S16x2) kernel ran, 0 for 32-bit    */
  int32_t warps_per_pair; /* 1; 2 or 4 in the wide-band tier (D > 1024, 32-bit)          */
  int32_t tier_pairs[3]; /* 16-bit kernel: pairs run at 32 / 16 / 8 slots per lane (the
                            slot tiers for D > 512 / 257..512 / <= 256 diagonals)         */
  int32_t input_chunks;  /* host inputs: chunks streamed under the kernel (1 for device)  */
  int32_t lpt_from_chunk; /* chunks from this one on are dispatched as one longest-first
                             group (they arrive before the queue reaches them)           */
  int32_t pin_off;     /* 32-slot front: the common low padding off = (-D) mod 16 of its
                          pairs when the pinned front ran (one capped slot), else -1     */
  int32_t rebase_iters; /* 16-bit kernels: iterations between re-centrings of the 32-slot
                          front (128, 64 or 32, the longest the 16-bit guard admits), 0
                          when the 16-bit kernels do not apply                           */
  int32_t pin_off8;    /* 16-slot front: the common low padding off = (-D) mod 8 of its pairs
                          when its pinned instantiation ran, else -1                     */
} agatha_stats_t;

/* Create a context on CUDA device `cuda_device`.  Fails with AGATHA_ECUDA when the
 * device is not an sm_100 part.  Host inputs stream to the device in chunks of ~48 MB of
 * ASCII; the environment variable AGATHA_CHUNK_BYTES (>= 256), read here, overrides the
 * chunk size (tests use it to exercise many chunks on small batches). */
int agatha_ctx_create(agatha_ctx_t** ctx, int cuda_device);
void agatha_ctx_destroy(agatha_ctx_t* ctx);

/* Align every pair of `batch` with `params`; write n_pairs results to `out` (host or
 * device memory per AGATHA_OUT_DEVICE).  Steps a1-a8 of DESIGN.md all run on the GPU. */
int agatha_align_batch(agatha_ctx_t* ctx, const agatha_batch_t* batch,
                       const agatha_params_t* params, agatha_result_t* out, void* cuda_stream);

/* Pack `len` ASCII bases (device memory) into 4-bit codes A0 C1 G2 T3 N4, 8 per uint32
 * word, earliest base in the low nibble (§2.2 l.279-285),
 * unused trailing nibbles zero.  `words` (device) receives ceil(len/8) words.  flags:
 * AGATHA_PACK_REVERSE packs back to front; AGATHA_N_MAP maps invalid bytes to N,
 * otherwise they yield AGATHA_ECHAR. */
int agatha_pack4(agatha_ctx_t* ctx, const uint8_t* ascii, uint64_t len, uint32_t* words,
                 uint32_t flags, void* cuda_stream);

/* The dispatch plan of step a2 for `batch` (device inputs and outputs): nominal[k] =
 * in-band in-table cell count of pair k (un-terminated), order = pair ids sorted by
 * descending nominal (ties in any order). */
int agatha_plan(agatha_ctx_t* ctx, const agatha_batch_t* batch, const agatha_params_t* params,
                uint32_t* order, uint32_t* nominal, void* cuda_stream);

/* Debug: per-anti-diagonal local maxima (Eq. 5) of pair `pair` of the last batch run on
 * this context, as computed by the kernel: for c in [0, cap) score[c] = H*, ref_i[c] =
 * i* (or -1 when the anti-diagonal is empty or was never reached).  Host outputs.
 * Requires the pair to be re-run: the call re-aligns `batch` with tracing on. */
int agatha_localmax_trace(agatha_ctx_t* ctx, const agatha_batch_t* batch,
                          const agatha_params_t* params, uint64_t pair, int32_t* score,
                          int32_t* ref_i, int64_t cap, void* cuda_stream);

/* NEXT #1: a shared pair counter for agatha_batch_t.queue.  _create allocates zeroed
 * device counters (int32 [0..2], one per slot tier, and the batch fingerprint at [8];
 * 256 bytes) on the context's device and returns
 * their CUDA IPC handle (64 bytes) for other processes; _open maps a handle from another
 * process (peer access over NVLink when on another GPU) into this context; _reset zeroes
 * the counters and the fingerprint on `cuda_stream` (before each batch);
 * _close releases a created (opened = 0) or opened (opened = 1) counter. */
int agatha_queue_create(agatha_ctx_t* ctx, int32_t** queue, uint8_t handle[64]);
int agatha_queue_open(agatha_ctx_t* ctx, const uint8_t handle[64], int32_t** queue);
int agatha_queue_reset(agatha_ctx_t* ctx, int32_t* queue, void* cuda_stream);
int agatha_queue_close(agatha_ctx_t* ctx, int32_t* queue, int opened);

/* NEXT #1: a FEDERATED batch for cross-GPU dynamic
 * balancing without replicated inputs.  The global batch is the concatenation, in owner
 * order, of n_owners (1..8) device batches: owners[o] holds owner o's ASCII sequences and
 * offsets (flags must include AGATHA_MEM_DEVICE; pointers may be peer-mapped memory of
 * another GPU or process, from agatha_ipc_open, read over NVLink).  Global pair g of
 * owner o is its local pair g - (pairs of owners 0..o-1).  Every participant passes the
 * same owners (its own mapping of them), params and `flags` (AGATHA_ORDER_INPUT,
 * _SINGLE_TIER, _FORCE_32BIT, _N_MAP), and the same `queue` (agatha_queue_*): the
 * persistent kernels claim global pairs from the one order, read a claimed pair's
 * inputs from its owner, and write its 24-byte record to row g of `out` (a DEVICE
 * buffer of 24 * total pairs, owned by the caller); rows the participant did not claim
 * are zero (merge as for agatha_batch_t.queue).  queue = NULL: this context aligns the
 * whole global batch.  The result of every pair equals agatha_align_batch's on the
 * concatenated batch.  Errors as agatha_align_batch; EINVAL also for a host-memory
 * owner or n_owners outside 1..8, ERANGE for 2^31 or more pairs in total. */
int agatha_align_federated(agatha_ctx_t* ctx, const agatha_batch_t* owners, int n_owners,
                           const agatha_params_t* params, agatha_result_t* out, int32_t* queue,
                           uint32_t flags, void* cuda_stream);

/* Device buffers shareable across processes (CUDA IPC): _alloc returns `bytes` of device
 * memory on the context's device and its 64-byte IPC handle; _open maps another
 * process's handle into this context (peer access over NVLink when on another GPU);
 * _close frees an allocated (opened = 0) or unmaps an opened (opened = 1) buffer. */
int agatha_ipc_alloc(agatha_ctx_t* ctx, uint64_t bytes, void** ptr, uint8_t handle[64]);
int agatha_ipc_open(agatha_ctx_t* ctx, const uint8_t handle[64], void** ptr);
int agatha_ipc_close(agatha_ctx_t* ctx, void* ptr, int opened);

int agatha_get_stats(const agatha_ctx_t* ctx, agatha_stats_t* stats);
const char* agatha_strerror(int code);
int agatha_version(void);

#ifdef __cplusplus
}
#endif
#endif /* AGATHA_H_ */
