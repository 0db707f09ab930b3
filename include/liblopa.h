/*
 * liblopa — the LoPA branch-construction and verification step (arXiv 2512.16229) as a
 * C-ABI library for NVIDIA B200 (sm_100a).
 *
 * Citation keys: P:n = line n of the paper's text; S:n = line n of SPEC.md.
 * "R<n>" = reading n in DESIGN.md §2 (where the paper is silent or ambiguous).
 *
 * What the library computes (one LoPA iteration, Alg. 1, after the forward):
 *   a1  Conf(i) = top-1 softmax probability of position i's logits, and the greedy token
 *       ("a confidence function Conf(.) assigns a score to each position i in M_t";
 *       R1 top-1 probability, R2 temperature 1, R3 greedy, R4 lowest token id on ties).
 *   a2  Eq. 2 branch confidence C(B_j) = mean of Conf over M_{B_j} (1.0 if
 *       empty, R8) and B* = argmax_j C(B_j) (ties -> lowest j, anchor first, R9).
 *   a3  Eq. 1 anchor fill on the winner's reused logits:
 *       S_high = {i in M : Conf(i) > tau}; I_fill = S_high, else {argmax_i Conf(i)}.
 *   a4  Alg. 1 step 2: top-k of M_{B0} by (conf desc, position asc) (R6),
 *       n_br = min(k, |M_{B0}|) + 1 (R7); B_j = B0 with p_j filled by its greedy token.
 *   a5  Branch parallelism: branches sharded over ranks, one NCCL all-gather of
 *       each rank's local best (score, id, row) per step (or, opt-in, the same exchange over
 *       CUDA-IPC peer memory: lopa_bp_step_p2p).
 * Beyond the step: windows of up to 256 positions with per-position Eq. 1
 * thresholds (the D2F multi-block window, NEXT-1), Eq. 2 variants (NEXT-2), the winner's
 * payload exchange (Commit-Winner-Cache, NEXT-3) and the LM-head projection on tcgen05 with
 * Conf fused into its epilogue (NEXT-4).
 *
 * Conventions (all calls):
 *   - Pointers named *_dev / documented "device" are device pointers into caller-owned
 *     memory.  The library allocates no device memory per call.
 *   - Every compute call is asynchronous, stream-ordered on `stream` (a cudaStream_t passed
 *     as void*; NULL = the legacy default stream) and returns a HOST status (lopa_status_t)
 *     describing argument validation and launch errors only.
 *   - Data-dependent errors are OR-ed into a caller-zeroed device word `dev_status`
 *     (LOPA_DEV_*); the host sees them after it synchronises.
 *   - Logits are bf16, row-major [n_rows][ld] with ld >= vocab, ld % 8 == 0 and a
 *     16-byte-aligned base (TMA bulk copies move 16-byte units).  Entries in [vocab, ld)
 *     are never interpreted.
 *   - Masks are uint8, 1 = masked (position still to be decoded); torch.bool is
 *     layout-compatible.  Tokens are int32 (V = 151936 > 2^16).
 *   - Branch tables are [max_branches][window] row-major; branch 0 is the anchor B0.
 *   - tau is fp32; a position is "high" iff (float)conf > tau (strict; R5, R14).
 *   - Workspace: lopa_workspace_bytes() bytes of device memory, zeroed by the caller ONCE
 *     before first use; the library keeps its state there (every successful call leaves the
 *     work counters zero again and advances the partial epoch that tells the reduction's
 *     partials of this call from stale ones), so it may be shared by every kind
 *     of call and by CUDA-graph replays.  A workspace must not be used by two calls that may
 *     run concurrently.  After a LOPA_ERR_CUDA return, zero it again.
 */
#ifndef LIBLOPA_H_
#define LIBLOPA_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#if defined(__GNUC__)
#pragma GCC visibility push(default)
#endif

#define LOPA_VERSION 10000 /* 1.0.0 */

typedef enum {
  LOPA_OK = 0,
  LOPA_ERR_INVALID_ARG = 1, /* null pointer, vocab < 1, window < 1, k < 0, tau not in (0,1],
                               ld < vocab, ld % 8 != 0, logits not 16-byte aligned, ...   */
  LOPA_ERR_UNSUPPORTED = 2, /* window > LOPA_MAX_WINDOW, branches > LOPA_MAX_BRANCHES,
                               rows > LOPA_MAX_ROWS, vocab > LOPA_MAX_VOCAB, device is not
                               sm_100                                                      */
  LOPA_ERR_CUDA = 3,        /* a CUDA runtime error (launch / capture)                     */
  LOPA_ERR_NCCL = 4         /* an NCCL error in the branch-parallel exchange               */
} lopa_status_t;

/* Device status bits (OR-ed into *dev_status). */
#define LOPA_DEV_EMPTY_MASK 1 /* Eq. 1 applied with nothing masked           */
#define LOPA_DEV_NONFINITE 2  /* a reduced row holds NaN or +inf, or is all -inf (R20);
                                 that row's conf / argmax are unspecified                   */
#define LOPA_DEV_PEER_TIMEOUT 4 /* lopa_bp_step_p2p: a peer's record did not arrive (bounded
                                   wait); that step decides nothing: n_branches_next = 0,
                                   the next tables are left untouched.  Check dev_status
                                   after every peer-memory step.                            */

#define LOPA_DEV_INTERNAL 8   /* internal protocol error: a partial of the reduction never
                                 arrived within the fold's bounded poll (a fault upstream)  */

#define LOPA_MAX_WINDOW 256   /* W <= 256 (the D2F multi-block window); W > 64 needs V <= 2^22 */
#define LOPA_MAX_BRANCHES 32  /* k + 1 <= 32: one lane per branch in the select             */
#define LOPA_MAX_ROWS 4096    /* rows per call: n_rows, or max_branches * window            */
#define LOPA_MAX_VOCAB (1 << 23) /* conf >= 1/V >= 2^-23 keeps the fp64 Eq. 2 sums exact       */

int lopa_version(void);
const char* lopa_status_string(int status);
/* The CUDA runtime's message for the last call of this thread that returned LOPA_ERR_CUDA
 * ("" if none).  The string is owned by the library and valid until the next such call. */
const char* lopa_last_cuda_error(void);
/* Whether the reduction kernel may copy its first logits rows before waiting for the previous
 * kernel on the stream (see the stream-order contract at lopa_step_args_t): 1 (the default) or
 * 0, for callers whose logits producer lets its dependents launch before its last logits store.
 * Process-wide, read at every launch; returns the previous setting. */
int lopa_set_logits_prefetch(int32_t enabled);
/* Debug: {registers/thread, max threads/block, static shared bytes, local bytes/thread, block
 * size launched} of the vocabulary-reduction kernel K1 this build uses. */
int lopa_debug_k1_attrs(int32_t* out5);
/* Debug, checked builds (-DLOPA_CHECKED, the library's own bounds / protocol checks): writes
 * {violations, first violating site, bitmask of violating sites} counted since the last call and
 * resets them.  Returns LOPA_ERR_UNSUPPORTED (zeros written) in product builds. */
int lopa_debug_check_read(uint32_t* out3);

/* Bytes of device workspace needed for up to max_rows rows of `vocab` logits. */
size_t lopa_workspace_bytes(int32_t max_rows, int32_t vocab);

/* Number of canonical segments a row of `vocab` logits is split into (the
 * fp32 reduction order is fixed per vocab, so conf bits depend only on the row's bytes). */
int32_t lopa_num_segments(int32_t vocab);

/* a1 — Conf(.) and greedy token of every selected row (R1-R4, R20).
 *   logits   device bf16 [n_rows][ld]
 *   row_mask device uint8 [n_rows] or NULL (NULL = reduce every row).  Rows with
 *            row_mask[r] == 0 are not read and conf[r] / argmax[r] are left untouched.
 *   conf     device float [n_rows]: 1 / sum_v exp(l_v - max_v l_v)
 *   argmax   device int32 [n_rows]: the lowest v with l_v = max
 *   dev_status device int32 (LOPA_DEV_NONFINITE)
 *   workspace  device, lopa_workspace_bytes(n_rows, vocab) bytes (see conventions)
 * n_rows = 0 is a no-op.  Errors: INVALID_ARG, UNSUPPORTED (n_rows > LOPA_MAX_ROWS), CUDA. */
int lopa_confidence(const void* logits, int64_t ld, int32_t n_rows, int32_t vocab,
                    const uint8_t* row_mask, float* conf, int32_t* argmax, int32_t* dev_status,
                    void* workspace, size_t workspace_bytes, void* stream);

/* a3 — Eq. 1 + Alg. 1 step 1.
 *   conf, argmax  device [window] (read only where mask[i] == 1)
 *   tokens, mask  device [window]: the state x_t, M_t
 *   tokens_out, mask_out device [window]: B0 (x_{B0}, M_{B0}); may alias tokens / mask.
 * If nothing is masked: LOPA_DEV_EMPTY_MASK is set and the state is copied unchanged. */
int lopa_anchor_fill(const float* conf, const int32_t* argmax, const int32_t* tokens,
                     const uint8_t* mask, int32_t window, float tau, int32_t* tokens_out,
                     uint8_t* mask_out, int32_t* dev_status, void* stream);

/* a3 with per-position thresholds (the D2F multi-block window; R25):
 * tau_pos device float [window] or NULL (NULL = tau everywhere). */
int lopa_anchor_fill_ex(const float* conf, const int32_t* argmax, const int32_t* tokens,
                        const uint8_t* mask, int32_t window, float tau, const float* tau_pos,
                        int32_t* tokens_out, uint8_t* mask_out, int32_t* dev_status,
                        void* stream);

/* a4 — Alg. 1 step 2.
 *   conf, argmax        device [window] (the anchor's confidences, read where mask_b0 == 1)
 *   tokens_b0, mask_b0  device [window]
 *   branch_tokens       device int32 [k+1][window]  (row 0 = B0, row j = B_j)
 *   branch_mask         device uint8 [k+1][window]
 *   lookahead_pos       device int32 [k] (p_1..p_n, -1 padded); may be NULL when k == 0
 *   n_branches          device int32 scalar: n = min(k, |M_B0|) + 1
 * Rows j > n - 1 of the branch tables are left untouched.  k = 0 is valid (n = 1). */
int lopa_spawn_branches(const float* conf, const int32_t* argmax, const int32_t* tokens_b0,
                        const uint8_t* mask_b0, int32_t window, int32_t k,
                        int32_t* branch_tokens, uint8_t* branch_mask, int32_t* lookahead_pos,
                        int32_t* n_branches, void* stream);

/* a2 — Eq. 2 + select.
 *   conf         device float [max_branches][window] (each branch's own verify conf)
 *   branch_mask  device uint8 [max_branches][window]
 *   n_branches   device int32 scalar (branches j >= *n_branches are absent)
 *   scores       device float [max_branches]: C(B_j) (fp64 sum in position order, rounded
 *                once to fp32); absent branches get -inf
 *   winner       device int32 scalar: smallest j with the largest fp32 score (R9) */
int lopa_verify_select(const float* conf, const uint8_t* branch_mask, const int32_t* n_branches,
                       int32_t max_branches, int32_t window, float* scores, int32_t* winner,
                       void* stream);

/* Branch-confidence metrics.  The Eq. 2 mean is the paper's default; the
 * two variants are the ones P:204 names.  All are computed from exact fp64 sums. */
#define LOPA_METRIC_MEAN 0            /* C(B_j) = mean of Conf over M_Bj (Eq. 2)                 */
#define LOPA_METRIC_SLIDING_MIN 1     /* min over length-w windows of M_Bj (position order) of the
                                         window mean; w clamped to |M_Bj| ("local quality")     */
#define LOPA_METRIC_BOTTOM_FRACTION 2 /* mean of the ceil(eta |M_Bj|) lowest confidences
                                         ("least confident segment")                            */

/* a2 with a metric: as lopa_verify_select, scores by `metric` / `metric_param`. */
int lopa_verify_select_ex(const float* conf, const uint8_t* branch_mask, const int32_t* n_branches,
                          int32_t max_branches, int32_t window, int32_t metric, float metric_param,
                          float* scores, int32_t* winner, void* stream);

/* One verify step (a1 -> a2 -> a3 -> a4): the streaming reduction kernel and the fold/decision
 * kernel, launched back to back (programmatic dependent launch) on `stream`.
 * Stream-order contract for `logits` (all calls that read logits): the reduction kernel starts
 * copying its first logits rows as soon as the previous kernel on the stream lets dependents
 * launch (griddepcontrol.launch_dependents; a kernel that never executes it does so at its end),
 * before waiting for that kernel's memory.  A kernel that writes the logits must therefore not
 * trigger its dependents before its last logits store (ordinary kernels, copies and liblopa's own
 * kernels satisfy this), or the caller turns the early copy off: lopa_set_logits_prefetch(0). */
typedef struct {
  /* inputs */
  const void* logits;            /* device bf16 [max_branches][window][ld]: verify logits     */
  int64_t ld;                    /* row stride in elements                                    */
  int32_t vocab;
  int32_t window;                /* W <= LOPA_MAX_WINDOW                                      */
  int32_t max_branches;          /* table capacity (k + 1 for a steady-state loop)           */
  const int32_t* n_branches;     /* device scalar: branches present in the tables / logits;
                                    0 (a complete block fed back, R21): row 0 passes through,
                                    n_branches_next = 0                                         */
  const int32_t* branch_tokens;  /* device int32 [max_branches][window]                      */
  const uint8_t* branch_mask;    /* device uint8 [max_branches][window]                      */
  int32_t k;                     /* lookahead budget for the next spawn, k + 1 <= LOPA_MAX_BRANCHES */
  float tau;                     /* Eq. 1 threshold, (0, 1]                                  */
  /* outputs (device) */
  float* conf;                   /* [max_branches][window]; written where masked             */
  int32_t* argmax;               /* [max_branches][window]; written where masked             */
  float* scores;                 /* [max_branches]                                          */
  int32_t* winner;               /* scalar j*                                                */
  int32_t* next_tokens;          /* [k+1][window]: B0..Bn of the next iteration              */
  uint8_t* next_mask;            /* [k+1][window]                                            */
  int32_t* lookahead_pos;        /* [k] (may be NULL if k == 0)                              */
  int32_t* n_branches_next;      /* scalar; 0 = the winner has no masked position (block
                                    complete, R21): next_tokens[0] / next_mask[0] = winner   */
  int32_t* dev_status;           /* scalar, LOPA_DEV_* bits                                  */
  void* workspace;
  size_t workspace_bytes;        /* >= lopa_workspace_bytes(max_branches * window, vocab)   */
  int32_t metric;                /* branch confidence: LOPA_METRIC_* (0 = Eq. 2 mean)        */
  float metric_param;            /* window w >= 1 (integer) or eta in (0, 1]; unused for mean */
  const float* tau_pos;          /* device float [window] per-position Eq. 1 thresholds, or
                                    NULL (= tau): the D2F window's tau_act / tau_conf         */
  const int32_t* window_dev;     /* NULL, or a device int32 scalar W_d in [1, window]: the step
                                    then runs on a window of W_d positions read on the device
                                    (the device-resident D2F loop, lopa_d2f_*): logits, tables,
                                    conf / argmax and next tables are laid out [.][W_d] inside
                                    their `window`-sized capacity; tau_pos [W_d]; `window` is
                                    the capacity (and sizes the workspace).  Only lopa_step.  */
} lopa_step_args_t;

/* Next tables must not alias the input tables.  Errors: INVALID_ARG, UNSUPPORTED, CUDA. */
int lopa_step(const lopa_step_args_t* args, void* stream);

/* ---------------------------------------------------------------- NEXT-1 on the device
 * The D2F block pipeline (readings R25 / R26) as device state plus a scheduler
 * kernel, so that a whole multi-block decode -- the forward, lopa_step on the active window
 * (args.window_dev = &sched[1], args.n_branches = &sched[2], args.tau_pos = tau_pos, tables =
 * branch_tokens / branch_mask), lopa_d2f_update -- runs with no host read and can be captured
 * in one CUDA graph.  Iterations after the last block is committed are no-ops (sched[3] = 1,
 * n_branches = 0: the step passes through, the scheduler and the harness forward return). */
typedef struct {
  int32_t gen_len;          /* generation length, a multiple of block_size                  */
  int32_t block_size;       /* B >= 1                                                        */
  int32_t k;                /* lookahead budget, k + 1 <= LOPA_MAX_BRANCHES                  */
  int32_t max_window;       /* in [block_size, LOPA_MAX_WINDOW]: active blocks * B stays <=  */
  double tau_add;           /* activate the next block when the newest active block's fill
                               ratio >= tau_add (compared exactly in double, R26 (b))        */
  float tau_act, tau_conf;  /* Eq. 1 thresholds of the newest / older active blocks (R25)   */
  int32_t trace_cap;        /* entries of `trace` (0 if trace is NULL)                       */
  /* caller-owned device buffers */
  int32_t* region_tokens;   /* [gen_len]: initial tokens in (masked positions), final out   */
  uint8_t* region_mask;     /* [gen_len]: 1 = still masked (set to 1 by lopa_d2f_init)       */
  int32_t* block_status;    /* [gen_len / B]: 0 inactive, 1 active, 2 committed              */
  int32_t* sched;           /* [8]: window start p0, window W, branches of the next step n,
                               done, forwards, committed blocks, -, -                         */
  float* tau_pos;           /* [max_window]: the window's per-position thresholds            */
  int32_t* branch_tokens;   /* [k + 1][max_window] capacity; the step's tables, [n][W]       */
  uint8_t* branch_mask;     /* [k + 1][max_window] capacity                                  */
  int32_t* commit_order;    /* [gen_len / B]: blocks in commit order (-1 = not yet)          */
  int32_t* trace;           /* [trace_cap][4] (p0, W, n, winner) per forward, or NULL        */
} lopa_d2f_t;

/* Region fully masked, block 0 active, first window = block 0 with one branch (the initial
 * predict).  Errors: INVALID_ARG (sizes, NULL buffers), CUDA. */
int lopa_d2f_init(const lopa_d2f_t* d, void* stream);
/* After a lopa_step on the window: B* -> region, rules (a) / (b), the next window's thresholds
 * and tables (spawned branches carried over; n_next = 0 -> the new window's initial predict).
 * winner / n_next / next_tokens / next_mask: that step's outputs ([k+1][W] layout). */
int lopa_d2f_update(const lopa_d2f_t* d, const int32_t* winner, const int32_t* n_next,
                    const int32_t* next_tokens, const uint8_t* next_mask, void* stream);
/* Harness (not the method): SYN-D2F logits [n][W][ld] of the device window, block b's positions
 * from block b's columns of each branch (DESIGN.md §3 "D2F loops"). */
int lopa_d2f_syn_forward(uint64_t seed, int32_t vocab, int64_t ld, int32_t extras,
                         const lopa_d2f_t* d, void* logits, void* stream);

/* ---------------------------------------------------------------- device-terminated loops
 * A CUDA graph whose body repeats on the device under a conditional WHILE node until a
 * condition word stops it: the Alg. 1 loop until the selected branch is complete (R21: the
 * step's n_branches_next = 0) or a D2F decode until every block is committed (sched[3] != 0),
 * with no host read and no fixed iteration count.
 *   lopa_while_begin: starts capturing `stream` into the loop body; the caller then issues the
 *     body (e.g. forward + lopa_step + table copies) on that stream; cond_word: device int32,
 *     read after each iteration: continue while it is non-zero (until_zero = 1) or zero
 *     (until_zero = 0), and at most max_iters iterations per launch.
 *   lopa_while_end: appends the condition kernel, ends the capture, instantiates the graph.
 *   lopa_while_launch: runs the whole loop (>= 1 iteration) on `stream` (NULL: the legacy
 *     default stream, as every other call); asynchronous.  lopa_while_iterations: iterations of the last launch (synchronous).
 * The body must not allocate or synchronise.  Errors: INVALID_ARG (order of calls), CUDA. */
typedef struct lopa_while lopa_while_t;
int lopa_while_begin(void* stream, const int32_t* cond_word, int32_t until_zero, int32_t max_iters,
                     lopa_while_t** out);
int lopa_while_end(lopa_while_t* w);
int lopa_while_launch(lopa_while_t* w, void* stream);
int lopa_while_iterations(const lopa_while_t* w, int32_t* out_host);
void lopa_while_destroy(lopa_while_t* w);

/* Harness: lopa_syn_generate for the branches present, the count read on the device: branch
 * tables (and out) hold the shard of global branches [branch_base, branch_base + max_branches);
 * rows of global branches >= *n_branches_dev are skipped.  The forward stand-in inside a
 * device-terminated loop (branch_base = 0 on one GPU, the rank's first branch under BP). */
int lopa_syn_generate_dev(uint64_t seed, int32_t block, int32_t vocab, int64_t ld, int32_t window,
                          int32_t max_branches, const int32_t* n_branches_dev, int32_t branch_base,
                          const int32_t* branch_tokens, const uint8_t* branch_mask, int32_t extras,
                          void* out, void* stream);

/* ---------------------------------------------------------------- branch parallelism (a5)
 * Global branch j lives on rank j / B_loc, B_loc = ceil(max_branches / world).
 * Each rank reduces only its branches' logits, scores them, and publishes one record
 * {its B_loc scores, its best (score, id), that branch's tokens/mask/conf/argmax row}.
 * One all-gather of the records replaces the (score, id) all-gather + winner-row broadcast
 * (the broadcast root is device data).  Every rank then runs the same
 * deterministic select, anchor and spawn, so the next branch tables are replicated.        */

/* Bytes of one rank's exchange record for `window` and `b_loc` local branches. */
size_t lopa_bp_record_bytes(int32_t window, int32_t b_loc);

/* Local half of a BP step on one rank: a1 + local Eq. 2 + local best -> record.
 *   args: as lopa_step, except `logits` holds ONLY this rank's branches
 *         [b_loc][window][ld], conf / argmax are [b_loc][window], and the next_* / winner /
 *         scores / lookahead / n_branches_next outputs are ignored (may be NULL).
 *   branch_base: global id of the first local branch (rank * b_loc); b_loc: local capacity.
 *   record: device, lopa_bp_record_bytes(window, b_loc) bytes. */
int lopa_bp_local(const lopa_step_args_t* args, int32_t branch_base, int32_t b_loc,
                  void* record, void* stream);

/* Global half: select over `world` records (contiguous, rank order), then anchor + spawn.
 * Writes args->scores [world * b_loc >= max_branches] (absent = -inf), winner,
 * next_tokens / next_mask / lookahead_pos / n_branches_next, dev_status. */
int lopa_bp_finish(const lopa_step_args_t* args, int32_t b_loc, int32_t world,
                   const void* records, void* stream);

typedef struct lopa_bp lopa_bp_t;
#define LOPA_BP_UNIQUE_ID_BYTES 128

/* Rank 0 creates the NCCL unique id; the caller ships it to the other ranks (torch PG). */
int lopa_bp_get_unique_id(void* unique_id_out /* LOPA_BP_UNIQUE_ID_BYTES */);
/* Collective over `world` ranks; device = the CUDA device of this rank. */
int lopa_bp_create(const void* unique_id, int32_t rank, int32_t world, int32_t device,
                   lopa_bp_t** out);
/* Full BP step: lopa_bp_local -> ncclAllGather(records) -> lopa_bp_finish, on `stream`.
 * records: device, world * lopa_bp_record_bytes(window, b_loc) bytes (this rank's slot is
 * records + rank * record_bytes). */
int lopa_bp_step(lopa_bp_t* bp, const lopa_step_args_t* args, int32_t b_loc, void* records,
                 void* stream);
/* Pending asynchronous NCCL error (ncclCommGetAsyncError), as LOPA_OK / LOPA_ERR_NCCL. */
int lopa_bp_check(lopa_bp_t* bp);
void lopa_bp_destroy(lopa_bp_t* bp);

/* Measurement: record a CUDA event pair around every K1 (vocabulary-reduction kernel) launch of
 * the next max_records lopa_step / lopa_confidence / lopa_bp_local calls (events recorded on the
 * call's stream).  lopa_profile_read synchronises, writes up to max durations in ms and the
 * count, and disables recording.  Errors: INVALID_ARG, CUDA. */
int lopa_profile_enable(int32_t max_records);
int lopa_profile_read(float* k1_ms, int32_t max, int32_t* n_out);

/* Measurement: K1 (the vocabulary-reduction kernel) alone, as launched inside lopa_step (one
 * CTA per SM but one), over the rows of a lopa_confidence call: it leaves only the per-group
 * partials in the workspace (no conf / argmax).  Lets bench.py time K1's average launch
 * duration with CUDA events around back-to-back launches.  Arguments and errors as
 * lopa_confidence. */
int lopa_debug_reduce_only(const void* logits_bf16, int64_t ld, int32_t n_rows, int32_t vocab,
                           const uint8_t* row_mask, int32_t* dev_status, void* workspace,
                           size_t workspace_bytes, void* stream);

/* Debug: per-CTA phase timeline (%globaltimer ns) of the last reduction launch, for builds
 * compiled with -DLOPA_TIMELINE; returns the slots per CTA written to out[n_ctas][slots], or 0.
 * Slots: 0 CTA start, 1 producer start, 2 first stage consumed, 3 last unit consumed,
 * 4 tail start, 5 tail end. */
int lopa_debug_timeline(unsigned long long* out, int n_ctas);
/* Debug: per-warp timeline of the warp-staged K1's last launch (experiment builds with
 * -DLOPA_LDG_TL only).  Returns the words written, minus the words needed if n_words is too
 * small, 0 if the build has no timeline. */
int lopa_debug_ldg_timeline(unsigned long long* out, int n_words);
/* Debug: per-item timeline of the TMA-form K1's last launch (-DLOPA_K1_TL builds only); same
 * return convention. */
int lopa_debug_k1_timeline(unsigned long long* out, int n_words);
/* Debug: per-step marks of chained steps (-DLOPA_CHAIN_TL builds only), [64][12] ns; cleared. */
int lopa_debug_chain_timeline(unsigned long long* out, int n_words);

/* ---------------------------------------------------------------- harness (not the method)
 * SYN-D2F synthetic logits for a batch of branch states (the stand-in for the dLLM forward;
 * DESIGN.md §3).  Holds none of LoPA's arithmetic.
 *   branch_tokens / branch_mask device [n_branches][window]; out device bf16 [n_branches]
 *   [window][ld]; entries in [vocab, ld) are written as 0.  extras: 0 or 1 (toy tie / flat
 *   rows). */
int lopa_syn_generate(uint64_t seed, int32_t block, int32_t vocab, int64_t ld, int32_t window,
                      int32_t n_branches, const int32_t* branch_tokens,
                      const uint8_t* branch_mask, int32_t extras, void* out, void* stream);

/* Branch parallelism over peer memory (the exchange of lopa_bp_step without NCCL): each rank
 * writes its record straight into every peer's record buffer over NVLink (CUDA IPC mapping)
 * and raises a per-rank epoch flag there (release at system scope); the finishing kernel
 * waits for every rank's flag of this step (acquire) and runs the same deterministic select /
 * anchor / spawn.  Records are double-buffered by epoch parity, so a rank may run one step
 * ahead of a slow reader.  Same results as lopa_bp_step.
 *   lopa_bp_p2p_alloc: allocates this rank's buffers for (window <= 256, b_loc) and, if
 *     payload_bytes > 0 (a multiple of 16), two parities of [b_loc][payload_bytes] payload
 *     slots; writes its IPC handle (LOPA_BP_IPC_HANDLE_BYTES) to handle_out; once per
 *     communicator.
 *   lopa_bp_p2p_open: all_handles = the world handles in rank order (gathered by the caller);
 *     maps every peer's buffers.
 *   lopa_bp_step_p2p: as lopa_bp_step (args, b_loc), on the P2P buffers: K1, then ONE kernel
 *     that computes the local record, stores it into every peer over NVLink, raises this rank's
 *     epoch flag there, waits for every rank's flag and runs the global select / anchor / spawn.
 *     The epoch lives in device memory, so the step may be captured in CUDA graphs (the
 *     Commit-Winner-Cache payload slots below stay host-driven).  A peer that never arrives
 *     within the bounded wait sets LOPA_DEV_PEER_TIMEOUT and ends the step with
 *     n_branches_next = 0 (tables untouched): callers check dev_status after every step.
 * Errors: LOPA_ERR_INVALID_ARG (order of calls, sizes), LOPA_ERR_CUDA (allocation, IPC). */
#define LOPA_BP_IPC_HANDLE_BYTES 64
int lopa_bp_p2p_alloc(lopa_bp_t* bp, int32_t window, int32_t b_loc, size_t payload_bytes,
                      void* handle_out);
int lopa_bp_p2p_open(lopa_bp_t* bp, const void* all_handles);
int lopa_bp_step_p2p(lopa_bp_t* bp, const lopa_step_args_t* args, int32_t b_loc, void* stream);

/* The branch-parallel step from hidden states (NEXT-4 with a5; P:293-298 with P:136):
 * this rank's rows -- branches [rank b_loc, (rank + 1) b_loc), i.e. b_loc * window rows of
 * `hidden` (device bf16 [b_loc * window][ld_hidden], the rank's slice of the verify forward)
 * -- through the LM head + Conf (as lopa_lmhead_confidence, into args->conf / args->argmax, the
 * rank's [b_loc][window] arrays; rows of absent branches are not reduced), then the exchange and
 * the global a2 -> a4 exactly as lopa_bp_step_p2p (peer memory opened: `records` unused, NULL)
 * or lopa_bp_step (NCCL: `records` = the [world][lopa_bp_record_bytes] device buffer).
 * args->logits is not read.  lmh_workspace: lopa_lmhead_workspace_bytes(b_loc * window) bytes.
 * Same results (bits) as lopa_step_lmhead on one GPU with the same hidden states. */
int lopa_bp_step_lmhead(lopa_bp_t* bp, const lopa_step_args_t* args, int32_t b_loc,
                        const void* hidden, int64_t ld_hidden, const void* weight, int64_t ld_weight,
                        int32_t hidden_dim, void* records, void* lmh_workspace,
                        size_t lmh_workspace_bytes, void* stream);

/* NEXT-3 over peer memory (Commit-Winner-Cache, without a collective): step e's
 * payloads (e.g. each local branch's KV features) are written by their owner into its payload
 * slots of parity e & 1 (lopa_bp_payload_slots: device pointer [b_loc][payload_bytes], NULL if
 * none) before that rank's lopa_bp_step_p2p(e); after it, lopa_bp_commit_winner_p2p copies the
 * winner's payload straight from its owner's slots into `out` (device, payload_bytes, 16-byte
 * aligned): one pass over NVLink, ordered by the step's acquire of the owner's flag.  The
 * parity double-buffering makes it safe for an owner to write step e + 1's payloads while
 * peers still pull step e's. */
void* lopa_bp_payload_slots(lopa_bp_t* bp, int32_t parity);
int lopa_bp_commit_winner_p2p(lopa_bp_t* bp, const int32_t* winner, void* out, void* stream);

/* NEXT-3 — Commit-Winner-Cache (Figure 3 phase 2): after a BP step
 * every rank holds the selected branch id in `winner` (device int32, e.g. args->winner of
 * lopa_bp_step); this makes the winner's payload (its KV features or any per-branch state of
 * payload_bytes bytes) available on every rank, without a host synchronisation.
 *   local_payloads device [b_loc][payload_bytes]: this rank's branches rank*b_loc .. +b_loc-1
 *   out            device [payload_bytes]: receives the winner's payload on every rank
 *   payload_bytes  a positive multiple of 16; both pointers 16-byte aligned
 * Mechanism: the owner contributes the payload, every other rank zeros, and one NCCL sum
 * all-reduce over 32-bit words reassembles it bit-exactly (integers: x + 0 = x).
 * Two launches on `stream` (a select kernel, then the all-reduce). */
int lopa_bp_commit_winner(lopa_bp_t* bp, const int32_t* winner, int32_t b_loc,
                          const void* local_payloads, size_t payload_bytes, void* out,
                          void* stream);

/* NEXT-4 — the LM-head projection with Conf fused into its epilogue: the logits
 * never reach HBM.  For each row r of the hidden states (the rows of the verify forward whose
 * position is masked; "parallel verification", P:207 logits reuse):
 *   logits[r][v] = sum_k hidden[r][k] * weight[v][k]     (bf16 inputs, fp32 accumulation)
 *   conf[r]      = 1 / sum_v exp(logits[r][v] - max_v logits[r][v])     (R1, R2)
 *   argmax[r]    = lowest v attaining the maximum                        (R3, R4)
 * The logits are kept in fp32 (never rounded to bf16); reading R27 in DESIGN.md gives the
 * tolerance against the exact (fp64) definition.
 *   hidden   device bf16 [rows][ld_hidden], 16-byte aligned, ld_hidden % 8 == 0
 *   weight   device bf16 [vocab][ld_weight] (nn.Linear layout: one row per token), same rules
 *   rows in [1, LOPA_MAX_ROWS]; hidden_dim a positive multiple of 64; vocab in
 *     [1, LOPA_MAX_VOCAB].  Up to 256 rows share one pass over the weights; more rows run in
 *     chunks of 256, one pass each.
 *   row_mask device uint8 [rows] or NULL: rows with row_mask[r] == 0 get conf NaN, argmax -1
 *   conf, argmax  device [rows]; a selected row whose logits contain NaN or +inf, or are all
 *            -inf, sets LOPA_DEV_NONFINITE (conf NaN, argmax -1); -inf logits are tokens of
 *            probability 0 (R20)
 *   workspace   lopa_lmhead_workspace_bytes(rows) bytes of device memory (no zeroing needed)
 * Two kernels (tcgen05 GEMM + epilogue, then a fold of the per-SM partials) on `stream`.
 * Passes of 129-256 rows run on CTA pairs and are launched programmatically dependent: they
 * request their first weight rows before the previous kernel on the stream has finished, so
 * `weight` must not be written by that kernel (it is a model parameter); `hidden` and the
 * workspace are read / written only after it. */
size_t lopa_lmhead_workspace_bytes(int32_t rows);
int lopa_lmhead_confidence(const void* hidden, int64_t ld_hidden, const void* weight,
                           int64_t ld_weight, int32_t rows, int32_t hidden_dim, int32_t vocab,
                           const uint8_t* row_mask, float* conf, int32_t* argmax,
                           int32_t* dev_status, void* workspace, size_t workspace_bytes,
                           void* stream);

/* The verify step of lopa_step (a1 -> a2 -> a3 -> a4) from the verify forward's HIDDEN STATES
 * instead of its logits: a1 is the fused LM-head + Conf above over the max_branches * window
 * rows (<= LOPA_MAX_ROWS) of `hidden` (bf16 [max_branches][window][ld_hidden], row b * window + i =
 * branch b, position i), restricted to the masked rows of present branches; then the same
 * decision kernel as lopa_step.  args->logits and args->ld are ignored; every other field of
 * `args` keeps its lopa_step meaning (conf / argmax receive the fused a1 results).
 * lmh_workspace: lopa_lmhead_workspace_bytes(rows) bytes.  Three kernels, PDL-chained. */
int lopa_step_lmhead(const lopa_step_args_t* args, const void* hidden, int64_t ld_hidden,
                     const void* weight, int64_t ld_weight, int32_t hidden_dim,
                     void* lmh_workspace, size_t lmh_workspace_bytes, void* stream);

#if defined(__GNUC__)
#pragma GCC visibility pop
#endif

#ifdef __cplusplus
}
#endif
#endif /* LIBLOPA_H_ */
