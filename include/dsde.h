/*
 * dsde.h — C-ABI of the B200-native DSDE speculative-verification hot path.
 *
 * DSDE = "Dynamic Speculative Decoding Engine", arXiv 2509.01083.
 * Citation keys: P:n = PAPER.md line n; S:n = SPEC.md line n; D1..D17 =
 * the readings of the paper listed in DESIGN.md §3.
 *
 * The library (libdsde.so) exports exactly the functions declared here.
 * Signatures use plain pointers, sizes and opaque handles only.
 *
 * Conventions for every entry point:
 *   - Pointers are DEVICE pointers on the calling thread's current CUDA
 *     device unless the parameter says "host".
 *   - Calls that take a `stream` (a cudaStream_t passed as void*) only
 *     enqueue work on it; none of them synchronises the host, allocates
 *     memory or copies device->host. NULL = the legacy default stream.
 *   - The caller owns every input, output and workspace buffer. The library
 *     owns dsde_state (device memory allocated in dsde_state_create, never in
 *     a hot call) and dsde_comm.
 *   - Calls on one dsde_state must be serialised (same stream, or ordered);
 *     separate states are independent.
 *   - Outputs are bit-deterministic for identical inputs and launch
 *     configuration (no float atomics; every reduction has a fixed order).
 *   - Synchronous argument errors return DSDE_ERR_ARG (or DSDE_ERR_STATE)
 *     and launch nothing. DSDE_ERR_CUDA / DSDE_ERR_NCCL mirror a failed
 *     launch / collective.
 *   - Data errors that can only be seen on the device (see dsde_verify) set
 *     a sticky error word in the state; read it with dsde_get_device_error.
 *     A device-side error never causes an out-of-bounds access.
 */
#ifndef DSDE_H_
#define DSDE_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define DSDE_ABI_VERSION 4

typedef enum {
    DSDE_OK = 0,
    DSDE_ERR_ARG = -1,    /* invalid argument; nothing launched              */
    DSDE_ERR_CUDA = -2,   /* CUDA launch / runtime error                     */
    DSDE_ERR_NCCL = -3,   /* NCCL unavailable or collective failed           */
    DSDE_ERR_STATE = -4,  /* B larger than the state's capacity, bad slot    */
    DSDE_ERR_DEVICE = -5  /* returned by dsde_get_device_error only          */
} dsde_status;

typedef enum { DSDE_F32 = 0, DSDE_BF16 = 1 } dsde_dtype;

/* Reserved padding token id written into unused emitted-token slots when a
 * sequence accepts fewer than k_i drafts ("a reserved padding token
 * ID prevents invalid token identifiers from propagating"). */
#define DSDE_PAD (-1)

/* Largest per-sequence speculation length accepted by dsde_verify. */
#define DSDE_MAX_SL 16
/* Largest KLD history window (n_long) a state can hold. */
#define DSDE_MAX_WINDOW 64

/* Device-side error codes (dsde_get_device_error). */
#define DSDE_DERR_NONE 0
#define DSDE_DERR_BAD_SL 1        /* k_i outside [1, DSDE_MAX_SL] or cu_sl not monotone */
#define DSDE_DERR_BAD_TOKEN 2     /* draft token outside [0, V)                          */
#define DSDE_DERR_NONFINITE 3     /* non-finite logits in a row                          */
#define DSDE_DERR_ROWS 4          /* cu_sl[B] != total_draft_rows                         */
#define DSDE_DERR_BAD_SLOT 5      /* state slot outside [0, max_seqs)                     */
#define DSDE_DERR_VP_FALLBACK 6   /* vocab-parallel: residual mass 0 (the D7 fallback to p needs the
                                     whole row on one GPU; not supported by dsde_vp_*)    */

/* Per-slot bits of the optional `flags` output of dsde_verify. */
#define DSDE_FLAG_ACCEPT_NEAR_TIE 1  /* |u_acc - min(1, p/q)| < 1e-6 at this position      */
#define DSDE_FLAG_SAMPLE_NEAR_TIE 2  /* |u_smp - C/R| < 1e-6 at a CDF edge of the draw (D23: also a
                                        proposal's u_prop at a CDF edge of p or u_keep within
                                        1e-6 of its keep probability)                        */
#define DSDE_FLAG_FALLBACK 4         /* residual mass 0: the token was drawn from p (D7)  */
#define DSDE_FLAG_PROPOSAL_FALLBACK 8 /* D23: none of the DSDE_RESAMPLE_PROPOSALS proposals was
                                        kept; the recovery token is the D7 draw              */

/* The recovery draw (the resample from normalize(max(0, p - q)) at the first
 * rejection; S:127, P:260 — the paper does not say how it is sampled):
 *   DSDE_RESAMPLE_FULL (default, D7): the inverse CDF over max(0, p - q) with
 *     u_smp (one pass over the drawn row's logits after the finalize).
 *   DSDE_RESAMPLE_PROPOSAL (D23): proposals v_j ~ p (the inverse CDF
 *     of D7 over p with u_prop of proposal j = 1, 2, ...), each kept with
 *     probability max(0, p_v - q_v) / p_v (u_keep < that); the first kept
 *     proposal is the token. Exact: a kept proposal is distributed as
 *     normalize(max(0, p - q)); each is kept with probability TV(p, q). If
 *     none of DSDE_RESAMPLE_PROPOSALS is kept, the D7 draw above decides
 *     (flag DSDE_FLAG_PROPOSAL_FALLBACK). (u_prop, u_keep) of proposal j:
 *     Philox4x32-10 keyed by the slot's seed at counter (j, 0, 0, 0), res53 of
 *     words 0-1 / 2-3 (D6 uses counter 0). A proposal needs p's slice masses
 *     (from the row stream) and one slice of the row, so the recovery draw
 *     costs ~1/TV slice scans instead of a pass over the row: faster when the
 *     draft is far from the target (low acceptance), slower when TV is small.
 * Both are exact samplers of the same distribution; they consume different
 * random numbers, so they emit different tokens for the same seeds. The
 * bonus draw (all drafts accepted) is D7 over p in both. The
 * vocabulary-parallel stages (dsde_vp_*) implement DSDE_RESAMPLE_FULL. */
#define DSDE_RESAMPLE_PROPOSAL 0
#define DSDE_RESAMPLE_FULL 1
#define DSDE_RESAMPLE_PROPOSALS 256

/* Adapter configuration; defaults from the paper / SPEC (dsde_config_default).
 * Validity (S:173-174 plus D11/D17): 0 < delta <= 1; 1 <= n_short < n_long
 * <= DSDE_MAX_WINDOW; sl_min >= 1; sl_min < sl_ceiling <= DSDE_MAX_SL;
 * epsilon > 0; calib_steps >= 0; 1 <= calib_sl <= sl_ceiling;
 * window_unit in {0,1}; cap_mode in {0,1}; greedy in {0,1}; masked in {0,1};
 * entropy_mode in {0,1}; entropy_gamma > 0; resample in {0,1}. */
typedef struct {
    double delta;      /* decay factor of Eq.5, 0.85                         */
    int n_short;       /* short window, 10                                   */
    int n_long;        /* long window, 30                                    */
    int sl_min;        /* SL_min, 2                                          */
    int sl_ceiling;    /* hard bound on the calibrated SL_max (D17), 8               */
    double epsilon;    /* Eq.1 epsilon, 1e-6                                 */
    int calib_steps;   /* preliminary steps of Eq.1 (D12), 5                  */
    int calib_sl;      /* SL used while calibrating (D12), 4                         */
    int window_unit;   /* 0 = per-token KLD observations (default), 1 = per-step means (D8) */
    int cap_mode;      /* 0 = no cap (cap = max SL^), 1 = Eq.11 mean / MSE cap (default)     */
    int greedy;        /* 0 = rejection sampling (default); 1 = T = 0 verification: accept iff
                          x_j = argmax t_j, emit the target argmax (
                          ties -> smallest token id, D18). Read by dsde_verify / dsde_step
                          from the state; KLDs, signal and cap are unchanged. */
    int device_rows;   /* 0 = total_draft_rows is exactly sum_i k_i (default). 1 = it is a row
                          capacity >= sum_i k_i: the kernels read sum_i k_i = cu_sl[B] on the device,
                          grids and workspace are sized for the capacity, and a sequence whose rows
                          end beyond it is a DSDE_DERR_BAD_SL device error. Output arrays are sized
                          for the capacity. The launch configuration of dsde_verify / dsde_step then
                          no longer depends on the SLs, so one captured CUDA graph serves every SL
                          pattern (the SLs are device data). */
    int masked;        /* 0 = every logit is finite (default). 1 = logits may be -inf (top-k / top-p
                          masks, D21): a -inf target logit has p = 0, a -inf draft
                          logit q = 0; KL(p||q) = +inf when the draft masks a token the target keeps;
                          a draft token with q(x) = 0 is DSDE_DERR_BAD_TOKEN. The stream then takes
                          the exact per-element path everywhere. Not combinable with the draft
                          entropy (dsde_set_draft_entropy): DSDE_ERR_ARG. */
    int entropy_mode;  /* 0 = KLD signal only (default). 1 = SL^ = min(Eq.8, SL_H) with the draft-entropy
                          predictor SL_H = clamp(rint(max(0, 1 - sqrt(gamma H)) (SL_max - SL_min)
                          + SL_min)), H = the mean draft entropy of the step (D22; "optionally combined
                          with entropy"). Needs dsde_set_draft_entropy (else DSDE_ERR_ARG). */
    double entropy_gamma; /* gamma of D22, 0.5 */
    int resample;      /* the recovery draw's reading: DSDE_RESAMPLE_FULL (default, D7) or
                          DSDE_RESAMPLE_PROPOSAL (D23); see DSDE_RESAMPLE_FULL above */
} dsde_config;

typedef struct dsde_state_s* dsde_state; /* per-sequence KLD ring, calibration, SL_max, error word */
typedef struct dsde_comm_s* dsde_comm;   /* an NCCL communicator; NULL = single GPU                 */

/* Fills *cfg (host) with the defaults above. */
void dsde_config_default(dsde_config* cfg);

/* Human-readable name of a status code (static string). */
const char* dsde_status_string(dsde_status s);

/* ABI version of the loaded library (== DSDE_ABI_VERSION). */
int dsde_abi_version(void);

/* ---------------------------------------------------------------------- */
/* State                                                                   */
/* ---------------------------------------------------------------------- */

/* Creates a state for up to max_seqs sequences (slots 0..max_seqs-1) on the
 * current device and zero-initialises it (synchronously). cfg is host memory
 * and is copied. Errors: DSDE_ERR_ARG for an invalid cfg or max_seqs < 1;
 * DSDE_ERR_CUDA if the allocation fails. */
dsde_status dsde_state_create(const dsde_config* cfg, int max_seqs, dsde_state* out);

/* Starts new requests: clears history, calibration and SL_max of the n slots
 * listed in `slots` (device int32[n]). Asynchronous on stream. */
dsde_status dsde_state_reset(dsde_state st, const int32_t* slots, int n, void* stream);

/* Frees the state (synchronises the device first). NULL is accepted. */
dsde_status dsde_state_destroy(dsde_state st);

/* Size in bytes of the state's per-sequence device image (export/import). */
size_t dsde_state_bytes(dsde_state st);

/* Copies the per-sequence device image to / from `buf` (device, >=
 * dsde_state_bytes bytes), asynchronously on stream. Used to checkpoint,
 * replay and teacher-force ("adapter state dump/restore"). */
dsde_status dsde_state_export(dsde_state st, void* buf, size_t bytes, void* stream);
dsde_status dsde_state_import(dsde_state st, const void* buf, size_t bytes, void* stream);

/* Reads (and does not clear) the sticky device error word: *code is one of
 * DSDE_DERR_*, *seq the batch index of the first offending sequence (-1 if
 * none). Host pointers. Synchronises the device. */
dsde_status dsde_get_device_error(dsde_state st, int32_t* code, int32_t* seq);

/* Clears the device error word (asynchronous on stream). */
dsde_status dsde_clear_device_error(dsde_state st, void* stream);

/* ---------------------------------------------------------------------- */
/* Verify: §8(a) steps a1-a4                                               */
/* ---------------------------------------------------------------------- */

/* Workspace bytes dsde_verify needs for these sizes (host function). */
size_t dsde_verify_workspace_size(int B, int total_draft_rows, int V, dsde_dtype dtype);

/* One batched speculative-verification step ("Ragged Q").
 *
 * Sequence i in [0,B) drafted k_i = cu_sl[i+1]-cu_sl[i] tokens
 * x_{i,0..k_i-1}. For every draft position j it computes, from
 * the target logits t (row cu_sl[i]+i+j) and draft logits d (row
 * cu_sl[i]+j), with p = softmax(t), q = softmax(d):
 *   kld[cu_sl[i]+j]  = KL(p || q) = sum_v p_v log(p_v/q_v)   (D1, D3)
 *   acc_j            = u_acc(i,j) < min(1, p(x_j)/q(x_j))     (D5)
 * and a_i = first j with !acc_j, else k_i (prefix shape). The final
 * token is drawn by inverse CDF in ascending token id (D7) from
 *   normalize(max(0, p - q)) of position a_i  if a_i < k_i (recovery), or
 *   p of target row k_i                       if a_i = k_i (bonus token),
 * using u_smp(i, a_i). The two uniforms of slot (i,j) are
 *   (u_acc, u_smp) = res53 pairs of Philox4x32-10(key = seed, ctr = 0)   (D6).
 *
 * Arguments:
 *   B, V              batch size (>= 1) and vocabulary size (>= 2).
 *   dtype             DSDE_BF16 or DSDE_F32 logits.
 *   total_draft_rows  host copy of cu_sl[B] = sum_i k_i (grid sizing without
 *                     a device->host read); checked on the device.
 *   cu_sl             int32[B+1], exclusive prefix sum of k_i, cu_sl[0] = 0.
 *   draft_tokens      int32[total_draft_rows], token x_{i,j} at cu_sl[i]+j.
 *   target_logits     [total_draft_rows + B, ld_t] row-major; row cu_sl[i]+i+j
 *                     for j in [0,k_i] (row k_i = the bonus position).
 *   draft_logits      [total_draft_rows, ld_d] row-major.
 *   ld_t, ld_d        leading dimensions in elements, >= V; base pointers and
 *                     rows must be 16-byte aligned.
 *   seeds             uint64[total_draft_rows + B], one per output slot
 *                     (i,j), j in [0,k_i], at index cu_sl[i]+i+j.
 *   accepted_len      out int32[B]: a_i in [0,k_i]; -1 for a sequence with a
 *                     device-detected data error.
 *   emitted_tokens    out int32[total_draft_rows + B]: slot cu_sl[i]+i+j holds
 *                     x_{i,j} for j < a_i, the drawn token at j = a_i, and
 *                     DSDE_PAD for j > a_i.
 *   kld               out float[total_draft_rows]: KL at every draft position,
 *                     including positions after the first rejection (D3).
 *   flags             optional out uint8[total_draft_rows + B] (NULL ok):
 *                     DSDE_FLAG_* bits per slot.
 *   workspace         device scratch of >= dsde_verify_workspace_size bytes,
 *                     256-byte aligned, not used concurrently by another call.
 *   st                state whose error word receives device-detected errors.
 *   stream            CUDA stream.
 * Device-detected data errors (sticky, first one wins): a token outside
 * [0,V) or non-finite logits in a row (DSDE_DERR_BAD_TOKEN / _NONFINITE: the
 * sequence gets accepted_len -1, all-pad tokens and NaN KLD; the others are
 * unaffected); k_i outside [1, DSDE_MAX_SL] or rows beyond the launch
 * (DSDE_DERR_BAD_SL, or DSDE_DERR_ROWS when cu_sl[B] != total_draft_rows:
 * that sequence gets accepted_len -1, the others are unaffected); a cu_sl that
 * is not a non-decreasing prefix starting at 0 (DSDE_DERR_BAD_SL: no row can be
 * attributed, every sequence gets accepted_len -1). No device error ever
 * causes an out-of-bounds access.
 *
 * Execution: two kernels on `stream`: the row stream k_stream_ldg (persistent
 * warps read every (draft row, 2048-token slice) of the target and draft
 * logits once and write slice partials to the workspace), then k_tail
 * (programmatic dependent launch; one CTA per sequence: fp64 row merge,
 * accept test, layout, draw, select). */
dsde_status dsde_verify(int B, int V, dsde_dtype dtype, int total_draft_rows,
                        const int32_t* cu_sl, const int32_t* draft_tokens,
                        const void* target_logits, int64_t ld_t,
                        const void* draft_logits, int64_t ld_d,
                        const uint64_t* seeds, int32_t* accepted_len,
                        int32_t* emitted_tokens, float* kld, uint8_t* flags,
                        void* workspace, size_t ws_bytes, dsde_state st, void* stream);

/* ---------------------------------------------------------------------- */
/* Vocabulary-parallel verification (the    */
/* 70B target on 8 GPUs implies a vocab-parallel LM head)                   */
/* ---------------------------------------------------------------------- */
/* Shard s of n holds columns [v0_s, v0_s + Vs_s) of every target and draft
 * row (the row layout of dsde_verify, only narrower): v0_s = s W with the
 * shard width W from dsde_vp_sizes (a multiple of the 2048-token bf16 /
 * 512-token fp32 stream slice) and the last shard the remainder; ld >= Vs_s.
 * The stages below, with the caller's exchanges between them, give outputs
 * bit-identical to dsde_verify on the unsharded rows (every partial and every
 * draw mass is the unsharded one, read in the unsharded order):
 *   dsde_vp_stream   (per shard)  -> its partial block, its (t_x, d_x) (zeros
 *                                   where another shard owns x);
 *     exchange: all-gather the blocks into part_all [n][total][ns_sh] (32 B
 *               entries), all-reduce (sum) xlog [total][2] floats;
 *   dsde_vp_finalize (every shard) -> accepted_len, emitted (all but the
 *                                   drawn token), kld, flags, rec [B] (64 B);
 *   dsde_vp_draw     (per shard)  -> its mass block [B][nd_sh] (16 B entries);
 *     exchange: all-gather into mass_all [n][B][nd_sh];
 *   dsde_vp_select   (every shard) -> tok [B]: the drawn token (global id, the
 *                                   sample flags << 24) on the shard owning
 *                                   the crossing slice, -1 elsewhere;
 *     exchange: all-reduce (max) tok;
 *   dsde_vp_place    (every shard) -> the drawn tokens into emitted / flags.
 * dsde_vp_verify runs the whole sequence over a dsde_comm (NCCL all-gather /
 * all-reduce; comm NULL = one shard). The signal and cap then run unchanged
 * (every shard holds every KLD: dsde_update_signal / dsde_next_sl).
 * Supported: the default sampling mode only (no greedy, temperature, masks,
 * draft entropy or device_rows on the state: DSDE_ERR_ARG); a residual of
 * mass 0 (the D7 fallback) is DSDE_DERR_VP_FALLBACK. Buffers are device
 * memory, 16-byte aligned; asynchronous on stream. */
dsde_status dsde_vp_sizes(int V, int nshards, dsde_dtype dtype, int* shard_width, int* ns_sh, int* nd_sh);
dsde_status dsde_vp_stream(dsde_state st, int B, int V, int nshards, int shard, dsde_dtype dtype,
                           int total_draft_rows, const int32_t* cu_sl, const int32_t* draft_tokens,
                           const void* target_shard, int64_t ld_t, const void* draft_shard, int64_t ld_d,
                           void* part_block, float* xlog, void* stream);
dsde_status dsde_vp_finalize(dsde_state st, int B, int V, int nshards, dsde_dtype dtype, int total_draft_rows,
                             const int32_t* cu_sl, const int32_t* draft_tokens, const void* part_all,
                             const float* xlog, const uint64_t* seeds, int32_t* accepted_len,
                             int32_t* emitted_tokens, float* kld, uint8_t* flags, void* rec, void* stream);
dsde_status dsde_vp_draw(dsde_state st, int B, int V, int nshards, int shard, dsde_dtype dtype, const void* rec,
                         const void* target_shard, int64_t ld_t, const void* draft_shard, int64_t ld_d,
                         void* mass_block, void* stream);
dsde_status dsde_vp_select(dsde_state st, int B, int V, int nshards, int shard, dsde_dtype dtype,
                           const void* rec, const void* mass_all, const void* target_shard, int64_t ld_t,
                           const void* draft_shard, int64_t ld_d, int32_t* tok, void* stream);
dsde_status dsde_vp_place(dsde_state st, int B, const void* rec, const int32_t* tok_all,
                          int32_t* emitted_tokens, uint8_t* flags, void* stream);
/* Workspace of dsde_vp_verify (256-byte aligned): the exchange buffers. */
size_t dsde_vp_workspace_size(int B, int total_draft_rows, int V, int nshards, dsde_dtype dtype);
dsde_status dsde_vp_verify(dsde_state st, int B, int V, dsde_dtype dtype, int total_draft_rows,
                           const int32_t* cu_sl, const int32_t* draft_tokens, const void* target_shard,
                           int64_t ld_t, const void* draft_shard, int64_t ld_d, const uint64_t* seeds,
                           int32_t* accepted_len, int32_t* emitted_tokens, float* kld, uint8_t* flags,
                           void* workspace, size_t ws_bytes, dsde_comm comm, void* stream);

/* Per-sequence sampling temperature (D20; P:312 evaluates T = 0 and 1, P:490
 * per-sequence temperature) of the following dsde_verify /
 * dsde_step calls on this state: `temperature` is device float[B] indexed by
 * batch position (read by every call; the caller owns it), NULL = T = 1 for
 * every sequence (the default). T > 0: p = softmax(t / T), q = softmax(d / T)
 * (KLDs, accept test and draws at T); T = 0: that sequence verifies greedily
 * (as dsde_config.greedy, D18, KLDs at T = 1). A negative or non-finite T is
 * a DSDE_DERR_NONFINITE device error for its sequence. */
dsde_status dsde_set_temperature(dsde_state st, const float* temperature);

/* Kernel timing of dsde_verify / dsde_step (instrumentation; off by
 * default). While enabled, every dsde_verify / dsde_step call on this state
 * records CUDA events on its stream before its first launch and after each of
 * its DSDE_VERIFY_PHASES phases: 0 = the row stream k_stream_ldg (a1),
 * 1 = the tail k_tail (a2-a4, and in dsde_step a5-a6 plus the single-GPU cap
 * a7), 2 and 3 = unused (read 0; dsde_step's multi-GPU cap kernels and
 * all-reduce are not inside the recorded phases). The tail is launched with
 * programmatic dependent launch, so the event between the two kernels also
 * covers the tail's start-up that overlaps the stream's drain.
 * dsde_profile_read blocks until the last recorded event completes, writes
 * the summed milliseconds of each phase over the calls recorded since the
 * previous read to ms[DSDE_VERIFY_PHASES] (host memory) and the call count to
 * *calls (may be NULL), then forgets them. Host functions; not thread-safe
 * per state. */
#define DSDE_VERIFY_PHASES 4
dsde_status dsde_profile_enable(dsde_state st, int enable);
dsde_status dsde_profile_read(dsde_state st, float* ms, int* calls);

/* ---------------------------------------------------------------------- */
/* Signal + SL prediction: §8(a) steps a5-a6                               */
/* ---------------------------------------------------------------------- */

/* Observes one verification step for B sequences and predicts SL^_i.
 * Per sequence (slot = slots[i]):
 *   1. append KL_{i,0..k_i-1} in position order to the history ring of
 *      capacity n_long, oldest evicted (Fig.5); with
 *      window_unit = 1 the step mean is appended instead (D8);
 *   2. mu_last = mean of this step's KLDs;
 *   3. for the first calib_steps observed steps accumulate SL_A,max = max
 *      a_i, the mean and max KLD; at the last one set SL_max by Eq.1
 *      rounded half-even and clamped to [sl_min+1, sl_ceiling] (D11, D12);
 *   4. Var_w over the most recent min(n, n_short) and min(n, n_long)
 *      observations with alpha_i = delta^(i-1), i = 1 most recent (Eq.5-7,
 *      P:214-223), by a weighted Welford recurrence in fp64;
 *   5. WVIR = Var_short / Var_long (Eq.4); WVIR = 1 while n < n_short
 *      (D9) or Var_long < 1e-12 (D10);
 *   6. SF = exp(2 mu_last) - 1 (Eq.3); penalty = SF * WVIR;
 *   7. SL^ = rint((1 - penalty)(SL_max - SL_min) + SL_min) if penalty <= 1,
 *      else SL_min (Eq.8), clamped to [SL_min, SL_max]; while
 *      calibrating SL^ = calib_sl.
 * Arguments: slots int32[B] state slots; cu_sl, kld, accepted_len as produced
 * by dsde_verify; sl_hat out int32[B]; diag optional out double[B][8] =
 * (mu_last, sf, var_short, var_long, wvir, penalty, x_pre_round, sl_max)
 * (var_* are NaN during warm-up; x_pre_round is NaN while calibrating).
 * A sequence whose accepted_len is -1 (verify data error) is left untouched
 * and gets sl_hat = sl_min. */
dsde_status dsde_update_signal(dsde_state st, int B, const int32_t* slots,
                               const int32_t* cu_sl, const float* kld,
                               const int32_t* accepted_len, int32_t* sl_hat,
                               double* diag, void* stream);

/* ---------------------------------------------------------------------- */
/* Adaptive cap and next SL: §8(a) step a7                                 */
/* ---------------------------------------------------------------------- */

/* Batch-wide cap (Eq.9-11) and next speculation lengths.
 * cap = round-half-even(sum_i SL^_i / N) over the N sequences of the batch
 * that have finished calibration, in exact int64 arithmetic (D14); with a
 * communicator the sum and N are all-reduced over all ranks first (the only
 * cross-GPU exchange of the path). cap_mode 0: cap = max SL^ (no cap).
 * N == 0: cap = sl_ceiling. Then
 *   next_sl_i = calibrating ? calib_sl : min(SL^_i, cap),
 *   next_sl_i = min(next_sl_i, budget_i) if budget != NULL.
 * Arguments: slots int32[B]; sl_hat int32[B] from dsde_update_signal; budget
 * optional int32[B] (remaining tokens, >= 1); next_sl out int32[B]; cap out
 * int32[1]; comm NULL for a single GPU. */
dsde_status dsde_next_sl(dsde_state st, int B, const int32_t* slots, const int32_t* sl_hat,
                         const int32_t* budget, int32_t* next_sl, int32_t* cap,
                         dsde_comm comm, void* stream);

/* ---------------------------------------------------------------------- */
/* Whole step: §8(a) steps a1-a7 in one call                               */
/* ---------------------------------------------------------------------- */

/* One DSDE decoding step of the batch: exactly
 *   dsde_verify(B, V, dtype, total_draft_rows, cu_sl, draft_tokens, ...);
 *   dsde_update_signal(st, B, slots, cu_sl, kld, accepted_len, sl_hat, diag);
 *   dsde_next_sl(st, B, slots, sl_hat, budget, next_sl, cap, comm);
 * with the same arguments, results, state updates and errors as those three
 * calls made in that order on `stream` (bit-identical outputs), but in two
 * kernels on one GPU: the row stream and the tail, whose CTA for sequence i
 * also updates its signal and predicts SL^ (a5-a6); the warp completing the
 * batch's last signal applies the cap (a7). With a communicator the cap's
 * exact partial is all-reduced over NCCL after the tail (two more launches +
 * the collective).
 * The workspace is the one dsde_verify takes. Errors: the union of the three
 * calls' synchronous checks (DSDE_ERR_ARG / DSDE_ERR_STATE) and
 * DSDE_ERR_CUDA / DSDE_ERR_NCCL. Calls on one state must be serialised. */
dsde_status dsde_step(dsde_state st, int B, int V, dsde_dtype dtype, int total_draft_rows,
                      const int32_t* slots, const int32_t* cu_sl, const int32_t* draft_tokens,
                      const void* target_logits, int64_t ld_t, const void* draft_logits,
                      int64_t ld_d, const uint64_t* seeds, const int32_t* budget,
                      int32_t* accepted_len, int32_t* emitted_tokens, float* kld, uint8_t* flags,
                      int32_t* sl_hat, double* diag, int32_t* next_sl, int32_t* cap,
                      void* workspace, size_t ws_bytes, dsde_comm comm, void* stream);

/* Draft entropy (the paper's optional entropy signal next to
 * the KLD). While entropy != NULL, every dsde_verify / dsde_step
 * call on this state also writes H(q_j) = -sum_v q_v log q_v, q = softmax of
 * draft row j, to entropy[j] for j in [0, sum_i k_i) (device memory, float,
 * sized for the rows of the calls; not owned). It is formed in the same
 * streaming pass (two extra per-slice sums of the draft's own softmax, merged
 * in fp64 with the row), at ~1e-6 relative accuracy. NULL (the default) turns
 * it off and the stream kernel compiled without it runs. Errors: DSDE_ERR_ARG
 * for a NULL state. Host-side setting, no stream work. */
dsde_status dsde_set_draft_entropy(dsde_state st, float* entropy);

/* Host-callable form of the cap rule used by dsde_next_sl (same code): the
 * cap from the global exact partial (sum of SL^, N, max SL^). Lets callers
 * that all-reduce the partial themselves (and the CPU tests) apply it. */
int32_t dsde_cap_value(const dsde_config* cfg, int64_t sum_sl_hat, int64_t n_active,
                       int64_t max_sl_hat);

/* ---------------------------------------------------------------------- */
/* Multi-GPU: one NCCL communicator over the ranks of one box              */
/* ---------------------------------------------------------------------- */

/* NCCL is resolved at run time from the process (the copy torch already
 * loaded, else libnccl.so.2); without it these return DSDE_ERR_NCCL. */
dsde_status dsde_comm_unique_id(uint8_t id[128]);                 /* host; rank 0 */
dsde_status dsde_comm_init(const uint8_t id[128], int nranks, int rank, dsde_comm* out);
dsde_status dsde_comm_destroy(dsde_comm comm);

#ifdef __cplusplus
}
#endif

#endif /* DSDE_H_ */
