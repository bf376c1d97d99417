/*
 * include/dash.h -- C ABI of libdash.so: DASH deterministic attention
 * backward for NVIDIA B200 (sm_100a).
 *
 * Paper: "DASH: Deterministic Attention Scheduling for High-Throughput
 * Reproducible LLM Training", arXiv 2601.21824.  "P:n" below is line n of
 * that paper's text; "AMB-k" is reading k of DESIGN.md §Readings.
 *
 * Conventions shared by every entry point
 * ---------------------------------------
 *  - Tensors q, k, v, o, dO, dq, dk, dv: bf16, layout [B, N, H, d], dense
 *    row-major (d fastest), 16-byte aligned.  lse: fp32 [B, H, N],
 *    natural-log logsumexp of the scaled scores (AMB-15).  These are
 *    Algorithm 1's "Q, K, V, O, dO in R^{N x d}, logsumexp L in R^N"
 *    for every (batch, head).
 *  - Supported: d in {64, 128}; N a positive multiple of 128 (the KV/Q tile
 *    size B_r = B_c = 128 of the schedule model, AMB-11); seqlen_q = seqlen_k;
 *    B * N * H < 2^31 rows.
 *  - softmax_scale <= 0 selects 1/sqrt(d) (AMB-1).
 *  - Device pointers are CUDA device pointers owned by the caller.  All
 *    scratch lives in the caller-provided workspace; the only device memory
 *    the library allocates is its schedule tables (a few KB per (device,
 *    schedule, n, mask), uploaded once on first use and cached), and
 *    dash_attn_bwd_host creates three library-owned streams per device on
 *    first use.  After a warm-up call the backward can be captured in a CUDA
 *    graph.  `stream` is a cudaStream_t (NULL = legacy
 *    default stream); every call is stream-ordered and asynchronous unless
 *    stated otherwise.  A workspace must not be used by two in-flight calls.
 *  - Errors are returned as dash_status; nothing is thrown across the ABI.
 *    DASH_ERR_INVALID_ARG: null pointer, misalignment, unsupported shape.
 *    DASH_ERR_UNSUPPORTED: a legal request this build cannot run (see each
 *    call).  DASH_ERR_WORKSPACE: workspace too small.  DASH_ERR_CUDA: a CUDA
 *    runtime error (cudaGetLastError after launch).  DASH_ERR_DEADLOCK: a
 *    ticket wait exceeded its bound in an earlier call on this workspace
 *    (reported by the next call that synchronises, see dash_check_workspace).
 */
#ifndef DASH_H_
#define DASH_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  DASH_OK = 0,
  DASH_ERR_INVALID_ARG = 1,
  DASH_ERR_UNSUPPORTED = 2,
  DASH_ERR_WORKSPACE = 3,
  DASH_ERR_CUDA = 4,
  DASH_ERR_DEADLOCK = 5
} dash_status;

typedef enum { DASH_MASK_FULL = 0, DASH_MASK_CAUSAL = 1 } dash_mask;

/* Q-tile visiting orders over the ordered dQ reduction (§3):
 *  NAIVE      -- ascending Q tiles, dQ reduced in ascending KV order; the
 *                FlashAttention-3 deterministic baseline.
 *  DESCENDING -- Descending Q-Tile Iteration, same reduction order (§3.3,
 *                P:91-103; AMB-6).
 *  SHIFT      -- Shift Scheduling: cyclic shift for the full mask,
 *                Symmetric Shift (KV pairs i, n-1-i, two phases) for the
 *                causal mask; dQ reduced in visit-step order. */
typedef enum {
  DASH_SCHED_NAIVE = 0,
  DASH_SCHED_DESCENDING = 1,
  DASH_SCHED_SHIFT = 2,
  /* dash_attn_bwd only: one of the three above, chosen per (mask, N, d) --
   * see dash_attn_bwd_resolve_schedule. */
  DASH_SCHED_AUTO = 3
} dash_schedule;

typedef struct {
  int batch;           /* B */
  int seqlen;          /* N (= seqlen_q = seqlen_k) */
  int heads;           /* H */
  int head_dim;        /* d */
  float softmax_scale; /* <= 0 -> 1/sqrt(d) */
} dash_shape;

/* Attention forward: o = softmax(scale * q k^T [+ causal mask]) v and the
 * natural-log logsumexp lse, i.e. the O and L that Algorithm 1 requires
 * (P:353).  Causal: key c is visible to query r iff c <= r.  Not the timed
 * path; numerically an fp32-accumulating kernel with bf16 output.
 * Returns DASH_ERR_INVALID_ARG / DASH_ERR_CUDA as described above. */
dash_status dash_attn_fwd(const dash_shape* shape, const void* q, const void* k, const void* v,
                          void* o, float* lse, int causal, void* stream);

/* Bytes of device workspace dash_attn_bwd needs for this problem: the W
 * interleaved fp32 dQ accumulators [W][B,H,N,d] (Alg.1 line 34's "dQ_i in
 * global memory"; AMB-27) -- W = dash_attn_bwd_acc_split(shape, ...) under the
 * current setting when deterministic != 0, W = 1 for the atomic variant --
 * D = rowsum(dO o O) and -L*log2(e) fp32 [B,H,N] (Alg.1 line 1, P:355;
 * AMB-2), one int32 ticket per (accumulator, b, h, Q sub-tile) (the "global
 * order"), the job counter and the error flag.  The accumulators
 * sit at offset 0.  Returns 0 for an invalid shape.  A workspace sized under
 * one W setting is rejected (DASH_ERR_WORKSPACE) by a call that needs more. */
size_t dash_attn_bwd_workspace_bytes(const dash_shape* shape, int causal, int schedule,
                                     int deterministic);

/* Attention backward (Algorithm 1).  Computes
 *   D = rowsum(dO o O); P = exp(scale*S - L); dS = P o (dP - D)
 *   dV = P^T dO;  dK = scale * dS^T Q;  dQ = scale * dS K
 * with each CTA owning a KV tile (dK, dV reduced on chip) and the dQ
 * partials of all KV tiles added into an fp32 accumulator.
 *  deterministic != 0: the adds into each dQ tile happen in the fixed order
 *    of `schedule`, enforced by a per-Q-tile ticket (acquire/release), so
 *    results are bitwise identical run to run and across (b, h) sharding.
 *  deterministic == 0: the atomic comparison variant (Fig.1) -- the
 *    same kernel with unordered reduce-adds; Q order still follows `schedule`.
 * dq, dk, dv are written (not accumulated); dq = bf16(scale * accumulator),
 * formed in the main kernel's tail or by a convert kernel after it (see
 * dash_attn_bwd_set_fused_dq).  o and lse must come from the
 * forward of the same inputs (dash_attn_fwd or any exact equivalent).
 * SHIFT with causal and an odd number of KV tiles runs the Symmetric Shift of
 * n_kv + 1 tiles without the phantom tile (DESIGN.md AMB-29).
 * SHIFT with the full mask and n_kv > 128 runs in groups of <= 128 KV tiles
 * (AMB-30); SHIFT causal with more than 128 tile pairs in groups of <= 128
 * pairs (AMB-35).
 * DASH_ERR_UNSUPPORTED: SHIFT needing more co-resident CTAs than the device
 * holds (one group: min(n_kv, 128) for full, min(ceil(n_kv/2), 128) for
 * causal; App. B of SURVEY.md, AMB-12).
 * DASH_ERR_WORKSPACE: workspace_bytes < dash_attn_bwd_workspace_bytes(). */
dash_status dash_attn_bwd(const dash_shape* shape, const void* q, const void* k, const void* v,
                          const void* o, const void* dout, const float* lse,
                          void* dq, void* dk, void* dv, int causal, int schedule,
                          int deterministic, void* workspace, size_t workspace_bytes,
                          void* stream);

/* End-to-end variant with HOST buffers: q, k, v, o, dout, lse are host
 * pointers (pinned memory recommended: pageable memory makes the copies
 * synchronous), dq, dk, dv host outputs, same layouts as dash_attn_bwd.
 * The (b, h) heads are split into chunks (batch ranges, or head ranges of one
 * batch when B is small) that stream through three device slots of
 * `workspace` on three library-owned streams: the H2D copy of chunk i+1, the
 * backward of chunk i and the D2H copy of chunk i-1 overlap.  A chunk is a
 * (b, h) shard, so the results are bit-identical to dash_attn_bwd on the
 * whole problem.  Work queued on `stream` before the call is waited for; the
 * call returns after the last copy has completed and `stream` is ordered
 * after it.  Workspace size: dash_attn_bwd_host_workspace_bytes() (three
 * chunk slots, each with its own dash_attn_bwd workspace).  Errors as
 * dash_attn_bwd; DASH_ERR_INVALID_ARG also for a null host pointer. */
size_t dash_attn_bwd_host_workspace_bytes(const dash_shape* shape, int causal, int schedule,
                                          int deterministic);
dash_status dash_attn_bwd_host(const dash_shape* shape, const void* q, const void* k,
                               const void* v, const void* o, const void* dout, const float* lse,
                               void* dq, void* dk, void* dv, int causal, int schedule,
                               int deterministic, void* workspace, size_t workspace_bytes,
                               void* stream);

/* Synchronises `stream` and reports DASH_ERR_DEADLOCK if a ticket wait of
 * the most recent dash_attn_bwd on this workspace exceeded its bound (see
 * dash_attn_bwd_set_watchdog): the kernel then raises a device-wide abort
 * flag, every warp role leaves, and the outputs are invalid.  Else DASH_OK.
 * Every dash_attn_bwd resets the flag at its start. */
dash_status dash_check_workspace(const dash_shape* shape, int causal, int schedule,
                                 int deterministic, const void* workspace, void* stream);

/* Host-side DAG model (§3.1-3.4): critical-path length of the
 * deterministic backward of `n_heads` heads executed on `n_sm` SMs under
 * `schedule`, each task a compute phase of weight c followed by a reduction
 * phase of weight r, dQ_j reduced in the schedule's order.  Jobs are claimed
 * head-major by the earliest-free SM, ties to the lowest SM index (AMB-7); a
 * reduction occupies its SM (AMB-24).  n_q must equal n_kv (AMB-11).
 * p == NULL selects {n_heads = 2, n_sm = n_kv, c = 1, r = 1}.
 * DASH_ERR_INVALID_ARG: n_q != n_kv, n_kv < 1, c < 1 or r < 1 (positive
 * weights: Lemma 1's premise), n_sm < 1, n_heads < 1.
 * SHIFT causal with odd n_kv: the n_kv + 1 schedule without the phantom tile
 * (AMB-29).
 * DASH_ERR_DEADLOCK: the schedule cannot finish on n_sm SMs (SHIFT with
 * fewer SMs than a head's jobs). */
typedef struct {
  int n_heads;
  int n_sm;
  int64_t c;
  int64_t r;
} dash_dag_params;

dash_status dash_schedule_critical_path(int schedule, int n_q, int n_kv, int mask,
                                        const dash_dag_params* p, int64_t* out_length);

/* The per-head schedule table the kernels use (§8(a) row a1): for each job
 * (in claim order) its tasks (kv tile, q tile) in visiting order and each
 * task's rank in its dQ tile's reduction order.  Arrays must hold
 * `capacity` tasks; *n_tasks / *n_jobs receive the counts (if capacity is
 * too small nothing is written and DASH_ERR_WORKSPACE is returned).
 * task_job[t] is the job index of task t; tasks of a job are contiguous. */
dash_status dash_schedule_table(int schedule, int n_kv, int mask, int capacity,
                                int32_t* task_job, int32_t* task_kv, int32_t* task_q,
                                int32_t* task_rank, int32_t* n_tasks, int32_t* n_jobs);

/* Per-kernel timing of dash_attn_bwd for measurement: between
 * dash_profile_begin() and dash_profile_end(), every dash_attn_bwd records
 * CUDA events on its own stream around its three kernels (preprocess, main,
 * dQ convert).  dash_profile_end synchronises those events and returns the
 * summed milliseconds of each kernel and the number of calls profiled.
 * Host-thread-global; not for concurrent use from several threads. */
dash_status dash_profile_begin(void);
dash_status dash_profile_end(double* ms_preprocess, double* ms_main, double* ms_convert,
                             int* n_calls);

/* Measurement variant of dash_attn_bwd (same arguments and results) that
 * also records, per CTA of the main kernel and per Q sub-tile x it processes
 * (x < trace_cap), clock64() stamps of the pipeline stages into `trace`
 * (device memory, uint64 [grid][trace_cap][32], grid = min(jobs, SMs),
 * zero-filled by the caller).  Slots: 0 S/dP MMAs issued, 1 P^T/dS^T seen
 * by the MMA issuer, 2 dQ MMA issued, 3 softmax start, 4 softmax done,
 * 5 dQ drain start, 6 dQ staged, 7 ticket acquired, 8 reduce issued,
 * 9 ticket released.  This is the DAG model's C/R phase timeline
 * (SURVEY.md §5 DASH_TRACE).  DASH_ERR_INVALID_ARG for a null trace. */
dash_status dash_attn_bwd_trace(const dash_shape* shape, const void* q, const void* k,
                                const void* v, const void* o, const void* dout, const float* lse,
                                void* dq, void* dk, void* dv, int causal, int schedule,
                                int deterministic, void* workspace, size_t workspace_bytes,
                                unsigned long long* trace, int trace_cap, void* stream);

/* The schedule dash_attn_bwd runs for `schedule` (DASH_SCHED_AUTO resolved,
 * others returned unchanged): with n = N / 128, SHIFT for n <= 32; causal
 * DESCENDING for n >= 64 at d = 128 and n >= 128 at d = 64 (SHIFT between);
 * full mask NAIVE for n > 32 -- the fastest of the paper's three measured on
 * B200.  Returns -1 for an invalid shape or schedule. */
int dash_attn_bwd_resolve_schedule(const dash_shape* shape, int causal, int schedule);

/* Number W of interleaved fp32 dQ accumulators the deterministic backward
 * with these arguments uses (AMB-27).  W = 1 is the paper's single global
 * order per dQ tile.  W in {2, 4, 8}: the contribution of rank k
 * is added, in rank order, into accumulator k mod W under that accumulator's
 * own ticket, and the convert kernel sums the accumulators in index order --
 * a fixed order, so results stay bitwise deterministic, while consecutive
 * adds into one accumulator are W schedule steps apart instead of one.
 * Automatic rule (depends on N, d and the kernel only -- never on B or H, so
 * (b, h) sharding cannot change it), with n = N / T tiles of T rows
 * (dash_attn_bwd_tile): single-CTA kernel (T = 128): W = 8 for n >= 256, 4
 * for n >= 64, else 2; CTA-pair kernel (T = 256): 1 for n <= 8, 2 for n <= 16,
 * 4 for n < 128, else 8.  shape == NULL returns the setting itself (0 =
 * automatic); an invalid shape or schedule returns 0.  The setting defaults
 * to automatic, or to the DASH_ACC_SPLIT environment variable;
 * dash_attn_bwd_set_acc_split(w), w in {0 (automatic), 1, 2, 4, 8}, changes it
 * for later calls (host-global, not for concurrent use; other values:
 * DASH_ERR_INVALID_ARG).  The atomic variant always uses one accumulator. */
int dash_attn_bwd_acc_split(const dash_shape* shape, int causal, int schedule);
dash_status dash_attn_bwd_set_acc_split(int w);

/* Verification variant of dash_attn_bwd (same arguments and results) that
 * also writes every dQ partial dQ_local = dS K_i (Alg.1 line 28; fp32,
 * unscaled) as it is handed to the ordered reduction: partials is device
 * memory, fp32 [B*H][n][N][d] with n = N / T KV tiles of T rows
 * (T = dash_attn_bwd_tile(shape, causal, schedule)), element
 * [bh][i][r][c] = the partial of KV tile i for query row r (rows of Q tiles
 * that KV tile i does not visit are left untouched; zero-fill first).  With
 * the schedule's ranks this lets
 * a test re-sum the partials in the paper's order on the host and compare dq
 * bit for bit (SURVEY.md §8(c) c4 "T5
 * replay").  partial_bytes must be >= dash_attn_bwd_dump_bytes(shape) (else
 * DASH_ERR_WORKSPACE); null/misaligned partials: DASH_ERR_INVALID_ARG. */
size_t dash_attn_bwd_dump_bytes(const dash_shape* shape, int causal, int schedule);
dash_status dash_attn_bwd_dump(const dash_shape* shape, const void* q, const void* k,
                               const void* v, const void* o, const void* dout, const float* lse,
                               void* dq, void* dk, void* dv, int causal, int schedule,
                               int deterministic, void* workspace, size_t workspace_bytes,
                               float* partials, size_t partial_bytes, void* stream);

/* Bound of one ticket wait of the ordered reduction, in SM clock cycles
 * (clock64); 0 restores the default (2^36, ~35 s at 1.965 GHz).  A wait that
 * exceeds it aborts the launch (dash_check_workspace -> DASH_ERR_DEADLOCK)
 * instead of hanging the GPU.  Host-global; DASH_ERR_INVALID_ARG if < 0. */
dash_status dash_attn_bwd_set_watchdog(long long cycles);

/* Verification only (the watchdog test): the next dash_attn_bwd issued by the
 * calling thread presets its first ticket to `poison` (0 = no fault) -- a
 * rank no ordered add ever reaches -- so a wait can only end through the
 * watchdog.  Always DASH_OK. */
dash_status dash_attn_bwd_inject_fault(int poison);

/* Schedule tile size T (B_r = B_c, AMB-11 / AMB-31) a dash_attn_bwd with
 * these arguments runs with: 256 -- the CTA-pair kernel (a cluster of two
 * CTAs per 256-row KV tile, cta_group::2 MMAs, one dQ partial per 256 KV
 * rows) -- at d = 128 when N is a multiple of 256 and N >= 4096 (full mask:
 * N >= 2048), else 128 (the single-CTA kernel, which measured faster on
 * shorter heads: more, shorter jobs); for SHIFT only when the head's jobs fit
 * the device's CTA pairs.  Depends on (N, d, mask, schedule) only, never on
 * B or H.  The schedules, ranks and the DAG model are those of the paper with
 * n = N / T tiles.  0 for an invalid shape or schedule. */
int dash_attn_bwd_tile(const dash_shape* shape, int causal, int schedule);

/* 0 = automatic (the rule above), 128 = always the single-CTA kernel, 256 =
 * the CTA-pair kernel wherever it applies (d = 128, N a multiple of 256, a
 * SHIFT head fits the device's pairs).  Host-global; DASH_ERR_INVALID_ARG for
 * other values.  DASH_TILE in the environment sets the initial value. */
dash_status dash_attn_bwd_set_tile(int tile);

/* dQ-plane budget.  The W fp32 dQ accumulators (AMB-27) of all B*H heads take
 * W * B*H*N*d*4 bytes of the workspace -- 32 GiB at BASELINE config 4 (B = 8,
 * H = 32, N = 32k, d = 128, W = 8).  When that exceeds the budget (default 4
 * GiB), dash_attn_bwd processes the flattened heads in chunks of
 * dash_attn_bwd_head_chunk(...) consecutive heads (main kernel + dQ convert
 * per chunk, one preprocess) that reuse one set of accumulator planes, and
 * dash_attn_bwd_workspace_bytes shrinks accordingly.  A chunk is a (b, h)
 * shard (heads are independent, §2.1): every per-head schedule, rank and
 * accumulation order is unchanged, so results are bit-identical for every
 * budget.  set_plane_budget(0) restores the default; host-global, applies to
 * later calls (a workspace sized under another budget may then be too small:
 * DASH_ERR_WORKSPACE).  head_chunk returns the heads per chunk (B*H when one
 * chunk suffices), 0 for an invalid shape or schedule. */
dash_status dash_attn_bwd_set_plane_budget(size_t bytes);
int dash_attn_bwd_head_chunk(const dash_shape* shape, int causal, int schedule, int deterministic);

/* dQ finalise (the fp32 accumulator of P:396 turned into
 * the bf16 dQ output).  mode 1 (default): from N = 2048 the main kernel
 * writes dq itself -- every reducer agent counts its completed jobs (release)
 * and CTAs whose jobs ran out convert the heads whose jobs all completed
 * (acquire), in the kernel's tail -- and below N = 2048 (short jobs, little
 * tail; measured faster there) the separate K4 convert kernel does.  mode 0:
 * always K4; mode 2: always in the main kernel.  Every mode forms
 * bf16(scale * (acc_0 + ... + acc_{W-1})) in the same order: results are
 * bit-identical.  Host-global, later calls; the workspace size does not
 * depend on it.  DASH_ERR_INVALID_ARG for another mode. */
dash_status dash_attn_bwd_set_fused_dq(int mode);
int dash_attn_bwd_fused_dq(void);

/* Device kernel launches one dash_attn_bwd with these arguments makes: 1
 * (preprocess) + per chunk of heads (dash_attn_bwd_head_chunk) the main
 * kernel and, unless the dQ finalise is fused for this shape, K4.  0 for an
 * invalid shape or schedule. */
int dash_attn_bwd_launch_count(const dash_shape* shape, int causal, int schedule,
                               int deterministic);

/* Shape-free form: 3 (preprocess, main, dQ convert), or 2 when the finalise
 * is always fused (mode 2), for heads that fit one chunk. */
int dash_attn_bwd_launches(int causal, int schedule, int deterministic);

/* Diagnostic code behind the calling thread's most recent DASH_ERR_CUDA (0 if
 * none yet): the cudaError_t of the failing runtime call; 10000 + cudaError_t
 * when the launch of the main backward kernel was refused; -1 when a TMA
 * tensor map could not be encoded (alignment / extent of a tensor). */
int dash_last_cuda_error(void);

const char* dash_status_string(dash_status s);
const char* dash_version(void);

#ifdef __cplusplus
}
#endif

#endif /* DASH_H_ */
