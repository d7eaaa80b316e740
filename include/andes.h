/*
 * andes.h -- C ABI of the B200-native Andes scheduling-decision library (libandes.so).
 *
 * The library computes, on one B200 (sm_100a), the per-iteration QoE-aware
 * scheduling decision of Andes (arXiv 2404.16283, "PAPER"):
 *   S1  QoE of every live request's delivered-token timeline   (Eq. 1-3)
 *   S3  QoE gain of serving vs waiting over Delta t, for every
 *       candidate batch size B                                 (Eq. 4)
 *   S4  priority = gain / context length and Algorithm 1's
 *       greedy packing for every B                             (Eq. 6)
 *   S5  best B
 *   S0/S2 selective triggering and batch-size range
 *   S6  preemption cap                                         (reading R18)
 * "P:Lnnn" = line nnn of the paper's text; "Rnn" = the numbered
 * readings of silent/ambiguous passages listed in DESIGN.md.
 *
 * Conventions (all entry points):
 *  - Every array pointer is DEVICE memory owned by the caller, unless the
 *    entry point's name ends in _host.  The library never frees caller memory.
 *  - Times are integer microseconds. Absolute times are int64; times relative
 *    to a request's arrival are uint32 (must be < 2^32 us, ~71.6 min).
 *  - `stream` is a cudaStream_t passed as void*. Device entry points are
 *    ASYNCHRONOUS on that stream: they validate host-side arguments, enqueue
 *    kernels and return; results are valid after the stream is synchronised.
 *  - Host-side validation errors return a negative AndesStatus before any launch.
 *  - The library never allocates, frees or synchronises inside a device entry
 *    point; its workspace is sized by andes_create's limits.
 *  - One context per stream; contexts are not thread-safe.
 *  - andes_qoe_eval / andes_gain_estimate / andes_schedule are stream-capture safe: a
 *    decision can be captured once into a CUDA graph and replayed (same pointers/params).
 *  - Device-side errors go to the context's sticky error word (mapped pinned host memory the
 *    kernels write; no copy or synchronisation is added to a call).  The first call on the
 *    context that starts after the failing kernel has run returns the error and clears the
 *    word (with back-to-back asynchronous calls that can be a later call than the next one):
 *      ANDES_E_CAPACITY: a workspace capacity was exceeded on the device -- more running
 *        requests than the decision holds (4096; 2048 per rank in the sharded decision), or a
 *        timestamp pool longer than limits.max_tokens.  Always checked; the failing decision is
 *        truncated and flags it with ANDES_F_TRUNCATED.
 *      ANDES_E_RANGE: a data precondition failed.  Checked only under ANDES_DEBUG_CHECKS
 *        (andes_schedule, andes_schedule_shard): period >= 1, 1 <= l_i <= M, tl_base
 *        nondecreasing with room for n_deliv, delivery times nondecreasing and <= now - a_i,
 *        ranks unique (exact), fewer than 2^20 tokens due per request.
 */
#ifndef ANDES_H
#define ANDES_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct AndesCtx AndesCtx; /* opaque; owns a device workspace sized at create */

typedef enum {
    ANDES_OK = 0,
    ANDES_E_INVAL = -1,    /* bad argument (null pointer, zero period, B out of range, ...) */
    ANDES_E_RANGE = -2,    /* a device-side data precondition failed (debug checks)        */
    ANDES_E_CUDA = -3,     /* a CUDA runtime error; see andes_last_error                   */
    ANDES_E_NCCL = -4,     /* the peer-memory all-gather timed out waiting for a peer       */
    ANDES_E_CAPACITY = -5, /* n, B_cap, token count or running-set size above the limits   */
    ANDES_NOT_TRIGGERED = 1 /* _host entry points only: the trigger did not fire           */
} AndesStatus;

/* Workspace limits, fixed at create. */
typedef struct {
    uint32_t max_requests; /* largest n of any call                                     */
    uint32_t max_B;        /* largest B_cap (<= 1024)                                   */
    uint64_t max_tokens;   /* largest timestamp-pool span (tl_base[n-1] + n_deliv[n-1]) */
    uint32_t max_running;  /* largest number of running requests (<= 4096; 0 = 4096)    */
    int32_t device;        /* CUDA device ordinal                                       */
} AndesLimits;

/* Request table (the paper's Request Tracker state), structure of arrays,
 * length n.  Storing requests in rank order is recommended (coalesced tie scans). */
typedef struct {
    uint32_t n;
    const int64_t *arrival_us;    /* a_i: arrival time (absolute)                                   */
    const uint32_t *ttft_us;      /* TTFT target (reading R1: I_1 = a + ttft)                */
    const uint32_t *period_us;    /* P_i = 1/consumption speed, >= 1 (I_j = I_1+(j-1)P) */
    const uint32_t *ctx_len;      /* l_i = prompt + generated tokens, 1 <= l_i <= M (Eq. 5)  */
    const uint32_t *n_deliv;      /* g_i: tokens delivered so far                                    */
    const uint32_t *max_total;    /* total-token cap; UINT32_MAX = unknown (reading R7)      */
    const uint32_t *start_off_us; /* o_i: delay before the first new token if served; NULL = all 0
                                     (P:L355 excludes preemption overhead; reading R6)               */
    const uint32_t *rank;         /* unique tie-break; smaller = earlier arrival = wins (reading R10) */
    const uint8_t *running;       /* 1 if in the current batch                                       */
    const uint64_t *tl_base;      /* element offset of request i's timestamps in tl_pool; must be
                                     nondecreasing in i with tl_base[i+1] >= tl_base[i] + n_deliv[i] */
    const uint32_t *tl_pool;      /* delivery timestamps, us since arrival, nondecreasing per request,
                                     each <= now - arrival; 16-byte aligned                           */
    uint64_t tl_len;              /* number of uint32 elements readable at tl_pool; must be >=
                                     tl_base[n-1] + n_deliv[n-1] (the scan reads it through a TMA
                                     tensor map bounded by tl_len)                                    */
} AndesRequests;

/* andes_qoe_eval modes */
#define ANDES_EVAL_INFLIGHT 0u /* QoE at eval time t: tokens due by t, clamp at t (reading R3) */
#define ANDES_EVAL_FINAL 1u    /* whole delivered timeline, no clamp (reading R19)                     */

/* andes_schedule flags */
#define ANDES_FORCE 1u        /* run the solver even if the trigger does not fire            */
#define ANDES_PRUNE 2u        /* restrict B to [B_min, B_max]; default [1, B_max] */
#define ANDES_DEBUG_CHECKS 4u /* device-side data precondition checks                         */
#define ANDES_LQSF 16u        /* priority = the raw gain (Least QoE Slack First; reading
                                 R21) instead of gain / l (Eq. 6); everything else unchanged  */
/* Appendix-A objectives (readings R22-R23; single-GPU andes_schedule only): the
 * item value of request i becomes
 *   ANDES_OBJ_MAXMIN : max(Q_min - Q_wait,i, 0), Q_min = min over the requests of their QoE now
 *   ANDES_OBJ_PERFECT: [1(Q_serve,i = 1) - 1(Q_wait,i = 1)] * 1(Q_now,i = 1)
 * where Q_now,i is the in-flight QoE at now (R3).  The call then runs a second timeline scan
 * (eval = now) before the decision.  At most one of the two. */
#define ANDES_OBJ_MAXMIN 32u
#define ANDES_OBJ_PERFECT 64u
/* Overhead-aware refiner (readings R24-R27), applied after the preemption cap: the
 * admits (greedy order) are paired with the minimal prefix of the remaining victims that makes
 * room in M; a pair's stall is its victims' preemption costs plus the admit's resumption cost
 * (recompute = prefill of l at prefill_tok_s, swap = l / swap_tok_s each way, the faster round
 * trip); the pair is kept iff the admit's gain exceeds the QoE the still-running requests lose
 * under that stall (in 2^-32 units); the first rejected pair cancels itself and the rest
 * (ANDES_F_REFINED in the flags).  The identity when the running set alone exceeds M. */
#define ANDES_REFINE 128u

/* Decision-time parameters. */
typedef struct {
    int64_t now_us;          /* decision time                                                  */
    uint32_t horizon_us;     /* Delta t (reading R8), >= 1                             */
    uint32_t B_cap;          /* candidate batch sizes are 1..B_cap, 1 <= B_cap <= max_B         */
    const uint32_t *tau_us;  /* DEVICE u32[B_cap]: token latency tau(B) at index B-1 (App. B)   */
    uint64_t kv_capacity;    /* M: KV-cache capacity in tokens (Eq. 5)                          */
    uint32_t preempt_cap;    /* max preemptions per decision; UINT32_MAX = off (reading R18)    */
    uint32_t cur_latency_us; /* current iteration latency (trigger)                     */
    uint32_t flags;          /* ANDES_FORCE | ANDES_PRUNE | ANDES_DEBUG_CHECKS | ANDES_LQSF |
                                ANDES_OBJ_MAXMIN | ANDES_OBJ_PERFECT | ANDES_REFINE            */
    uint32_t prefill_tok_s;  /* refiner: prefill / recomputation throughput (tokens/s; 0 = free) */
    uint32_t swap_tok_s;     /* refiner: swap bandwidth (tokens/s; 0 = no swapping)             */
    const int64_t *now_dev;  /* i64[1] in DEVICE or mapped pinned HOST memory, optional (NULL:
                                now_us).  When set, the decision time is read (once, by the call's
                                first kernel) when the call runs, so one captured CUDA graph of a
                                serving iteration can be replayed at a new time every iteration
                                (write the time, replay).  andes_schedule only; ignored by
                                andes_schedule_host and the sharded decision.                    */
} AndesSchedParams;

/* scalars[] layout of AndesDecision */
#define ANDES_SC_B_STAR 0   /* chosen batch size B* (0 = empty decision / not triggered)   */
#define ANDES_SC_REALIZED 1 /* number of requests served after the cap                      */
#define ANDES_SC_N_ADMIT 2
#define ANDES_SC_N_PREEMPT 3
#define ANDES_SC_B_LO 4
#define ANDES_SC_B_HI 5
#define ANDES_SC_FLAGS 6  /* ANDES_F_* below                                                 */
#define ANDES_SC_K_STAR 7 /* Algorithm 1 prefix length at B* (before the cap)                */
#define ANDES_SC_COUNT 8
#define ANDES_F_TRIGGERED 1u
#define ANDES_F_CAP_HIT 2u
#define ANDES_F_CAP_OVERRIDDEN 4u
#define ANDES_F_SLOW_PATH 8u /* informational: a capacity fallback path ran */
#define ANDES_F_TRUNCATED 16u /* the running set exceeded the decision's capacity (4096): the victim
                                 list was truncated; the next call returns ANDES_E_CAPACITY        */
#define ANDES_F_REFINED 32u  /* the overhead-aware refiner rewrote the decision (ANDES_REFINE)   */

/* Decision outputs (DEVICE memory owned by the caller). */
typedef struct {
    uint8_t *serve_mask;   /* [n]  final serve set x (Alg. 1 output P:L512, after the cap)     */
    uint32_t *admit_idx;   /* [B_cap] admitted/resumed requests, greedy order                  */
    uint32_t *preempt_idx; /* [n]  preempted requests, victim order (reading R18)              */
    uint32_t *scalars;     /* [ANDES_SC_COUNT]                                                 */
    int64_t *V;            /* [B_cap] V(B) = sum of llrint(gain*2^32) over S_B; INT64_MIN if B
                              was not a candidate (reading R9)                                   */
    uint32_t *kstar;       /* [B_cap] Algorithm 1 prefix length per B; 0 if not a candidate    */
    /* Optional zero-copy export (andes_schedule): MAPPED pinned HOST memory (cudaHostAlloc; with
     * UVA every pinned allocation is mapped) that the call's last kernel fills with the decision's
     * head, so a serving loop reads it after a stream sync without a copy: scalars (32 B) at 0,
     * V (8 B_cap) at 32, admit_idx (4 B_cap) at 32 + 8 B_cap, the first min(n_preempt,
     * export_preempt) preempt_idx entries at 32 + 12 B_cap, then at 32 + 12 B_cap +
     * 4 export_preempt the next batch as an index list -- the requests served after the decision,
     * scalars[ANDES_SC_REALIZED] of them (kept running ones, then admits), at most export_served
     * -- which the engine runs and which can feed the next andes_tracker_append_dev directly
     * (idx = that list, count = the realized scalar), and last, 8-byte aligned after the list,
     * a completion word set to 1 behind a system-scope fence: a host that clears it before the
     * call may poll it instead of synchronising the stream.  NULL: no export. */
    void *export_host;
    uint32_t export_preempt;
    uint32_t export_served;
} AndesDecision;

/* QoE outputs of andes_qoe_eval (DEVICE memory; any pointer may be NULL). */
typedef struct {
    float *q;         /* [n] QoE (Eq. 3) rounded to fp32                        */
    double *q64;      /* [n] QoE in fp64 (1 - S_delay/S_whole, RN; R4: 1 if S_whole = 0) */
    int64_t *s_delay; /* [n] S_delay in us (Eq. 1), exact                        */
    int64_t *s_whole; /* [n] S_whole in us (Eq. 2), exact                        */
    uint32_t *m;      /* [n] number of tokens evaluated                           */
} AndesQoeOut;

/* Create/destroy a context on limits->device. Allocates the device workspace. */
int andes_create(AndesCtx **ctx, const AndesLimits *limits);
int andes_destroy(AndesCtx *ctx);

/* Human-readable description of the last error on ctx (never NULL). */
const char *andes_last_error(const AndesCtx *ctx);

/* S1: QoE of every request (Eq. 1-3).  INFLIGHT: at relative time
 * t_i = eval_time_us - a_i over the m_i = min(#{j: I_j <= t_i}, max_total) due
 * tokens, actual consumption clamped at t_i, undelivered due tokens at t_i
 * (readings R1-R5).  FINAL: over all n_deliv tokens without clamp (R19).
 * Errors: ANDES_E_INVAL (null req/out/arrays, mode), ANDES_E_CAPACITY (n or token
 * span above limits), ANDES_E_CUDA. */
int andes_qoe_eval(AndesCtx *ctx, const AndesRequests *req, int64_t eval_time_us, uint32_t mode,
                   const AndesQoeOut *out, void *stream);

/* Sweep of independent scenarios (BASELINE config 5; end-of-trace QoE): FINAL-mode QoE of
 * every request (m = g, no clamp; reading R19), then per scenario s the mean over its requests
 * with g >= 1, where scenario s holds requests [scen_off[s], scen_off[s+1]) (DEVICE u32[S+1],
 * nondecreasing, scen_off[S] <= n).  mean_out f64[S] (0 when no request has a token),
 * count_out u32[S] optional (requests averaged).  The mean is a fixed-order fp64 reduction
 * (deterministic; within 1e-12 relative of the exact mean of the per-request fp64 QoE).
 * Errors: ANDES_E_INVAL, ANDES_E_CAPACITY, ANDES_E_CUDA. */
int andes_qoe_scenario_mean(AndesCtx *ctx, const AndesRequests *req, const uint32_t *scen_off, uint32_t S,
                            double *mean_out, uint32_t *count_out, void *stream);

/* S3 materialised for an explicit list of B (parity and inspection):
 * gain_out f64[nB*n] = Q_serve,i(B) - Q_wait,i (Eq. 4), key_out f32[nB*n] =
 * float(gain / l_i) with -0 -> +0 (Eq. 6, reading R9); row b is B = B_list_host[b]
 * (HOST array, 1 <= B <= B_cap).  qwait_out f64[n] optional.  Q_serve uses one new
 * token every tau(B) starting at now + o_i (reading R6).  Either output may be NULL.
 * Errors: ANDES_E_INVAL, ANDES_E_CAPACITY (nB > max_B), ANDES_E_CUDA. */
int andes_gain_estimate(AndesCtx *ctx, const AndesRequests *req, int64_t now_us, uint32_t horizon_us,
                        const uint32_t *tau_us, uint32_t B_cap, const uint32_t *B_list_host, uint32_t nB,
                        double *gain_out, float *key_out, double *qwait_out, void *stream);

/* S0-S6: one full scheduling decision.  Asynchronous: the trigger outcome is
 * reported in scalars[ANDES_SC_FLAGS] & ANDES_F_TRIGGERED; when it does not fire
 * serve_mask = running and every other output is zero.  Errors: ANDES_E_INVAL,
 * ANDES_E_CAPACITY, ANDES_E_RANGE (previous call's debug check failed), ANDES_E_CUDA. */
int andes_schedule(AndesCtx *ctx, const AndesRequests *req, const AndesSchedParams *p, AndesDecision *out,
                   void *stream);

/* Same decision with every pointer in req, p->tau_us and out in HOST memory:
 * copies the inputs host->device into the context workspace, runs the decision,
 * copies the outputs back and synchronises `stream`.  Returns ANDES_NOT_TRIGGERED
 * when the trigger did not fire (outputs still written).  Requires the context
 * to have been created with max_tokens covering the pool. */
int andes_schedule_host(AndesCtx *ctx, const AndesRequests *req_host, const AndesSchedParams *p_host,
                        AndesDecision *out_host, void *stream);

/* ---- Request Tracker update ---------------------------------------------------
 * Device-resident tracker state: the mutable views of the AndesRequests arrays a serving loop
 * updates between decisions (DEVICE memory owned by the caller).  Each timeline must have room
 * to grow: request i may hold tl_base[i+1] - tl_base[i] tokens (the last one tl_len - tl_base).
 * Timelines should start 16-byte aligned (the scan's fast path); appending keeps them so. */
typedef struct {
    uint32_t n;
    const int64_t *arrival_us;
    const uint64_t *tl_base;
    uint32_t *tl_pool;
    uint64_t tl_len;
    uint32_t *n_deliv;
    uint32_t *ctx_len;
    uint8_t *running;
} AndesTracker;

/* One iteration's deliveries: token k (k < count) of request idx[k] reached its client at absolute
 * time t_abs[k]; idx/t_abs are DEVICE arrays in which a request's tokens are consecutive and in
 * time order.  Appends t_abs[k] - a_i to the request's timeline, n_deliv[i] += 1, ctx_len[i] += 1
 * (a generated token extends the context l_i of Eq. 5).  serve_mask (DEVICE u8[n], optional, e.g.
 * the decision's output) becomes the running set.  Asynchronous on stream, capture safe.  A token
 * without room in its timeline is dropped and the next call returns ANDES_E_CAPACITY.
 * Errors: ANDES_E_INVAL (NULL arrays). */
int andes_tracker_append(AndesCtx *ctx, const AndesTracker *t, const uint32_t *idx, const int64_t *t_abs,
                         uint32_t count, const uint8_t *serve_mask, void *stream);

/* The same update with the token count read on the device (*count_dev, DEVICE u32, at most
 * max_count; idx / t_abs hold max_count slots), so that a serving iteration -- the copy of its
 * deltas into idx / t_abs / count_dev, this update and andes_schedule -- can be captured once
 * into a CUDA graph and replayed with new deltas every iteration.  A count above max_count
 * appends none of the tokens and the next call returns ANDES_E_CAPACITY.
 * Errors: ANDES_E_INVAL (NULL arrays). */
int andes_tracker_append_dev(AndesCtx *ctx, const AndesTracker *t, const uint32_t *idx, const int64_t *t_abs,
                             const uint32_t *count_dev, uint32_t max_count, const uint8_t *serve_mask,
                             void *stream);

/* ---- Serving-loop simulator --------------------------------------
 * A trace is served iteration by iteration with andes_schedule in the loop, on the device:
 * at time now, the live requests (arrived, a_i <= now, and unfinished, g_i < out_i; rank = trace
 * index; running = served in the previous iteration; l_i = prompt_i + g_i; the output length is
 * unknown to the scheduler, max_total = UINT32_MAX, reading R7) are scheduled (S0-S6, forced);
 * every served request receives one token at now' = now + tau(min(realized, B_cap)) (at least
 * one; zero preemption overhead, as BASELINE config 1's driver), appended to its timeline; the
 * served set becomes the running set; now = now'.  With no live request the clock jumps to the
 * next arrival.  Runs until every request has its whole output or max_iters iterations.
 * The end-of-trace QoE (reading R19) is then andes_qoe_eval(FINAL) on the trace table.
 * All arrays DEVICE memory owned by the caller; the host loop reads a 32-byte control block once
 * per iteration (the call is synchronous on `stream`).  The context must hold n requests,
 * tl_len tokens and B_cap. */
typedef struct {
    uint32_t n;                    /* trace requests, arrival order (arrival_us nondecreasing)   */
    const int64_t *arrival_us;
    const uint32_t *ttft_us, *period_us;
    const uint32_t *prompt_len;    /* prompt tokens (context before the first output token)      */
    const uint32_t *output_len;    /* tokens the request will receive (>= 1)                     */
    const uint64_t *tl_base;       /* timeline offsets: room for output_len[i] tokens each,
                                      16-byte aligned starts recommended                          */
    uint32_t *tl_pool;             /* out: delivery times (us since arrival)                      */
    uint64_t tl_len;
    uint32_t *n_deliv;             /* out: tokens delivered (zeroed by the call)                  */
    uint8_t *served;               /* scratch [n]                                                 */
    void *workspace;               /* scratch of andes_sim_workspace(n) bytes, 16-byte aligned   */
} AndesSim;

typedef struct {
    const uint32_t *tau_us;  /* DEVICE u32[B_cap] */
    uint32_t B_cap;
    uint64_t kv_capacity;
    uint32_t horizon_us;
    uint32_t preempt_cap;
    uint32_t flags;          /* andes_schedule flags (ANDES_LQSF, objectives, ...); FORCE implied */
    uint32_t max_iters;
} AndesSimParams;

typedef struct {            /* HOST */
    uint64_t iterations;    /* decisions taken                                  */
    int64_t start_us, end_us;
    uint32_t finished;      /* requests that received their whole output        */
    uint32_t pad;
} AndesSimStats;

uint64_t andes_sim_workspace(uint32_t n);
/* Errors: ANDES_E_INVAL, ANDES_E_CAPACITY (n, tokens or B_cap above the context limits), any
 * error of andes_schedule, ANDES_E_CUDA. */
int andes_simulate(AndesCtx *ctx, const AndesSim *sim, const AndesSimParams *p, AndesSimStats *stats, void *stream);

/* ---- Multi-GPU decision ------------------------------------------
 * One process per GPU; rank g holds a contiguous range of the population (its requests have
 * global indices base_g .. base_g + n_g - 1, base_g = n_0 + ... + n_{g-1}; the rank fields must
 * be unique over all ranks).  The decision runs as ANDES_SHARD_STEPS asynchronous steps on the
 * caller's stream.  After step s (s = 0..3) the caller all-gathers every rank's send block of
 * xbytes[s] bytes, in rank order, into each rank's recv buffer of world * xbytes[s] bytes
 * (ncclAllGather / torch.distributed.all_gather_into_tensor on the same stream), and passes that
 * recv buffer to step s + 1:
 *   step 0: request prep + timeline scan (S1), round-0 block: trigger inputs, l histogram
 *   step 1: global trigger and B range (S0, S2), gain state and key bounds (S3), round-1 block:
 *           the rank's lower-bound key histogram
 *   step 2: global theta, survivors, exact keys at every B, round-2 block: per B the rank's
 *           top-min(B, survivors) in Algorithm 1's order
 *   step 3: merge of the ranks' lists, Algorithm 1's walk, V(B), B* (S4, S5), round-3 block:
 *           the rank's preemption victims at B*
 *   step 4: preemption cap (S6) and outputs.
 * Outputs: scalars, V, kstar are replicated (identical on every rank); admit_idx and
 * preempt_idx hold GLOBAL request indices (identical on every rank; preempt_idx must hold the
 * global victim count, at most 4096); serve_mask covers this rank's n requests.  The decision
 * equals andes_schedule on the concatenated population bit for bit (all payloads are integers).
 * Limits: world <= ANDES_MAX_WORLD, running requests per rank <= 2048 (else ANDES_E_CAPACITY on
 * the next call).  Send and recv buffers are DEVICE memory owned by the caller, 16-byte aligned. */
#define ANDES_SHARD_ROUNDS 4
#define ANDES_SHARD_STEPS 5
#define ANDES_MAX_WORLD 8
typedef struct {
    uint32_t world;                       /* number of ranks, 1..ANDES_MAX_WORLD             */
    uint32_t rank;                        /* this rank, < world                             */
    uint32_t B_cap;                       /* must equal AndesSchedParams.B_cap of the calls */
    uint32_t pad;
    uint64_t xbytes[ANDES_SHARD_ROUNDS];  /* send block bytes after step s                  */
} AndesShard;

/* Fills *out for (world, rank, B_cap).  Errors: ANDES_E_INVAL. */
int andes_shard_init(AndesCtx *ctx, uint32_t world, uint32_t rank, uint32_t B_cap, AndesShard *out);

/* One step (0..ANDES_SHARD_STEPS-1) of the sharded decision; `local` is this rank's request
 * table (DEVICE memory, as for andes_schedule).  recv: NULL for step 0, else the gathered blocks
 * of round step-1.  send: this rank's block of round `step` (steps 0..3; NULL for step 4).
 * Every step must be issued with the same req / params / out.  Errors: ANDES_E_INVAL,
 * ANDES_E_CAPACITY, ANDES_E_RANGE, ANDES_E_CUDA. */
int andes_schedule_shard(AndesCtx *ctx, const AndesShard *shard, uint32_t step, const AndesRequests *local,
                         const AndesSchedParams *p, AndesDecision *out, const void *recv, void *send,
                         void *stream);

/* ---- Peer-memory all-gather for the sharded decision (no NCCL) ---------------------------
 * The four exchanges of andes_schedule_shard as device collectives over CUDA IPC mappings: each
 * rank's arena (G flags, two parities of G slots of max_block bytes) lives in its own device
 * memory and is written by every peer directly (P2P stores over NVLink between the GPUs of a node;
 * on one GPU, processes sharing the device).  Setup: andes_comm_create returns this rank's IPC
 * handle (ANDES_COMM_HANDLE_BYTES); the caller exchanges the handles (any host channel, e.g.
 * torch.distributed.all_gather_object) and passes all of them, in rank order, to
 * andes_comm_connect.  andes_comm_allgather(send, recv, bytes): every rank's send block (DEVICE,
 * bytes <= max_block, a multiple of 16, the same bytes on every rank; send and recv 16-byte
 * aligned) into recv (DEVICE, world * bytes, rank order); two kernels on the stream (push +
 * publish, wait + pull), capture safe; all ranks must issue the same all-gathers in the same
 * order, and one communicator's all-gathers must be ordered on one stream.  A wait longer than 10 s for a peer is flagged and the next
 * call returns ANDES_E_NCCL.  Errors: ANDES_E_INVAL, ANDES_E_CUDA. */
#define ANDES_COMM_HANDLE_BYTES 64
typedef struct AndesComm AndesComm;
int andes_comm_create(AndesComm **out, int device, uint32_t world, uint32_t rank, uint64_t max_block,
                      void *handle_out);
int andes_comm_connect(AndesComm *comm, const void *handles);
int andes_comm_allgather(AndesComm *comm, const void *send, void *recv, uint64_t bytes, void *stream);
int andes_comm_destroy(AndesComm *comm);

/* ---- Exact reference solver (NEXT-4; Algorithm 2) --------------------------
 * The 3D dynamic program for Eq. 5 at target batch size B over n items with integer values
 * value[i] (e.g. llrint(gain_i 2^32), reading R9, so that the optimum is exact) and weights
 * weight[i] (context lengths l_i), capacity M: x[n] (u8) = Algorithm 2's solution (its line order:
 * "not served" then "served" on strict improvement, the first maximum of dp[N][B][:], the
 * backtracking), *best = its value (INT64_MIN when no B items fit), Vb[B+1] (optional) = the
 * best value for every b <= B (max over m of dp[N][b][:]).  O(n (B+1)(M+1)) work in one CTA:
 * meant for small instances (greedy-vs-exact quality checks), not for the decision path.
 * All pointers DEVICE memory; workspace (8-byte aligned) of andes_knapsack_dp_workspace(n, B, M)
 * bytes owned by the caller.  Asynchronous on stream.  Errors: ANDES_E_INVAL, ANDES_E_CAPACITY. */
uint64_t andes_knapsack_dp_workspace(uint32_t n, uint32_t B, uint64_t M);
int andes_knapsack_dp(AndesCtx *ctx, const int64_t *value, const uint32_t *weight, uint32_t n, uint32_t B,
                      uint64_t M, void *workspace, uint64_t workspace_bytes, uint8_t *x, int64_t *best,
                      int64_t *Vb, void *stream);

/* Per-stage timing.  When enabled, andes_schedule records a CUDA event before its first
 * and after each of its kernels on the call's stream (also under stream capture, so a
 * captured CUDA graph of a decision carries the event-record nodes).  andes_profile_read
 * blocks until the last recorded event completes and writes the elapsed milliseconds of
 * each stage.  andes_schedule: [0] reset + prep + trigger/B range (S0, S2), [1] timeline scan
 * (S1), [2] per-request state and key bounds (S3a), [3] candidate keys for every B (S3b),
 * [4] Algorithm 1 per B + best B + cap + serve mask (S4-S6), [5] unused (0).
 * andes_qoe_eval: [0] prep, [1] timeline scan, [2] QoE finalize, [3..5] unused.
 * Errors: ANDES_E_INVAL (profiling off / nothing recorded), ANDES_E_CUDA. */
#define ANDES_N_STAGES 6
int andes_profile_enable(AndesCtx *ctx, int enable);
int andes_profile_read(AndesCtx *ctx, float *stage_ms);

/* Library version string, e.g. "andes-b200 0.1 sm_100a". */
const char *andes_version(void);

#ifdef __cplusplus
}
#endif
#endif /* ANDES_H */
