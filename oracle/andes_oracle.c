/*
 * oracle/andes_oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * A plain, slow, literal CPU implementation of the Andes per-iteration
 * scheduling decision (arXiv 2404.16283).  Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference legs may load this library.
 * It shares no code, header, table or helper with the CUDA product path
 * (paper_2404_16283_b200/); it defines its own structs below.
 *
 * Build: gcc -O2 -ffp-contract=off -fno-fast-math -shared -fPIC
 *        (IEEE-754 binary64 round-to-nearest via SSE2, no contraction).
 *
 * Citations: P:Lnnn = /root/reference/PAPER.md line nnn (the paper);
 *            DESIGN.md "Readings" R1..R19 = how silent/ambiguous points are read.
 *
 * What each function follows
 *   due_count     O1  -- "QoE can be computed on requests in any state",
 *                        reading R3 (m = number of tokens due by t, capped by max_total).
 *   qoe_walk      O2  -- Eq. 1-3 walked token by token; ideal
 *                        timeline (reading R1), actual consumption
 *                        recurrence (reading R2), clamp at t (R3),
 *                        S_whole = 0 -> QoE 1 (R4).
 *   gain          O3-O5 -- Eq. 4 with Q_wait = no new tokens
 *                         and Q_serve(B) = one new token every tau(B)
 *                        (P:L391 footnote, App. B, reading R6);
 *                        priority Eq. 6.
 *   schedule      O6-O9 -- selective triggering (R15), batch-size
 *                        range (R16), Algorithm 1 step by step with
 *                        `break` (R10/R11), best B (R13),
 *                        preemption cap (reading R18; pairing after paper
 *                        section 4.3).
 *
 * Parity status: O2 is pinned by closed forms of Fig. 5 (tests/test_oracle_pins.py)
 * and worked examples; O7 by brute force and Algorithm 2; O9 "preemption cap" has
 * no paper text -- it is pinned only by DESIGN.md's definition (reading R18) and
 * the derived golden decision G1 (tests/golden/g1_decision.json).
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <math.h>
#include <pthread.h>

#define ORC_MAX_THREADS 256

#define ORC_OK 0
#define ORC_E_INVAL (-1)
#define ORC_E_NOMEM (-6)
#define ORC_NOT_TRIGGERED 1

#define ORC_FORCE 1u
#define ORC_PRUNE 2u
#define ORC_LQSF 16u /* priority = the raw gain (Least QoE Slack First; SPEC lqsf_policy) */
/* Appendix A objectives, readings R22-R23: the item value (gain) of request i is
 *   MAXMIN : max(Q_min - Q_wait,i, 0), Q_min = min over the live requests of their QoE now;
 *   PERFECT: [1(Q_serve,i = 1) - 1(Q_wait,i = 1)] * 1(Q_now,i = 1);
 * Q_now,i = the in-flight QoE at the decision time (O1-O2 with t = now - a_i, reading R3). */
#define ORC_MAXMIN 32u
#define ORC_PERFECT 64u
/* Overhead-aware refiner (readings R24-R27), applied to the decision after S6. */
#define ORC_REFINE 128u
#define ORC_FLAG_REFINED 32u

#define ORC_FLAG_TRIGGERED 1u
#define ORC_FLAG_CAP_HIT 2u
#define ORC_FLAG_CAP_OVERRIDDEN 4u

typedef struct {
    uint32_t n;
    const int64_t *arrival_us;    /* a_i, absolute microseconds */
    const uint32_t *ttft_us;      /* TTFT target */
    const uint32_t *period_us;    /* P_i = 1/speed in microseconds */
    const uint32_t *ctx_len;      /* l_i */
    const uint32_t *n_deliv;      /* g_i */
    const uint32_t *max_total;    /* cap on total tokens; UINT32_MAX = unknown */
    const uint32_t *start_off_us; /* o_i; NULL = all zero */
    const uint32_t *rank;         /* unique; smaller wins ties */
    const uint8_t *running;       /* 1 = in the current batch */
    const uint64_t *tl_base;      /* offset of request i's timestamps in tl_pool */
    const uint32_t *tl_pool;      /* delivery times, microseconds since arrival */
} orc_requests;

typedef struct {
    int64_t now_us;
    uint32_t horizon_us;     /* Delta t */
    const uint32_t *tau_us;  /* tau(B) for B = 1..B_cap at index B-1 */
    uint32_t B_cap;
    uint64_t kv_capacity;    /* M */
    uint32_t preempt_cap;    /* UINT32_MAX = off */
    uint32_t cur_latency_us; /* current iteration latency (trigger) */
    uint32_t flags;          /* ORC_FORCE | ORC_PRUNE | ORC_LQSF | ORC_MAXMIN | ORC_PERFECT | ORC_REFINE */
    uint32_t prefill_tok_s;  /* refiner: recomputation / prefill throughput, tokens per second */
    uint32_t swap_tok_s;     /* refiner: swap bandwidth, tokens per second (0 = no swapping) */
} orc_params;

typedef struct {
    uint8_t *serve_mask;   /* [n] final serve set */
    uint32_t *admit_idx;   /* [n] admitted requests, greedy order */
    uint32_t *preempt_idx; /* [n] preempted requests, victim order */
    uint32_t *scalars;     /* [8]: B_star, realized, n_admit, n_preempt, B_lo, B_hi, flags, k_star(B*) */
    int64_t *V;            /* [B_cap] objective V(B) in units of 2^-32; INT64_MIN if not evaluated */
    uint32_t *kstar;       /* [B_cap] Algorithm 1 prefix length per B; 0 if not evaluated */
} orc_decision;

/* ------------------------------------------------------------------ O1 */
/* Number of tokens due by relative time t (reading R3): token j is due when
 * its ideal time I_j = ttft + (j-1) P is <= t; capped by max_total (R7). */
static int64_t due_count(int64_t t, int64_t ttft, int64_t P, uint32_t max_total)
{
    int64_t m;
    if (t < ttft)
        m = 0;
    else
        m = (t - ttft) / P + 1; /* t - ttft >= 0: C division is floor here */
    if (m > (int64_t)max_total)
        m = (int64_t)max_total;
    return m;
}

/* ------------------------------------------------------------------ O2 */
/* Eq. 1-3 over the first m tokens of the delivery list D[0..n).
 *   I_j   = ttft + (j-1) P                                  (R1)
 *   A_1   = max(D_1, I_1);  A_j = max(D_j, A_{j-1} + P)      (R2)
 *   T~_j  = min(A_j, t) for delivered j; t for undelivered   (R3 clamp)
 *           (final_mode: T~_j = A_j, m = n, no clamp; R19)
 *   S_delay = sum_j (T~_j - I_j)                             (Eq. 1)
 *   S_whole = sum_j (T~_m - I_j)                             (Eq. 2)
 * T is caller scratch of length >= m. */
static void qoe_walk(const int64_t *D, int64_t n, int64_t ttft, int64_t P, int64_t t,
                     int64_t m, int final_mode, int64_t *T, int64_t *S_delay, int64_t *S_whole)
{
    int64_t j, A = 0, sd = 0, sw = 0;
    for (j = 1; j <= m; j++) {
        int64_t I = ttft + (j - 1) * P;
        if (j <= n) {
            int64_t d = D[j - 1];
            if (j == 1)
                A = d > I ? d : I;
            else
                A = d > A + P ? d : A + P;
            if (final_mode)
                T[j - 1] = A;
            else
                T[j - 1] = A < t ? A : t;
        } else {
            T[j - 1] = t;
        }
    }
    for (j = 1; j <= m; j++) {
        int64_t I = ttft + (j - 1) * P;
        sd += T[j - 1] - I;
        sw += T[m - 1] - I;
    }
    *S_delay = sd;
    *S_whole = sw;
}

/* Eq. 3; S_whole = 0 -> 1 (reading R4). */
static double qoe_value(int64_t S_delay, int64_t S_whole)
{
    if (S_whole == 0)
        return 1.0;
    return 1.0 - (double)S_delay / (double)S_whole;
}

int oracle_qoe_walk(const uint32_t *D_us, uint32_t n, int64_t ttft, int64_t P, int64_t t,
                    int64_t m, int final_mode, int64_t *S_delay, int64_t *S_whole, double *Q)
{
    int64_t *D, *T;
    int64_t j;
    if (P < 1 || m < 0)
        return ORC_E_INVAL;
    if (final_mode)
        m = n;
    D = (int64_t *)malloc(sizeof(int64_t) * (n + 1));
    T = (int64_t *)malloc(sizeof(int64_t) * (m + 1));
    if (!D || !T) {
        free(D);
        free(T);
        return ORC_E_NOMEM;
    }
    for (j = 0; j < n; j++)
        D[j] = D_us[j];
    qoe_walk(D, n, ttft, P, t, m, final_mode, T, S_delay, S_whole);
    *Q = qoe_value(*S_delay, *S_whole);
    free(D);
    free(T);
    return ORC_OK;
}

/* QoE of every request at absolute time eval_time_us (O1+O2), or of its whole
 * delivered timeline (final_mode, reading R19). Outputs may be NULL. */
/* O1+O2 for requests [lo, hi). */
static int qoe_eval_range(const orc_requests *r, uint32_t lo, uint32_t hi, int64_t eval_time_us, int final_mode,
                          double *q_out, int64_t *sd_out, int64_t *sw_out, uint32_t *m_out)
{
    uint32_t i;
    uint64_t maxg = 1;
    int64_t maxm = 1;
    int64_t *D, *T;
    for (i = lo; i < hi; i++) {
        int64_t t = eval_time_us - r->arrival_us[i];
        int64_t m = final_mode ? r->n_deliv[i] : due_count(t, r->ttft_us[i], r->period_us[i], r->max_total[i]);
        if (r->n_deliv[i] > maxg)
            maxg = r->n_deliv[i];
        if (m > maxm)
            maxm = m;
    }
    D = (int64_t *)malloc(sizeof(int64_t) * maxg);
    T = (int64_t *)malloc(sizeof(int64_t) * (size_t)maxm);
    if (!D || !T) {
        free(D);
        free(T);
        return ORC_E_NOMEM;
    }
    for (i = lo; i < hi; i++) {
        int64_t t = eval_time_us - r->arrival_us[i];
        int64_t g = r->n_deliv[i], j, sd, sw;
        int64_t m = final_mode ? g : due_count(t, r->ttft_us[i], r->period_us[i], r->max_total[i]);
        for (j = 0; j < g; j++)
            D[j] = r->tl_pool[r->tl_base[i] + (uint64_t)j];
        qoe_walk(D, g, r->ttft_us[i], r->period_us[i], t, m, final_mode, T, &sd, &sw);
        if (q_out)
            q_out[i] = qoe_value(sd, sw);
        if (sd_out)
            sd_out[i] = sd;
        if (sw_out)
            sw_out[i] = sw;
        if (m_out)
            m_out[i] = (uint32_t)m;
    }
    free(D);
    free(T);
    return ORC_OK;
}

typedef struct {
    const orc_requests *r;
    uint32_t lo, hi;
    int64_t eval_time_us;
    int final_mode, rc;
    double *q;
    int64_t *sd, *sw;
    uint32_t *m;
} qrange_t;

static void *qrange_worker(void *arg)
{
    qrange_t *a = (qrange_t *)arg;
    a->rc = qoe_eval_range(a->r, a->lo, a->hi, a->eval_time_us, a->final_mode, a->q, a->sd, a->sw, a->m);
    return NULL;
}

/* QoE of every request at absolute time eval_time_us (O1+O2), or of its whole delivered
 * timeline (final_mode, reading R19).  Outputs may be NULL.  The requests are independent;
 * nthreads > 1 splits them into contiguous ranges over threads (same per-request values). */
int oracle_qoe_eval_mt(const orc_requests *r, int64_t eval_time_us, int final_mode, double *q_out,
                       int64_t *sd_out, int64_t *sw_out, uint32_t *m_out, int nthreads)
{
    qrange_t a[ORC_MAX_THREADS];
    pthread_t th[ORC_MAX_THREADS];
    uint32_t i;
    int t, nt = nthreads < 1 ? 1 : (nthreads > ORC_MAX_THREADS ? ORC_MAX_THREADS : nthreads);
    for (i = 0; i < r->n; i++)
        if (r->period_us[i] < 1)
            return ORC_E_INVAL;
    if ((uint32_t)nt > r->n)
        nt = r->n ? (int)r->n : 1;
    for (t = 0; t < nt; t++) {
        a[t].r = r;
        a[t].lo = (uint32_t)((uint64_t)r->n * t / nt);
        a[t].hi = (uint32_t)((uint64_t)r->n * (t + 1) / nt);
        a[t].eval_time_us = eval_time_us;
        a[t].final_mode = final_mode;
        a[t].q = q_out;
        a[t].sd = sd_out;
        a[t].sw = sw_out;
        a[t].m = m_out;
        th[t] = 0;
        if (nt == 1 || pthread_create(&th[t], NULL, qrange_worker, &a[t]) != 0) {
            th[t] = 0;
            qrange_worker(&a[t]);
        }
    }
    for (t = 0; t < nt; t++)
        if (th[t])
            pthread_join(th[t], NULL);
    for (t = 0; t < nt; t++)
        if (a[t].rc != ORC_OK)
            return a[t].rc;
    return ORC_OK;
}

int oracle_qoe_eval(const orc_requests *r, int64_t eval_time_us, int final_mode,
                    double *q_out, int64_t *sd_out, int64_t *sw_out, uint32_t *m_out)
{
    return oracle_qoe_eval_mt(r, eval_time_us, final_mode, q_out, sd_out, sw_out, m_out, 1);
}

/* ------------------------------------------------------------------ O3-O5 */
typedef struct {
    int64_t *D; /* scratch deliveries */
    int64_t *T; /* scratch consumption times */
} scratch_t;

static int64_t request_due(const orc_requests *r, uint32_t i, int64_t now, uint32_t horizon)
{
    int64_t t = now + (int64_t)horizon - r->arrival_us[i];
    return due_count(t, r->ttft_us[i], r->period_us[i], r->max_total[i]);
}

/* Q_wait (O3): the real timeline only -- waiting "does not generate any tokens". */
static double q_wait(const orc_requests *r, uint32_t i, int64_t now, uint32_t horizon, scratch_t *s)
{
    int64_t t = now + (int64_t)horizon - r->arrival_us[i];
    int64_t m = request_due(r, i, now, horizon);
    int64_t g = r->n_deliv[i], j, sd, sw;
    for (j = 0; j < g; j++)
        s->D[j] = r->tl_pool[r->tl_base[i] + (uint64_t)j];
    qoe_walk(s->D, g, r->ttft_us[i], r->period_us[i], t, m, 0, s->T, &sd, &sw);
    return qoe_value(sd, sw);
}

/* Q_serve(B) (O4): the real timeline followed by hypothetical deliveries at
 * (now - a) + o + k * tau(B), k = 1..m-g (reading R6). */
static double q_serve(const orc_requests *r, uint32_t i, int64_t now, uint32_t horizon,
                      uint32_t tau_B, scratch_t *s)
{
    int64_t t = now + (int64_t)horizon - r->arrival_us[i];
    int64_t m = request_due(r, i, now, horizon);
    int64_t g = r->n_deliv[i], j, k, sd, sw, n;
    int64_t o = r->start_off_us ? r->start_off_us[i] : 0;
    for (j = 0; j < g; j++)
        s->D[j] = r->tl_pool[r->tl_base[i] + (uint64_t)j];
    n = g;
    for (k = 1; k <= m - g; k++)
        s->D[n++] = (now - r->arrival_us[i]) + o + k * (int64_t)tau_B;
    qoe_walk(s->D, n, r->ttft_us[i], r->period_us[i], t, m, 0, s->T, &sd, &sw);
    return qoe_value(sd, sw);
}

/* O5: gain = Q_serve - Q_wait (Eq. 4); priority = gain / l (Eq. 6);
 * key = float(priority), -0 canonicalised to +0 (reading R9);
 * objective units: llrint(gain * 2^32) (reading R9). */
static float priority_key(double gain, uint32_t l)
{
    double prio = gain / (double)l;
    float key = (float)prio;
    if (key == 0.0f)
        key = 0.0f;
    return key;
}

/* LQSF reading (R21): the same decision with the raw gain (Eq. 4) as the priority
 * instead of gain / l (Eq. 6): key = float(gain), -0 canonicalised to +0. */
static float lqsf_key(double gain)
{
    float key = (float)gain;
    if (key == 0.0f)
        key = 0.0f;
    return key;
}

static int64_t gain_fixed(double gain)
{
    return llrint(gain * 4294967296.0);
}

static int alloc_scratch(const orc_requests *r, int64_t now, uint32_t horizon, scratch_t *s)
{
    uint32_t i;
    int64_t need = 1;
    for (i = 0; i < r->n; i++) {
        int64_t m = request_due(r, i, now, horizon);
        int64_t g = r->n_deliv[i];
        int64_t len = g > m ? g : m;
        if (len > need)
            need = len;
    }
    s->D = (int64_t *)malloc(sizeof(int64_t) * (size_t)(need + 1));
    s->T = (int64_t *)malloc(sizeof(int64_t) * (size_t)(need + 1));
    if (!s->D || !s->T) {
        free(s->D);
        free(s->T);
        return ORC_E_NOMEM;
    }
    return ORC_OK;
}

/* Gains and keys for an explicit list of B (row b of the outputs = B_list[b]). */
typedef struct {
    const orc_requests *r;
    int64_t now;
    uint32_t horizon, lo, hi, nB;
    const uint32_t *tau_us, *B_list;
    double *gain_out, *qwait_out;
    float *key_out;
    int rc;
} grange_t;

/* Gains and keys of requests [lo, hi) (O3-O5). */
static void *grange_worker(void *arg)
{
    grange_t *a = (grange_t *)arg;
    const orc_requests *r = a->r;
    uint32_t i, b;
    scratch_t s;
    a->rc = ORC_OK;
    if (alloc_scratch(r, a->now, a->horizon, &s) != ORC_OK) {
        a->rc = ORC_E_NOMEM;
        return NULL;
    }
    for (i = a->lo; i < a->hi; i++) {
        double qw = q_wait(r, i, a->now, a->horizon, &s);
        if (a->qwait_out)
            a->qwait_out[i] = qw;
        for (b = 0; b < a->nB; b++) {
            double gain = q_serve(r, i, a->now, a->horizon, a->tau_us[a->B_list[b] - 1], &s) - qw;
            if (a->gain_out)
                a->gain_out[(size_t)b * r->n + i] = gain;
            if (a->key_out)
                a->key_out[(size_t)b * r->n + i] = priority_key(gain, r->ctx_len[i]);
        }
    }
    free(s.D);
    free(s.T);
    return NULL;
}

/* Gains and keys for an explicit list of B (row b of the outputs = B_list[b]).  The requests
 * are independent; nthreads > 1 splits them into contiguous ranges over threads. */
int oracle_gain_estimate_mt(const orc_requests *r, int64_t now, uint32_t horizon, const uint32_t *tau_us,
                            uint32_t B_cap, const uint32_t *B_list, uint32_t nB, double *gain_out,
                            float *key_out, double *qwait_out, int nthreads)
{
    grange_t a[ORC_MAX_THREADS];
    pthread_t th[ORC_MAX_THREADS];
    uint32_t b;
    int t, nt = nthreads < 1 ? 1 : (nthreads > ORC_MAX_THREADS ? ORC_MAX_THREADS : nthreads);
    for (b = 0; b < nB; b++)
        if (B_list[b] < 1 || B_list[b] > B_cap)
            return ORC_E_INVAL;
    if ((uint32_t)nt > r->n)
        nt = r->n ? (int)r->n : 1;
    for (t = 0; t < nt; t++) {
        a[t].r = r;
        a[t].now = now;
        a[t].horizon = horizon;
        a[t].lo = (uint32_t)((uint64_t)r->n * t / nt);
        a[t].hi = (uint32_t)((uint64_t)r->n * (t + 1) / nt);
        a[t].nB = nB;
        a[t].tau_us = tau_us;
        a[t].B_list = B_list;
        a[t].gain_out = gain_out;
        a[t].qwait_out = qwait_out;
        a[t].key_out = key_out;
        th[t] = 0;
        if (nt == 1 || pthread_create(&th[t], NULL, grange_worker, &a[t]) != 0) {
            th[t] = 0;
            grange_worker(&a[t]);
        }
    }
    for (t = 0; t < nt; t++)
        if (th[t])
            pthread_join(th[t], NULL);
    for (t = 0; t < nt; t++)
        if (a[t].rc != ORC_OK)
            return a[t].rc;
    return ORC_OK;
}

int oracle_gain_estimate(const orc_requests *r, int64_t now, uint32_t horizon, const uint32_t *tau_us,
                         uint32_t B_cap, const uint32_t *B_list, uint32_t nB, double *gain_out,
                         float *key_out, double *qwait_out)
{
    return oracle_gain_estimate_mt(r, now, horizon, tau_us, B_cap, B_list, nB, gain_out, key_out, qwait_out, 1);
}

/* ------------------------------------------------------------------ O6-O9 */
typedef struct {
    uint32_t idx;
    uint32_t rank;
    float key;
} item_t;

/* Greedy order: descending priority, ties to the smaller rank (reading R10). */
static int cmp_greedy(const void *pa, const void *pb)
{
    const item_t *a = (const item_t *)pa, *b = (const item_t *)pb;
    if (a->key > b->key)
        return -1;
    if (a->key < b->key)
        return 1;
    if (a->rank < b->rank)
        return -1;
    if (a->rank > b->rank)
        return 1;
    return 0;
}

/* Victim order: the exact reverse of the greedy order (reading R18). */
static int cmp_victim(const void *pa, const void *pb)
{
    return -cmp_greedy(pa, pb);
}

static int cmp_u32(const void *pa, const void *pb)
{
    uint32_t a = *(const uint32_t *)pa, b = *(const uint32_t *)pb;
    return a < b ? -1 : (a > b ? 1 : 0);
}

/* ------------------------------------------------------------------ refiner (NEXT-1) */
/* R24 overhead model (SPEC preemption_overhead / select_mechanism), integer us:
 *   recompute: preempt 0, resume l * 1e6 / prefill_tok_s (one prefill of the context);
 *   swap     : preempt = resume = l * 1e6 / swap_tok_s;
 * the mechanism with the smaller round trip, ties to swap.  A queued request's admission costs
 * its prefill (recompute resume). */
static void overhead_us(const orc_params *p, uint32_t l, int queued, int64_t *pre, int64_t *res)
{
    int64_t rc = p->prefill_tok_s ? (int64_t)l * 1000000 / p->prefill_tok_s : 0;
    int64_t sw = p->swap_tok_s ? (int64_t)l * 1000000 / p->swap_tok_s : -1;
    if (queued || sw < 0 || rc < 2 * sw) {
        *pre = 0;
        *res = rc;
    } else {
        *pre = sw;
        *res = sw;
    }
}

/* The R24 overhead model itself, exported for the pins (SPEC preemption_overhead /
 * select_mechanism examples): *pre / *res in microseconds. */
int oracle_overhead_us(uint32_t prefill_tok_s, uint32_t swap_tok_s, uint32_t l, int queued, int64_t *pre, int64_t *res)
{
    orc_params p;
    memset(&p, 0, sizeof p);
    p.prefill_tok_s = prefill_tok_s;
    p.swap_tok_s = swap_tok_s;
    overhead_us(&p, l, queued, pre, res);
    return ORC_OK;
}

/* R25-R27: walk the admits (greedy order); each takes the minimal prefix of the remaining
 * victims (victim order) that makes room in M; its stall D = the victims' preempt costs + its
 * own resume cost; loss = sum over the requests still running after the pair of
 * llrint((Q_now - Q(now + D)) 2^32), Q(now + D) = the in-flight QoE at now + D with no new
 * token (Q_wait with Delta t = D); keep the pair iff llrint(gain 2^32) > loss; the first
 * rejected pair cancels it and every later one.  Identity when the running set alone exceeds M. */
static int refine(const orc_requests *r, const orc_params *p, const double *gain, orc_decision *out)
{
    scratch_t sc = {NULL, NULL}, *s = &sc;
    int64_t Dmax = 0, c_pre, c_res;
    uint32_t n = r->n, i, k, n_adm = out->scalars[2], n_pre = out->scalars[3];
    uint32_t *adm = NULL, *pre = NULL, vp = 0, na = 0, nv = 0;
    uint8_t *kept = NULL;
    double *qnow = NULL;
    uint64_t W = 0, M = p->kv_capacity;
    int rc = ORC_OK;
    for (i = 0; i < n; i++)
        if (r->running[i])
            W += r->ctx_len[i];
    if (W > M)
        return ORC_OK;
    adm = (uint32_t *)malloc(sizeof(uint32_t) * (n_adm + 1));
    pre = (uint32_t *)malloc(sizeof(uint32_t) * (n_pre + 1));
    kept = (uint8_t *)calloc(n ? n : 1, 1);
    qnow = (double *)malloc(sizeof(double) * (n ? n : 1));
    if (!adm || !pre || !kept || !qnow) {
        rc = ORC_E_NOMEM;
        goto out;
    }
    memcpy(adm, out->admit_idx, sizeof(uint32_t) * n_adm);
    memcpy(pre, out->preempt_idx, sizeof(uint32_t) * n_pre);
    /* every pair's stall is at most the sum of all the costs: scratch for that horizon */
    for (k = 0; k < n_adm; k++) {
        overhead_us(p, r->ctx_len[adm[k]], r->n_deliv[adm[k]] == 0, &c_pre, &c_res);
        Dmax += c_res;
    }
    for (k = 0; k < n_pre; k++) {
        overhead_us(p, r->ctx_len[pre[k]], 0, &c_pre, &c_res);
        Dmax += c_pre;
    }
    if (Dmax > 0xFFFFFFFFll || alloc_scratch(r, p->now_us, (uint32_t)Dmax, s) != ORC_OK) {
        rc = Dmax > 0xFFFFFFFFll ? ORC_E_INVAL : ORC_E_NOMEM;
        goto out;
    }
    for (i = 0; i < n; i++) {
        kept[i] = r->running[i];
        if (kept[i])
            qnow[i] = q_wait(r, i, p->now_us, 0, s);
    }
    for (k = 0; k < n_adm; k++) {
        uint32_t a = adm[k], v0 = vp, v;
        uint64_t Wk = W;
        int64_t D, c_pre, c_res, loss = 0;
        while (Wk + r->ctx_len[a] > M && vp < n_pre)
            Wk -= r->ctx_len[pre[vp++]];
        if (Wk + r->ctx_len[a] > M) /* no room even with every remaining victim */
            break;
        overhead_us(p, r->ctx_len[a], r->n_deliv[a] == 0, &c_pre, &c_res);
        D = c_res;
        for (v = v0; v < vp; v++) {
            overhead_us(p, r->ctx_len[pre[v]], 0, &c_pre, &c_res);
            D += c_pre;
            kept[pre[v]] = 0;
        }
        for (i = 0; i < n; i++)
            if (kept[i])
                loss += gain_fixed(qnow[i] - q_wait(r, i, p->now_us, (uint32_t)D, s));
        if (gain_fixed(gain[a]) > loss) {
            W = Wk + r->ctx_len[a];
            na = k + 1;
            nv = vp;
        } else {
            for (v = v0; v < vp; v++)
                kept[pre[v]] = 1;
            break;
        }
    }
    /* outputs: accepted admits and victims; everything else stays as the status quo */
    for (i = 0; i < n; i++)
        out->serve_mask[i] = r->running[i] ? 1 : 0;
    for (k = 0; k < nv; k++) {
        out->serve_mask[pre[k]] = 0;
        out->preempt_idx[k] = pre[k];
    }
    for (k = 0; k < na; k++) {
        out->serve_mask[adm[k]] = 1;
        out->admit_idx[k] = adm[k];
    }
    {
        uint32_t realized = 0;
        for (i = 0; i < n; i++)
            realized += out->serve_mask[i];
        out->scalars[1] = realized;
    }
    out->scalars[2] = na;
    out->scalars[3] = nv;
    out->scalars[6] |= ORC_FLAG_REFINED;
out:
    free(adm);
    free(pre);
    free(kept);
    free(qnow);
    free(sc.D);
    free(sc.T);
    return rc;
}


/* S3 + S4 at one candidate B: every request's gain (O4/O5 or the objective's item value,
 * readings R21-R23), its priority key, the full comparison sort in greedy order (R10) and
 * Algorithm 1's walk with `break` (R11).  items[] / gain[] receive the sorted order
 * and the gains; *V_out = sum of llrint(gain 2^32) over S_B, *c_out = |S_B|. */
static void per_B(const orc_requests *r, const orc_params *p, uint32_t B, const double *qw,
                  const double *qnow, double qmin, scratch_t *s, item_t *items, double *gain,
                  int64_t *V_out, uint32_t *c_out)
{
    uint32_t n = r->n, i, k, c = 0;
    uint64_t W = 0, M = p->kv_capacity;
    int64_t V = 0;
    for (i = 0; i < n; i++) {
        if (p->flags & ORC_MAXMIN) {
            double v = qmin - qw[i];
            gain[i] = v > 0.0 ? v : 0.0;
        } else if (p->flags & ORC_PERFECT) {
            double qs = q_serve(r, i, p->now_us, p->horizon_us, p->tau_us[B - 1], s);
            gain[i] = ((qs == 1.0 ? 1.0 : 0.0) - (qw[i] == 1.0 ? 1.0 : 0.0)) * (qnow[i] == 1.0 ? 1.0 : 0.0);
        } else {
            gain[i] = q_serve(r, i, p->now_us, p->horizon_us, p->tau_us[B - 1], s) - qw[i];
        }
        items[i].idx = i;
        items[i].rank = r->rank[i];
        items[i].key = (p->flags & ORC_LQSF) ? lqsf_key(gain[i]) : priority_key(gain[i], r->ctx_len[i]);
    }
    qsort(items, n, sizeof(item_t), cmp_greedy);
    /* Algorithm 1: take while within M and B, else break. */
    for (k = 0; k < n; k++) {
        uint32_t l = r->ctx_len[items[k].idx];
        if (W + l <= M && c + 1 <= B) {
            W += l;
            c += 1;
            V += gain_fixed(gain[items[k].idx]);
        } else {
            break;
        }
    }
    *V_out = V;
    *c_out = c;
}

typedef struct {
    const orc_requests *r;
    const orc_params *p;
    const double *qw, *qnow;
    double qmin;
    orc_decision *out;
    uint32_t B_lo, B_hi, stride, first;
    int rc;
} bloop_t;

/* One worker: B = B_lo + first, + stride, ... (its own scratch; writes only V[B-1], kstar[B-1]). */
static void *bloop_worker(void *arg)
{
    bloop_t *a = (bloop_t *)arg;
    uint32_t n = a->r->n, B;
    scratch_t s = {NULL, NULL};
    item_t *items = (item_t *)malloc(sizeof(item_t) * n);
    double *gain = (double *)malloc(sizeof(double) * n);
    a->rc = ORC_OK;
    if (!items || !gain || alloc_scratch(a->r, a->p->now_us, a->p->horizon_us, &s) != ORC_OK) {
        a->rc = ORC_E_NOMEM;
    } else {
        for (B = a->B_lo + a->first; B <= a->B_hi; B += a->stride) {
            int64_t V;
            uint32_t c;
            per_B(a->r, a->p, B, a->qw, a->qnow, a->qmin, &s, items, gain, &V, &c);
            a->out->V[B - 1] = V;
            a->out->kstar[B - 1] = c;
        }
    }
    free(items);
    free(gain);
    free(s.D);
    free(s.T);
    return NULL;
}

static int run_B_loop(const orc_requests *r, const orc_params *p, uint32_t B_lo, uint32_t B_hi,
                      const double *qw, const double *qnow, double qmin, orc_decision *out, int nthreads)
{
    bloop_t a[ORC_MAX_THREADS];
    pthread_t th[ORC_MAX_THREADS];
    int t, nt = nthreads < 1 ? 1 : (nthreads > ORC_MAX_THREADS ? ORC_MAX_THREADS : nthreads);
    if ((uint32_t)nt > B_hi - B_lo + 1)
        nt = (int)(B_hi - B_lo + 1);
    for (t = 0; t < nt; t++) {
        a[t].r = r;
        a[t].p = p;
        a[t].qw = qw;
        a[t].qnow = qnow;
        a[t].qmin = qmin;
        a[t].out = out;
        a[t].B_lo = B_lo;
        a[t].B_hi = B_hi;
        a[t].stride = (uint32_t)nt;
        a[t].first = (uint32_t)t;
    }
    if (nt == 1) {
        bloop_worker(&a[0]);
        return a[0].rc;
    }
    for (t = 0; t < nt; t++)
        if (pthread_create(&th[t], NULL, bloop_worker, &a[t]) != 0) {
            a[t].rc = ORC_E_NOMEM;
            bloop_worker(&a[t]); /* run it here instead */
            th[t] = 0;
        }
    for (t = 0; t < nt; t++)
        if (th[t])
            pthread_join(th[t], NULL);
    for (t = 0; t < nt; t++)
        if (a[t].rc != ORC_OK)
            return a[t].rc;
    return ORC_OK;
}

int oracle_schedule_mt(const orc_requests *r, const orc_params *p, orc_decision *out, int nthreads);

int oracle_schedule(const orc_requests *r, const orc_params *p, orc_decision *out)
{
    return oracle_schedule_mt(r, p, out, 1);
}

/* The decision (O6-O9).  nthreads > 1 splits the independent per-B walks over threads. */
int oracle_schedule_mt(const orc_requests *r, const orc_params *p, orc_decision *out, int nthreads)
{
    uint32_t n = r->n, i, B, k;
    uint64_t run_l = 0, M = p->kv_capacity;
    uint32_t minP = UINT32_MAX;
    int triggered;
    uint32_t B_lo, B_hi, k_M, B_star = 0, best_k = 0;
    int64_t best_V = INT64_MIN;
    item_t *best_items = NULL, *vict = NULL;
    uint32_t *sorted_l = NULL;
    double *qw = NULL, *best_gain = NULL, *qnow = NULL, qmin = 1.0;
    uint8_t *in_S = NULL;
    scratch_t s = {NULL, NULL};
    int rc = ORC_OK;

    if (p->B_cap < 1 || M < 1 || !p->tau_us)
        return ORC_E_INVAL;
    memset(out->scalars, 0, sizeof(uint32_t) * 8);
    for (B = 1; B <= p->B_cap; B++) {
        out->V[B - 1] = INT64_MIN;
        out->kstar[B - 1] = 0;
    }
    for (i = 0; i < n; i++) {
        if (r->period_us[i] < 1 || r->ctx_len[i] < 1 || r->ctx_len[i] > M)
            return ORC_E_INVAL;
        if (r->running[i])
            run_l += r->ctx_len[i];
        if (r->period_us[i] < minP)
            minP = r->period_us[i];
    }

    /* S0 selective triggering (reading R15): occupancy strictly above
     * 90% (10*W > 9*M), or iteration latency above the most stringent reader's
     * period, or forced. */
    triggered = (p->flags & ORC_FORCE) != 0 || 10 * run_l > 9 * M || (n > 0 && p->cur_latency_us > minP);
    if (!triggered) {
        uint32_t c = 0;
        for (i = 0; i < n; i++) {
            out->serve_mask[i] = r->running[i] ? 1 : 0;
            c += out->serve_mask[i];
        }
        out->scalars[1] = c;
        return ORC_NOT_TRIGGERED;
    }
    out->scalars[6] = ORC_FLAG_TRIGGERED;
    for (i = 0; i < n; i++)
        out->serve_mask[i] = 0;
    if (n == 0)
        return ORC_OK;

    /* S2 batch-size range (readings R16/R17). B_max: add the shortest
     * contexts until M is reached. */
    sorted_l = (uint32_t *)malloc(sizeof(uint32_t) * n);
    best_items = (item_t *)malloc(sizeof(item_t) * n);
    vict = (item_t *)malloc(sizeof(item_t) * n);
    qw = (double *)malloc(sizeof(double) * n);
    best_gain = (double *)malloc(sizeof(double) * n);
    in_S = (uint8_t *)calloc(n, 1);
    if (!sorted_l || !best_items || !vict || !qw || !best_gain || !in_S) {
        rc = ORC_E_NOMEM;
        goto done;
    }
    memcpy(sorted_l, r->ctx_len, sizeof(uint32_t) * n);
    qsort(sorted_l, n, sizeof(uint32_t), cmp_u32);
    {
        uint64_t W = 0;
        k_M = 0;
        for (i = 0; i < n; i++) {
            if (W + sorted_l[i] > M)
                break;
            W += sorted_l[i];
            k_M++;
        }
    }
    B_hi = p->B_cap;
    if (n < B_hi)
        B_hi = n;
    if (k_M < B_hi)
        B_hi = k_M;
    B_lo = 1;
    if (p->flags & ORC_PRUNE) {
        /* B_min: the largest B whose tau(B) keeps pace with the most stringent
         * reader (non-strict, reading R16); 1 if none; capped at B_hi. */
        for (B = 1; B <= B_hi; B++)
            if (p->tau_us[B - 1] <= minP)
                B_lo = B;
    }
    out->scalars[4] = B_lo;
    out->scalars[5] = B_hi;
    if (B_hi == 0)
        goto done;

    if (alloc_scratch(r, p->now_us, p->horizon_us, &s) != ORC_OK) {
        rc = ORC_E_NOMEM;
        goto done;
    }
    for (i = 0; i < n; i++)
        qw[i] = q_wait(r, i, p->now_us, p->horizon_us, &s);
    if (p->flags & (ORC_MAXMIN | ORC_PERFECT)) {
        qnow = (double *)malloc(sizeof(double) * (n ? n : 1));
        if (!qnow) {
            rc = ORC_E_NOMEM;
            goto done;
        }
        for (i = 0; i < n; i++) {
            qnow[i] = q_wait(r, i, p->now_us, 0, &s); /* Q at t = now - a_i (no new token) */
            if (i == 0 || qnow[i] < qmin)
                qmin = qnow[i];
        }
    }

    /* S3/S4 for every candidate B: gains, priorities, Algorithm 1 (per_B below).  The B
     * values are independent; with nthreads > 1 they are split over threads (SURVEY.md 8(d)(ii):
     * the integer outputs V(B), k*(B) do not depend on the split). */
    if (run_B_loop(r, p, B_lo, B_hi, qw, qnow, qmin, out, nthreads) != ORC_OK) {
        rc = ORC_E_NOMEM;
        goto done;
    }
    /* S5 best B; ties go to the larger B (reading R13): B ascends, so >=. */
    for (B = B_lo; B <= B_hi; B++)
        if (out->V[B - 1] >= best_V) {
            best_V = out->V[B - 1];
            B_star = B;
        }
    /* S_{B*}: the greedy order and gains at B* (the same per_B walk, recomputed once) */
    {
        int64_t Vb;
        uint32_t cb;
        per_B(r, p, B_star, qw, qnow, qmin, &s, best_items, best_gain, &Vb, &cb);
        best_k = cb;
    }
    out->scalars[0] = B_star;
    out->scalars[7] = best_k;

    /* S6 preemption cap (reading R18, after the refiner's pairing P:L576-581). */
    {
        uint32_t n_vict = 0, n_adm = 0, n_pre = 0, c0 = 0, kk;
        uint64_t W0 = 0;
        uint32_t cap = p->preempt_cap;
        for (k = 0; k < best_k; k++)
            in_S[best_items[k].idx] = 1;
        for (k = 0; k < n; k++) { /* victims R \ S, in victim order */
            uint32_t idx = best_items[k].idx;
            if (r->running[idx] && !in_S[idx])
                vict[n_vict++] = best_items[k];
        }
        qsort(vict, n_vict, sizeof(item_t), cmp_victim);
        if (cap == UINT32_MAX || n_vict <= cap) {
            for (k = 0; k < best_k; k++) { /* admits S \ R in greedy order */
                uint32_t idx = best_items[k].idx;
                out->serve_mask[idx] = 1;
                if (!r->running[idx])
                    out->admit_idx[n_adm++] = idx;
            }
            for (k = 0; k < n_vict; k++)
                out->preempt_idx[n_pre++] = vict[k].idx;
        } else {
            out->scalars[6] |= ORC_FLAG_CAP_HIT;
            for (i = 0; i < n; i++)
                out->serve_mask[i] = r->running[i] ? 1 : 0;
            for (k = 0; k < cap; k++) {
                out->serve_mask[vict[k].idx] = 0;
                out->preempt_idx[n_pre++] = vict[k].idx;
            }
            for (i = 0; i < n; i++)
                if (out->serve_mask[i]) {
                    W0 += r->ctx_len[i];
                    c0 += 1;
                }
            if (W0 > M) {
                /* memory beats the cap: keep preempting in victim order */
                out->scalars[6] |= ORC_FLAG_CAP_OVERRIDDEN;
                for (kk = cap; kk < n_vict && W0 > M; kk++) {
                    out->serve_mask[vict[kk].idx] = 0;
                    out->preempt_idx[n_pre++] = vict[kk].idx;
                    W0 -= r->ctx_len[vict[kk].idx];
                    c0 -= 1;
                }
            } else {
                for (k = 0; k < best_k; k++) { /* admit in greedy order, break at first misfit */
                    uint32_t idx = best_items[k].idx;
                    uint32_t l = r->ctx_len[idx];
                    if (r->running[idx])
                        continue;
                    if (W0 + l <= M && c0 + 1 <= B_star) {
                        out->serve_mask[idx] = 1;
                        out->admit_idx[n_adm++] = idx;
                        W0 += l;
                        c0 += 1;
                    } else {
                        break;
                    }
                }
            }
        }
        {
            uint32_t realized = 0;
            for (i = 0; i < n; i++)
                realized += out->serve_mask[i];
            out->scalars[1] = realized;
        }
        out->scalars[2] = n_adm;
        out->scalars[3] = n_pre;
    }
    if ((p->flags & ORC_REFINE) && B_star)
        rc = refine(r, p, best_gain, out);

done:
    free(sorted_l);
    free(best_items);
    free(vict);
    free(qw);
    free(qnow);
    free(best_gain);
    free(in_S);
    free(s.D);
    free(s.T);
    return rc;
}
