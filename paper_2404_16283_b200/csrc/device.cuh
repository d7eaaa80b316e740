// device.cuh -- internal device-side definitions of libandes (sm_100a).
//
// Everything here is product code; it shares nothing with oracle/.
// Notation follows PAPER.md section 3.1 / 4.1 and DESIGN.md "Closed forms":
//   I_j  = ttft + (j-1) P                        ideal consumption time (reading R1)
//   lat_j = d_j - I_j,  delta_j = max(0, max_{k<=j} lat_k)   actual-minus-ideal (R2)
//   delta~_j = min(delta_j, t - I_j)             clamped at the evaluation time (R3)
//   S_delay = sum_j delta~_j,  S_whole = m delta~_m + P m(m-1)/2     (Eq. 1-2)
#pragma once
#include <cstdint>
#include <cuda.h>
#include <cuda_runtime.h>

namespace andes {

// ---------------------------------------------------------------- constants
constexpr int kScanThreads = 128;                 // 4 independent warps per CTA
constexpr int kScanItems = 32;                    // one 128-byte row of the pool per lane
constexpr int kWTile = 32 * kScanItems;           // tokens per warp-tile (4 KiB, one TMA box)
constexpr int kTile = kWTile;                     // tiling unit of tile_meta / tile_status
constexpr int kWWinCap = 32;                      // window entries (+ sentinel) per warp
constexpr int kOvfCap = 128;                      // the CTA's shared overflow window (dense tiles)
constexpr int kCarryDirect = 4096;                // head segments up to this long: carry read directly
constexpr int kWarpSmem = 2 * kWTile * 4;               // double-buffered warp-tile
constexpr int kScanDynSmem = (kScanThreads / 32) * kWarpSmem + 1024;  // + 1 KiB alignment slack (swizzle)
constexpr int kSelectThreads = 1024;
constexpr int kMaxB = 1024;
constexpr int kMaxRunning = 4096;
constexpr int kStageRun = kMaxRunning / 2;        // running requests handled by the per-B cap staging
constexpr uint32_t kHistL = 4096;                 // exact histogram of l < 4095 (+ overflow bucket)
constexpr uint32_t kHistK = 4096;                 // key histograms: top 12 bits of the ordered key
constexpr uint32_t kCandCap = 2559;               // survivor capacity of the pruned path (k_select scratch)
constexpr uint32_t kRunOrdAt = 3584;              // k_select scratch: running order / prefix sums (512 slots)

// tile status words (decoupled look-back), see k_qoe_scan
constexpr unsigned long long kStAgg = 1ull << 62;
constexpr unsigned long long kStPrefix = 2ull << 62;
constexpr unsigned long long kStMask = 3ull << 62;
constexpr unsigned long long kFlagBit = 1ull << 32;

// device error word bits.  Data preconditions (set only under ANDES_DEBUG_CHECKS): period,
// context length, tl_base order, timestamps, rank uniqueness, tokens due; capacity (always):
// running set above the workspace limits, timestamp pool above limits.max_tokens.
constexpr uint32_t kErrPeriod = 1u, kErrCtx = 2u, kErrBase = 4u, kErrTimes = 8u, kErrRank = 16u,
                   kErrRunning = 32u, kErrDue = 64u, kErrTokens = 128u;
constexpr uint32_t kErrCapacity = kErrRunning | kErrTokens;

// ---------------------------------------------------------------- views
struct ReqView {
  uint32_t n;
  const int64_t* __restrict__ arrival;
  const uint32_t* __restrict__ ttft;
  const uint32_t* __restrict__ period;
  const uint32_t* __restrict__ ctx_len;
  const uint32_t* __restrict__ n_deliv;
  const uint32_t* __restrict__ max_total;
  const uint32_t* __restrict__ start_off;  // may be null
  const uint32_t* __restrict__ rank;
  const uint8_t* __restrict__ running;
  const uint64_t* __restrict__ tl_base;
  const uint32_t* __restrict__ tl_pool;
  uint64_t tl_len;  // readable elements at tl_pool
};

// Mutable view of the tracker arrays (andes_tracker_append).
struct TrackerView {
  uint32_t n;
  const int64_t* arrival;
  const uint64_t* tl_base;
  uint32_t* tl_pool;
  uint64_t tl_len;
  uint32_t* n_deliv;
  uint32_t* ctx_len;
  uint8_t* running;
};

// Serving-loop simulator (sim.cu): the control block read by the host once per iteration, and
// the trace + live-table view.
struct SimCtl {
  int64_t now;           // the iteration's time (after k_sim_step: the next one)
  int64_t next_arrival;  // first request not yet arrived (INT64_MAX if none)
  uint32_t n_live;       // live requests (k_sim_live)
  uint32_t finished;     // arrived requests that have received their whole output
  uint32_t pad[2];
};
struct SimView {
  uint32_t n;
  const int64_t* arrival;
  const uint32_t *ttft, *period, *prompt, *out_len;
  const uint64_t* tl_base;
  uint32_t* tl_pool;
  uint64_t tl_len;
  uint32_t* g;
  uint8_t* served;
  // live table (k_sim_live), in trace order
  int64_t* l_arr;
  uint32_t *l_ttft, *l_period, *l_ctx, *l_g, *l_rank, *l_idx, *l_maxtot;
  uint8_t* l_run;
  uint64_t* l_base;
  SimCtl* ctl;
};

// Per-tile descriptor of the timeline scan (written by prep): the request owning the tile's
// first position and the source of its head-segment carry.
struct alignas(16) TileMeta {
  unsigned long long hbase;  // tl_base of r0
  uint32_t r0;               // last request with tl_base <= tile start
  uint32_t flags;            // bit 0: gap before r0 (dummy window entry); bits 1-2: carry mode
  uint32_t hcnt;             // tokens of r0 before the tile (direct carry)
  uint32_t httft, hP, pad;
};

// Per-request record of the timeline scan (written by prep).
struct alignas(16) ScanRec {
  unsigned long long base;  // tl_base
  uint32_t lim;             // tokens to scan: min(g, m) (FINAL: g)
  uint32_t P, ttft;
  uint32_t trel;            // evaluation time - arrival (FINAL: unused)
  uint32_t ek;              // edge kind of the last valid token: 1 delta_g (g < m), 2 delta~_m
  uint32_t pad;
};

// Small per-call globals (zeroed by one memset node per call).
struct Globals {
  unsigned long long run_l;      // sum of l over running requests
  unsigned long long pool_end;   // tl_base[n-1] + n_deliv[n-1]
  uint32_t ntiles;               // scan tiles
  uint32_t inv_minP;             // UINT32_MAX - min_i P_i (atomicMax)
  uint32_t n_run;                // running requests appended to run_list
  uint32_t done;                 // select CTAs finished (last-block pattern)
  uint32_t B_lo, B_hi;           // candidate range
  uint32_t triggered;
  uint32_t err;                  // this call's error bits (kErr*); also raised to Work::err_map
  uint32_t slow;                 // slow-path flags
  uint32_t tile_ctr;             // dynamic tile counter of the timeline scan
  uint32_t prep_done;            // prep CTAs finished (last-block pattern)
  uint32_t run_ctr;              // k_state: running requests appended to run_st / run_idx
  uint32_t tau_lo, tau_hi;       // min / max tau(B) over the candidate range
  uint32_t theta;                // ordered-key threshold: >= B_hi requests have LB >= theta
  uint32_t n_surv;               // requests with UB >= theta (candidates)
  uint32_t overflow;             // n_surv above the candidate capacity: full-N fallback
  uint32_t cand_ctr;             // candidate slot counter
  // multi-GPU decision (shard.cu); run_l / inv_minP hold the global values after step 1
  uint32_t shard_base;           // global index of this rank's first request
  uint32_t n_global;             // requests over all ranks
  uint32_t n_run_global;         // running requests over all ranks
  uint32_t shard_Bstar;          // B* (step 3 -> step 4)
  uint32_t unal;                 // prep: some timeline does not start on a 16-byte boundary
  uint32_t sel_ready;            // k_select, B-independent keys: B_hi's sorted list is published
  unsigned long long qmin_bits;  // max-min objective: ~(fp64 bits of min_i Q_now,i) (Q >= 0: the bit
                                 // patterns are ordered; inverted so that the zeroed word is "none")
  uint32_t rf_npairs;            // refiner: feasible admit/victim pairs
  uint32_t max_rank;             // prep (decisions): max_i rank_i (the exact-zero rank histogram's scale)
};

static_assert(sizeof(Globals) == 128, "Globals: one 128-byte line, one warp snapshot");

// Second line of the per-call globals (zeroed with them): grid-barrier words of the fused
// decision kernel and the counters of a call's second timeline scan.
struct Globals2 {
  uint32_t arrive_a, ready_a, arrive_b, ready_b;  // k_decide grid barriers
  uint32_t theta, zcut, n_surv, overflow;         // k_decide: survivor cut published at barrier A
  uint32_t tile_ctr_b;                            // the decision scan's chunk counter after a scan at now
  uint32_t qnow_ctr;                              // Q_now chunks claimed by the decision scan's idle warps
  uint32_t rf_done;                               // refiner: k_refine_loss CTAs finished (last block)
  uint32_t pad0;
  unsigned long long best_vb;                     // S5: max over B of pack_vb(V(B), B) (select CTAs)
  long long tshift;                               // *now_dev - now_ref, read once by prep (now_dev calls)
  uint32_t pad[16];
};
static_assert(sizeof(Globals2) == 128, "Globals2: one 128-byte line");

// S5 (ties to the larger B, reading R13) as one 64-bit atomicMax: V(B) (|V| < 2^43: a sum
// of at most 1024 values llrint(gain 2^32) with |gain| <= 1) offset to be positive, then B in the
// low 11 bits, so the larger packed value is the larger V, or on equal V the larger B; 0 = none.
__host__ __device__ __forceinline__ unsigned long long pack_vb(long long V, uint32_t B) {
  return ((unsigned long long)(V + (1ll << 43)) << 11) | (unsigned long long)B;
}

// Block snapshot of the Globals line: warp 0 loads it (one request per CTA) and the block reads
// shared memory.  Every thread of a many-CTA grid loading the same global words instead queues
// on one L2 slice; in k_select that skewed the CTA starts by 6 us.  Ends with __syncthreads().
__device__ __forceinline__ void snap_globals(const Globals* g, Globals* s) {
  if (threadIdx.x < 32)
    reinterpret_cast<uint32_t*>(s)[threadIdx.x] = __ldcg(reinterpret_cast<const uint32_t*>(g) + threadIdx.x);
  __syncthreads();
}

// B-independent per-request state for the gain closed form,
// written once per decision by k_state and read by the candidate / select / cap kernels.
struct alignas(16) PackedState {
  long long w0, c0, spre, cw, dto;
  double qw;
  uint32_t m, K, P, h0, l, rank;
  double qx;  // objective scalar: max-min -> its (B-independent) gain; perfect-count -> Q_now
};
static_assert(sizeof(PackedState) == 80, "PackedState layout");

// objectives (include/andes.h ANDES_OBJ_*): 0 = Andes (Eq. 4), 1 = max-min, 2 = perfect count
constexpr uint32_t kObjAndes = 0, kObjMaxMin = 1, kObjPerfect = 2;

// ---------------------------------------------------------------- multi-GPU exchange blocks
// Round 0: one rank's trigger / batch-size-range inputs.
struct ShardSummary {
  uint32_t n, n_run, minP, has_ovf;  // has_ovf: ovf[] holds this rank's smallest long contexts
  unsigned long long run_l;
  uint32_t pad[2];
  uint32_t hist[kHistL];             // l histogram (last bin: l >= kHistL - 1)
  uint32_t ovf[kMaxB];               // smallest l >= kHistL - 1, ascending, UINT32_MAX padded
};
// Round 2: one entry of a rank's local top-B list of candidate B (Algorithm 1's order).
struct alignas(8) XEntry {
  unsigned long long comp;  // composite (key desc, rank asc); 0 = padding
  long long gfix;           // llrint(gain 2^32)
  uint32_t l;               // context length
  uint32_t gidx;            // global request index | 0x80000000 if running
};
static_assert(sizeof(XEntry) == 24, "XEntry layout");
// Round 3: one rank's preemption victims at B* (running requests outside S_{B*}).
struct VictimX {
  unsigned long long comp;
  uint32_t l, gidx;
};
struct ShardVictims {
  uint32_t count, pad[3];
  VictimX v[kStageRun];
};
__host__ __device__ __forceinline__ size_t tri_off(uint32_t B) { return (size_t)B * (B - 1) / 2; }

struct Work;
__host__ __device__ inline Globals2* globals2(const Work& w);

struct Work {
  uint32_t* m;               // [N] tokens due at the evaluation time
  unsigned long long* spre;  // [N] sum of clamped delays of delivered due tokens
  uint32_t* edge;            // [N] delta_g (g < m) or delta~_m (g >= m)
  TileMeta* tile_meta;       // [tiles] per-tile descriptor
  unsigned long long* tile_status;  // [tiles]
  unsigned long long* tile_status_now;  // [tiles] look-back status of the objectives' scan at now
  uint32_t* hist_l;          // [kHistL] histogram of min(l, kHistL-1) (self-cleaning)
  uint32_t* hist_lb;         // [kHistK] histogram of lower-bound keys (self-cleaning)
  uint32_t* hist_ub;         // [kHistK] histogram of upper-bound keys (self-cleaning)
  uint32_t* run_list;        // [max_running]
  ScanRec* srec;             // [N] timeline-scan records
  PackedState* st;           // [N]
  uint32_t* ub;              // [N] ordered upper-bound key over the candidate B range
  uint32_t* zr;              // [N] rank bucket of a request whose key is exactly 0 for every B, else ~0
  uint32_t* hist_zr;         // [kHistK] histogram of zr (self-cleaning)
  uint32_t* cand_idx;        // [S_cap] request index of candidate slot (bit 31: running)
  PackedState* cand_st;      // [S_cap] the survivors' states, contiguous (one load in k_select)
  PackedState* run_st;       // [kMaxRunning] the running requests' states (k_state, any order)
  uint32_t* run_idx;         // [kMaxRunning] their request indices
  uint32_t* keyrow;          // [max_B][N] fallback: ordered keys of every request per B
  uint32_t* sel;             // [max_B][kMaxB] Algorithm 1 prefix per B, greedy order
  unsigned long long* sel_thr;  // [max_B] composite of the k*-th selected request per B
  uint32_t* stage_pre;       // [max_B][kStageRun] preempt list per candidate B (cap applied)
  uint32_t* stage_adm;       // [max_B][kMaxB] admit list per candidate B
  uint4* stage_sc;           // [max_B] {n_pre, n_adm, realized, flags} per candidate B
  XEntry* xm;                // [tri(max_B + 1)] merged Algorithm 1 prefixes per B (multi-GPU)
  Globals* g;
  unsigned long long* trace; // optional %globaltimer stamps (internal debugging), may be null
  uint32_t N_cap;            // row stride of keyrow
  uint32_t tiles_cap;        // capacity of tile_owner / tile_status
  uint32_t S_cap;            // survivor capacity of cand_idx
  uint32_t lqsf;             // this call's priority: 0 gain / l (Eq. 6), 1 raw gain (ANDES_LQSF)
  uint32_t obj;              // this call's objective (kObj*)
  uint32_t lb_ns;            // look-back wait bound (ns) before the direct head read (ANDES_LOOKBACK_NS)
  // objectives that need the QoE now (Appendix A): the decision-time scan's outputs
  uint32_t* m_now;           // [N]
  unsigned long long* spre_now;  // [N]
  uint32_t* edge_now;        // [N]
  ScanRec* srec_now;         // [N]
  double* qnow;              // [N] QoE at the decision time
  // overhead-aware refiner (refine.cu)
  uint32_t* vmark;           // [N] 1 + victim position of a preempted request, else 0
  uint32_t* rf_vend;         // [kMaxB] victims consumed after pair k
  long long* rf_D;           // [kMaxB] stall of pair k (us)
  long long* rf_loss;        // [kMaxB] QoE loss of pair k in units of 2^-32
  // error reporting: mapped pinned host word (the context's sticky error word, read and cleared
  // by the host at the start of the next call; no copy node, no synchronisation)
  uint32_t* err_map;
  // debug checks: open-addressing set of ranks (2 N_cap slots, self-cleaning), rank uniqueness
  unsigned long long* rank_set;
  // decision time read on the device (AndesSchedParams.now_dev): every time argument of the
  // call's kernels (passed for now_ref) is shifted by *now_dev - now_ref; NULL: no shift
  const long long* now_dev;
  long long now_ref;
};


__host__ __device__ inline Globals2* globals2(const Work& w) { return reinterpret_cast<Globals2*>(w.g + 1); }
// the shift k_reset_now published (every kernel of a now_dev call)
__device__ __forceinline__ long long tshift(const Work& w) { return w.now_dev ? __ldcg(&globals2(w)->tshift) : 0ll; }

// ---------------------------------------------------------------- error reporting
// Raise error bits: into this call's Globals word (read by the decision's own kernels, e.g. the
// ANDES_F_TRUNCATED flag) and into the mapped host word the next call reports.  Error paths only.
__device__ __forceinline__ void raise_err(const Work& w, uint32_t bits) {
  atomicOr(&w.g->err, bits);
  if (w.err_map) {
    volatile uint32_t* h = w.err_map;
    *h = *h | bits;
  }
}

// ---------------------------------------------------------------- small helpers
__host__ __device__ __forceinline__ uint32_t umin32(uint32_t a, uint32_t b) { return a < b ? a : b; }
__device__ __forceinline__ uint32_t ordered_key(float f) {
  // monotone map float -> u32 (larger float -> larger u32); -0 is canonicalised earlier
  uint32_t u = __float_as_uint(f);
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
__device__ __forceinline__ float key_from_ordered(uint32_t u) {
  return __uint_as_float((u & 0x80000000u) ? (u & 0x7fffffffu) : ~u);
}
// composite sort key: descending priority, then ascending rank (reading R10)
__device__ __forceinline__ unsigned long long composite(uint32_t okey, uint32_t rank) {
  return ((unsigned long long)okey << 32) | (unsigned long long)(0xFFFFFFFFu - rank);
}

// due tokens at relative time t (reading R3): 0 if t < ttft, else floor((t - ttft)/P) + 1,
// capped by max_total (reading R7).
__device__ __forceinline__ uint32_t due_count(int64_t t, uint32_t ttft, uint32_t P, uint32_t max_total) {
  if (t < (int64_t)ttft) return 0;
  const unsigned long long d = (unsigned long long)(t - (int64_t)ttft);
  // 32-bit division when the span fits (always, for times below 2^32 us): the 64-bit one is a
  // called subroutine
  unsigned long long q = ((d >> 32) == 0ull ? (unsigned long long)((uint32_t)d / P) : d / P) + 1ull;
  if (q > max_total) q = max_total;
  return (uint32_t)q;
}

// clamp(floor(num/div), 0, cap) for div > 0, cap < 2^20, exact.
// fp32 quotient estimate (abs error < 0.25 on quotients < 2^20) + one integer fix-up.
__device__ __forceinline__ int64_t qdiv_clamped(int64_t num, int64_t div, int64_t cap) {
  if (num <= 0) return 0;
  if (num >= cap * div) return cap;
  float qf = floorf(__fdividef((float)num, (float)div));
  int64_t q = (int64_t)qf;
  int64_t r = num - q * div;
  if (r < 0) q -= 1;
  else if (r >= div) q += 1;
  return q;
}

// sum_{k=a+1..b} (w0 - k P)
__device__ __forceinline__ int64_t sum_down(int64_t a, int64_t b, int64_t w0, int64_t P) {
  int64_t c = b - a;
  return c * w0 - P * ((c * (a + b + 1)) >> 1);
}
// sum_{k=a+1..b} (c0 + k e)
__device__ __forceinline__ int64_t sum_up(int64_t a, int64_t b, int64_t c0, int64_t e) {
  int64_t c = b - a;
  return c * c0 + e * ((c * (a + b + 1)) >> 1);
}

// Eq. 3 with reading R4, IEEE binary64 round-to-nearest, no contraction.
__device__ __forceinline__ double qoe_value(int64_t sd, int64_t sw) {
  if (sw == 0) return 1.0;
  return __dsub_rn(1.0, __ddiv_rn(__ll2double_rn(sd), __ll2double_rn(sw)));
}

// ---------------------------------------------------------------- per-request gain state
// B-independent part of Q_wait / Q_serve(B) for one request.
struct GainState {
  int64_t w0;      // t - ttft - (g-1) P      : t - I_{g+k} = w0 - k P
  int64_t c0;      // (now-a) + o - ttft - (g-1) P : lateness of new token k = c0 + k e
  int64_t spre;    // sum_{j<=min(g,m)} delta~_j
  int64_t cw;      // P m (m-1) / 2
  int64_t dto;     // Delta t - o  (= w0 - c0)
  uint32_t m, K;   // due tokens, undelivered due tokens (K = m - g if m > g else 0)
  uint32_t P;
  uint32_t h0;     // delta_g (0 if g == 0)
  double qw;       // Q_wait (Eq. 3 on the real timeline)
};

__device__ __forceinline__ GainState make_state(const ReqView& r, const Work& w, uint32_t i, int64_t now,
                                                uint32_t horizon) {
  GainState s;
  const int64_t a = r.arrival[i];
  const int64_t t = now + (int64_t)horizon - a;
  const uint32_t g = r.n_deliv[i];
  const uint32_t m = w.m[i];
  const uint32_t P = r.period[i];
  const int64_t ttft = r.ttft[i];
  const int64_t o = r.start_off ? (int64_t)r.start_off[i] : 0;
  s.m = m;
  s.P = P;
  s.spre = (int64_t)w.spre[i];
  s.cw = (int64_t)P * (((int64_t)m * ((int64_t)m - 1)) >> 1);
  s.w0 = t - ttft - ((int64_t)g - 1) * (int64_t)P;
  s.c0 = (now - a) + o - ttft - ((int64_t)g - 1) * (int64_t)P;
  s.dto = (int64_t)horizon - o;
  if (m == 0) {
    s.K = 0;
    s.h0 = 0;
    s.qw = 1.0;
  } else if (g >= m) {
    s.K = 0;
    s.h0 = 0;
    const int64_t dm = (int64_t)w.edge[i];
    s.qw = qoe_value(s.spre, (int64_t)m * dm + s.cw);
  } else {
    s.K = m - g;
    s.h0 = (g == 0) ? 0u : w.edge[i];
    const int64_t K = s.K;
    const int64_t sd = s.spre + sum_down(0, K, s.w0, P);
    const int64_t dm = s.w0 - K * (int64_t)P;  // = t - I_m
    s.qw = qoe_value(sd, (int64_t)m * dm + s.cw);
  }
  return s;
}

__device__ __forceinline__ GainState unpack_state(const PackedState& p) {
  GainState s;
  s.w0 = p.w0; s.c0 = p.c0; s.spre = p.spre; s.cw = p.cw; s.dto = p.dto;
  s.m = p.m; s.K = p.K; s.P = p.P; s.h0 = p.h0; s.qw = p.qw;
  return s;
}

// Q_serve(B) for tau = tau(B) (requires s.K >= 1): new token k delivered at
// (now - a) + o + k tau, i.e. lateness c0 + k e with e = tau - P.
__device__ __forceinline__ void serve_area(const GainState& s, uint32_t tau, int64_t& sd, int64_t& sw) {
  const int64_t K = s.K, P = s.P, w0 = s.w0, c0 = s.c0, h0 = s.h0;
  const int64_t e = (int64_t)tau - P;
  int64_t sum, dm;
  if (e < 0) {
    // delta_{g+k} = h = max(h0, c0 + e) for every k >= 1
    const int64_t h = max(h0, c0 + e);
    const int64_t ks = qdiv_clamped(w0 - h, P, K);
    sum = h * ks + sum_down(ks, K, w0, P);
    dm = min(h, w0 - K * P);
  } else {
    const int64_t kx = min(qdiv_clamped(w0 - h0, P, K), qdiv_clamped(s.dto, (int64_t)tau, K));
    int64_t nflat;
    if (e == 0)
      nflat = (c0 <= h0) ? kx : 0;
    else
      nflat = qdiv_clamped(h0 - c0, e, kx);
    sum = h0 * nflat + sum_up(nflat, kx, c0, e) + sum_down(kx, K, w0, P);
    dm = min(max(h0, c0 + K * e), w0 - K * P);
  }
  sd = s.spre + sum;
  sw = (int64_t)s.m * dm + s.cw;
}

// gain = Q_serve(B) - Q_wait (Eq. 4); 0 exactly when no undelivered token is due.
__device__ __forceinline__ double gain_at(const GainState& s, uint32_t tau) {
  if (s.K == 0) return 0.0;
  int64_t sd, sw;
  serve_area(s, tau, sd, sw);
  return __dsub_rn(qoe_value(sd, sw), s.qw);
}

// Q_serve(tau) == 1 exactly (S_delay = 0; Eq. 3): for the perfect-count objective
__device__ __forceinline__ bool serve_perfect(const GainState& s, uint32_t tau) {
  if (s.K == 0) return s.qw == 1.0;
  int64_t sd, sw;
  serve_area(s, tau, sd, sw);
  return qoe_value(sd, sw) == 1.0;
}

// the item value (knapsack gain) of the call's objective at tau(B) (Appendix A, P:L1160-1177;
// readings R22-R23): Andes Q_serve - Q_wait (Eq. 4); max-min max(Q_min - Q_wait, 0) (stored in
// qx); perfect count [1(Q_serve = 1) - 1(Q_wait = 1)] * 1(Q_now = 1) (Q_now stored in qx)
__device__ __forceinline__ double gain_obj(const GainState& s, double qx, uint32_t tau, uint32_t obj) {
  if (obj == kObjMaxMin) return qx;
  if (obj == kObjPerfect) {
    if (qx != 1.0) return 0.0;
    return (serve_perfect(s, tau) ? 1.0 : 0.0) - (s.qw == 1.0 ? 1.0 : 0.0);
  }
  return gain_at(s, tau);
}

// priority key (Eq. 6, reading R9): float(gain / l), -0 -> +0; with the LQSF objective (reading
// R21) the raw gain (Eq. 4) is the priority: float(gain)
__device__ __forceinline__ float prio_key(double gain, uint32_t l, uint32_t lqsf = 0u) {
  float k = lqsf ? __double2float_rn(gain) : __double2float_rn(__ddiv_rn(gain, (double)l));
  return (__float_as_uint(k) << 1) == 0u ? 0.0f : k;
}

__device__ __forceinline__ long long gain_fixed(double gain) {
  return __double2ll_rn(__dmul_rn(gain, 4294967296.0));
}

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
#define ANDES_TRACE(w, slot)                                  \
  do {                                                        \
    if ((w).trace && threadIdx.x == 0) (w).trace[(slot)] = gtimer(); \
  } while (0)

// ---------------------------------------------------------------- sync primitives
__device__ __forceinline__ unsigned long long ld_acquire(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
// Self-contained status words (flag + value in one 64-bit word): relaxed strong accesses suffice,
// no fence is needed because nothing else is published through them.
__device__ __forceinline__ unsigned long long ld_relaxed(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_relaxed(unsigned long long* p, unsigned long long v) {
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// Programmatic dependent launch (every decision kernel is launched with
// cudaLaunchAttributeProgrammaticStreamSerialization): a kernel lets its stream successor start
// launching early, and waits for its predecessor's completion (and memory) before reading it.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

}  // namespace andes
