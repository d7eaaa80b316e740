// select.cu -- S3-S6 of the decision: gains for every candidate B (Eq. 4/6), Algorithm 1 per B,
// best B, preemption cap (reading R18), serve-mask materialisation.
//
// Exact selection with bound-and-prune:
//   k_state   per request: the B-independent state, and rigorous lower/upper bounds of its
//             priority key over every candidate B.  S_delay and S_whole of Q_serve are
//             nondecreasing in tau (deliveries only move later), and every rounded operation of
//             the key (RN division, RN subtraction, RN64->RN32) is monotone, so evaluating the
//             same fp chain at (S_delay(tau_lo), S_whole(tau_hi)) / (S_delay(tau_hi),
//             S_whole(tau_lo)) bounds the computed key of every B with tau in [tau_lo, tau_hi].
//             Histograms of the bounds follow.
//   k_compact theta from the lower-bound histogram: >= B_max requests have key >= theta at every
//             B, so the exact top-B of every B lies among the requests whose upper bound is
//             >= theta ("survivors"); compacts them.
//   k_select  one CTA per B: exact keys of the survivors at B, their order by rank counting
//             (key desc, rank asc), Algorithm 1 walk, V(B), and B's preemption-cap
//             result staged; the last CTA picks B* and writes the outputs.
// If the survivors exceed the capacity, k_select evaluates every request at its B and
// radix-selects instead (slow path, flagged).
#include "block.cuh"
#include "device.cuh"
#include "launch.h"

#include <cstdlib>

namespace andes {

// ---------------------------------------------------------------- gain_estimate (parity API)
__global__ void k_gain_estimate(ReqView r, Work w, int64_t now, uint32_t horizon, const uint32_t* __restrict__ tau,
                                const uint32_t* __restrict__ B_list, uint32_t nB, double* gain_out, float* key_out,
                                double* qwait_out) {
  pdl_wait();
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < r.n; i += gridDim.x * blockDim.x) {
    const GainState s = make_state(r, w, i, now, horizon);
    const uint32_t l = r.ctx_len[i];
    if (qwait_out) qwait_out[i] = s.qw;
    for (uint32_t b = 0; b < nB; ++b) {
      const double gn = gain_at(s, tau[B_list[b] - 1]);
      if (gain_out) gain_out[(size_t)b * r.n + i] = gn;
      if (key_out) key_out[(size_t)b * r.n + i] = prio_key(gn, l);
    }
  }
}

// ---------------------------------------------------------------- S3a: state + key bounds
constexpr int kStateThreads = 256;
constexpr int kCandThreads = 256;

// ordered key of a zero priority, and the shift that maps ranks to the 4096 buckets of hist_zr
constexpr uint32_t kOKey0 = 0x80000000u;  // ordered_key(+0.0f)
__device__ __forceinline__ uint32_t zr_shift(uint32_t max_rank) {
  const uint32_t bits = 32u - __clz(max_rank | 1u);
  return bits > 12u ? bits - 12u : 0u;
}

// Per request: the B-independent state (k_state's output array st), the running requests'
// contiguous copy, rigorous key bounds over the candidate tau range and the CTA's bound
// histograms (s_hlb / s_hub: kHistK words each in shared memory), flushed to the global ones.
// CTA `cta` of `ncta` handles requests cta*NT + tid, + ncta*NT, ...
template <int NT>
__device__ void state_phase(const ReqView& r, const Work& w, int64_t now, uint32_t horizon, const Globals& sg,
                            uint32_t* s_hlb, uint32_t* s_hub, uint32_t cta, uint32_t ncta) {
  const uint32_t tid = threadIdx.x;
  const uint32_t tlo = sg.tau_lo, thi = sg.tau_hi;
  const uint32_t zs = zr_shift(sg.max_rank);
  for (uint32_t q = tid; q < kHistK; q += NT) {
    s_hlb[q] = 0u;
    s_hub[q] = 0u;
  }
  __syncthreads();
  for (uint32_t i = cta * NT + tid; i < r.n; i += ncta * NT) {
    const GainState s = make_state(r, w, i, now, horizon);
    PackedState p;
    p.w0 = s.w0; p.c0 = s.c0; p.spre = s.spre; p.cw = s.cw; p.dto = s.dto; p.qw = s.qw;
    p.m = s.m; p.K = s.K; p.P = s.P; p.h0 = s.h0; p.l = r.ctx_len[i]; p.rank = r.rank[i];
    p.qx = 0.0;
    if (w.obj == kObjMaxMin) {
      const double qmin = __longlong_as_double((long long)~__ldcg(&w.g->qmin_bits));  // stored inverted
      const double v = __dsub_rn(qmin, s.qw);
      p.qx = v > 0.0 ? v : 0.0;
    } else if (w.obj == kObjPerfect) {
      p.qx = w.qnow[i];
    }
    w.st[i] = p;
    if (r.running[i]) {  // a contiguous copy for k_select's cap staging (order irrelevant)
      const uint32_t slot = atomicAdd(&w.g->run_ctr, 1u);
      if (slot < (uint32_t)kMaxRunning) {
        w.run_st[slot] = p;
        w.run_idx[slot] = i;
      }
    }
    uint32_t lb, ub;
    if (w.obj != kObjAndes) {
      // max-min: one gain for every B; perfect count: 1(Q_serve = 1) is nonincreasing in tau
      lb = ordered_key(prio_key(gain_obj(s, p.qx, thi, w.obj), p.l, w.lqsf));
      ub = ordered_key(prio_key(gain_obj(s, p.qx, tlo, w.obj), p.l, w.lqsf));
    } else if (s.K == 0) {
      lb = ub = ordered_key(0.0f);  // gain exactly 0 for every B
    } else {
      int64_t sd_lo, sw_lo, sd_hi, sw_hi;
      serve_area(s, tlo, sd_lo, sw_lo);
      serve_area(s, thi, sd_hi, sw_hi);
      const double q_ub = qoe_value(sd_lo, sw_hi);
      const double q_lb = (sw_lo == 0) ? 0.0 : qoe_value(sd_hi, sw_lo);
      ub = ordered_key(prio_key(__dsub_rn(q_ub, s.qw), p.l, w.lqsf));
      lb = ordered_key(prio_key(__dsub_rn(q_lb, s.qw), p.l, w.lqsf));
    }
    w.ub[i] = ub;
    // a key exactly 0 at every B of the range (reading R10: ties by rank): only the B_hi smallest
    // ranks of these can ever be selected, so the compaction may prune the rest (rank histogram)
    const bool zero = lb == kOKey0 && ub == kOKey0;
    const uint32_t zb = zero ? p.rank >> zs : 0xFFFFFFFFu;
    w.zr[i] = zb;
    if (zero) atomicAdd(&w.hist_zr[zb], 1u);
    atomicAdd(&s_hlb[lb >> 20], 1u);
    atomicAdd(&s_hub[ub >> 20], 1u);
  }
  __syncthreads();
  for (uint32_t q = tid; q < kHistK; q += NT) {
    if (s_hlb[q]) atomicAdd(&w.hist_lb[q], s_hlb[q]);
    if (s_hub[q]) atomicAdd(&w.hist_ub[q], s_hub[q]);
  }
}

__global__ void __launch_bounds__(kStateThreads) k_state(ReqView r, Work w, int64_t now, uint32_t horizon) {
  __shared__ uint32_t s_hlb[kHistK], s_hub[kHistK];
  __shared__ Globals s_g;
  pdl_wait();
  snap_globals(w.g, &s_g);
  if (!s_g.triggered || s_g.B_hi == 0) return;
  if (blockIdx.x < 512) ANDES_TRACE(w, 3000 + 2 * blockIdx.x);
  state_phase<kStateThreads>(r, w, now + tshift(w), horizon, s_g, s_hlb, s_hub, blockIdx.x, gridDim.x);
  if (blockIdx.x < 512) ANDES_TRACE(w, 3000 + 2 * blockIdx.x + 1);
}

// ---------------------------------------------------------------- S3b: candidates

// theta = lower edge of the highest LB bucket b* with #(LB in buckets >= b*) >= B_hi, and the
// survivor count #(UB bucket >= b*); computed redundantly by every CTA of k_compact from the
// completed histograms (16 KB each, L2-resident), so no CTA waits on a last-block reduction.
// lb_src: G lower-bound histograms (stride kHistK), summed (multi-GPU: one per rank).
// s_h: kHistK words of shared scratch.
template <uint32_t NT>
__device__ __forceinline__ void theta_of(const Work& w, const uint32_t* lb_src, uint32_t G, uint32_t need,
                                         uint32_t& cut, uint32_t& nsurv, uint32_t* s_h) {
  constexpr uint32_t kPer = kHistK / NT;  // buckets per thread, descending
  __shared__ uint32_t s_w[NT / 32], s_cut, s_sv[NT / 32];
  const uint32_t tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  // coalesced loads of both histograms; survivors partial sums by bucket later
  // kPer independent loads per histogram (one round trip each, not kPer in sequence)
  uint32_t hu[kPer], v[kPer];
#pragma unroll
  for (uint32_t q = 0; q < kPer; ++q) {
    v[q] = __ldcg(&lb_src[q * NT + tid]);
    hu[q] = __ldcg(&w.hist_ub[q * NT + tid]);
  }
  for (uint32_t g = 1; g < G; ++g) {
#pragma unroll
    for (uint32_t q = 0; q < kPer; ++q) v[q] += __ldcg(&lb_src[(size_t)g * kHistK + q * NT + tid]);
  }
#pragma unroll
  for (uint32_t q = 0; q < kPer; ++q) s_h[q * NT + tid] = v[q];
  __syncthreads();
  uint32_t h[kPer], cnt = 0;
#pragma unroll
  for (uint32_t q = 0; q < kPer; ++q) {
    h[q] = s_h[kHistK - 1 - (tid * kPer + q)];
    cnt += h[q];
  }
  uint32_t inc = cnt;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t v = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= (uint32_t)o) inc += v;
  }
  if (lane == 31) s_w[wid] = inc;
  if (tid == 0) s_cut = 0u;
  __syncthreads();
  uint32_t wpre = 0;
  for (uint32_t k = 0; k < wid; ++k) wpre += s_w[k];
  const uint32_t ex = wpre + inc - cnt;
  if (ex < need && ex + cnt >= need) {
    uint32_t c2 = ex;
#pragma unroll
    for (uint32_t q = 0; q < kPer; ++q) {
      c2 += h[q];
      if (c2 >= need) {
        s_cut = kHistK - 1 - (tid * kPer + q);
        break;
      }
    }
  }
  __syncthreads();
  cut = s_cut;
  uint32_t sv = 0;
#pragma unroll
  for (uint32_t q = 0; q < kPer; ++q) sv += (q * NT + tid >= cut) ? hu[q] : 0u;
  for (int o = 16; o; o >>= 1) sv += __shfl_xor_sync(0xffffffffu, sv, o);
  if (lane == 0) s_sv[wid] = sv;
  __syncthreads();
  nsurv = 0;
  for (uint32_t k = 0; k < NT / 32; ++k) nsurv += s_sv[k];
}

// The exact-zero rank cut: the smallest bucket z* with #(exact zeros in buckets <= z*) >= need
// (every exact zero beyond it is pruned; non-zeros carry zr = ~0 and are never pruned), and
// the survivor count reduced by the pruned ones.  Computed redundantly by every CTA.
template <uint32_t NT>
__device__ __forceinline__ void zero_rank_cut(const Work& w, uint32_t need, uint32_t& zcut, uint32_t& nsurv) {
  constexpr uint32_t kPer = kHistK / NT;  // buckets per thread, ascending
  __shared__ uint32_t s_w[NT / 32], s_zc, s_kept;
  const uint32_t tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  uint32_t h[kPer], cnt = 0;
#pragma unroll
  for (uint32_t q = 0; q < kPer; ++q) {
    h[q] = __ldcg(w.hist_zr + tid * kPer + q);
    cnt += h[q];
  }
  uint32_t inc = cnt;
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t v = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= (uint32_t)o) inc += v;
  }
  if (lane == 31) s_w[wid] = inc;
  if (tid == 0) s_zc = 0xFFFFFFFFu;
  __syncthreads();
  uint32_t wpre = 0, tot = 0;
  for (uint32_t k = 0; k < NT / 32; ++k) {
    if (k < wid) wpre += s_w[k];
    tot += s_w[k];
  }
  const uint32_t ex = wpre + inc - cnt;
  if (ex < need && ex + cnt >= need) {
    uint32_t c2 = ex;
#pragma unroll
    for (uint32_t q = 0; q < kPer; ++q) {
      c2 += h[q];
      if (c2 >= need) {
        s_zc = tid * kPer + q;
        s_kept = c2;
        break;
      }
    }
  }
  __syncthreads();
  zcut = s_zc;
  if (zcut != 0xFFFFFFFFu) nsurv -= tot - s_kept;
  __syncthreads();
}

// theta, the exact-zero rank cut and the survivor count from the completed histograms (every
// thread of the CTA gets them; s_h: kHistK words of shared scratch).  lb_src: G lower-bound
// histograms (multi-GPU: one per rank), else the local one.
template <uint32_t NT>
__device__ __forceinline__ void survivor_cut(const Work& w, const uint32_t* lb_src, uint32_t G, uint32_t B_hi,
                                             uint32_t& theta, uint32_t& zcut, uint32_t& ns, uint32_t* s_h) {
  uint32_t cut;
  theta_of<NT>(w, lb_src ? lb_src : w.hist_lb, lb_src ? G : 1u, B_hi, cut, ns, s_h);
  theta = cut << 20;
  // exact zeros beyond the B_hi smallest ranks never make any top-B (single GPU only: the
  // multi-GPU path has no global rank histogram)
  zcut = 0xFFFFFFFFu;
  if (!lb_src && theta <= kOKey0) zero_rank_cut<NT>(w, B_hi, zcut, ns);
}

// Compaction of the survivors (UB >= theta, not pruned by the zero-rank cut) into cand_idx /
// cand_st, warp-aggregated appends; CTA `cta` of `ncta` scans blocks of NT requests.
template <uint32_t NT>
__device__ void compact_phase(const ReqView& r, const Work& w, uint32_t theta, uint32_t zcut, uint32_t cta,
                              uint32_t ncta) {
  const uint32_t lane = threadIdx.x & 31;
  for (uint32_t i0 = cta * NT; i0 < r.n; i0 += ncta * NT) {
    const uint32_t i = i0 + threadIdx.x;
    const bool surv = (i < r.n) && (w.ub[i] >= theta) && (zcut == 0xFFFFFFFFu || w.zr[i] == 0xFFFFFFFFu || w.zr[i] <= zcut);
    const uint32_t bal = __ballot_sync(0xffffffffu, surv);
    if (!bal) continue;
    uint32_t base = 0;
    if (lane == 0) base = atomicAdd(&w.g->cand_ctr, (uint32_t)__popc(bal));
    base = __shfl_sync(0xffffffffu, base, 0);
    if (surv) {
      const uint32_t slot = base + __popc(bal & ((1u << lane) - 1u));
      w.cand_idx[slot] = i | (r.running[i] ? 0x80000000u : 0u);
      w.cand_st[slot] = w.st[i];
    }
  }
}

__global__ void __launch_bounds__(kCandThreads) k_compact(ReqView r, Work w, const uint32_t* lb_src, uint32_t G) {
  pdl_wait();
  __shared__ Globals s_g;
  __shared__ uint32_t s_h[kHistK];
  if (blockIdx.x < 512) ANDES_TRACE(w, 8100 + 2 * blockIdx.x);
  snap_globals(w.g, &s_g);
  if (!s_g.triggered || s_g.B_hi == 0) return;
  uint32_t theta, zcut, ns;
  survivor_cut<kCandThreads>(w, lb_src, G, s_g.B_hi, theta, zcut, ns, s_h);
  if (blockIdx.x == 0) ANDES_TRACE(w, 2210);
  const bool ovf = ns > w.S_cap;  // S_cap <= kCandCap < kRankCap: survivors fit k_select's scratch
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    w.g->theta = theta;
    w.g->n_surv = ns;
    w.g->overflow = ovf ? 1u : 0u;
    if (ovf) atomicOr(&w.g->slow, 2u);
  }
  if (ovf) return;
  compact_phase<kCandThreads>(r, w, theta, zcut, blockIdx.x, gridDim.x);
  if (blockIdx.x < 512) ANDES_TRACE(w, 8100 + 2 * blockIdx.x + 1);
}

__device__ __forceinline__ uint32_t ld_acquire_u32(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_u32(uint32_t* p, uint32_t v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// ---------------------------------------------------------------- S4: Algorithm 1 per B
struct SelectArgs {
  ReqView r;
  Work w;
  int64_t now;
  uint32_t horizon;
  const uint32_t* tau;
  uint32_t B_cap;
  uint64_t M;
  uint32_t preempt_cap;
  SchedOut o;
  XEntry* xsend;  // multi-GPU step 2: this rank's local top-B lists (no walk / cap here)
};

struct FinSmem {
  unsigned long long* key;   // [kVictCap] victim sort keys
  uint32_t* idx;             // [kVictCap] victim request indices
  unsigned long long* vcum;  // [kVictCap] prefix sums of victim l / sort scratch
  uint32_t* adm;             // [kSortCap] S_{B*} in greedy order
  unsigned long long* acum;  // [kSortCap] admit prefix sums
  uint32_t* aflag;           // [kSortCap] admits (S \ R) in greedy order
};
__device__ void finalize_decision(const SelectArgs& A, const FinSmem& F);

// ---------------------------------------------------------------- S5 + S6 + outputs (one CTA)
// serve_mask already holds the running set (written by prep); the decision edits only the
// admitted and the preempted entries.
__device__ void finalize_decision(const SelectArgs& A, const FinSmem& F) {
  __shared__ uint32_t s_Bstar, s_kstar, s_nv, s_na;
  __shared__ unsigned long long s_thr, s_W0;
  __shared__ long long s_bv[kSelThreads / 32];
  __shared__ uint32_t s_bb[kSelThreads / 32];
  __shared__ unsigned long long s_tmp[kSelThreads / 32];
  unsigned long long* const s_key = F.key;
  uint32_t* const s_idx = F.idx;
  uint32_t* const s_adm = F.adm;
  unsigned long long* const s_acum = F.acum;
  uint32_t* const s_aflag = F.aflag;
  unsigned long long* const s_vcum = F.vcum;
  const ReqView& r = A.r;
  const Work& w = A.w;
  const uint32_t tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  uint32_t* sc = A.o.scalars;
  ANDES_TRACE(w, 2100);
  const bool trig = __ldcg(&w.g->triggered) != 0;
  const uint32_t B_lo = __ldcg(&w.g->B_lo), B_hi = __ldcg(&w.g->B_hi);
  const uint32_t n_run_all = __ldcg(&w.g->n_run);
  const uint32_t n_run = min(n_run_all, (uint32_t)kMaxRunning);
  if (n_run_all > (uint32_t)kMaxRunning && tid == 0) raise_err(w, kErrRunning);
  if (!trig) {
    if (tid == 0) {
      for (int q = 0; q < 8; ++q) sc[q] = 0u;
      sc[1] = n_run_all;
    }
    return;
  }
  // S5: largest V over candidate B, ties to the larger B (reading R13)
  {
    long long bv = (long long)0x8000000000000000ull;
    uint32_t bb = 0;
    for (uint32_t B = B_lo + tid; B <= B_hi; B += kSelThreads) {
      const long long v = __ldcg(A.o.V + (B - 1));
      if (bb == 0 || v > bv || (v == bv && B > bb)) {
        bv = v;
        bb = B;
      }
    }
    for (int o = 16; o; o >>= 1) {
      const long long v2 = __shfl_xor_sync(0xffffffffu, bv, o);
      const uint32_t b2 = __shfl_xor_sync(0xffffffffu, bb, o);
      if (b2 != 0 && (bb == 0 || v2 > bv || (v2 == bv && b2 > bb))) {
        bv = v2;
        bb = b2;
      }
    }
    if (lane == 0) {
      s_bv[wid] = bv;
      s_bb[wid] = bb;
    }
    __syncthreads();
    if (tid == 0) {
      bv = s_bv[0];
      bb = s_bb[0];
      for (uint32_t q = 1; q < kSelThreads / 32; ++q)
        if (s_bb[q] != 0 && (bb == 0 || s_bv[q] > bv || (s_bv[q] == bv && s_bb[q] > bb))) {
          bv = s_bv[q];
          bb = s_bb[q];
        }
      s_Bstar = bb;
      s_kstar = bb ? __ldcg(A.o.kstar + (bb - 1)) : 0u;
      s_thr = bb ? __ldcg(w.sel_thr + (bb - 1)) : ~0ull;
      s_nv = 0;
      s_W0 = 0;
    }
    __syncthreads();
  }
  ANDES_TRACE(w, 2101);
  const uint32_t Bs = s_Bstar, ks = s_kstar;
  const unsigned long long thr = s_thr;
  const uint32_t tB = Bs ? A.tau[Bs - 1] : 0u;
  // victims R \ S_{B*}: running requests whose composite at B* is below the k*-th selected
  // composite (composites are unique), keyed for the (key asc, rank desc) order
  {
    unsigned long long wl = 0;
    for (uint32_t q = tid; q < n_run; q += kSelThreads) {
      const uint32_t i = w.run_list[q];
      wl += r.ctx_len[i];
      const unsigned long long c = Bs ? comp_of(w.st[i], tB, w.lqsf, w.obj) : 0ull;
      if (ks == 0 || c < thr) {
        const uint32_t slot = atomicAdd(&s_nv, 1u);
        s_key[slot] = ~c;  // descending of ~ = ascending of the composite
        s_idx[slot] = i;
      }
    }
    for (int o = 16; o; o >>= 1) wl += __shfl_xor_sync(0xffffffffu, wl, o);
    if (lane == 0 && wl) atomicAdd(&s_W0, wl);
  }
  // admits S \ R in greedy order: ordered compaction of S_{B*}
  const uint32_t* selg = w.sel + (size_t)(Bs ? Bs - 1 : 0) * kMaxB;
  for (uint32_t q = tid; q < ks; q += kSelThreads) {
    const uint32_t i = __ldcg(selg + q);
    s_adm[q] = i;
    s_acum[q] = r.running[i] ? 0ull : 1ull;
  }
  __syncthreads();
  const uint32_t nv = s_nv;
  uint32_t size = 1;
  while (size < nv) size <<= 1;
  for (uint32_t q = nv + tid; q < size; q += kSelThreads) {
    s_key[q] = 0ull;
    s_idx[q] = 0xFFFFFFFFu;
  }
  block_inclusive_scan(s_acum, ks, s_tmp);
  for (uint32_t q = tid; q < ks; q += kSelThreads)
    if (s_acum[q] != (q ? s_acum[q - 1] : 0ull)) s_aflag[s_acum[q] - 1] = s_adm[q];
  if (tid == 0) s_na = ks ? (uint32_t)s_acum[ks - 1] : 0u;
  __syncthreads();
  const uint32_t na = s_na;  // s_aflag[0..na) = admits in greedy order
  if (nv <= 2u * kSelThreads) {
    // victim order by rank counting (sort keys are unique): position = #larger keys
    uint32_t* const s_tmpidx = reinterpret_cast<uint32_t*>(s_vcum);
    for (uint32_t q = tid; q < nv; q += kSelThreads) {
      const unsigned long long c = s_key[q];
      uint32_t pos = 0;
      for (uint32_t f = 0; f < nv; ++f) pos += (s_key[f] > c) ? 1u : 0u;
      s_tmpidx[pos] = s_idx[q];
    }
    __syncthreads();
    for (uint32_t q = tid; q < nv; q += kSelThreads) s_idx[q] = s_tmpidx[q];
    __syncthreads();
  } else {
    bitonic_sort<kSelThreads>(s_key, s_idx, size, true);
  }
  ANDES_TRACE(w, 2102);
  const uint32_t cap = A.preempt_cap;
  const bool cap_hit = !(cap == 0xFFFFFFFFu || nv <= cap);
  uint32_t n_pre, n_adm, flags = 1u, realized;
  if (!cap_hit) {
    n_pre = nv;
    n_adm = na;
    realized = ks;
  } else {
    flags |= 2u;
    // W0 after preempting the first cap victims; memory beats the cap (reading R18 step 5)
    for (uint32_t q = tid; q < nv; q += kSelThreads) s_vcum[q] = r.ctx_len[s_idx[q]];
    __syncthreads();
    block_inclusive_scan(s_vcum, nv, s_tmp);
    const unsigned long long W0 = s_W0 - (cap ? s_vcum[cap - 1] : 0ull);
    const uint32_t c0 = n_run - cap;
    if (W0 > A.M) {
      flags |= 4u;
      // smallest e >= 1 with s_W0 - vcum[cap + e - 1] <= M
      __shared__ uint32_t s_e;
      if (tid == 0) s_e = nv;
      __syncthreads();
      for (uint32_t q = cap + tid; q < nv; q += kSelThreads)
        if (s_W0 - s_vcum[q] <= A.M) atomicMin(&s_e, q + 1);
      __syncthreads();
      n_pre = s_e;
      n_adm = 0;
      realized = n_run - n_pre;
    } else {
      // admit in greedy order while W0 + l <= M and c0 + 1 <= B*, break at the first misfit
      for (uint32_t q = tid; q < na; q += kSelThreads) s_acum[q] = r.ctx_len[s_aflag[q]];
      __syncthreads();
      block_inclusive_scan(s_acum, na, s_tmp);
      __shared__ uint32_t s_a;
      if (tid == 0) s_a = 0;
      __syncthreads();
      uint32_t mine = 0;
      for (uint32_t q = tid; q < na; q += kSelThreads)
        mine += (W0 + s_acum[q] <= A.M && c0 + q + 1 <= Bs) ? 1u : 0u;
      for (int o = 16; o; o >>= 1) mine += __shfl_xor_sync(0xffffffffu, mine, o);
      if (lane == 0 && mine) atomicAdd(&s_a, mine);
      __syncthreads();
      n_pre = cap;
      n_adm = s_a;
      realized = c0 + n_adm;
    }
  }
  for (uint32_t q = tid; q < n_pre; q += kSelThreads) {
    const uint32_t i = s_idx[q];
    A.o.preempt_idx[q] = i;
    A.o.serve_mask[i] = 0;
  }
  for (uint32_t q = tid; q < n_adm; q += kSelThreads) {
    const uint32_t i = s_aflag[q];
    A.o.admit_idx[q] = i;
    A.o.serve_mask[i] = 1;
  }
  if (tid == 0) {
    if (__ldcg(&w.g->slow)) flags |= 8u;
    if (__ldcg(&w.g->err) & kErrRunning) flags |= 16u;
    sc[0] = Bs;
    sc[1] = realized;
    sc[2] = n_adm;
    sc[3] = n_pre;
    sc[4] = B_lo;
    sc[5] = B_hi;
    sc[6] = flags;
    sc[7] = ks;
  }
  ANDES_TRACE(w, 2105);
}


// Preemption cap (reading R18) for candidate B, precomputed by B's select CTA so that the final
// step only picks B* and copies: victims R \ S_B (running requests whose composite at B is below
// the k*-th selected composite) sorted by (key asc, rank desc); admits S_B \ R in greedy order;
// then the cap walk.  Staged per B: preempt list, admit list, {n_pre, n_adm, realized, flags}.
// Requires n_run <= kStageRun (the last CTA falls back to finalize_decision otherwise).
__device__ void stage_cap(const SelectArgs& A, uint32_t B, uint32_t tB, uint32_t kstar, unsigned long long thr,
                          const uint32_t* s_sel, unsigned long long* vkey, uint32_t* vidx, unsigned long long* vcum,
                          unsigned long long* acum, uint32_t* aflag, bool rpre, const unsigned long long* rk,
                          const uint32_t* rx, const uint32_t* rlen, uint32_t n_run, const uint32_t* lsel) {
  __shared__ uint32_t s_nv, s_na, s_e, s_a;
  __shared__ unsigned long long s_W0;
  __shared__ unsigned long long s_tmp[kSelThreads / 32];
  const ReqView& r = A.r;
  const Work& w = A.w;
  const uint32_t tid = threadIdx.x, lane = tid & 31;
  if (tid == 0) {
    s_nv = 0;
    s_W0 = 0;
    s_e = 0;
    s_a = 0;
  }
  __syncthreads();
  {
    unsigned long long wl = 0;
    if (rpre) {
      // composites precomputed by the caller in shared memory (n_run <= kSelThreads)
      if (tid < n_run) {
        wl = rlen[tid];
        const unsigned long long c = rk[tid];
        if (kstar == 0 || c < thr) {
          const uint32_t slot = atomicAdd(&s_nv, 1u);
          vkey[slot] = ~c;
          vidx[slot] = tid;  // the running slot: index rx[], length rlen[] (shared memory)
        }
      }
    } else {
      for (uint32_t q = tid; q < n_run; q += kSelThreads) {
        const uint32_t i = __ldcg(w.run_list + q);
        const PackedState st = w.st[i];
        wl += st.l;
        const unsigned long long c = comp_of(st, tB, w.lqsf, w.obj);
        if (kstar == 0 || c < thr) {
          const uint32_t slot = atomicAdd(&s_nv, 1u);
          vkey[slot] = ~c;  // descending of ~c = ascending composite
          vidx[slot] = i;
        }
      }
    }
    for (int o = 16; o; o >>= 1) wl += __shfl_xor_sync(0xffffffffu, wl, o);
    if (lane == 0 && wl) atomicAdd(&s_W0, wl);
  }
  // acum[q] (q < kstar) = 1 for a waiting selected request, written by the caller's V loop
  __syncthreads();
  block_inclusive_scan(acum, kstar, s_tmp);
  for (uint32_t q = tid; q < kstar; q += kSelThreads)
    if (acum[q] != (q ? acum[q - 1] : 0ull)) {
      aflag[acum[q] - 1] = s_sel[q];
      aflag[kSortCap + acum[q] - 1] = lsel[q];  // its l (upper half of aflag's 2 kSortCap words)
    }
  if (tid == 0) s_na = kstar ? (uint32_t)acum[kstar - 1] : 0u;
  // victim order by rank counting (keys unique)
  const uint32_t nv = s_nv;
  {
    uint32_t* const tmp = reinterpret_cast<uint32_t*>(vcum);
    for (uint32_t q = tid; q < nv; q += kSelThreads) {
      const unsigned long long c = vkey[q];
      uint32_t pos = 0;
#pragma unroll 4
      for (uint32_t f = 0; f < nv; ++f) pos += (vkey[f] > c) ? 1u : 0u;
      tmp[pos] = vidx[q];
    }
    __syncthreads();
    for (uint32_t q = tid; q < nv; q += kSelThreads) vidx[q] = tmp[q];
    __syncthreads();
  }
  const uint32_t na = s_na;
  const uint32_t cap = A.preempt_cap;
  const bool cap_hit = !(cap == 0xFFFFFFFFu || nv <= cap);
  uint32_t n_pre, n_adm, flags = 1u, realized;
  if (!cap_hit) {
    n_pre = nv;
    n_adm = na;
    realized = kstar;
  } else {
    flags |= 2u;
    for (uint32_t q = tid; q < nv; q += kSelThreads) vcum[q] = rpre ? rlen[vidx[q]] : r.ctx_len[vidx[q]];
    __syncthreads();
    block_inclusive_scan(vcum, nv, s_tmp);
    const unsigned long long W0a = s_W0;
    const unsigned long long W0 = W0a - (cap ? vcum[cap - 1] : 0ull);
    const uint32_t c0 = n_run - cap;
    if (W0 > A.M) {
      flags |= 4u;  // memory beats the cap: keep preempting in victim order
      if (tid == 0) s_e = nv;
      __syncthreads();
      for (uint32_t q = cap + tid; q < nv; q += kSelThreads)
        if (W0a - vcum[q] <= A.M) atomicMin(&s_e, q + 1);
      __syncthreads();
      n_pre = s_e;
      n_adm = 0;
      realized = n_run - n_pre;
    } else {
      for (uint32_t q = tid; q < na; q += kSelThreads) acum[q] = aflag[kSortCap + q];
      __syncthreads();
      block_inclusive_scan(acum, na, s_tmp);
      uint32_t mine = 0;
      for (uint32_t q = tid; q < na; q += kSelThreads) mine += (W0 + acum[q] <= A.M && c0 + q + 1 <= B) ? 1u : 0u;
      for (int o = 16; o; o >>= 1) mine += __shfl_xor_sync(0xffffffffu, mine, o);
      if (lane == 0 && mine) atomicAdd(&s_a, mine);
      __syncthreads();
      n_pre = cap;
      n_adm = s_a;
      realized = c0 + n_adm;
    }
  }
  uint32_t* pre = w.stage_pre + (size_t)(B - 1) * kStageRun;
  uint32_t* adm = w.stage_adm + (size_t)(B - 1) * kMaxB;
  for (uint32_t q = tid; q < n_pre; q += kSelThreads) pre[q] = rpre ? rx[vidx[q]] : vidx[q];
  for (uint32_t q = tid; q < n_adm; q += kSelThreads) adm[q] = aflag[q];
  if (tid == 0) w.stage_sc[B - 1] = make_uint4(n_pre, n_adm, realized, flags);
}

// stage_cap for the common case (no survivor overflow, n_run <= kSelThreads): the running
// requests were already put in ascending composite order at B (rord, with the prefix sums rcum of
// their l) during the survivors' rank counting, so the victims R \ S_B -- the running requests
// whose composite is below the k*-th selected one (composites are unique) -- are its first nv
// entries, in victim order (key asc, rank desc), and every cap quantity is a prefix sum:
//   W(after preempting the first p victims) = W_run - rcum[p - 1].
// sel / run8 / lsel: S_B in greedy order (request index, running flag, l); rk / rx: the running
// requests' composites / indices by running slot; aflag: 2 kSortCap words of scratch (admit
// index, admit l); acum: kSortCap words of scratch (admit prefix sums).
__device__ void stage_cap_fast(const SelectArgs& A, uint32_t B, uint32_t kstar, unsigned long long thr,
                               const uint32_t* sel, const uint8_t* run8, const uint32_t* lsel,
                               const unsigned long long* rk, const uint32_t* rx, const uint32_t* rord,
                               const unsigned long long* rcum, uint32_t n_run, uint32_t* aflag,
                               unsigned long long* acum) {
  __shared__ uint32_t s_wadm[kSelThreads / 32];
  __shared__ unsigned long long s_tmp2[kSelThreads / 32];
  const Work& w = A.w;
  const uint32_t tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  // victims: count of running composites below thr (all of them when k* = 0)
  const uint32_t nv =
      (uint32_t)__syncthreads_count(tid < n_run && (kstar == 0 || rk[tid] < thr));
  // admits S_B \ R in greedy order: positions q = 2 tid, 2 tid + 1 (k* <= kSortCap = 2 kSelThreads)
  const uint32_t q0 = 2 * tid;
  const bool a0 = q0 < kstar && !run8[q0], a1 = q0 + 1 < kstar && !run8[q0 + 1];
  const uint32_t mine = (a0 ? 1u : 0u) + (a1 ? 1u : 0u);
  uint32_t inc = mine;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t v = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= (uint32_t)o) inc += v;
  }
  if (lane == 31) s_wadm[wid] = inc;
  __syncthreads();
  uint32_t wpre = 0, na = 0;
  for (uint32_t k2 = 0; k2 < kSelThreads / 32; ++k2) {
    wpre += k2 < wid ? s_wadm[k2] : 0u;
    na += s_wadm[k2];
  }
  {
    uint32_t a = wpre + inc - mine;
    if (a0) {
      aflag[a] = sel[q0];
      aflag[kSortCap + a] = lsel[q0];
      ++a;
    }
    if (a1) {
      aflag[a] = sel[q0 + 1];
      aflag[kSortCap + a] = lsel[q0 + 1];
    }
  }
  const uint32_t cap = A.preempt_cap;
  const bool cap_hit = !(cap == 0xFFFFFFFFu || nv <= cap);
  uint32_t n_pre, n_adm, flags = 1u, realized;
  if (!cap_hit) {
    n_pre = nv;
    n_adm = na;
    realized = kstar;
    __syncthreads();  // aflag complete
  } else {
    flags |= 2u;
    const unsigned long long Wrun = rcum[n_run - 1];  // nv > cap >= 0 implies n_run >= 1
    const unsigned long long W0 = Wrun - (cap ? rcum[cap - 1] : 0ull);
    const uint32_t c0 = n_run - cap;
    if (W0 > A.M) {
      flags |= 4u;  // memory beats the cap: keep preempting in victim order (reading R18 step 5)
      // the first p >= cap + 1 with Wrun - rcum[p - 1] <= M (rcum increases), else all nv
      const uint32_t over =
          (uint32_t)__syncthreads_count(tid + cap < nv && Wrun - rcum[tid + cap] > A.M) +
          (uint32_t)__syncthreads_count(tid + cap + kSelThreads < nv && Wrun - rcum[tid + cap + kSelThreads] > A.M);
      n_pre = umin32(nv, cap + over + 1u);
      n_adm = 0;
      realized = n_run - n_pre;
    } else {
      // admit in greedy order while W0 + l <= M and c0 + 1 <= B, break at the first misfit: the
      // count of admit prefix sums that stay within both (prefix sums strictly increase)
      __syncthreads();  // aflag complete
      for (uint32_t q = tid; q < na; q += kSelThreads) acum[q] = aflag[kSortCap + q];
      __syncthreads();
      block_inclusive_scan(acum, na, s_tmp2);
      n_adm = (uint32_t)__syncthreads_count(tid < na && W0 + acum[tid] <= A.M && c0 + tid + 1 <= B) +
              (uint32_t)__syncthreads_count(tid + kSelThreads < na && W0 + acum[tid + kSelThreads] <= A.M &&
                                            c0 + tid + kSelThreads + 1 <= B);
      n_pre = cap;
      realized = c0 + n_adm;
    }
  }
  uint32_t* pre = w.stage_pre + (size_t)(B - 1) * kStageRun;
  uint32_t* adm = w.stage_adm + (size_t)(B - 1) * kMaxB;
  for (uint32_t q = tid; q < n_pre; q += kSelThreads) pre[q] = rx[rord[q]];
  for (uint32_t q = tid; q < n_adm; q += kSelThreads) adm[q] = aflag[q];
  if (tid == 0) w.stage_sc[B - 1] = make_uint4(n_pre, n_adm, realized, flags);
}

// S5 + copy of B*'s staged cap result into the outputs (last CTA of k_select).
__device__ bool finalize_fast(const SelectArgs& A) {
  __shared__ uint32_t s_Bstar;
  const ReqView& r = A.r;
  const Work& w = A.w;
  const uint32_t tid = threadIdx.x;
  const uint32_t B_lo = __ldcg(&w.g->B_lo), B_hi = __ldcg(&w.g->B_hi);
  // B* from the select CTAs' packed atomicMax (no reduction over V here)
  if (tid == 0) s_Bstar = (uint32_t)(__ldcg(&globals2(w)->best_vb) & 2047ull);
  __syncthreads();
  const uint32_t Bs = s_Bstar;
  if (Bs == 0) return false;  // no candidate B: general path
  const uint4 sc4 = __ldcg(w.stage_sc + (Bs - 1));
  const uint32_t n_pre = sc4.x, n_adm = sc4.y;
  const uint32_t* pre = w.stage_pre + (size_t)(Bs - 1) * kStageRun;
  const uint32_t* adm = w.stage_adm + (size_t)(Bs - 1) * kMaxB;
  for (uint32_t q = tid; q < n_pre; q += kSelThreads) {
    const uint32_t i = __ldcg(pre + q);
    A.o.preempt_idx[q] = i;
    A.o.serve_mask[i] = 0;
  }
  for (uint32_t q = tid; q < n_adm; q += kSelThreads) {
    const uint32_t i = __ldcg(adm + q);
    A.o.admit_idx[q] = i;
    A.o.serve_mask[i] = 1;
  }
  if (tid == 0) {
    uint32_t flags = sc4.w;
    if (__ldcg(&w.g->slow)) flags |= 8u;
    uint32_t* sc = A.o.scalars;
    sc[0] = Bs;
    sc[1] = sc4.z;
    sc[2] = n_adm;
    sc[3] = n_pre;
    sc[4] = B_lo;
    sc[5] = B_hi;
    sc[6] = flags;
    sc[7] = __ldcg(A.o.kstar + (Bs - 1));
  }
  (void)r;
  return true;
}

// CTA b handles B = b + 1: top min(B, n) requests by (key desc, rank asc), then Algorithm 1
// (P:L514-529): take while the running sum of l stays <= M (count <= B by construction), break
// at the first misfit; V(B) = sum of llrint(gain 2^32) over the taken prefix; then B's cap result
// is staged (stage_cap) and the last CTA to finish picks B* and writes the outputs.
// descending bitonic sort of one 64-bit value per lane across the warp (shuffles only)
__device__ __forceinline__ unsigned long long warp_sort_desc(unsigned long long v) {
  const uint32_t lane = threadIdx.x & 31;
#pragma unroll 1
  for (uint32_t k = 2; k <= 32; k <<= 1) {
#pragma unroll 1
    for (uint32_t j = k >> 1; j > 0; j >>= 1) {
      const unsigned long long o = __shfl_xor_sync(0xffffffffu, v, j);
      const bool keep_max = ((lane & k) == 0) == ((lane & j) == 0);
      v = keep_max ? (v > o ? v : o) : (v < o ? v : o);
    }
  }
  return v;
}
// number of entries > c in a 32-entry chunk sorted descending (0-padded: never larger)
__device__ __forceinline__ uint32_t count_gt32(const unsigned long long* ch, unsigned long long c) {
  uint32_t p = 0;
#pragma unroll
  for (uint32_t st = 16; st; st >>= 1)
    if (ch[p + st - 1] > c) p += st;
  return p + (ch[p] > c ? 1u : 0u);
}

// k_select's shared scratch (file scope: allocated in the kernels that use it)
__shared__ unsigned long long s_sel_ps[kSortCap];
__shared__ long long s_sel_gf[kSortCap];
__shared__ uint32_t s_sel_k, s_sel_last;
__shared__ long long s_sel_red[32];
__shared__ uint8_t s_sel_run8[kSortCap];  // running flag of the ordered survivors (pruned path)
__shared__ uint32_t s_sel_lsel[kSortCap];  // l of the ordered candidates (the walk's loads)
__shared__ long long s_sel_vsum;           // V(B) accumulator

// S4 for one candidate B (CTA-wide): the top min(B, n) requests by (key desc, rank asc), then
// Algorithm 1: take while the running sum of l stays <= M (count <= B by
// construction), break at the first misfit; V(B) = sum of llrint(gain 2^32) over the taken
// prefix; then B's cap result is staged (stage_cap).  Multi-GPU step 2 (A.xsend): publishes this
// rank's top list of B instead.  s_g: the snapshot of the call's globals after the compaction.
__device__ void select_one_B(const SelectArgs& A, uint32_t B, const Globals& s_g) {
  extern __shared__ unsigned char s_dyn[];
  unsigned long long* s_key = reinterpret_cast<unsigned long long*>(s_dyn);
  uint32_t* s_idx = reinterpret_cast<uint32_t*>(s_dyn + sizeof(unsigned long long) * kVictCap);
  unsigned long long* s_vc = reinterpret_cast<unsigned long long*>(s_idx + kVictCap);
  unsigned long long* const s_ps = s_sel_ps;
  long long* const s_gf = s_sel_gf;
  uint32_t& s_k = s_sel_k;
  long long* const s_red = s_sel_red;
  uint8_t* const s_run8 = s_sel_run8;
  uint32_t* const s_lsel = s_sel_lsel;
  long long& s_vsum = s_sel_vsum;
  const ReqView& r = A.r;
  const Work& w = A.w;
  const uint32_t tid = threadIdx.x;
  const uint32_t n = r.n;
  const bool trig = s_g.triggered != 0;
  const uint32_t B_lo = s_g.B_lo, B_hi = s_g.B_hi;
  const bool ovf = s_g.overflow != 0;
  const uint32_t ns = s_g.n_surv;
  const uint32_t n_run = s_g.n_run;
  ANDES_TRACE(w, 2 * (B - 1));

  if (!trig || B < B_lo || B > B_hi) {
    if (tid == 0) {
      A.o.V[B - 1] = (long long)0x8000000000000000ull;
      A.o.kstar[B - 1] = 0u;
    }
  } else {
    const uint32_t tB = A.tau[B - 1];
    // running requests' composites at B, evaluated in the survivors' pass (stage_cap's fast
    // path), in their own scratch past s_vc
    const bool rpre = !A.xsend && !ovf && n_run <= (uint32_t)kSelThreads;
    unsigned long long* const s_rk = s_vc + kVictCap;
    uint32_t* const s_rx = reinterpret_cast<uint32_t*>(s_rk + kSelThreads);
    uint32_t* const s_rl = s_rx + kSelThreads;
    // multi-GPU: a rank's local top list may be shorter than B (survivors are global)
    const uint32_t k = A.xsend ? min(B, ovf ? n : ns) : min(B, n);
    uint32_t cnt;
    if (ovf) {
      // overflow fallback: exact keys of every request at B (row B of keyrow), radix select.
      // Max-min keys do not depend on B (reading R22): k_state's upper bound is the exact key,
      // so every CTA selects from it directly (4 B per request instead of the 80-byte states).
      const bool bind = w.obj == kObjMaxMin;
      uint32_t* keys = bind ? w.ub : w.keyrow + (size_t)(B - 1) * w.N_cap;
      if (!bind)
        for (uint32_t i = tid; i < n; i += kSelThreads) keys[i] = okey_of(w.st[i], tB, w.lqsf, w.obj);
      __syncthreads();
      // B-independent keys: the order is the same for every B, so the CTA of B_hi selects once
      // and publishes its sorted list (row B_hi of sel); the other CTAs take prefixes of it.  A
      // CTA whose wait exceeds 200 us (the producer not yet resident: more CTAs than slots)
      // selects for itself, so no wait can block forever.
      uint32_t* const shared_list = w.sel + (size_t)(B_hi - 1) * kMaxB;
      bool have = false;
      if (bind && !A.xsend && B != B_hi) {
        if (tid == 0) {
          const unsigned long long t0 = gtimer();
          uint32_t ready = 0;
          while ((ready = ld_acquire_u32(&w.g->sel_ready)) == 0u && gtimer() - t0 < 200000ull) {
          }
          s_k = ready;
        }
        __syncthreads();
        have = s_k != 0u;
        if (have) {
          for (uint32_t q = tid; q < k; q += kSelThreads) {
            const uint32_t i = __ldcg(shared_list + q);
            s_idx[q] = i;
            s_key[q] = composite(keys[i], r.rank[i]);
          }
          __syncthreads();
          cnt = k;
        }
      }
      if (!have) {
        cnt = select_top_k(
            n, k,
            [&](uint32_t e, bool low) -> unsigned long long {
              return low ? composite(keys[e], r.rank[e]) : ((unsigned long long)keys[e] << 32);
            },
            [&](uint32_t e) { return e; }, s_key, s_idx);
        if (bind && !A.xsend && B == B_hi) {
          for (uint32_t q = tid; q < cnt; q += kSelThreads) shared_list[q] = s_idx[q];
          __threadfence();
          __syncthreads();
          if (tid == 0) st_release_u32(&w.g->sel_ready, 1u);
        }
      }
    } else {
      // exact keys of the survivors at B (S3 for this B), then their order by rank counting:
      // position = number of larger composites (unique); two composites per 16-byte load,
      // the odd tail padded with 0 (never larger).  Scratch: composites past the first
      // kSortCap slots of s_key, gfix in s_vc, request indices past kSortCap in s_idx.
      unsigned long long* s_all = s_key + kSortCap;
      uint32_t* s_ri = s_idx + kSortCap;
      long long* s_gall = reinterpret_cast<long long*>(s_vc);
      // indices first (one coalesced round trip), then the states: each iteration of the second
      // loop is independent, so its loads overlap instead of chaining behind the index load
      // survivors and running requests from their contiguous copies (k_compact / k_state): one
      // round trip, no index-then-state chain
      const uint32_t nr = rpre ? n_run : 0u;
#pragma unroll 2
      for (uint32_t e = tid; e < ns + nr; e += kSelThreads) {
        const bool sv = e < ns;
        const uint32_t iv = sv ? __ldcg(w.cand_idx + e) : __ldcg(w.run_idx + (e - ns));
        const PackedState p = *(sv ? w.cand_st + e : w.run_st + (e - ns));
        if (sv) s_ri[e] = iv;
        else s_rx[e - ns] = iv;
        const double gn = gain_of(p, tB, w.obj);
        const unsigned long long c = composite(ordered_key(prio_key(gn, p.l, w.lqsf)), p.rank);
        if (sv) {
          s_all[e] = c;
          s_gall[e] = gain_fixed(gn);
        } else {
          s_rk[e - ns] = c;
          s_rl[e - ns] = p.l;
        }
      }
      if (tid == 0) s_all[ns] = 0ull;
      __syncthreads();
      if (B == 256) ANDES_TRACE(w, 2400);
      if (B == 256 && w.trace && tid == 0) w.trace[2410] = ns;
      // positions from sorted 32-entry chunks (round 2): every thread keeps its elements'
      // composites in registers, every warp sorts 32-entry chunks of the survivors' and of the
      // running requests' composites in place (bitonic, shuffles), and an element's position is
      // the number of larger composites, summed over the chunks by binary searches: O(n log 32)
      // per element instead of the O(n) count (4 us per CTA)
      {
        const uint32_t lane = tid & 31, wid = tid >> 5;
        constexpr uint32_t kPer = (kCandCap + kSelThreads - 1) / kSelThreads;  // survivors per thread
        unsigned long long cs[kPer];
#pragma unroll
        for (uint32_t u = 0; u < kPer; ++u) {
          const uint32_t e = tid + u * kSelThreads;
          cs[u] = e < ns ? s_all[e] : 0ull;
        }
        const uint32_t tr = kSelThreads - 1 - tid;  // this thread's running request (top down)
        const unsigned long long cr = (rpre && tr < n_run) ? s_rk[tr] : 0ull;
        __syncthreads();
        const uint32_t nch_s = (ns + 31) >> 5, nch_r = rpre ? (n_run + 31) >> 5 : 0u;
#pragma unroll 1
        for (uint32_t ch = wid; ch < nch_s + nch_r; ch += kSelThreads / 32) {
          const bool sv = ch < nch_s;
          const uint32_t e = (sv ? ch : ch - nch_s) * 32 + lane;
          unsigned long long* const arr = sv ? s_all : s_rk;
          const unsigned long long c = e < (sv ? ns : n_run) ? arr[e] : 0ull;
          arr[e] = warp_sort_desc(c);  // (chunk padding 0: never larger)
        }
        __syncthreads();
#pragma unroll
        for (uint32_t u = 0; u < kPer; ++u) {
          const uint32_t e = tid + u * kSelThreads;
          if (e >= ns) break;
          const unsigned long long c = cs[u];
          const uint32_t le = __ldcg(&w.cand_st[e].l);  // its l for the walk
          uint32_t pos = 0;
#pragma unroll 1
          for (uint32_t ch = 0; ch < nch_s; ++ch) pos += count_gt32(s_all + 32 * ch, c);
          if (pos < k) {
            s_key[pos] = c;
            s_idx[pos] = s_ri[e] & 0x7FFFFFFFu;
            s_run8[pos] = (uint8_t)(s_ri[e] >> 31);
            s_gf[pos] = s_gall[e];
            s_lsel[pos] = le;
          }
        }
        if (rpre) {
          // ascending position = n_run - 1 - (number of larger composites); l placed by position
          if (tr < n_run) {
            uint32_t gt = 0;
#pragma unroll 1
            for (uint32_t ch = 0; ch < nch_r; ++ch) gt += count_gt32(s_rk + 32 * ch, cr);
            const uint32_t pos = n_run - 1u - gt;
            s_idx[kRunOrdAt + pos] = tr;
            s_vc[kRunOrdAt + pos] = s_rl[tr];
          }
          __syncthreads();
          if (wid == 0) {  // inclusive prefix sums of l in ascending order (per lane, then a warp scan)
            const uint32_t per = (n_run + 31) >> 5, q0 = lane * per, q1 = min(q0 + per, n_run);
            unsigned long long part = 0;
            for (uint32_t q = q0; q < q1; ++q) part += s_vc[kRunOrdAt + q];
            unsigned long long inc = part;
            for (int o = 1; o < 32; o <<= 1) {
              const unsigned long long u2 = __shfl_up_sync(0xffffffffu, inc, o);
              if (lane >= (uint32_t)o) inc += u2;
            }
            unsigned long long run = inc - part;
            for (uint32_t q = q0; q < q1; ++q) {
              run += s_vc[kRunOrdAt + q];
              s_vc[kRunOrdAt + q] = run;
            }
          }
        }
      }
      __syncthreads();
      if (B == 256) ANDES_TRACE(w, 2401);
      cnt = k;
    }
    if (A.xsend) {
      // multi-GPU step 2: publish this rank's top-k of B in order (padded to B); the merge of
      // all ranks' lists and Algorithm 1's walk run in k_shard_merge
      const uint32_t base = s_g.shard_base;
      XEntry* dst = A.xsend + tri_off(B);
      for (uint32_t q = tid; q < B; q += kSelThreads) {
        XEntry x;
        if (q < cnt) {
          const uint32_t i = s_idx[q];
          x.comp = s_key[q];
          x.gfix = ovf ? gain_fixed(gain_of(w.st[i], tB, w.obj)) : s_gf[q];
          x.l = r.ctx_len[i];
          x.gidx = (base + i) | (r.running[i] ? 0x80000000u : 0u);
        } else {
          x.comp = 0ull;
          x.gfix = 0;
          x.l = 0u;
          x.gidx = 0xFFFFFFFFu;
        }
        dst[q] = x;
      }
      return;
    }
    // Algorithm 1 walk (greedy order): k* = number of leading prefix sums of l that stay <= M;
    // prefix sums strictly increase (l >= 1), so this is exactly the walk with `break`.
    if (B == 256) ANDES_TRACE(w, 2402);
    // the walk block-wide (one warp alone is starved by the SM's other CTA): thread t holds
    // positions 2t, 2t+1 (cnt <= kSortCap = 2 kSelThreads); warp scan of l, warp totals through
    // shared memory, and k* = the number of prefix sums <= M by two counting barriers
    static_assert(kSortCap <= 2 * kSelThreads, "walk: two positions per thread");
    uint32_t kstar;
    {
      const uint32_t lane = tid & 31, wid = tid >> 5, q0 = 2 * tid;
      // l of the ordered candidates: placed by the pruned path's rank count, else loaded here
      unsigned long long l0 = 0, l1 = 0;
      if (ovf) {
        l0 = q0 < cnt ? r.ctx_len[s_idx[q0]] : 0ull;
        l1 = q0 + 1 < cnt ? r.ctx_len[s_idx[q0 + 1]] : 0ull;
        if (q0 < cnt) s_lsel[q0] = (uint32_t)l0;
        if (q0 + 1 < cnt) s_lsel[q0 + 1] = (uint32_t)l1;
      } else {
        l0 = q0 < cnt ? s_lsel[q0] : 0u;
        l1 = q0 + 1 < cnt ? s_lsel[q0 + 1] : 0u;
      }
      if (tid == 0) s_vsum = 0;
      unsigned long long inc = l0 + l1;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const unsigned long long u = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= (uint32_t)o) inc += u;
      }
      unsigned long long* const s_wsum = reinterpret_cast<unsigned long long*>(s_red);
      if (lane == 31) s_wsum[wid] = inc;
      __syncthreads();
      if (B == 256) ANDES_TRACE(w, 2403);
      unsigned long long off = 0;
      for (uint32_t k2 = 0; k2 < wid; ++k2) off += s_wsum[k2];
      const unsigned long long p1 = off + inc, p0 = p1 - l1;
      kstar = (uint32_t)__syncthreads_count(q0 < cnt && p0 <= A.M) +
              (uint32_t)__syncthreads_count(q0 + 1 < cnt && p1 <= A.M);
    }
    if (B == 256) ANDES_TRACE(w, 2406);
    long long v = 0;
    for (uint32_t q = tid; q < kstar; q += kSelThreads) {
      const uint32_t i = s_idx[q];
      v += ovf ? gain_fixed(gain_of(w.st[i], tB, w.obj)) : s_gf[q];
      w.sel[(size_t)(B - 1) * kMaxB + q] = i;
      // stage_cap's admit flags (s_ps is free after the walk)
      s_ps[q] = (ovf ? r.running[i] != 0 : s_run8[q] != 0) ? 0ull : 1ull;
    }
    if (B == 256) ANDES_TRACE(w, 2407);
    // V(B): warp sums, one shared 64-bit atomic per warp, one barrier
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if ((tid & 31) == 0 && v) atomicAdd(reinterpret_cast<unsigned long long*>(&s_vsum), (unsigned long long)v);
    __syncthreads();
    v = s_vsum;
    if (B == 256) ANDES_TRACE(w, 2408);
    const unsigned long long thr = kstar ? s_key[kstar - 1] : ~0ull;  // k*-th composite
    if (tid == 0) {
      A.o.V[B - 1] = v;
      if (!A.xsend) atomicMax(&globals2(w)->best_vb, pack_vb(v, B));
      A.o.kstar[B - 1] = kstar;
      w.sel_thr[B - 1] = thr;
    }
    if (B == 256) ANDES_TRACE(w, 2404);
    if (rpre) {
      stage_cap_fast(A, B, kstar, thr, s_idx, s_run8, s_lsel, s_rk, s_rx, s_idx + kRunOrdAt, s_vc + kRunOrdAt,
                     n_run, reinterpret_cast<uint32_t*>(s_gf), s_ps);
    } else if (n_run <= (uint32_t)kStageRun) {
      // victims and their prefix sums live past the first kStageRun slots of s_key / s_idx
      stage_cap(A, B, tB, kstar, thr, s_idx, s_key + kStageRun, s_idx + kStageRun, s_vc,
                s_ps, reinterpret_cast<uint32_t*>(s_gf), rpre, s_rk, s_rx, s_rl, n_run, s_lsel);
    }
    if (B == 256) ANDES_TRACE(w, 2405);
  }
  ANDES_TRACE(w, 2 * (B - 1) + 1);
}

// S5 + S6 by the last of `ncta` CTAs to finish (last-block pattern): B* = argmax V (ties to the
// larger B) and its staged cap result copied into the outputs, or the general finalize.
__device__ void select_finish(const SelectArgs& A, const Globals& s_g, uint32_t ncta) {
  extern __shared__ unsigned char s_dyn[];
  unsigned long long* s_key = reinterpret_cast<unsigned long long*>(s_dyn);
  uint32_t* s_idx = reinterpret_cast<uint32_t*>(s_dyn + sizeof(unsigned long long) * kVictCap);
  unsigned long long* s_vc = reinterpret_cast<unsigned long long*>(s_idx + kVictCap);
  const Work& w = A.w;
  const uint32_t tid = threadIdx.x;
  const bool trig = s_g.triggered != 0;
  const uint32_t n_run = s_g.n_run;
  __threadfence();
  __syncthreads();
  if (tid == 0) s_sel_last = (atomicAdd(&w.g->done, 1u) == ncta - 1) ? 1u : 0u;
  __syncthreads();
  if (!s_sel_last) return;
  __threadfence();
  ANDES_TRACE(w, 2100);
  if (trig && n_run <= (uint32_t)kStageRun && finalize_fast(A)) {
    ANDES_TRACE(w, 2105);
    return;
  }
  FinSmem F;
  F.key = s_key;
  F.idx = s_idx;
  F.vcum = s_vc;
  F.acum = s_sel_ps;
  F.adm = reinterpret_cast<uint32_t*>(s_sel_gf);
  F.aflag = reinterpret_cast<uint32_t*>(s_sel_gf) + kSortCap;
  finalize_decision(A, F);
}

// the key histograms were consumed by the compaction: self-clean them for the next call
__device__ __forceinline__ void clean_key_hists(const Work& w) {
  for (uint32_t q = blockIdx.x * blockDim.x + threadIdx.x; q < kHistK; q += gridDim.x * blockDim.x) {
    w.hist_lb[q] = 0u;
    w.hist_ub[q] = 0u;
    w.hist_zr[q] = 0u;
  }
}

// CTA b handles B = B_cap - b (largest B, the longest walk, scheduled first); the last CTA to
// finish picks B* and writes the outputs.
__global__ void __launch_bounds__(kSelThreads) k_select(SelectArgs A) {
  __shared__ Globals s_g;
  const uint32_t B = gridDim.x - blockIdx.x;
  ANDES_TRACE(A.w, 9200 + B - 1);
  pdl_wait();
  clean_key_hists(A.w);
  snap_globals(A.w.g, &s_g);
  select_one_B(A, B, s_g);
  if (A.xsend) return;
  select_finish(A, s_g, gridDim.x);
}

// ---------------------------------------------------------------- fused post-scan decision
// S3-S6 of a single-GPU decision in ONE cooperative kernel (all CTAs co-resident): the phases of
// k_state, k_compact and k_select separated by grid-wide barriers instead of kernel boundaries
// (each boundary cost a ~3-4 us launch gap plus the next grid's ramp-up):
//   A  per-request state and key bounds (state_phase), bound histograms
//   -- barrier: the last CTA to arrive computes theta / the zero-rank cut / the survivor count
//      once and releases the others
//   B  survivor compaction (compact_phase)
//   -- barrier
//   C  one candidate B per CTA (B = B_cap - b, b + grid, ...): select_one_B; S5/S6 by the last
//      CTA (select_finish)
// Grid-barrier words live in the second 128-byte line of the per-call globals (Globals2).

__device__ __forceinline__ void spin_until_set(const uint32_t* flag) {
  while (ld_acquire_u32(flag) == 0u) __nanosleep(20);
}

__global__ void __launch_bounds__(kSelThreads, 2) k_decide(SelectArgs A) {
  extern __shared__ unsigned char s_dyn[];
  __shared__ Globals s_g;
  __shared__ uint32_t s_flag;
  const ReqView& r = A.r;
  const Work& w = A.w;
  Globals2* ds = globals2(w);
  const uint32_t tid = threadIdx.x, G = gridDim.x;
  pdl_wait();
  snap_globals(w.g, &s_g);
  if (s_g.triggered && s_g.B_hi != 0) {
    // ---- phase A: state and key bounds (histograms in the dynamic shared buffer)
    uint32_t* s_hlb = reinterpret_cast<uint32_t*>(s_dyn);
    if (blockIdx.x < 512) ANDES_TRACE(w, 3000 + 2 * blockIdx.x);
    state_phase<kSelThreads>(r, w, A.now + tshift(w), A.horizon, s_g, s_hlb, s_hlb + kHistK, blockIdx.x, G);
    if (blockIdx.x < 512) ANDES_TRACE(w, 3000 + 2 * blockIdx.x + 1);
    // ---- barrier A; the last arriver computes the survivor cut
    __threadfence();
    __syncthreads();
    if (tid == 0) s_flag = (atomicAdd(&ds->arrive_a, 1u) == G - 1) ? 1u : 0u;
    __syncthreads();
    if (s_flag) {
      __threadfence();
      ANDES_TRACE(w, 2200);
      uint32_t theta, zcut, ns;
      survivor_cut<kSelThreads>(w, nullptr, 1u, s_g.B_hi, theta, zcut, ns, reinterpret_cast<uint32_t*>(s_dyn));
      const bool ovf = ns > w.S_cap;
      if (tid == 0) {
        ds->theta = theta;
        ds->zcut = zcut;
        ds->n_surv = ns;
        ds->overflow = ovf ? 1u : 0u;
        w.g->theta = theta;
        w.g->n_surv = ns;
        w.g->overflow = ovf ? 1u : 0u;
        if (ovf) atomicOr(&w.g->slow, 2u);
        __threadfence();
        st_release_u32(&ds->ready_a, 1u);
      }
      ANDES_TRACE(w, 2201);
    } else if (tid == 0) {
      spin_until_set(&ds->ready_a);
    }
    __syncthreads();
    // ---- phase B: survivor compaction
    const uint32_t theta = __ldcg(&ds->theta), zcut = __ldcg(&ds->zcut);
    if (blockIdx.x < 512) ANDES_TRACE(w, 8100 + 2 * blockIdx.x);
    if (!__ldcg(&ds->overflow)) compact_phase<kSelThreads>(r, w, theta, zcut, blockIdx.x, G);
    if (blockIdx.x < 512) ANDES_TRACE(w, 8100 + 2 * blockIdx.x + 1);
    // ---- barrier B
    __threadfence();
    __syncthreads();
    if (tid == 0) {
      if (atomicAdd(&ds->arrive_b, 1u) == G - 1) {
        __threadfence();
        st_release_u32(&ds->ready_b, 1u);
        ANDES_TRACE(w, 2210);
      } else {
        spin_until_set(&ds->ready_b);
      }
    }
    __syncthreads();
  }
  // ---- phase C: Algorithm 1 per B, S5/S6
  clean_key_hists(w);
  snap_globals(w.g, &s_g);
  for (uint32_t b = blockIdx.x; b < A.B_cap; b += G) {
    ANDES_TRACE(w, 9200 + A.B_cap - b - 1);
    select_one_B(A, A.B_cap - b, s_g);
  }
  select_finish(A, s_g, G);
}

// ---------------------------------------------------------------- host launchers
void launch_gain_estimate(const LaunchCfg& L, const ReqView& r, const Work& w, int64_t now, uint32_t horizon,
                          const uint32_t* tau, const uint32_t* B_list_dev, uint32_t nB, double* gain_out,
                          float* key_out, double* qwait_out) {
  if (r.n == 0) return;
  const uint32_t blocks = umin32((r.n + 255) / 256, L.sm_count * 8);
  launch_pdl(k_gain_estimate, blocks, 256, 0, L.stream, r, w, now, horizon, tau, B_list_dev, nB, gain_out, key_out,
             qwait_out);
}

void launch_state(const LaunchCfg& L, const ReqView& r, const Work& w, int64_t now, uint32_t horizon) {
  const uint32_t blocks = r.n ? umin32((r.n + kStateThreads - 1) / kStateThreads, L.sm_count * 4) : 1u;
  launch_pdl(k_state, blocks, kStateThreads, 0, L.stream, r, w, now, horizon);
}

void launch_compact(const LaunchCfg& L, const ReqView& r, const Work& w, const uint32_t* lb_src, uint32_t G) {
  const uint32_t cblocks = r.n ? umin32((r.n + kCandThreads - 1) / kCandThreads, L.sm_count) : 1u;
  launch_pdl(k_compact, cblocks, kCandThreads, 0, L.stream, r, w, lb_src, G);
}

// victims keys + indices + prefix sums (the fused S5/S6 tail needs all three)
// + the running requests' composites / indices / lengths (n_run <= kSelThreads)
static size_t select_smem() {
  return (2 * sizeof(unsigned long long) + sizeof(uint32_t)) * kVictCap +
         (sizeof(unsigned long long) + 2 * sizeof(uint32_t)) * kSelThreads;
}

static int g_decide_per_sm = 0;  // co-resident k_decide CTAs per SM (cooperative grid limit)

void init_kernels() {
  cudaFuncSetAttribute(k_select, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)select_smem());
  cudaFuncSetAttribute(k_decide, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)select_smem());
  int nb = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k_decide, kSelThreads, select_smem()) != cudaSuccess) nb = 0;
  g_decide_per_sm = nb;
}

// The fused post-scan decision (k_decide) when every CTA can be co-resident: a grid of
// max(B_cap, enough CTAs for the requests) up to the cooperative limit, one candidate B per CTA
// when B_cap fits.  Returns false (nothing launched) when it cannot run; the caller then launches
// k_state, k_compact and k_select.  Off by default (ANDES_FUSED=1 turns it on): on config 3 its two
// grid barriers (~1.7 us each, plus the single-CTA survivor cut) cost as much as the two kernel
// boundaries they replace (84 vs 78 us per decision, tools/time_decision.py).
bool launch_decide(const LaunchCfg& L, const ReqView& r, const Work& w, int64_t now, uint32_t horizon,
                   const uint32_t* tau, uint32_t B_cap, uint64_t M, uint32_t preempt_cap, const SchedOut& o) {
  static const bool off = [] {
    const char* v = getenv("ANDES_FUSED");
    return !(v && v[0] == '1');
  }();
  const uint32_t limit = (uint32_t)g_decide_per_sm * L.sm_count;
  if (off || limit == 0) return false;
  const uint32_t want = umin32(limit, (r.n + kSelThreads - 1) / kSelThreads);
  const uint32_t grid = umin32(limit, B_cap > want ? B_cap : want);
  SelectArgs A{r, w, now, horizon, tau, B_cap, M, preempt_cap, o, nullptr};
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid ? grid : 1u);
  cfg.blockDim = dim3(kSelThreads);
  cfg.dynamicSmemBytes = select_smem();
  cfg.stream = L.stream;
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeCooperative;
  at[0].val.cooperative = 1;
  at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl_enabled() ? 2 : 1;
  return cudaLaunchKernelEx(&cfg, k_decide, A) == cudaSuccess;
}

void launch_select(const LaunchCfg& L, const ReqView& r, const Work& w, int64_t now, uint32_t horizon,
                   const uint32_t* tau, uint32_t B_cap, uint64_t M, uint32_t preempt_cap, const SchedOut& o,
                   XEntry* xsend) {
  SelectArgs A{r, w, now, horizon, tau, B_cap, M, preempt_cap, o, xsend};
  launch_pdl(k_select, B_cap, kSelThreads, select_smem(), L.stream, A);
}

}  // namespace andes
