// refine.cu -- the overhead-aware refiner (NEXT-1; readings R24-R27), applied to the
// decision after the preemption cap (S6) when ANDES_REFINE is set.
//
//   k_refine_pairs  one CTA: the admits (greedy order) are paired with the minimal prefix of the
//                   remaining victims (victim order) that makes room in M; each pair's stall
//                   D_k = its victims' preempt costs + the admit's resume cost (R24 model);
//   k_refine_loss   one warp per (still-running request i, pair k): the QoE drop of i under the
//                   stall, llrint((Q_now,i - Q_i(now + D_k)) 2^32), summed per pair in int64
//                   (deterministic); Q_i(t) is the in-flight QoE at t with no new token;
//   refine_final    the last CTA of k_refine_loss: the first pair whose admit's gain does not
//                   exceed its loss cancels itself and every later pair; the outputs are rewritten.
// The pairs' acceptance is a prefix (the refiner stops at the first rejection), so every pair's
// loss can be evaluated in parallel assuming its predecessors were accepted.
#include "block.cuh"
#include "device.cuh"
#include "launch.h"

namespace andes {

constexpr uint32_t kRefineThreads = 256;

// R24: recompute (preempt 0, resume l / prefill rate) or swap (l / swap rate both ways), the
// smaller round trip, ties to swap; a queued request's admission costs its prefill.  Integer us.
__device__ __forceinline__ void overhead_us(uint32_t l, bool queued, uint32_t prefill, uint32_t swap, long long& pre,
                                            long long& res) {
  const long long rc = prefill ? (long long)l * 1000000ll / prefill : 0ll;
  const long long sw = swap ? (long long)l * 1000000ll / swap : -1ll;
  if (queued || sw < 0 || rc < 2 * sw) {
    pre = 0;
    res = rc;
  } else {
    pre = sw;
    res = sw;
  }
}

// In-place inclusive prefix sums of v[0..cnt) by a kRefineThreads CTA (contiguous runs per thread).
template <class T>
__device__ void refine_scan(T* v, uint32_t cnt, T* s_part) {
  const uint32_t tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const uint32_t per = (cnt + kRefineThreads - 1) / kRefineThreads;
  const uint32_t lo = min(cnt, tid * per), hi = min(cnt, lo + per);
  T part = 0;
  for (uint32_t q = lo; q < hi; ++q) part += v[q];
  T inc = part;
  for (int o = 1; o < 32; o <<= 1) {
    const T u = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= (uint32_t)o) inc += u;
  }
  if (lane == 31) s_part[wid] = inc;
  __syncthreads();
  T off = 0;
  for (uint32_t k = 0; k < wid; ++k) off += s_part[k];
  T run = off + inc - part;
  for (uint32_t q = lo; q < hi; ++q) {
    run += v[q];
    v[q] = run;
  }
  __syncthreads();
}

// The pairing of P:L565-598 (R24), in parallel: with AL = prefix sums of the admits' l and LV of
// the victims' l (victim order), admit k needs the first vp(k) victims, vp(k) = the smallest j
// with W0 + AL[k] - LV[j] <= M (monotone in k, so exactly the serial walk's victim pointer), and
// is feasible iff LV[nv] suffices; the first infeasible admit ends the pairs.  Its stall D_k =
// the preempt costs of victims vp(k-1) .. vp(k)-1 (prefix sums PV) + its own resume cost.
__global__ void __launch_bounds__(kRefineThreads) k_refine_pairs(ReqView r, Work w, SchedOut o, uint64_t M,
                                                                 uint32_t prefill, uint32_t swap) {
  extern __shared__ unsigned char s_dyn[];
  unsigned long long* s_LV = reinterpret_cast<unsigned long long*>(s_dyn);  // [kMaxRunning + 1]
  long long* s_PV = reinterpret_cast<long long*>(s_LV + kMaxRunning + 1);   // [kMaxRunning + 1]
  __shared__ unsigned long long s_AL[kMaxB];
  __shared__ long long s_res[kMaxB];
  __shared__ uint32_t s_vp[kMaxB];
  __shared__ unsigned long long s_pu[kRefineThreads / 32];
  __shared__ long long s_pl[kRefineThreads / 32];
  __shared__ uint32_t s_np;
  pdl_wait();
  const uint32_t tid = threadIdx.x;
  const bool trig = __ldcg(&w.g->triggered) != 0;
  const uint32_t Bs = o.scalars[0];
  const uint32_t na = trig && Bs ? o.scalars[2] : 0u, nv = trig && Bs ? min(o.scalars[3], (uint32_t)kMaxRunning) : 0u;
  const unsigned long long W0 = __ldcg(&w.g->run_l);
  for (uint32_t k = tid; k < kMaxB; k += kRefineThreads) w.rf_loss[k] = 0;
  for (uint32_t q = tid; q < na; q += kRefineThreads) {
    const uint32_t a = o.admit_idx[q];
    const uint32_t la = r.ctx_len[a];
    long long pre, res;
    overhead_us(la, r.n_deliv[a] == 0u, prefill, swap, pre, res);
    s_AL[q] = la;
    s_res[q] = res;
  }
  for (uint32_t v = tid; v < nv; v += kRefineThreads) {
    const uint32_t i = o.preempt_idx[v];
    const uint32_t lv = r.ctx_len[i];
    long long pre, res;
    overhead_us(lv, false, prefill, swap, pre, res);
    s_LV[v + 1] = lv;
    s_PV[v + 1] = pre;
    w.vmark[i] = v + 1u;  // 1 + victim position of request i (cleared by refine_final)
  }
  if (tid == 0) {
    s_LV[0] = 0ull;
    s_PV[0] = 0ll;
    s_np = (W0 <= M) ? na : 0u;  // identity when the running set alone exceeds M
  }
  __syncthreads();
  refine_scan(s_AL, na, s_pu);
  refine_scan(s_LV + 1, nv, s_pu);
  refine_scan(s_PV + 1, nv, s_pl);
  for (uint32_t k = tid; k < na; k += kRefineThreads) {
    const unsigned long long need = W0 + s_AL[k];  // LV[j] >= need - M
    uint32_t vp = 0;
    if (need > M) {
      const unsigned long long t = need - M;
      uint32_t lo = 0, hi = nv + 1;  // first j in [0, nv] with LV[j] >= t, nv + 1 if none
      while (lo < hi) {
        const uint32_t mid = (lo + hi) >> 1;
        if (s_LV[mid] >= t) hi = mid;
        else lo = mid + 1;
      }
      vp = lo;
    }
    s_vp[k] = vp;
    if (vp > nv) atomicMin(&s_np, k);
  }
  __syncthreads();
  const uint32_t np = s_np;
  for (uint32_t k = tid; k < np; k += kRefineThreads) {
    const uint32_t vp = s_vp[k], vq = k ? s_vp[k - 1] : 0u;
    w.rf_vend[k] = vp;
    w.rf_D[k] = (s_PV[vp] - s_PV[vq]) + s_res[k];
  }
  if (tid == 0) w.g->rf_npairs = np;
}

// Q of request i at relative time t with its delivered timeline only (Eq. 1-3, readings R1-R3),
// by one warp: lateness max-scan over the delivered tokens, clamped sums for the two times.
__device__ void walk_two(const ReqView& r, uint32_t i, long long t1, long long t2, double& q1, double& q2) {
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t g = r.n_deliv[i], P = r.period[i], ttft = r.ttft[i], mt = r.max_total[i];
  const unsigned long long base = r.tl_base[i];
  const uint32_t m1 = due_count(t1, ttft, P, mt), m2 = due_count(t2, ttft, P, mt);
  const uint32_t lim = min(g, max(m1, m2));
  long long s1 = 0, s2 = 0;     // sums of min(delta_j, t - I_j) over delivered due tokens
  uint32_t carry = 0, dm1 = 0, dm2 = 0;  // lateness carried; delta at m1 / m2 (when delivered)
  for (uint32_t j0 = 0; j0 < lim; j0 += 32) {
    const uint32_t j = j0 + lane;
    const uint32_t I = ttft + j * P;
    const uint32_t d = j < lim ? r.tl_pool[base + j] : I;
    uint32_t v = d > I ? d - I : 0u;  // lateness (>= 0)
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      const uint32_t u = __shfl_up_sync(0xffffffffu, v, off);
      if (lane >= (uint32_t)off) v = max(v, u);
    }
    const uint32_t dj = max(carry, v);  // delta_{j+1}
    if (j < lim) {
      if (j < m1) s1 += min((long long)dj, t1 - (long long)I);
      if (j < m2) s2 += min((long long)dj, t2 - (long long)I);
      if (j + 1 == m1) dm1 = dj;
      if (j + 1 == m2) dm2 = dj;
    }
    carry = max(carry, __shfl_sync(0xffffffffu, v, 31));
  }
  for (int off = 16; off; off >>= 1) {
    s1 += __shfl_xor_sync(0xffffffffu, s1, off);
    s2 += __shfl_xor_sync(0xffffffffu, s2, off);
    dm1 = max(dm1, __shfl_xor_sync(0xffffffffu, dm1, off));
    dm2 = max(dm2, __shfl_xor_sync(0xffffffffu, dm2, off));
  }
  auto finish = [&](uint32_t m, long long t, long long sp, uint32_t dm) -> double {
    if (m == 0) return 1.0;
    const long long Pl = P;
    const long long cw = Pl * (((long long)m * ((long long)m - 1)) >> 1);
    if (g >= m) {
      const long long Im = (long long)ttft + ((long long)m - 1) * Pl;
      const long long dtm = min((long long)dm, t - Im);
      return qoe_value(sp, (long long)m * dtm + cw);
    }
    const long long K = m - g;
    const long long w0 = t - (long long)ttft - ((long long)g - 1) * Pl;
    return qoe_value(sp + sum_down(0, K, w0, Pl), (long long)m * (w0 - K * Pl) + cw);
  };
  q1 = finish(m1, t1, s1, dm1);
  q2 = finish(m2, t2, s2, dm2);
}

// The first pair whose admit's gain does not exceed its loss cancels itself and every later pair
// (R27); the outputs are rewritten.  One CTA: the last CTA of k_refine_loss.
__device__ void refine_final(const ReqView& r, const Work& w, const SchedOut& o, const uint32_t* tau, uint64_t M) {
  __shared__ uint32_t s_na;
  const uint32_t tid = threadIdx.x;
  const bool trig = __ldcg(&w.g->triggered) != 0;
  const uint32_t Bs = o.scalars[0];
  if (!trig || Bs == 0) return;
  const uint32_t n_adm = o.scalars[2], n_pre = min(o.scalars[3], (uint32_t)kMaxRunning);
  for (uint32_t v = tid; v < n_pre; v += kRefineThreads) w.vmark[o.preempt_idx[v]] = 0u;  // self-clean
  if (__ldcg(&w.g->run_l) > M) return;  // the running set alone exceeds M: identity (R25)
  const uint32_t np = __ldcg(&w.g->rf_npairs);
  if (tid == 0) s_na = np;
  __syncthreads();
  const uint32_t tB = tau[Bs - 1];
  for (uint32_t k = tid; k < np; k += kRefineThreads) {
    const long long gf = gain_fixed(gain_of(w.st[o.admit_idx[k]], tB, w.obj));
    if (!(gf > (long long)__ldcg(w.rf_loss + k))) atomicMin(&s_na, k);
  }
  __syncthreads();
  const uint32_t na = s_na, nv = na ? __ldcg(w.rf_vend + (na - 1)) : 0u;
  for (uint32_t q = na + tid; q < n_adm; q += kRefineThreads) o.serve_mask[o.admit_idx[q]] = 0;
  for (uint32_t v = nv + tid; v < n_pre; v += kRefineThreads) o.serve_mask[o.preempt_idx[v]] = 1;
  if (tid == 0) {
    o.scalars[1] = __ldcg(&w.g->n_run) - nv + na;
    o.scalars[2] = na;
    o.scalars[3] = nv;
    o.scalars[6] |= 32u;  // ANDES_F_REFINED
  }
}

__global__ void __launch_bounds__(kRefineThreads) k_refine_loss(ReqView r, Work w, int64_t now, SchedOut o,
                                                                const uint32_t* tau, uint64_t M) {
  __shared__ Globals s_g;
  pdl_wait();
  now += tshift(w);  // (AndesSchedParams.now_dev)
  snap_globals(w.g, &s_g);
  const uint32_t np = s_g.rf_npairs;
  const uint32_t n_run = min(s_g.n_run, (uint32_t)kMaxRunning);
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, W = (gridDim.x * blockDim.x) >> 5;
  for (uint32_t pr = gw; np && pr < n_run * np; pr += W) {
    const uint32_t q = pr / np, k = pr - q * np;
    const uint32_t i = __ldcg(w.run_list + q);
    const uint32_t vm = __ldcg(w.vmark + i);
    if (vm && vm - 1u < __ldcg(w.rf_vend + k)) continue;  // preempted by pairs <= k
    const long long a = r.arrival[i];
    double qn, qd;
    walk_two(r, i, now - a, now + __ldcg(w.rf_D + k) - a, qn, qd);
    if (lane == 0) {
      const long long lf = gain_fixed(__dsub_rn(qn, qd));
      if (lf) atomicAdd(reinterpret_cast<unsigned long long*>(w.rf_loss + k), (unsigned long long)lf);
    }
  }
  // the last CTA to finish takes the acceptance decision (k_refine_final's work, last-block)
  __shared__ uint32_t s_last;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) s_last = atomicAdd(&globals2(w)->rf_done, 1u) == gridDim.x - 1 ? 1u : 0u;
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  refine_final(r, w, o, tau, M);
}

static size_t refine_pairs_smem() { return 2 * sizeof(unsigned long long) * (kMaxRunning + 1); }

void init_refine_kernels() {
  cudaFuncSetAttribute(k_refine_pairs, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)refine_pairs_smem());
}

void launch_refine(const LaunchCfg& L, const ReqView& r, const Work& w, const SchedOut& o, int64_t now,
                   const uint32_t* tau, uint64_t M, uint32_t prefill, uint32_t swap) {
  launch_pdl(k_refine_pairs, 1, kRefineThreads, refine_pairs_smem(), L.stream, r, w, o, M, prefill, swap);
  launch_pdl(k_refine_loss, L.sm_count * 4, kRefineThreads, 0, L.stream, r, w, now, o, tau, M);
}

}  // namespace andes
