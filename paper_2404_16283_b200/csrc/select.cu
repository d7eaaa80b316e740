// select.cu -- S3-S6 of the decision: gains for every candidate B (Eq. 4/6), Algorithm 1
// per B via an exact radix threshold-select on the (priority desc, rank asc) composite
// key, best B, preemption cap (reading R18), serve-mask materialisation.
#include "device.cuh"
#include "launch.h"

namespace andes {

// ---------------------------------------------------------------- gain_estimate (parity API)
__global__ void k_gain_estimate(ReqView r, Work w, int64_t now, uint32_t horizon, const uint32_t* __restrict__ tau,
                                const uint32_t* __restrict__ B_list, uint32_t nB, double* gain_out, float* key_out,
                                double* qwait_out) {
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

// ---------------------------------------------------------------- S3: keys for every B
// One thread per request; the B-independent state (Q_wait, constants) is built once and the
// closed form of Q_serve(B) is evaluated for every candidate B in [B_lo, B_hi].
__global__ void __launch_bounds__(256) k_gain_keys(ReqView r, Work w, int64_t now, uint32_t horizon,
                                                   const uint32_t* __restrict__ tau, uint32_t B_cap) {
  __shared__ uint32_t s_tau[kMaxB];
  if (!w.g->triggered) return;
  const uint32_t B_lo = w.g->B_lo, B_hi = w.g->B_hi;
  for (uint32_t q = threadIdx.x; q < B_cap; q += blockDim.x) s_tau[q] = tau[q];
  __syncthreads();
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < r.n; i += gridDim.x * blockDim.x) {
    const GainState s = make_state(r, w, i, now, horizon);
    const uint32_t l = r.ctx_len[i];
    uint32_t* out = w.keyrow + i;
    if (s.K == 0) {
      const uint32_t z = ordered_key(0.0f);
      for (uint32_t B = B_lo; B <= B_hi; ++B) out[(size_t)(B - 1) * w.N_cap] = z;
      continue;
    }
    for (uint32_t B = B_lo; B <= B_hi; ++B) {
      const double gn = gain_at(s, s_tau[B - 1]);
      out[(size_t)(B - 1) * w.N_cap] = ordered_key(prio_key(gn, l));
    }
  }
}

// ---------------------------------------------------------------- block helpers
template <int NT>
__device__ __forceinline__ long long block_sum_ll(long long v, long long* red) {
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  __syncthreads();
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  long long t = 0;
  if (threadIdx.x < 32) {
    t = (threadIdx.x < NT / 32) ? red[threadIdx.x] : 0;
    for (int o = 16; o; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
    if (threadIdx.x == 0) red[0] = t;
  }
  __syncthreads();
  t = red[0];
  __syncthreads();
  return t;
}

// In-place bitonic sort of (key, idx) pairs in shared memory, size = power of two.
// descending = true sorts by key descending.
template <int NT>
__device__ void bitonic_sort(unsigned long long* key, uint32_t* idx, uint32_t size, bool descending) {
  for (uint32_t k = 2; k <= size; k <<= 1) {
    for (uint32_t j = k >> 1; j > 0; j >>= 1) {
      for (uint32_t t = threadIdx.x; t < size; t += NT) {
        const uint32_t p = t ^ j;
        if (p > t) {
          const bool up = ((t & k) == 0) == descending;  // region direction
          const unsigned long long a = key[t], b = key[p];
          if ((a < b) == up) {
            key[t] = b;
            key[p] = a;
            const uint32_t x = idx[t];
            idx[t] = idx[p];
            idx[p] = x;
          }
        }
      }
      __syncthreads();
    }
  }
}

constexpr int kSelThreads = 512;
constexpr int kSortCap = kMaxB;        // candidates per B
constexpr int kVictCap = kMaxRunning;  // victims at B*

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
};

__device__ void finalize_decision(const SelectArgs& A, unsigned long long* s_key, uint32_t* s_idx);

// ---------------------------------------------------------------- S4: Algorithm 1 per B
// CTA b handles B = b + 1.  Exact MSB-first radix select (8-bit digits) of the
// k = min(B, n)-th largest composite (priority key, ~rank) over all n requests, then the
// top k are sorted and walked exactly as Algorithm 1: take while the running
// sum of l stays <= M (count <= B holds by construction), break at the first misfit.
__global__ void __launch_bounds__(kSelThreads) k_select(SelectArgs A) {
  extern __shared__ unsigned char s_dyn[];
  unsigned long long* s_key = reinterpret_cast<unsigned long long*>(s_dyn);
  uint32_t* s_idx = reinterpret_cast<uint32_t*>(s_dyn + sizeof(unsigned long long) * kVictCap);
  __shared__ uint32_t s_hist[256];
  __shared__ uint32_t s_cnt;
  __shared__ unsigned long long s_prefix;
  __shared__ uint32_t s_need;
  __shared__ int s_stop;
  __shared__ long long s_red[32];
  __shared__ uint32_t s_last;

  const ReqView& r = A.r;
  const Work& w = A.w;
  const uint32_t tid = threadIdx.x;
  const uint32_t B = blockIdx.x + 1;
  const uint32_t n = r.n;
  const bool trig = w.g->triggered != 0;
  const uint32_t B_lo = w.g->B_lo, B_hi = w.g->B_hi;

  if (!trig || B < B_lo || B > B_hi) {
    if (tid == 0) {
      A.o.V[B - 1] = (long long)0x8000000000000000ull;
      A.o.kstar[B - 1] = 0u;
    }
  } else {
    const uint32_t* keys = w.keyrow + (size_t)(B - 1) * w.N_cap;
    const uint32_t k = min(B, n);
    unsigned long long prefix = 0ull, mask = 0ull;
    uint32_t need = k;
    for (int shift = 56; shift >= 0; shift -= 8) {
      for (uint32_t q = tid; q < 256; q += kSelThreads) s_hist[q] = 0u;
      __syncthreads();
      const bool lowpass = shift < 32;
      for (uint32_t i = tid; i < n; i += kSelThreads) {
        const unsigned long long c = lowpass ? composite(keys[i], r.rank[i]) : ((unsigned long long)keys[i] << 32);
        if ((c & mask) == prefix) atomicAdd(&s_hist[(uint32_t)(c >> shift) & 255u], 1u);
      }
      __syncthreads();
      if (tid < 32) {
        // lane L covers buckets 255-8L .. 248-8L (descending)
        uint32_t cnt[8], tot = 0;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          cnt[j] = s_hist[255 - 8 * tid - j];
          tot += cnt[j];
        }
        uint32_t inc = tot;
        for (int o = 1; o < 32; o <<= 1) {
          const uint32_t v = __shfl_up_sync(0xffffffffu, inc, o);
          if (tid >= (uint32_t)o) inc += v;
        }
        const uint32_t exc = inc - tot;
        if (exc < need && inc >= need) {
          uint32_t above = exc;
          for (int j = 0; j < 8; ++j) {
            if (above + cnt[j] >= need) {
              const uint32_t bucket = 255 - 8 * tid - j;
              s_prefix = prefix | ((unsigned long long)bucket << shift);
              s_need = need - above;
              s_stop = (cnt[j] == need - above) ? 1 : 0;
              break;
            }
            above += cnt[j];
          }
        }
      }
      __syncthreads();
      prefix = s_prefix;
      need = s_need;
      mask |= 255ull << shift;
      if (s_stop) break;
    }
    // collect the k elements with composite >= prefix
    const unsigned long long theta = prefix;
    if (tid == 0) s_cnt = 0;
    __syncthreads();
    for (uint32_t i = tid; i < n; i += kSelThreads) {
      const uint32_t okey = keys[i];
      if (((unsigned long long)okey << 32 | 0xFFFFFFFFull) < theta) continue;  // cheap reject
      const unsigned long long c = composite(okey, r.rank[i]);
      if (c >= theta) {
        const uint32_t slot = atomicAdd(&s_cnt, 1u);
        if (slot < kSortCap) {
          s_key[slot] = c;
          s_idx[slot] = i;
        }
      }
    }
    __syncthreads();
    const uint32_t cnt = min(s_cnt, (uint32_t)kSortCap);
    uint32_t size = 1;
    while (size < cnt) size <<= 1;
    for (uint32_t q = cnt + tid; q < size; q += kSelThreads) {
      s_key[q] = 0ull;
      s_idx[q] = 0xFFFFFFFFu;
    }
    __syncthreads();
    bitonic_sort<kSelThreads>(s_key, s_idx, size, true);
    // Algorithm 1 walk: prefix sums of l in greedy order (<= 1024 elements, 2 per thread)
    __shared__ unsigned long long s_ps[kSortCap];
    for (uint32_t q = tid; q < cnt; q += kSelThreads) s_ps[q] = r.ctx_len[s_idx[q]];
    __syncthreads();
    for (uint32_t off = 1; off < cnt; off <<= 1) {
      unsigned long long v0 = 0, v1 = 0;
      const uint32_t q0 = tid, q1 = tid + kSelThreads;
      if (q0 < cnt && q0 >= off) v0 = s_ps[q0 - off];
      if (q1 < cnt && q1 >= off) v1 = s_ps[q1 - off];
      __syncthreads();
      if (q0 < cnt) s_ps[q0] += v0;
      if (q1 < cnt) s_ps[q1] += v1;
      __syncthreads();
    }
    // k* = number of leading prefix sums <= M (l >= 1: prefix sums strictly increase)
    if (tid == 0) s_cnt = 0;
    __syncthreads();
    uint32_t mine = 0;
    for (uint32_t q = tid; q < cnt; q += kSelThreads) mine += (s_ps[q] <= A.M) ? 1u : 0u;
    if (mine) atomicAdd(&s_cnt, mine);
    __syncthreads();
    const uint32_t kstar = s_cnt;
    long long v = 0;
    const uint32_t tB = A.tau[B - 1];
    for (uint32_t q = tid; q < kstar; q += kSelThreads) {
      const uint32_t i = s_idx[q];
      const GainState s = make_state(r, w, i, A.now, A.horizon);
      v += gain_fixed(gain_at(s, tB));
      w.sel[(size_t)(B - 1) * kMaxB + q] = i;
    }
    v = block_sum_ll<kSelThreads>(v, s_red);
    if (tid == 0) {
      A.o.V[B - 1] = v;
      A.o.kstar[B - 1] = kstar;
    }
  }
  // last CTA finalises the decision
  __threadfence();
  __syncthreads();
  if (tid == 0) s_last = (atomicAdd(&w.g->done, 1u) == gridDim.x - 1) ? 1u : 0u;
  __syncthreads();
  if (s_last) {
    __threadfence();
    finalize_decision(A, s_key, s_idx);
  }
}

// ---------------------------------------------------------------- S5 + S6 (one CTA)
__device__ void finalize_decision(const SelectArgs& A, unsigned long long* s_key, uint32_t* s_idx) {
  __shared__ uint32_t s_Bstar, s_kstar, s_nv;
  const ReqView& r = A.r;
  const Work& w = A.w;
  const uint32_t tid = threadIdx.x;
  uint32_t* sc = A.o.scalars;
  const bool trig = w.g->triggered != 0;
  const uint32_t B_lo = w.g->B_lo, B_hi = w.g->B_hi;
  const uint32_t n_run = min(w.g->n_run, (uint32_t)kMaxRunning);
  if (w.g->n_run > (uint32_t)kMaxRunning && tid == 0) atomicOr(&w.g->err, kErrRunning);
  if (!trig) {
    if (tid == 0) {
      for (int q = 0; q < 8; ++q) sc[q] = 0u;
      sc[1] = w.g->n_run;
    }
    return;
  }
  if (tid == 0) {
    // S5: largest V over candidate B, ties to the larger B (reading R13)
    uint32_t Bs = 0;
    long long best = 0;
    for (uint32_t B = B_lo; B <= B_hi; ++B) {
      const long long v = __ldcg(A.o.V + (B - 1));
      if (Bs == 0 || v >= best) {
        best = v;
        Bs = B;
      }
    }
    s_Bstar = Bs;
    s_kstar = Bs ? __ldcg(A.o.kstar + (Bs - 1)) : 0u;
  }
  __syncthreads();
  const uint32_t Bs = s_Bstar, ks = s_kstar;
  const uint32_t* sel = w.sel + (size_t)(Bs ? Bs - 1 : 0) * kMaxB;
  for (uint32_t q = tid; q < ks; q += kSelThreads) w.mark[__ldcg(sel + q)] = 1u;
  if (tid == 0) s_nv = 0;
  __syncthreads();
  // victims: running requests outside S_{B*}, ordered by (key asc, rank desc)
  for (uint32_t q = tid; q < n_run; q += kSelThreads) {
    const uint32_t i = w.run_list[q];
    if (!(w.mark[i] & 1u)) {
      const uint32_t slot = atomicAdd(&s_nv, 1u);
      const uint32_t okey = Bs ? w.keyrow[(size_t)(Bs - 1) * w.N_cap + i] : 0u;
      s_key[slot] = ~composite(okey, r.rank[i]);  // descending of ~ = ascending of composite
      s_idx[slot] = i;
    }
  }
  __syncthreads();
  const uint32_t nv = s_nv;
  uint32_t size = 1;
  while (size < nv) size <<= 1;
  for (uint32_t q = nv + tid; q < size; q += kSelThreads) {
    s_key[q] = 0ull;
    s_idx[q] = 0xFFFFFFFFu;
  }
  __syncthreads();
  bitonic_sort<kSelThreads>(s_key, s_idx, size, true);
  if (tid == 0) {
    // S6 preemption cap (reading R18), sequential over <= B* admits and nv victims
    uint32_t flags = 1u;  // triggered
    uint32_t n_adm = 0, n_pre = 0, realized = 0;
    const uint32_t cap = A.preempt_cap;
    if (cap == 0xFFFFFFFFu || nv <= cap) {
      for (uint32_t q = 0; q < ks; ++q) {
        const uint32_t i = sel[q];
        if (!r.running[i]) A.o.admit_idx[n_adm++] = i;
      }
      for (uint32_t q = 0; q < nv; ++q) A.o.preempt_idx[n_pre++] = s_idx[q];
      realized = ks;
    } else {
      flags |= 2u;
      unsigned long long W0 = 0;
      uint32_t c0 = 0;
      for (uint32_t q = 0; q < n_run; ++q) {
        W0 += r.ctx_len[w.run_list[q]];
        ++c0;
      }
      for (uint32_t q = 0; q < cap; ++q) {
        const uint32_t i = s_idx[q];
        w.mark[i] |= 2u;
        A.o.preempt_idx[n_pre++] = i;
        W0 -= r.ctx_len[i];
        --c0;
      }
      if (W0 > A.M) {
        flags |= 4u;  // memory beats the cap
        for (uint32_t q = cap; q < nv && W0 > A.M; ++q) {
          const uint32_t i = s_idx[q];
          w.mark[i] |= 2u;
          A.o.preempt_idx[n_pre++] = i;
          W0 -= r.ctx_len[i];
          --c0;
        }
      } else {
        for (uint32_t q = 0; q < ks; ++q) {
          const uint32_t i = sel[q];
          if (r.running[i]) continue;
          const uint32_t l = r.ctx_len[i];
          if (W0 + l <= A.M && c0 + 1 <= Bs) {
            w.mark[i] |= 4u;
            A.o.admit_idx[n_adm++] = i;
            W0 += l;
            ++c0;
          } else {
            break;
          }
        }
      }
      realized = c0;
    }
    if (w.g->slow) flags |= 8u;
    if (w.g->err & kErrRunning) flags |= 16u;
    sc[0] = Bs;
    sc[1] = realized;
    sc[2] = n_adm;
    sc[3] = n_pre;
    sc[4] = B_lo;
    sc[5] = B_hi;
    sc[6] = flags;
    sc[7] = ks;
  }
}

// ---------------------------------------------------------------- serve mask
__global__ void k_mask(ReqView r, Work w, SchedOut o) {
  const bool trig = w.g->triggered != 0;
  const bool cap_hit = (__ldcg(o.scalars + 6) & 2u) != 0;
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < r.n; i += gridDim.x * blockDim.x) {
    const uint8_t mk = w.mark[i];
    const uint8_t run = r.running[i];
    uint8_t x;
    if (!trig) x = run ? 1 : 0;
    else if (cap_hit) x = ((run && !(mk & 2u)) || (mk & 4u)) ? 1 : 0;
    else x = (mk & 1u) ? 1 : 0;
    o.serve_mask[i] = x;
    if (mk) w.mark[i] = 0;
  }
}

// ---------------------------------------------------------------- host launchers
void launch_gain_estimate(const LaunchCfg& L, const ReqView& r, const Work& w, int64_t now, uint32_t horizon,
                          const uint32_t* tau, const uint32_t* B_list_dev, uint32_t nB, double* gain_out,
                          float* key_out, double* qwait_out) {
  if (r.n == 0) return;
  const uint32_t blocks = umin32((r.n + 255) / 256, L.sm_count * 8);
  k_gain_estimate<<<blocks, 256, 0, L.stream>>>(r, w, now, horizon, tau, B_list_dev, nB, gain_out, key_out,
                                                qwait_out);
}

void launch_gain_keys(const LaunchCfg& L, const ReqView& r, const Work& w, int64_t now, uint32_t horizon,
                      const uint32_t* tau, uint32_t B_cap) {
  if (r.n == 0) return;
  const uint32_t blocks = (r.n + 255) / 256;
  k_gain_keys<<<blocks, 256, 0, L.stream>>>(r, w, now, horizon, tau, B_cap);
}

static size_t select_smem() { return (sizeof(unsigned long long) + sizeof(uint32_t)) * kVictCap; }

void init_kernels() {
  cudaFuncSetAttribute(k_select, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)select_smem());
}

void launch_select(const LaunchCfg& L, const ReqView& r, const Work& w, int64_t now, uint32_t horizon,
                   const uint32_t* tau, uint32_t B_cap, uint64_t M, uint32_t preempt_cap, const SchedOut& o) {
  SelectArgs A{r, w, now, horizon, tau, B_cap, M, preempt_cap, o};
  k_select<<<B_cap, kSelThreads, select_smem(), L.stream>>>(A);
}

void launch_mask(const LaunchCfg& L, const ReqView& r, const Work& w, const SchedOut& o) {
  if (r.n == 0) return;
  const uint32_t blocks = umin32((r.n + 255) / 256, L.sm_count * 8);
  k_mask<<<blocks, 256, 0, L.stream>>>(r, w, o);
}

}  // namespace andes
