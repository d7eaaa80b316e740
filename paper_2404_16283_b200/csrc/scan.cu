// scan.cu -- S0/S1/S2 of the decision: per-request preparation, the token-parallel
// QoE timeline scan (K1) and the trigger / batch-size-range step.
//
// K1 computes, for every request i and the evaluation time t_i ("QoE can be
// computed on requests in any state"), over its delivered due tokens j <= min(g, m):
//     delta_j  = max(0, max_{k<=j} (d_k - I_k))        (actual consumption, reading R2)
//     S_pre    = sum_j min(delta_j, t - I_j)           (Eq. 1 restricted to delivered tokens)
//     edge     = delta_g (g < m) or delta~_m (g >= m)
// The timestamp pool is streamed once: tiles of kTile tokens are staged into shared
// memory with cp.async.bulk (TMA bulk copy, mbarrier completion), double-buffered,
// by a persistent grid; the prefix max crosses tile boundaries through a single-pass
// decoupled look-back on the segmented-max monoid (flag = segment start, value = max).
#include "device.cuh"
#include "launch.h"

namespace andes {

// ---------------------------------------------------------------- prep
// One pass over the requests: m_i, zeroed accumulators, tile owners, and for a
// decision the trigger inputs (sum of running l, min period), the l histogram for
// B_max and the running list.
__global__ void k_prep(ReqView r, Work w, int64_t eval_abs, uint32_t final_mode, uint32_t sched,
                       uint64_t kv_cap, uint32_t debug) {
  const uint32_t n = r.n;
  uint32_t local_err = 0;
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const uint32_t g = r.n_deliv[i];
    const uint32_t P = r.period[i];
    uint32_t m;
    if (final_mode) {
      m = g;
    } else {
      const int64_t t = eval_abs - r.arrival[i];
      m = due_count(t, r.ttft[i], P ? P : 1u, r.max_total[i]);
    }
    w.m[i] = m;
    w.spre[i] = 0ull;
    w.edge[i] = 0u;
    // tile ownership: tiles whose start position p satisfies base_i <= p < base_{i+1}
    const unsigned long long base = r.tl_base[i];
    const unsigned long long next = (i + 1 < n) ? r.tl_base[i + 1] : base + g;
    const uint32_t t_lo = (i == 0) ? 0u : (uint32_t)((base + kTile - 1) / kTile);
    uint32_t t_hi = (uint32_t)((next + kTile - 1) / kTile);
    if (t_hi > w.tiles_cap) {  // pool span above limits.max_tokens: refuse (flagged), never overrun
      t_hi = w.tiles_cap;
      local_err |= kErrTokens;
    }
    for (uint32_t t = t_lo; t < t_hi; ++t) w.tile_owner[t] = i;
    if (i + 1 == n) {
      w.g->ntiles = min((uint32_t)((base + g + kTile - 1) / kTile), w.tiles_cap);
      w.g->pool_end = min(base + g, (unsigned long long)w.tiles_cap * kTile);
    }
    if (debug) {
      if (P == 0) local_err |= kErrPeriod;
      if (i + 1 < n && next < base + g) local_err |= kErrBase;
      if (!final_mode && m >= (1u << 20)) local_err |= kErrDue;
    }
    if (sched) {
      const uint32_t l = r.ctx_len[i];
      atomicMax(&w.g->inv_minP, 0xFFFFFFFFu - P);
      atomicAdd(&w.hist_l[l < kHistL - 1 ? l : kHistL - 1], 1u);
      if (r.running[i]) {
        atomicAdd(&w.g->run_l, (unsigned long long)l);
        const uint32_t slot = atomicAdd(&w.g->n_run, 1u);
        if (slot < kMaxRunning) w.run_list[slot] = i;
      }
      if (debug && (l == 0 || l > kv_cap)) local_err |= kErrCtx;
    }
  }
  if (local_err) atomicOr(&w.g->err, local_err);
}

// ---------------------------------------------------------------- bounds (1 CTA)
// S0 selective triggering (reading R15) and S2 batch-size range
// (reading R16): B_max = number of shortest contexts that fit in M,
// B_min = largest B with tau(B) <= min_i P_i (only with ANDES_PRUNE).
__global__ void __launch_bounds__(1024) k_bounds(ReqView r, Work w, const uint32_t* __restrict__ tau,
                                                 uint32_t B_cap, uint64_t M, uint32_t cur_latency,
                                                 uint32_t flags) {
  __shared__ unsigned long long s_cnt[1024];
  __shared__ unsigned long long s_sum[1024];
  __shared__ uint32_t s_kM;
  const uint32_t tid = threadIdx.x;
  const uint32_t n = r.n;
  const uint32_t minP = 0xFFFFFFFFu - w.g->inv_minP;
  const unsigned long long run_l = w.g->run_l;
  const bool trig = (flags & 1u) || (10ull * run_l > 9ull * M) || (n > 0 && cur_latency > minP);
  // per-thread slice of the exact l histogram: buckets [64 tid, 64 tid + 64)
  constexpr uint32_t kPer = kHistL / 1024;
  unsigned long long c = 0, s = 0;
  for (uint32_t b = tid * kPer; b < (tid + 1) * kPer; ++b) {
    const uint32_t h = w.hist_l[b];
    c += h;
    s += (unsigned long long)h * b;
  }
  s_cnt[tid] = c;
  s_sum[tid] = s;
  if (tid == 0) s_kM = 0xFFFFFFFFu;
  __syncthreads();
  // inclusive scans (Hillis-Steele; 10 steps)
  for (uint32_t off = 1; off < 1024; off <<= 1) {
    unsigned long long a = 0, b2 = 0;
    if (tid >= off) { a = s_cnt[tid - off]; b2 = s_sum[tid - off]; }
    __syncthreads();
    s_cnt[tid] += a;
    s_sum[tid] += b2;
    __syncthreads();
  }
  // k_M = max k with sum of the k smallest l <= M, needed only up to min(B_cap, n)
  const uint32_t need = min(B_cap, n);
  {
    const unsigned long long c_ex = tid ? s_cnt[tid - 1] : 0ull;
    const unsigned long long s_ex = tid ? s_sum[tid - 1] : 0ull;
    // the thread whose slice contains the crossing (count reaches need or sum exceeds M)
    const bool crosses = (s_cnt[tid] >= need || s_sum[tid] > M) && (c_ex < need && s_ex <= M);
    if (crosses) {
      unsigned long long k = c_ex, W = s_ex;
      bool stop = false;
      for (uint32_t b = tid * kPer; b < (tid + 1) * kPer && !stop; ++b) {
        const uint32_t h = w.hist_l[b];
        if (b == kHistL - 1 && h) break;  // overflow bucket: exact values needed, slow path below
        for (uint32_t q = 0; q < h; ++q) {
          if (k >= need || W + b > M) { stop = true; break; }
          W += b;
          ++k;
        }
      }
      if (stop || k >= need) s_kM = (uint32_t)(k < need ? k : (unsigned long long)need);
      else s_kM = 0xFFFFFFFEu;  // reached the overflow bucket
    }
  }
  __syncthreads();
  if (s_kM == 0xFFFFFFFFu) s_kM = 0;  // (not reachable for n >= 1 unless all l are in overflow)
  __syncthreads();
  uint32_t kM = s_kM;
  if (kM == 0xFFFFFFFEu || (kM == 0 && n > 0 && s_cnt[1023] > 0)) {
    // Slow path (l >= 65535 among the smallest): repeated exact minima over all requests.
    __shared__ unsigned long long s_red[32];
    __shared__ unsigned long long s_taken_key;
    unsigned long long k = 0, W = 0;
    for (uint32_t b = 0; b < kHistL - 1; ++b) {  // all small l first (they all fit: see crossing)
      const uint32_t h = w.hist_l[b];
      k += h;
      W += (unsigned long long)h * b;
    }
    unsigned long long last = 0;  // (l << 32 | i) of the last taken large element
    bool first = true;
    while (k < need) {
      unsigned long long best = ~0ull;
      for (uint32_t i = tid; i < n; i += blockDim.x) {
        const uint32_t l = r.ctx_len[i];
        if (l < kHistL - 1) continue;
        const unsigned long long key = ((unsigned long long)l << 32) | i;
        if ((first || key > last) && key < best) best = key;
      }
      for (int o = 16; o; o >>= 1) best = min(best, __shfl_xor_sync(0xffffffffu, best, o));
      if ((tid & 31) == 0) s_red[tid >> 5] = best;
      __syncthreads();
      if (tid == 0) {
        unsigned long long b2 = ~0ull;
        for (int q = 0; q < 32; ++q) b2 = min(b2, s_red[q]);
        s_taken_key = b2;
      }
      __syncthreads();
      const unsigned long long b2 = s_taken_key;
      __syncthreads();
      if (b2 == ~0ull || W + (b2 >> 32) > M) break;
      W += b2 >> 32;
      ++k;
      last = b2;
      first = false;
    }
    kM = (uint32_t)k;
    if (tid == 0) atomicOr(&w.g->slow, 1u);
  }
  // self-clean the histogram for the next call (after every reader above)
  __syncthreads();
  for (uint32_t b = tid; b < kHistL; b += blockDim.x) w.hist_l[b] = 0u;
  if (tid == 0) {
    const uint32_t B_hi = min(min(B_cap, n), kM);
    uint32_t B_lo = 1;
    if (flags & 2u) {
      for (uint32_t B = 1; B <= B_hi; ++B)
        if (tau[B - 1] <= minP) B_lo = B;
    }
    w.g->B_hi = B_hi;
    w.g->B_lo = (B_hi == 0) ? 1u : min(B_lo, B_hi);
    w.g->triggered = trig ? 1u : 0u;
  }
}

// ---------------------------------------------------------------- K1 timeline scan
namespace {

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(phase)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

// segmented max monoid on (flag, value): combine(a, b) with a earlier than b
__device__ __forceinline__ unsigned long long seg_combine(unsigned long long a, unsigned long long b) {
  if (b & kFlagBit) return b;
  const uint32_t v = max((uint32_t)a, (uint32_t)b);
  return (a & kFlagBit) | v;
}

struct ScanArgs {
  ReqView r;
  Work w;
  int64_t eval_abs;
};

// Issue the bulk copy of tile t into buffer buf (one elected thread).
__device__ __forceinline__ void issue_tile(const ScanArgs& A, uint32_t t, unsigned long long pool_end,
                                           uint32_t* buf, uint64_t* bar) {
  const unsigned long long p0 = (unsigned long long)t * kTile;
  const unsigned long long pend = min(p0 + (unsigned long long)kTile, pool_end);
  const uint32_t cnt = (uint32_t)(pend - p0);
  const uint32_t bulk = (cnt / 4u) * 16u;  // 16-byte multiple
  mbar_expect_tx(bar, bulk);
  if (bulk) bulk_g2s(buf, A.r.tl_pool + p0, bulk, bar);
}

}  // namespace

template <bool kFinal>
__global__ void __launch_bounds__(kScanThreads) k_qoe_scan(ScanArgs A) {
  __shared__ alignas(128) uint32_t s_tile[2][kTile];
  __shared__ alignas(8) uint64_t s_bar[2];
  __shared__ unsigned long long s_win[kWindowCap + 1];
  __shared__ unsigned long long s_warp[kScanThreads / 32];
  __shared__ unsigned long long s_carry;
  __shared__ uint32_t s_r0, s_wn;

  const ReqView& r = A.r;
  const Work& w = A.w;
  const uint32_t tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const uint32_t ntiles = w.g->ntiles;
  const unsigned long long pool_end = w.g->pool_end;
  const uint32_t n = r.n;

  if (tid == 0) {
    mbar_init(&s_bar[0], 1);
    mbar_init(&s_bar[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  uint32_t phase[2] = {0u, 0u};
  uint32_t t = blockIdx.x;
  if (tid == 0 && t < ntiles) issue_tile(A, t, pool_end, s_tile[0], &s_bar[0]);
  uint32_t buf = 0;

  for (; t < ntiles; t += gridDim.x, buf ^= 1u) {
    const unsigned long long p0 = (unsigned long long)t * kTile;
    const unsigned long long pend = min(p0 + (unsigned long long)kTile, pool_end);
    // prefetch the next tile of this CTA into the other buffer (its previous generic-proxy
    // reads/writes were ordered by the trailing __syncthreads; fence them against the
    // async-proxy bulk write)
    if (tid == 0 && t + gridDim.x < ntiles) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      issue_tile(A, t + gridDim.x, pool_end, s_tile[buf ^ 1u], &s_bar[buf ^ 1u]);
    }

    // request window: requests r0 .. r_end own the positions of this tile
    if (tid == 0) {
      const uint32_t r0 = w.tile_owner[t];
      const uint32_t r_end = (t + 1 < ntiles) ? w.tile_owner[t + 1] : n - 1;
      s_r0 = r0;
      s_wn = r_end - r0 + 1;
    }
    __syncthreads();
    const uint32_t r0 = s_r0, wn = s_wn;
    const bool win_ok = wn <= kWindowCap;
    if (win_ok)
      for (uint32_t q = tid; q <= wn; q += kScanThreads)
        s_win[q] = (r0 + q < n) ? r.tl_base[r0 + q] : ~0ull;
    // tail tokens not covered by the 16-byte bulk copy
    {
      const uint32_t cnt = (uint32_t)(pend - p0);
      const uint32_t bulk_tok = (cnt / 4u) * 4u;
      if (tid < cnt - bulk_tok) s_tile[buf][bulk_tok + tid] = r.tl_pool[p0 + bulk_tok + tid];
    }
    mbar_wait(&s_bar[buf], phase[buf]);
    phase[buf] ^= 1u;
    __syncthreads();

    // ---- locate this thread's first owner
    const unsigned long long my0 = p0 + (unsigned long long)tid * kScanItems;
    auto base_of = [&](uint32_t rr) -> unsigned long long {
      if (rr >= n) return ~0ull;
      if (win_ok && rr >= r0 && rr - r0 <= wn) return s_win[rr - r0];
      return r.tl_base[rr];
    };
    uint32_t rr;
    {
      // largest rr in [r0, r0+wn-1] with base(rr) <= my0
      uint32_t lo = r0, hi = r0 + wn - 1;
      while (lo < hi) {
        const uint32_t mid = lo + (hi - lo + 1) / 2;
        if (base_of(mid) <= my0) lo = mid;
        else hi = mid - 1;
      }
      rr = lo;
    }
    // ---- load my items
    uint32_t d[kScanItems];
    {
      const uint4* src = reinterpret_cast<const uint4*>(&s_tile[buf][tid * kScanItems]);
#pragma unroll
      for (int q = 0; q < kScanItems / 4; ++q) {
        const uint4 v = src[q];
        d[4 * q + 0] = v.x;
        d[4 * q + 1] = v.y;
        d[4 * q + 2] = v.z;
        d[4 * q + 3] = v.w;
      }
    }
    // ---- pass 1: lat+ per valid item and the thread aggregate
    uint32_t lat[kScanItems];
    uint32_t valid = 0;  // bit per item
    uint32_t start = 0;  // bit per item: k == 0
    unsigned long long agg = 0ull;
    {
      uint32_t cur = rr;
      unsigned long long cb = base_of(cur), nb = base_of(cur + 1);
      uint32_t lim = 0, P = 1, ttft = 0;
      auto load_req = [&](uint32_t q) {
        if (q < n) {
          const uint32_t g = r.n_deliv[q];
          const uint32_t m = w.m[q];
          lim = kFinal ? g : min(g, m);
          P = r.period[q];
          ttft = r.ttft[q];
        } else {
          lim = 0;
        }
      };
      load_req(cur);
#pragma unroll
      for (int j = 0; j < kScanItems; ++j) {
        const unsigned long long pos = my0 + j;
        lat[j] = 0;
        if (pos >= pend) continue;
        while (pos >= nb) {
          ++cur;
          cb = nb;
          nb = base_of(cur + 1);
          load_req(cur);
        }
        const unsigned long long k = pos - cb;
        if (k < lim) {
          const unsigned long long I = (unsigned long long)ttft + k * P;
          const unsigned long long dd = d[j];
          const uint32_t lp = dd > I ? (uint32_t)(dd - I) : 0u;
          lat[j] = lp;
          valid |= 1u << j;
          if (k == 0) {
            start |= 1u << j;
            agg = kFlagBit | lp;
          } else {
            agg = (agg & kFlagBit) | max((uint32_t)agg, lp);
          }
        }
      }
    }
    // ---- block-wide exclusive scan of thread aggregates
    unsigned long long incl = agg;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const unsigned long long v = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= (uint32_t)o) incl = seg_combine(v, incl);
    }
    if (lane == 31) s_warp[wid] = incl;
    unsigned long long excl = __shfl_up_sync(0xffffffffu, incl, 1);
    if (lane == 0) excl = 0ull;
    __syncthreads();
    unsigned long long warp_prefix = 0ull;
    for (uint32_t q = 0; q < wid; ++q) warp_prefix = seg_combine(warp_prefix, s_warp[q]);
    excl = seg_combine(warp_prefix, excl);
    // ---- tile look-back (thread 0)
    if (tid == 0) {
      unsigned long long tile_agg = 0ull;
      for (uint32_t q = 0; q < kScanThreads / 32; ++q) tile_agg = seg_combine(tile_agg, s_warp[q]);
      unsigned long long acc = 0ull;
      if (t > 0) {
        st_release(&w.tile_status[t], kStAgg | tile_agg);
        for (int64_t j = (int64_t)t - 1; j >= 0; --j) {
          unsigned long long s;
          do {
            s = ld_acquire(&w.tile_status[j]);
          } while ((s & kStMask) == 0ull);
          acc = seg_combine(s & ~kStMask, acc);
          if ((s & kStMask) == kStPrefix || (acc & kFlagBit)) break;
        }
      }
      st_release(&w.tile_status[t], kStPrefix | seg_combine(acc, tile_agg));
      s_carry = acc;
    }
    __syncthreads();
    const unsigned long long carry = seg_combine(s_carry, excl);

    // ---- pass 2: clamped delays, per-request partial sums, edges
    {
      uint32_t cur = rr;
      unsigned long long cb = base_of(cur), nb = base_of(cur + 1);
      uint32_t g = 0, m = 0, P = 1, ttft = 0;
      int64_t trel = 0;
      auto load_req = [&](uint32_t q) {
        if (q < n) {
          g = r.n_deliv[q];
          m = kFinal ? g : w.m[q];
          P = r.period[q];
          ttft = r.ttft[q];
          if (!kFinal) trel = A.eval_abs - r.arrival[q];
        }
      };
      load_req(cur);
      uint32_t pm = (uint32_t)carry;
      unsigned long long sum = 0ull;
      bool have = false;
#pragma unroll
      for (int j = 0; j < kScanItems; ++j) {
        if (!((valid >> j) & 1u)) continue;
        const unsigned long long pos = my0 + j;
        if (pos >= nb) {
          if (have && sum) atomicAdd(&w.spre[cur], sum);
          sum = 0ull;
          have = false;
          while (pos >= nb) {
            ++cur;
            cb = nb;
            nb = base_of(cur + 1);
          }
          load_req(cur);
        }
        const uint32_t k = (uint32_t)(pos - cb);
        pm = ((start >> j) & 1u) ? lat[j] : max(pm, lat[j]);
        uint32_t dt;
        if (kFinal) {
          dt = pm;
        } else {
          const int64_t u = trel - ((int64_t)ttft + (int64_t)k * P);  // t - I_{k+1} >= 0
          dt = (int64_t)pm < u ? pm : (uint32_t)u;
        }
        sum += dt;
        have = true;
        if (!kFinal && k + 1 == g && g < m) w.edge[cur] = pm;  // delta_g
        if (k + 1 == m && g >= m) w.edge[cur] = dt;           // delta~_m (FINAL: delta_g)
      }
      if (have && sum) atomicAdd(&w.spre[cur], sum);
    }
    __syncthreads();  // buffers and window reused by the next tile
  }
}

// ---------------------------------------------------------------- qoe finalize
// S_delay / S_whole / QoE per request from K1's state (DESIGN.md "Closed forms":
// undelivered due tokens sit at t, Eq. 1-3).
__global__ void k_qoe_final(ReqView r, Work w, int64_t eval_abs, uint32_t final_mode, float* q,
                            double* q64, int64_t* sdo, int64_t* swo, uint32_t* mo) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < r.n; i += gridDim.x * blockDim.x) {
    const uint32_t g = r.n_deliv[i], m = w.m[i];
    const int64_t P = r.period[i];
    const int64_t spre = (int64_t)w.spre[i];
    int64_t sd = 0, sw = 0;
    const int64_t cw = P * (((int64_t)m * ((int64_t)m - 1)) >> 1);
    if (m == 0) {
      sd = sw = 0;
    } else if (g >= m) {
      sd = spre;
      sw = (int64_t)m * (int64_t)w.edge[i] + cw;
    } else {
      const int64_t t = eval_abs - r.arrival[i];
      const int64_t K = m - g;
      const int64_t w0 = t - (int64_t)r.ttft[i] - ((int64_t)g - 1) * P;
      sd = spre + sum_down(0, K, w0, P);
      sw = (int64_t)m * (w0 - K * P) + cw;
    }
    const double qq = qoe_value(sd, sw);
    if (q) q[i] = __double2float_rn(qq);
    if (q64) q64[i] = qq;
    if (sdo) sdo[i] = sd;
    if (swo) swo[i] = sw;
    if (mo) mo[i] = m;
  }
  (void)final_mode;
}

// ---------------------------------------------------------------- host launchers
void launch_prep(const LaunchCfg& L, const ReqView& r, const Work& w, int64_t eval_abs, bool final_mode,
                 bool sched, uint64_t kv_cap, bool debug) {
  if (r.n == 0) return;
  const uint32_t blocks = umin32((r.n + 255) / 256, L.sm_count * 8);
  k_prep<<<blocks, 256, 0, L.stream>>>(r, w, eval_abs, final_mode ? 1u : 0u, sched ? 1u : 0u, kv_cap,
                                       debug ? 1u : 0u);
}

void launch_bounds(const LaunchCfg& L, const ReqView& r, const Work& w, const uint32_t* tau, uint32_t B_cap,
                   uint64_t M, uint32_t cur_latency, uint32_t flags) {
  k_bounds<<<1, 1024, 0, L.stream>>>(r, w, tau, B_cap, M, cur_latency, flags);
}

void launch_scan(const LaunchCfg& L, const ReqView& r, const Work& w, int64_t eval_abs, bool final_mode) {
  if (r.n == 0) return;
  ScanArgs A{r, w, eval_abs};
  if (final_mode)
    k_qoe_scan<true><<<L.scan_grid, kScanThreads, 0, L.stream>>>(A);
  else
    k_qoe_scan<false><<<L.scan_grid, kScanThreads, 0, L.stream>>>(A);
}

void launch_qoe_final(const LaunchCfg& L, const ReqView& r, const Work& w, int64_t eval_abs, bool final_mode,
                      float* q, double* q64, int64_t* sd, int64_t* sw, uint32_t* m) {
  if (r.n == 0) return;
  const uint32_t blocks = umin32((r.n + 255) / 256, L.sm_count * 8);
  k_qoe_final<<<blocks, 256, 0, L.stream>>>(r, w, eval_abs, final_mode ? 1u : 0u, q, q64, sd, sw, m);
}

int scan_blocks_per_sm() {
  int b = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, k_qoe_scan<false>, kScanThreads, 0);
  int b2 = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b2, k_qoe_scan<true>, kScanThreads, 0);
  return b < b2 ? b : b2;
}

}  // namespace andes
