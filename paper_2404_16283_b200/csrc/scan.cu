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
#include <cuda.h>

#include <cstdlib>

#include "device.cuh"
#include "launch.h"

namespace andes {

// ---------------------------------------------------------------- prep (+ S0/S2 in the last CTA)
constexpr int kPrepThreads = 256;
#ifndef ANDES_TOK_UNROLL
#define ANDES_TOK_UNROLL 4
#endif
constexpr int kTokUnroll = ANDES_TOK_UNROLL;  // unroll of the aligned path's token loops
#ifndef ANDES_STATIC_PCT
#define ANDES_STATIC_PCT 95
#endif
constexpr uint32_t kStaticPct = ANDES_STATIC_PCT;  // share of the scan's chunks assigned statically

__device__ __forceinline__ void bounds_sync() { asm volatile("bar.sync 2, %0;" ::"n"(kScanThreads) : "memory"); }

// S0 selective triggering (reading R15) and S2 batch-size range (P:L545-551,
// reading R16), run by the last prep CTA once every request has been counted:
//   B_max = number of shortest contexts that fit in M (exact l histogram, overflow slow path),
//   B_min = largest B with tau(B) <= min_i P_i (only with ANDES_PRUNE), and the tau range
//   over [B_lo, B_hi] used by the gain bounds.
__device__ void bounds_block(const ReqView& r, const Work& w, const uint32_t* __restrict__ tau, uint32_t B_cap,
                             uint64_t M, uint32_t cur_latency, uint32_t flags) {
  constexpr uint32_t NT = kScanThreads, kPer = kHistL / NT;
  __shared__ unsigned long long s_cnt[NT], s_sum[NT];
  __shared__ uint32_t s_kM, s_Blo, s_tlo, s_thi;
  const uint32_t tid = threadIdx.x, n = r.n;
  const uint32_t minP = 0xFFFFFFFFu - __ldcg(&w.g->inv_minP);
  const unsigned long long run_l = __ldcg(&w.g->run_l);
  const bool trig = (flags & 1u) || (10ull * run_l > 9ull * M) || (n > 0 && cur_latency > minP);
  const uint32_t need = min(B_cap, n);
  uint32_t hv[kPer];
  unsigned long long c = 0, sm = 0;
#pragma unroll
  for (uint32_t q = 0; q < kPer; ++q) {
    const uint32_t b = tid * kPer + q;
    hv[q] = __ldcg(&w.hist_l[b]);
    if (b < kHistL - 1) {
      c += hv[q];
      sm += (unsigned long long)hv[q] * b;
    } else {
      c += hv[q];  // overflow bucket: counted, value unknown (>= kHistL - 1)
      sm += (unsigned long long)hv[q] * b;
    }
  }
  s_cnt[tid] = c;
  s_sum[tid] = sm;
  if (tid == 0) {
    s_kM = 0xFFFFFFFFu;
    s_Blo = 1;
    s_tlo = 0xFFFFFFFFu;
    s_thi = 0;
  }
  bounds_sync();
  for (uint32_t off = 1; off < NT; off <<= 1) {
    unsigned long long a = 0, b2 = 0;
    if (tid >= off) { a = s_cnt[tid - off]; b2 = s_sum[tid - off]; }
    bounds_sync();
    s_cnt[tid] += a;
    s_sum[tid] += b2;
    bounds_sync();
  }
  {
    const unsigned long long c_ex = tid ? s_cnt[tid - 1] : 0ull;
    const unsigned long long s_ex = tid ? s_sum[tid - 1] : 0ull;
    const bool crosses = (s_cnt[tid] >= need || s_sum[tid] > M) && (c_ex < need && s_ex <= M);
    if (crosses) {
      unsigned long long k = c_ex, W = s_ex;
      bool stop = false, ovf = false;
      for (uint32_t q = 0; q < kPer && !stop; ++q) {
        const uint32_t b = tid * kPer + q;
        const uint32_t h = hv[q];
        if (b == kHistL - 1 && h) { ovf = true; break; }
        // take min(h, need - k, floor((M - W) / b)) contexts of length b
        unsigned long long take = min((unsigned long long)h, need - k);
        if (b > 0) take = min(take, (M - W) / b);
        W += take * b;
        k += take;
        if (take < h) stop = true;
      }
      s_kM = ovf && !stop && k < need ? 0xFFFFFFFEu : (uint32_t)min(k, (unsigned long long)need);
    }
  }
  bounds_sync();
  uint32_t kM = s_kM == 0xFFFFFFFFu ? 0u : s_kM;
  if (kM == 0xFFFFFFFEu) {
    // Slow path: the shortest contexts reach the overflow bucket (l >= kHistL - 1); take
    // exact successive minima over all requests (rare: needs B_max contexts that long).
    __shared__ unsigned long long s_red[NT / 32], s_best;
    unsigned long long k = 0, W = 0;
    for (uint32_t b = 0; b < kHistL - 1; ++b) {
      const uint32_t h = __ldcg(&w.hist_l[b]);
      k += h;
      W += (unsigned long long)h * b;
    }
    unsigned long long last = 0;
    bool first = true;
    while (k < need) {
      unsigned long long best = ~0ull;
      for (uint32_t i = tid; i < n; i += NT) {
        const uint32_t l = r.ctx_len[i];
        if (l < kHistL - 1) continue;
        const unsigned long long key = ((unsigned long long)l << 32) | i;
        if ((first || key > last) && key < best) best = key;
      }
      for (int o = 16; o; o >>= 1) best = min(best, __shfl_xor_sync(0xffffffffu, best, o));
      if ((tid & 31) == 0) s_red[tid >> 5] = best;
      bounds_sync();
      if (tid == 0) {
        unsigned long long b2 = ~0ull;
        for (uint32_t q = 0; q < NT / 32; ++q) b2 = min(b2, s_red[q]);
        s_best = b2;
      }
      bounds_sync();
      const unsigned long long b2 = s_best;
      bounds_sync();
      if (b2 == ~0ull || W + (b2 >> 32) > M) break;
      W += b2 >> 32;
      ++k;
      last = b2;
      first = false;
    }
    kM = (uint32_t)k;
    if (tid == 0) atomicOr(&w.g->slow, 1u);
  }
  const uint32_t B_hi = min(need, kM);
  // B_min (reading R16) and the tau range of the candidate B
  if (flags & 2u) {
    uint32_t best = 1;
    for (uint32_t B = 1 + tid; B <= B_hi; B += NT)
      if (tau[B - 1] <= minP) best = max(best, B);
    atomicMax(&s_Blo, best);
  }
  bounds_sync();
  const uint32_t B_lo = (B_hi == 0) ? 1u : min(s_Blo, B_hi);
  {
    uint32_t lo = 0xFFFFFFFFu, hi = 0;
    for (uint32_t B = B_lo + tid; B <= B_hi; B += NT) {
      lo = min(lo, tau[B - 1]);
      hi = max(hi, tau[B - 1]);
    }
    atomicMin(&s_tlo, lo);
    atomicMax(&s_thi, hi);
  }
  // self-clean the l histogram for the next call
  for (uint32_t b = tid; b < kHistL; b += NT) w.hist_l[b] = 0u;
  bounds_sync();
  if (tid == 0) {
    w.g->B_hi = B_hi;
    w.g->B_lo = B_lo;
    w.g->tau_lo = s_tlo;
    w.g->tau_hi = s_thi;
    w.g->triggered = trig ? 1u : 0u;
  }
}

// One pass over the requests: m_i, zeroed accumulators, scan records, tile owners, and for a
// decision the trigger inputs (sum of running l, min period), the l histogram for B_max,
// the running list and the status-quo serve mask (bounds_block then runs in the scan's CTA 0).
// dual: also the records of a second in-flight evaluation at now_abs (the Appendix-A objectives'
// Q_now) into m_now / spre_now / edge_now / srec_now and tile_status_now; the tile descriptors
// serve both scans (a head whose tokens due at now end before a tile contributes nothing there).
__global__ void __launch_bounds__(kPrepThreads) k_prep(ReqView r, Work w, int64_t eval_abs, uint32_t final_mode,
                                                      uint32_t sched, uint64_t kv_cap, uint32_t debug,
                                                      uint8_t* __restrict__ serve_mask, int64_t now_abs,
                                                      uint32_t dual, uint32_t eval) {
  __shared__ uint32_t s_hl[kHistL];
  __shared__ uint32_t s_minP, s_maxR;
  __shared__ unsigned long long s_runl;
  const uint32_t n = r.n;
  uint32_t local_err = 0, local_unal = 0;
  pdl_wait();
  if (w.now_dev) {
    // AndesSchedParams.now_dev: the shift the call's reset kernel read (k_reset_now)
    const int64_t sh = tshift(w);
    eval_abs += sh;
    now_abs += sh;
  }
  if (blockIdx.x < 512) ANDES_TRACE(w, 7000 + 2 * blockIdx.x);
  if (sched) {
    for (uint32_t q = threadIdx.x; q < kHistL; q += blockDim.x) s_hl[q] = 0u;
    if (threadIdx.x == 0) {
      s_minP = 0xFFFFFFFFu;
      s_maxR = 0u;
      s_runl = 0;
    }
    __syncthreads();
  }
  uint32_t my_minP = 0xFFFFFFFFu, my_maxR = 0u;
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
    if (!eval) {  // (andes_qoe_eval: the scan builds its records from the request table)
      ScanRec sr;
      sr.base = r.tl_base[i];
      sr.lim = min(g, m);
      sr.P = P;
      sr.ttft = r.ttft[i];
      sr.trel = final_mode ? 0u : (uint32_t)(eval_abs - r.arrival[i]);
      sr.ek = (!final_mode && g < m) ? 1u : 2u;
      sr.pad = 0u;
      w.srec[i] = sr;
      if (dual) {
        const uint32_t mn = due_count(now_abs - r.arrival[i], sr.ttft, P ? P : 1u, r.max_total[i]);
        w.m_now[i] = mn;
        w.spre_now[i] = 0ull;
        w.edge_now[i] = 0u;
        sr.lim = min(g, mn);
        sr.trel = (uint32_t)(now_abs - r.arrival[i]);
        sr.ek = g < mn ? 1u : 2u;
        w.srec_now[i] = sr;
      }
    }
    // tile ownership: tiles whose start position p satisfies base_i <= p < base_{i+1}
    const unsigned long long base = r.tl_base[i];
    const unsigned long long next = (i + 1 < n) ? r.tl_base[i + 1] : base + g;
    const uint32_t t_lo = (i == 0) ? 0u : (uint32_t)((base + kWTile - 1) / kWTile);
    uint32_t t_hi = (uint32_t)((next + kWTile - 1) / kWTile);
    if (t_hi > w.tiles_cap) {  // pool span above limits.max_tokens: refuse (flagged), never overrun
      t_hi = w.tiles_cap;
      local_err |= kErrTokens;
    }
    for (uint32_t t = t_lo; t < t_hi; ++t) {
      // descriptor of tile t (its start position p0 lies in [base_i, base_{i+1})): first request,
      // gap flag, and the head segment's carry source (0 none, 1 direct, 2 look-back)
      const unsigned long long p0 = (unsigned long long)t * kWTile;
      TileMeta tm;
      tm.hbase = base;
      tm.r0 = i;
      uint32_t mode = 0, hcnt = 0;
      if (base < p0) {
        const unsigned long long span = p0 - base;
        const uint32_t lim = final_mode ? g : min(g, m);
        if ((unsigned long long)lim > span) {
          hcnt = (uint32_t)span;
          mode = (span <= (unsigned long long)kCarryDirect) ? 1u : 2u;
        }
      }
      tm.flags = (base > p0 ? 1u : 0u) | (mode << 1);
      tm.hcnt = hcnt;
      tm.httft = r.ttft[i];
      tm.hP = P;
      tm.pad = 0;
      w.tile_meta[t] = tm;
      w.tile_status[t] = 0ull;  // look-back status of this call (read only by the scan, after prep)
      if (dual) w.tile_status_now[t] = 0ull;
    }
    if (i + 1 == n) {
      unsigned long long pe = min(base + g, (unsigned long long)w.tiles_cap * kWTile);
      if (pe > r.tl_len) {  // pool shorter than the spans it claims: refuse (flagged), never overread
        pe = r.tl_len;
        local_err |= kErrTokens;
      }
      w.g->ntiles = (uint32_t)((pe + kWTile - 1) / kWTile);
      w.g->pool_end = pe;
    }
    if (g && (base & 3ull)) local_unal = 1u;
    if (debug) {
      if (P == 0) local_err |= kErrPeriod;
      if (i + 1 < n && next < base + g) local_err |= kErrBase;
      if (!final_mode && m >= (1u << 20)) local_err |= kErrDue;
    }
    if (sched) {
      const uint32_t l = r.ctx_len[i];
      my_minP = min(my_minP, P);
      my_maxR = max(my_maxR, r.rank[i]);
      serve_mask[i] = r.running[i] ? 1 : 0;  // status quo; the decision edits only the changes
      atomicAdd(&s_hl[l < kHistL - 1 ? l : kHistL - 1], 1u);
      if (r.running[i]) {
        atomicAdd(&s_runl, (unsigned long long)l);
        const uint32_t slot = atomicAdd(&w.g->n_run, 1u);
        if (slot < kMaxRunning) w.run_list[slot] = i;
      }
      if (debug && (l == 0 || l > kv_cap)) local_err |= kErrCtx;
    }
  }
  if (local_err) raise_err(w, local_err);
  if (__any_sync(0xffffffffu, local_unal) && (threadIdx.x & 31) == 0) atomicOr(&w.g->unal, 1u);
  if (!sched) return;
  for (int o = 16; o; o >>= 1) {
    my_minP = min(my_minP, __shfl_xor_sync(0xffffffffu, my_minP, o));
    my_maxR = max(my_maxR, __shfl_xor_sync(0xffffffffu, my_maxR, o));
  }
  if ((threadIdx.x & 31) == 0) {
    atomicMin(&s_minP, my_minP);
    atomicMax(&s_maxR, my_maxR);
  }
  __syncthreads();
  for (uint32_t q = threadIdx.x; q < kHistL; q += blockDim.x)
    if (s_hl[q]) atomicAdd(&w.hist_l[q], s_hl[q]);
  if (threadIdx.x == 0) {
    atomicMax(&w.g->inv_minP, 0xFFFFFFFFu - s_minP);
    if (s_maxR) atomicMax(&w.g->max_rank, s_maxR);
    if (s_runl) atomicAdd(&w.g->run_l, s_runl);
  }
  if (blockIdx.x < 512) ANDES_TRACE(w, 7000 + 2 * blockIdx.x + 1);
}

// ---------------------------------------------------------------- K1 timeline scan
namespace {

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
// 32-bit shared-address forms (addresses computed once per warp; no generic->shared
// conversions on the per-tile path)
__device__ __forceinline__ void mbar_expect_tx_s(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait_s(uint32_t bar, uint32_t phase) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, 1000000;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(bar),
      "r"(phase)
      : "memory");
}
__device__ __forceinline__ void st_shared_u32(uint32_t addr, uint32_t v) {
  asm volatile("st.shared.u32 [%0], %1;" ::"r"(addr), "r"(v) : "memory");
}
// TMA: one [32 rows x 32 u32] box of the pool (one warp-tile), 128-byte swizzled
__device__ __forceinline__ void tma_tile(const CUtensorMap* tmap, uint32_t dst, uint32_t row0, uint32_t bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::
          "r"(dst),
      "l"(reinterpret_cast<uint64_t>(tmap)), "r"(0), "r"(row0), "r"(bar)
      : "memory");
}
__device__ __forceinline__ uint4 ld_shared_v4(uint32_t addr) {
  uint4 v;
  asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(addr));
  return v;
}
__device__ __forceinline__ uint32_t ld_shared_u32(uint32_t addr) {
  uint32_t v;
  asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(addr));
  return v;
}

// segmented max monoid on (flag, value): combine(a, b) with a earlier than b
__device__ __forceinline__ unsigned long long seg_combine(unsigned long long a, unsigned long long b) {
  if (b & kFlagBit) return b;
  const uint32_t v = max((uint32_t)a, (uint32_t)b);
  return (a & kFlagBit) | v;
}

// The head request's carry read directly from its hcnt earlier tokens (tile descriptor mode 1,
// and the look-back's fallback): max_j (d_j - I_j)^+ with I_j = ttft + j P (readings R1-R2).
// Warp-wide; every lane returns the value.
__device__ __noinline__ uint32_t head_carry(const uint32_t* __restrict__ pool, unsigned long long hbase,
                                            uint32_t hcnt, uint32_t httft, uint32_t hP, uint32_t lane) {
  uint32_t cm = 0u;
  for (uint32_t k0 = 0; k0 < hcnt; k0 += 8 * 32) {  // 8 independent loads in flight per lane
    uint32_t d[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const uint32_t kk = k0 + u * 32 + lane;
      d[u] = kk < hcnt ? __ldg(&pool[hbase + kk]) : 0u;
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const uint32_t kk = k0 + u * 32 + lane;
      const uint32_t I = httft + kk * hP;
      if (kk < hcnt) cm = max(cm, max(d[u], I) - I);
    }
  }
  for (int o = 16; o; o >>= 1) cm = max(cm, __shfl_xor_sync(0xffffffffu, cm, o));
  return cm;
}

// Decoupled look-back for tile t (descriptor mode 2), 32 predecessors per step (lane k reads
// tile t-1-k): stop at the newest inclusive prefix or segment head, combine older-to-newer with
// a shuffle tree.  Only tiles from the one holding the head request's first token are read (that
// tile's aggregate carries the segment flag, so the walk always stops there).  Predecessors are
// claimed after t (chunks run from the pool's end), so a predecessor may belong to a warp that
// is itself waiting, or to this warp's own next tile: a wait longer than w.lb_ns (20 us unless
// ANDES_LOOKBACK_NS says otherwise) gives up and reads the head's earlier tokens directly (the
// same value), so no wait blocks forever.
__device__ __noinline__ unsigned long long lookback(const ReqView& r, const Work& w, uint32_t t, uint32_t lane) {
  const TileMeta* tmp = w.tile_meta + t;
  const unsigned long long hbase = tmp->hbase;
  const int64_t hs = (int64_t)(hbase / (unsigned long long)kWTile);
  const unsigned long long t0 = gtimer();
  unsigned long long acc = 0ull;
  for (int64_t jhi = (int64_t)t - 1;; jhi -= 32) {
    const int64_t j = jhi - (int64_t)lane;
    unsigned long long s = kStPrefix;  // before the head's first tile: not needed (empty)
    bool late = false;
    if (j >= hs) {
      while (((s = ld_relaxed(&w.tile_status[j])) & kStMask) == 0ull) {
        if (gtimer() - t0 >= (unsigned long long)w.lb_ns) {
          late = true;
          break;
        }
      }
    }
    if (__any_sync(0xffffffffu, late))
      return kFlagBit | head_carry(r.tl_pool, hbase, tmp->hcnt, tmp->httft, tmp->hP, lane);
    const bool stop = (s & kStMask) == kStPrefix || (s & kFlagBit);
    const uint32_t bal = __ballot_sync(0xffffffffu, stop);
    const uint32_t kst = bal ? (uint32_t)(__ffs(bal) - 1) : 31u;
    unsigned long long v = (lane <= kst) ? (s & ~kStMask) : 0ull;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const unsigned long long u = __shfl_down_sync(0xffffffffu, v, o);
      if (lane + o < 32) v = seg_combine(u, v);
    }
    acc = seg_combine(__shfl_sync(0xffffffffu, v, 0), acc);
    if (bal) return acc;
  }
}

// byte offset of tile-local token x in a 128B-swizzled [rows x 32] u32 tile
__device__ __forceinline__ uint32_t swz(uint32_t x) {
  const uint32_t row = x >> 5, chunk = (x >> 2) & 7u;
  return (row << 7) | ((chunk ^ (row & 7u)) << 4) | ((x & 3u) << 2);
}

// Q_now of request i (the Appendix-A objectives' QoE at the decision time, reading R3) from the
// scan at now (m_now / spre_now / edge_now), stored in qnow; returns ~(fp64 bits) for the min.
__device__ __forceinline__ unsigned long long qnow_of(const ReqView& r, const Work& w, uint32_t i, int64_t now) {
  const uint32_t g = r.n_deliv[i], m = w.m_now[i];
  const int64_t P = r.period[i];
  const int64_t spre = (int64_t)w.spre_now[i];
  const int64_t cw = P * (((int64_t)m * ((int64_t)m - 1)) >> 1);
  int64_t sd = 0, sw = 0;
  if (m == 0) {
    sd = sw = 0;
  } else if (g >= m) {
    sd = spre;
    sw = (int64_t)m * (int64_t)w.edge_now[i] + cw;
  } else {
    const int64_t t = now - r.arrival[i];
    const int64_t K = m - g;
    const int64_t w0 = t - (int64_t)r.ttft[i] - ((int64_t)g - 1) * P;
    sd = spre + sum_down(0, K, w0, P);
    sw = (int64_t)m * (w0 - K * P) + cw;
  }
  const double q = qoe_value(sd, sw);
  w.qnow[i] = q;
  return ~(unsigned long long)__double_as_longlong(q);
}

// raise the objective's Q_min (stored inverted, atomicMax) unless the word already holds it
__device__ __forceinline__ void qmin_raise(const Work& w, unsigned long long best) {
  if (best && best > __ldcg(&w.g->qmin_bits)) atomicMax(&w.g->qmin_bits, best);
}

struct ScanArgs {
  ReqView r;
  Work w;
  int64_t eval_abs;
  // decision only: S0/S2 bounds computed by CTA 0 before it joins the scan
  uint32_t sched;
  const uint32_t* tau;
  uint32_t B_cap;
  uint64_t M;
  uint32_t cur_latency, flags;
  uint32_t* tile_ctr;  // the chunk counter of this scan (a call's second scan has its own)
  uint32_t qnow;       // objectives: idle warps finish Q_now from the scan at now (k_qnow's work)
  int64_t now_abs;
};

// kEval (andes_qoe_eval): the scan builds request i's record from the request table instead of
// reading prep's copy (srec): the request-table fields are loaded one unit ahead (RawRec) and
// converted when the unit is processed, so the prefetch never waits for its loads.
struct RawRec {
  unsigned long long base;
  long long arr;
  uint32_t g, P, ttft, mt;
};
template <bool kFinal>
__device__ __forceinline__ RawRec raw_of(const ReqView& r, uint32_t i) {
  RawRec x;
  x.base = r.tl_base[i];
  x.g = r.n_deliv[i];
  x.P = r.period[i];
  x.ttft = r.ttft[i];
  x.arr = kFinal ? 0ll : r.arrival[i];
  x.mt = kFinal ? 0u : r.max_total[i];
  return x;
}
// prep's record (k_prep, the same arithmetic)
template <bool kFinal>
__device__ __forceinline__ ScanRec rec_from_raw(int64_t eval_abs, const RawRec& x) {
  ScanRec s;
  s.base = x.base;
  s.P = x.P;
  s.ttft = x.ttft;
  s.pad = 0u;
  uint32_t m;
  if (kFinal) {
    m = x.g;
    s.trel = 0u;
    s.ek = 2u;
  } else {
    const int64_t t = eval_abs - x.arr;
    m = due_count(t, x.ttft, x.P ? x.P : 1u, x.mt);
    s.trel = (uint32_t)t;
    s.ek = x.g < m ? 1u : 2u;
  }
  s.lim = min(x.g, m);
  return s;
}
template <bool kEval, bool kFinal>
__device__ __forceinline__ ScanRec rec_of(const ScanArgs& A, uint32_t i) {
  if constexpr (kEval) return rec_from_raw<kFinal>(A.eval_abs, raw_of<kFinal>(A.r, i));
  else return A.w.srec[i];
}
template <bool kEval>
struct PipeRec {
  using T = ScanRec;
};
template <>
struct PipeRec<true> {
  using T = RawRec;
};

// One request of a tile's window in tile-local coordinates (x = position - p0).
struct Entry {
  int32_t ls;     // local start (base - p0), clamped to [-1, kWTile + 1]
  int32_t vend;   // local end of the valid tokens (base + lim - p0), clamped to [-1, kWTile]
  uint32_t A;     // ideal time of local position 0: ttft + (p0 - base) P (mod 2^32); I(x) = A + x P
  uint32_t trel;  // t - arrival: clamp of the consumption times (R3)
  uint32_t P;
  uint32_t ek;    // edge kind (1 = delta_g, 2 = delta~_m) when the last valid token is in this tile, else 0
  uint32_t ridx;  // request index (0xFFFFFFFF: dummy / sentinel)
  uint32_t pad;
};
static_assert(sizeof(Entry) == 32, "Entry is two 16-byte shared-memory vectors");

template <int kT = kWTile>
__device__ __forceinline__ Entry entry_of(const ScanRec& s, uint32_t ri, unsigned long long p0) {
  Entry e;
  const long long ls = (long long)s.base - (long long)p0;
  const long long ve = ls + (long long)s.lim;
  e.ls = (int32_t)max(-1ll, min(ls, (long long)kT + 1));
  e.vend = (int32_t)max(-1ll, min(ve, (long long)kT));
  e.A = s.ttft + (uint32_t)(unsigned long long)(-ls) * s.P;
  e.trel = s.trel;
  e.pad = 0;
  e.P = s.P;
  e.ek = (ve >= 1 && ve <= (long long)kT) ? s.ek : 0u;
  e.ridx = ri;
  return e;
}

__device__ __forceinline__ Entry null_entry(bool sentinel) {
  Entry e;
  e.ls = sentinel ? kWTile + 1 : -1;
  e.vend = -1;
  e.A = 0; e.trel = 0; e.P = 0; e.ek = 0; e.ridx = 0xFFFFFFFFu; e.pad = 0;
  return e;
}

// Window = requests r0 .. r0+wn-1-dummy overlapping the tile (entry 0 is a dummy when a gap
// precedes r0), from their raw scan records (warp-staged in shared memory, or global memory
// when the tile overlaps more than kWWinCap requests).
template <bool kEval, bool kFinal>
struct RawWin {
  const ScanArgs* A;
  unsigned long long p0;
  uint32_t r0, dummy, wn;
  __device__ __forceinline__ int32_t start(uint32_t q) const {
    if (q >= wn) return kWTile + 1;
    if (dummy && q == 0) return -1;
    const unsigned long long base = kEval ? A->r.tl_base[r0 + q - dummy] : A->w.srec[r0 + q - dummy].base;
    const long long ls = (long long)base - (long long)p0;
    return (int32_t)max(-1ll, min(ls, (long long)kWTile + 1));
  }
  __device__ __forceinline__ Entry get(uint32_t q) const {
    if (q >= wn || (dummy && q == 0)) return null_entry(q >= wn);
    return entry_of(rec_of<kEval, kFinal>(*A, r0 + q - dummy), r0 + q - dummy, p0);
  }
};

// One warp-tile: 32 lanes x 32 tokens.  Tokens of request q at local position x have ideal
// time I(x) = e.A + x P; the actual consumption time follows A_x = max(d_x, A_{x-1} + P)
// (reading R2) and is clamped at t (R3).  Pass 1 builds the segmented max of lat+ (the carry
// monoid), pass 2 sums T~ per piece and subtracts the closed-form sum of I.

template <bool kFinal, class Win>
__device__ __forceinline__ unsigned long long warp_tile(const ScanArgs& A, const Win& win, uint32_t tile_s, uint32_t wn,
                                                        uint32_t t, uint32_t mode, uint32_t cdirect, uint32_t swz_on) {
  const Work& w = A.w;
  const uint32_t lane = threadIdx.x & 31;
  const int32_t x0 = (int32_t)(lane * kScanItems);
  uint32_t q0;
  {
    uint32_t lo = 0, hi = wn - 1;
    while (lo < hi) {
      const uint32_t mid = (lo + hi + 1) >> 1;
      if (win.start(mid) <= x0) lo = mid;
      else hi = mid - 1;
    }
    q0 = lo;
  }
  const uint32_t rowb = tile_s + (lane << 7), rsw = swz_on ? (lane & 7u) : 0u;  // plain tiles: no XOR
  const Entry e0 = win.get(q0);
  const bool starts_here = e0.ls == x0;
  // Pieces that start in this row are final after one pass.  The row's first piece, when it
  // continues a request from an earlier row, is computed with zero carry-in; its sum and edge
  // are held back until the carry is known and recomputed only if the carry is non-zero
  // (A_x = max(Z_x, I_x + c), Z the zero-carry recurrence).
  const bool held = !starts_here && x0 < e0.vend;
  unsigned long long h_sum = 0ull;
  int32_t h_xe = x0;
  uint32_t h_edge = 0u;  // edge value of the held piece (valid when its vend is in this row)
  bool h_has_edge = false;

  auto flush = [&](const Entry& e, int32_t xs, int32_t xe, unsigned long long sumT) {
    const uint32_t nn = (uint32_t)(xe - xs);
    const uint32_t Is = e.A + (uint32_t)xs * e.P;
    const unsigned long long sumI =
        (unsigned long long)nn * Is + (unsigned long long)e.P * (((unsigned long long)nn * (nn - 1)) >> 1);
    const unsigned long long d = sumT - sumI;
    if (d) atomicAdd(&w.spre[e.ridx], d);
  };
  auto edge_val = [&](const Entry& e, uint32_t Acur, uint32_t tcl) -> uint32_t {
    const uint32_t Il = e.A + (uint32_t)(e.vend - 1) * e.P;
    return (e.ek == 1u) ? Acur - Il : min(Acur, tcl) - Il;
  };

  unsigned long long agg;
  {
    Entry e = e0;
    uint32_t q = q0;
    int32_t ns = win.start(q + 1);
    bool live = x0 < e.vend;
    bool first = held;
    uint32_t P = live ? e.P : 0u;
    uint32_t tcl = live ? (kFinal ? 0xFFFFFFFFu : e.trel) : 0u;
    uint32_t Acur = e.A + (uint32_t)x0 * e.P - e.P;  // zero-carry baseline I(x0) - P
    uint32_t flag = starts_here ? 1u : 0u, vfz = 0;
    int32_t xs = x0;
    unsigned long long sumT = 0ull;
    int32_t ev = live ? min(e.vend, ns) : ns;
#pragma unroll 1
    for (uint32_t g = 0; g < kScanItems / 4; ++g) {
      const uint4 dv = ld_shared_v4(rowb | ((g ^ rsw) << 4));
      const int32_t gx = x0 + (int32_t)(4 * g);
      if (ev - gx >= 4) {
        Acur = max(Acur + P, dv.x);
        sumT += min(Acur, tcl);
        Acur = max(Acur + P, dv.y);
        sumT += min(Acur, tcl);
        Acur = max(Acur + P, dv.z);
        sumT += min(Acur, tcl);
        Acur = max(Acur + P, dv.w);
        sumT += min(Acur, tcl);
        continue;
      }
      const uint32_t dd[4] = {dv.x, dv.y, dv.z, dv.w};
#pragma unroll
      for (int jj = 0; jj < 4; ++jj) {
        const int32_t x = gx + jj;
        if (x == ev) {
          if (live && x == e.vend) {
            const uint32_t ev_val = e.ek ? edge_val(e, Acur, tcl) : 0u;
            if (first) {
              h_sum = sumT;
              h_xe = x;
              h_has_edge = e.ek != 0u;
              h_edge = ev_val;
              first = false;
            } else {
              flush(e, xs, x, sumT);
              if (e.ek) w.edge[e.ridx] = ev_val;
            }
            vfz = Acur - (e.A + (uint32_t)(x - 1) * e.P);
            live = false;
            P = 0;
            tcl = 0;
          }
          if (x == ns) {
            do {
              ++q;
              ns = win.start(q + 1);
            } while (ns <= x);
            e = win.get(q);
            live = x < e.vend;
            P = live ? e.P : 0u;
            tcl = live ? (kFinal ? 0xFFFFFFFFu : e.trel) : 0u;
            Acur = e.A + (uint32_t)x * e.P - e.P;
            xs = x;
            sumT = 0ull;
            flag = 1u;
            vfz = 0;
          }
          ev = live ? min(e.vend, ns) : ns;
        }
        Acur = max(Acur + P, dd[jj]);
        sumT += min(Acur, tcl);
      }
    }
    const int32_t xe = x0 + kScanItems;
    if (live) {
      const bool has_edge = e.vend == xe && e.ek;
      const uint32_t ev_val = has_edge ? edge_val(e, Acur, tcl) : 0u;
      if (first) {
        h_sum = sumT;
        h_xe = xe;
        h_has_edge = has_edge;
        h_edge = ev_val;
      } else {
        flush(e, xs, xe, sumT);
        if (has_edge) w.edge[e.ridx] = ev_val;
      }
    }
    const uint32_t v = live ? Acur - (e.A + (uint32_t)(xe - 1) * e.P) : vfz;
    agg = (flag ? kFlagBit : 0ull) | v;
  }
  // ---- warp scan + tile carry
  unsigned long long incl = agg;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const unsigned long long v = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= (uint32_t)o) incl = seg_combine(v, incl);
  }
  unsigned long long excl = __shfl_up_sync(0xffffffffu, incl, 1);
  if (lane == 0) excl = 0ull;
  const unsigned long long tile_agg = __shfl_sync(0xffffffffu, incl, 31);
  unsigned long long acc = 0ull;
  if (mode == 2u) {
    // decoupled look-back, 32 predecessors per step (lane k reads tile t-1-k): stop at the
    // newest inclusive prefix or segment head; combine older-to-newer with a shuffle tree
    if (lane == 0) st_relaxed(&w.tile_status[t], kStAgg | tile_agg);
    acc = lookback(A.r, w, t, lane);
  } else if (mode == 1u) {
    acc = kFlagBit | cdirect;
  }
  const unsigned long long prefix = seg_combine(acc, tile_agg);
  if (lane == 0) st_relaxed(&w.tile_status[t], kStPrefix | prefix);
  const uint32_t carry = (uint32_t)seg_combine(acc, excl);

  // ---- the held first piece, now that its carry-in is known
  if (held) {
    if (carry != 0u) {
      const uint32_t P = e0.P;
      const uint32_t tcl = kFinal ? 0xFFFFFFFFu : e0.trel;
      uint32_t Acur = e0.A + (uint32_t)x0 * P - P + carry;
      unsigned long long sumT = 0ull;
      const uint32_t nh = (uint32_t)(h_xe - x0);  // 1..32 tokens
#pragma unroll 1
      for (uint32_t g = 0; 4 * g < nh; ++g) {
        const uint4 dv = ld_shared_v4(rowb | ((g ^ rsw) << 4));
        const uint32_t dd[4] = {dv.x, dv.y, dv.z, dv.w};
#pragma unroll
        for (int jj = 0; jj < 4; ++jj) {
          if (4 * g + jj < nh) {
            Acur = max(Acur + P, dd[jj]);
            sumT += min(Acur, tcl);
          }
        }
      }
      h_sum = sumT;
      if (h_has_edge) h_edge = edge_val(e0, Acur, tcl);
    }
    flush(e0, x0, h_xe, h_sum);
    if (h_has_edge) w.edge[e0.ridx] = h_edge;
  }
  return prefix;
}

// ---- aligned fast path: every request starting in the tile starts on a 16-byte boundary
// (token index multiple of 4), so every 4-token group belongs to one request.  The tile's valid
// tokens are cut into pieces (request ∩ tile, up to its valid end) and the pieces into
// sub-ranges of SR tokens (SR chosen per tile so that <= 32 sub-ranges exist); lane u owns
// sub-range u, so no lane ever meets a request boundary (no event path, no divergence):
//   pass 1  zero-carry recurrence over the sub-range -> its lateness at the last token (tokens
//           past the valid end read as d = 0, which keeps the lateness constant);
//   scan    segmented max over the sub-ranges (flag = a piece that starts in the tile), seeded
//           with the tile's carry-in -> every sub-range's exact carry;
//   pass 2  the recurrence again from the carry: sum of T~ = min(A, t) over the valid tokens,
//           the edge value at the request's last valid token, one 64-bit atomic per sub-range.
// Returns false (nothing done) when the tile has too many pieces for one round.
// e: this lane's request of the tile (lane q = request r0 + q, q < wn <= 24, zero-length ones
// included), in tile-local coordinates.
// A dense tile is processed in batches of up to 31 requests (first_batch / last_batch): the
// running prefix seeds the next batch (mode 1); only a single-batch tile publishes its aggregate
// early, and only the last batch publishes the tile's prefix (both only when pub: a look-back
// can reach this tile).  Modes 0 and 1 only: a tile that
// looks back (mode 2) takes the row path.
// Sub-range length SR(np) of the aligned path for np pieces in a tile: sum ceil(len/SR) <=
// kWTile/SR + np <= 32, and SR is an odd number of 16-byte chunks (the sub-ranges of one piece
// then start in distinct shared-memory banks); mg = ceil(2^32 / SR), so that ceil(x / SR) =
// umulhi(x + SR - 1, mg) exactly for x < 2^32 / SR (here x <= 2 kWTile).
struct SubRangeTab {
  uint32_t sr[33], mg[33];
};
constexpr SubRangeTab make_subrange_tab(uint32_t tokens = kWTile) {
  SubRangeTab t{};
  for (uint32_t np = 0; np <= 32; ++np) {
    const uint32_t d = np < 32 ? 32u - np : 1u;
    const uint32_t sr = 4u * (((tokens / 4u + d - 1u) / d) | 1u);
    t.sr[np] = sr;
    t.mg[np] = (uint32_t)((0x100000000ull + sr - 1u) / sr);
  }
  return t;
}
__constant__ SubRangeTab kSubRange = make_subrange_tab();
__constant__ SubRangeTab kSubRange2 = make_subrange_tab(2 * kWTile);  // two-tile units
static_assert(make_subrange_tab(2 * kWTile).sr[31] <= 4 * kWTile, "SR table (2 tiles)");
static_assert(make_subrange_tab().sr[31] <= 2 * kWTile && make_subrange_tab().sr[0] == 4u * 9u, "SR table");

template <bool kFinal, int TW = 1, bool kHead = false>
__device__ __forceinline__ void warp_tile_aligned(const ScanArgs& A, const Entry& e, uint32_t tile_s, uint32_t t,
                                                  uint32_t mode, uint32_t cdirect, unsigned long long& prefix,
                                                  bool first_batch, bool last_batch, bool pub) {
  const Work& w = A.w;
  const uint32_t lane = threadIdx.x & 31;
  constexpr int32_t kT = TW * kWTile;  // tokens of the unit (TW warp-tiles)
  const int32_t ps = max(e.ls, 0), pe = max(ps, min(e.vend, kT));
  const uint32_t len = (uint32_t)(pe - ps);
  const uint32_t np = __popc(__ballot_sync(0xffffffffu, len != 0u));
  // sub-range length from the table (no division on the hot path): <= 32 sub-ranges in total
  const uint32_t SR = TW == 1 ? kSubRange.sr[np] : kSubRange2.sr[np];
  const uint32_t cnt = __umulhi(len + SR - 1u, TW == 1 ? kSubRange.mg[np] : kSubRange2.mg[np]);  // ceil(len / SR)
  uint32_t incl = cnt;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t v = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= (uint32_t)o) incl += v;
  }
  const uint32_t U = __shfl_sync(0xffffffffu, incl, 31);
  // sub-range u = lane: its piece q = first entry with incl[q] > u
  const uint32_t u = lane;
  uint32_t q = 0;
#pragma unroll
  for (uint32_t st = 16; st; st >>= 1) {
    const uint32_t v = __shfl_sync(0xffffffffu, incl, q + st - 1);
    if (v <= u) q += st;
  }
  q = min(q, 31u);
  const bool active = u < U;
  // the piece's parameters from its lane (ls and the edge kind share one word)
  const uint32_t q_off = __shfl_sync(0xffffffffu, incl - cnt, q);
  const uint32_t qA = __shfl_sync(0xffffffffu, e.A, q), qP = __shfl_sync(0xffffffffu, e.P, q);
  const uint32_t qtrel = __shfl_sync(0xffffffffu, e.trel, q);
  const uint32_t qridx = __shfl_sync(0xffffffffu, e.ridx, q);
  const int32_t qvend = __shfl_sync(0xffffffffu, e.vend, q);
  const uint32_t lsek = __shfl_sync(0xffffffffu, ((uint32_t)(e.ls + 1) << 2) | e.ek, q);
  const int32_t qls = (int32_t)(lsek >> 2) - 1;
  const uint32_t qek = lsek & 3u;
  const int32_t q_ps = max(qls, 0), q_pe = max(q_ps, min(qvend, kT));
  const uint32_t k = u - q_off;
  const int32_t xs = active ? q_ps + (int32_t)(SR * k) : 0;
  const int32_t xe = active ? min(xs + (int32_t)SR, q_pe) : 0;
  const uint32_t P = active ? qP : 0u;
  const uint32_t tcl = kFinal ? 0xFFFFFFFFu : qtrel;
  // kHead (unaligned timelines: a piece may start inside a 4-token group): the sub-range's first
  // hn <= 3 tokens, up to the next 16-byte boundary, form a head group processed first
  uint32_t hn = 0, h0 = 0, h1 = 0, h2 = 0;
  int32_t xa = xs;
  if constexpr (kHead) {
    const uint32_t mis = (uint32_t)xs & 3u;
    hn = (active && mis) ? min(4u - mis, (uint32_t)(xe - xs)) : 0u;
    if (hn) {
      const uint4 v = ld_shared_v4(tile_s + (((uint32_t)xs >> 2) << 4));
      h0 = mis == 1u ? v.y : mis == 2u ? v.z : v.w;
      h1 = mis == 1u ? v.z : v.w;
      h2 = v.w;
    }
    xa = xs + (int32_t)hn;
  }
  // full 4-token groups of the sub-range, then at most one partial group (the valid end)
  const uint32_t nfull = active ? (uint32_t)(xe - xa) >> 2 : 0u;
  const uint32_t ntail = active ? (uint32_t)(xe - xa) & 3u : 0u;
  const uint32_t gmax = __reduce_max_sync(0xffffffffu, nfull);
  const uint32_t Is = qA + (uint32_t)xs * P;  // ideal time of the sub-range's first token
  // the tile is in plain row-major layout here (no swizzle): chunk c at tile_s + 16 c
  const uint32_t a0 = tile_s + (((uint32_t)xa >> 2) << 4);
  // the tail group's tokens (loaded once, used by both passes); missing tokens read as 0
  uint32_t t0 = 0, t1 = 0, t2 = 0;
  if (ntail) {
    const uint4 v = ld_shared_v4(a0 + (nfull << 4));
    t0 = v.x;
    t1 = ntail > 1 ? v.y : 0u;
    t2 = ntail > 2 ? v.z : 0u;
  }
  // ---- pass 1: zero-carry lateness at the sub-range's end.  The groups every active lane has
  // (gi < nmin, warp-uniform) run unpredicated; the few that only some lanes have, predicated.
  const uint32_t nmin = min(gmax, __reduce_min_sync(0xffffffffu, active ? nfull : 0xFFFFFFFFu));
  uint32_t a = Is - P;
  // Two-tile units (large pools) and FINAL mode: pass 1 also sums the zero-carry consumption
  // times A(0) over the valid tokens (mod 2^32), and pass 2 is skipped wherever the carry and the
  // clamp at t allow a closed form or that sum (below).
  // One-tile units (the decision's 64K-request scan) keep the plain two passes: there the extra
  // pass-1 work measured slower (decision +1 us) than the skipped pass saves.
#ifndef ANDES_NO_P2SKIP
  constexpr bool kSkip = TW == 2 || kFinal;
#else
  constexpr bool kSkip = false;
#endif
  uint32_t s0 = 0u, d1 = 0u;  // (kSkip) the zero-carry sum; the sub-range's first token
  // kUnc: pass 1 sums A(0) unclamped (two adds per four tokens instead of four mins more); the
  // sum is then used only where no token of the sub-range reaches past t (below).
  // ANDES_CLAMPED_S0: the clamped sum min(A(0), t) instead (A/B)
#ifndef ANDES_CLAMPED_S0
  constexpr bool kUnc = true;
#else
  constexpr bool kUnc = false;
#endif
  auto cl = [&](uint32_t x) -> uint32_t { return kUnc ? x : min(x, tcl); };
  if constexpr (kSkip) {
    d1 = active ? ld_shared_u32(tile_s + ((uint32_t)xs << 2)) : 0u;
    if (kHead && hn) {
      a = max(a + P, h0);
      s0 = cl(a);
      if (hn > 1u) {
        a = max(a + P, h1);
        s0 += cl(a);
      }
      if (hn > 2u) {
        a = max(a + P, h2);
        s0 += cl(a);
      }
    }
#pragma unroll kTokUnroll
    for (uint32_t gi = 0; gi < nmin; ++gi) {
      const uint4 v = ld_shared_v4(a0 + (gi << 4));
      const uint32_t A0 = max(a + P, v.x), A1 = max(A0 + P, v.y), A2 = max(A1 + P, v.z), A3 = max(A2 + P, v.w);
      a = A3;
      s0 += cl(A0) + cl(A1) + cl(A2) + cl(A3);
    }
    for (uint32_t gi = nmin; gi < gmax; ++gi) {
      if (gi < nfull) {
        const uint4 v = ld_shared_v4(a0 + (gi << 4));
        const uint32_t A0 = max(a + P, v.x), A1 = max(A0 + P, v.y), A2 = max(A1 + P, v.z), A3 = max(A2 + P, v.w);
        a = A3;
        s0 += cl(A0) + cl(A1) + cl(A2) + cl(A3);
      }
    }
    if (ntail) {
      const uint32_t A0 = max(a + P, t0), A1 = max(A0 + P, t1), A2 = max(A1 + P, t2);
      s0 += cl(A0) + (ntail > 1 ? cl(A1) : 0u) + (ntail > 2 ? cl(A2) : 0u);
      a = A2;
    }
  } else {
    if (kHead && hn) {
      a = max(a + P, h0);
      if (hn > 1u) a = max(a + P, h1);
      if (hn > 2u) a = max(a + P, h2);
    }
#pragma unroll kTokUnroll
    for (uint32_t gi = 0; gi < nmin; ++gi) {
      const uint4 v = ld_shared_v4(a0 + (gi << 4));
      a = max(a + P, v.x);
      a = max(a + P, v.y);
      a = max(a + P, v.z);
      a = max(a + P, v.w);
    }
    for (uint32_t gi = nmin; gi < gmax; ++gi) {
      if (gi < nfull) {
        const uint4 v = ld_shared_v4(a0 + (gi << 4));
        a = max(a + P, v.x);
        a = max(a + P, v.y);
        a = max(a + P, v.z);
        a = max(a + P, v.w);
      }
    }
    if (ntail) {
      a = max(a + P, t0);
      a = max(a + P, t1);
      a = max(a + P, t2);
    }
  }
  const uint32_t nslots = hn + 4u * nfull + (ntail ? 3u : 0u);  // processed token slots
  const uint32_t dz = nslots ? a - (Is + (nslots - 1u) * P) : 0u;
  // a request starts in this sub-range; idle lanes (after every sub-range) are the identity
  const bool flag = active && k == 0 && qls >= 0;
  // warp segmented max-scan on 32-bit values, the segment flags in a ballot: lane i's inclusive
  // value is the max over lanes [s_i, i], s_i the last flagged lane <= i (0 if none)
  const uint32_t F = __ballot_sync(0xffffffffu, flag);
  const uint32_t fb = F & (0xFFFFFFFFu >> (31u - lane));  // flags of lanes 0..lane
  const int32_t sgs = fb ? 31 - __clz(fb) : -1;
  uint32_t sv = dz;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t u = __shfl_up_sync(0xffffffffu, sv, o);
    if ((int32_t)lane - o >= sgs) sv = max(sv, u);
  }
  uint32_t excl_v = __shfl_up_sync(0xffffffffu, sv, 1);
  if (lane == 0) excl_v = 0u;
  const bool excl_flag = (F & ((1u << lane) - 1u)) != 0u;  // a segment starts in lanes 0..lane-1
  const unsigned long long tile_agg =
      (F ? kFlagBit : 0ull) | (unsigned long long)__shfl_sync(0xffffffffu, sv, 31);
  // ---- the tile's carry-in (direct read or decoupled look-back), as in warp_tile; the aggregate
  // is published first so that successors looking back never wait on this tile's second pass
  // (a unit of TW tiles publishes into each of its tiles' words: a look-back combines with max,
  // so seeing the same unit twice is harmless)
  if (pub && first_batch && last_batch && lane < (uint32_t)TW) st_relaxed(&w.tile_status[t + lane], kStAgg | tile_agg);
  unsigned long long acc = 0ull;
  // (a tile that looks back (mode 2) takes the row path: this one sees modes 0 and 1 only)
  if (mode == 1u) acc = kFlagBit | cdirect;
  prefix = seg_combine(acc, tile_agg);
  if (pub && last_batch && lane < (uint32_t)TW) st_relaxed(&w.tile_status[t + lane], kStPrefix | prefix);
  const uint32_t carry = flag ? 0u : excl_flag ? excl_v : max((uint32_t)acc, excl_v);
  // ---- pass 2: consumption times from the carry, sums, edge.
  // Sum of T~ = min(A, t) over the sub-range.  Only S = sum(T~ - I) is needed, and every term is
  // at most the lateness at the sub-range's last token, max(dz, carry) (the lateness max is
  // nondecreasing): when nn * max(dz, carry) < 2^32 for every lane (warp-uniform), the sums run
  // in 32-bit arithmetic modulo 2^32 and S = (sum T~ - sum I) mod 2^32 is exact; else 64-bit.
  uint32_t Ac = Is - P + carry;
  const uint32_t nn_all = active ? (uint32_t)max(xe - xs, 0) : 0u;
  const bool fits32 = __all_sync(0xffffffffu, (unsigned long long)nn_all * max(dz, carry) < (1ull << 32));
  if (kSkip && fits32) {
    // The lateness with carry c is max(c, L(0)), L(0) the zero-carry lateness (nondecreasing from
    // L1 at the first token to dz at the last), so per lane:
    //   c >= dz   A(c) = I + c at every token: closed form, the clamp point by one division
    //             (with c replaced by dz when L(0) is constant);
    //   c <= L1   A(c) = A(0) at every token: the sum is pass 1's s0;
    //   else      A(c) = A(0) from the first token with A(0) >= I + c on: walk up to it only,
    //             correcting s0 by min(I + c, t) - min(A(0), t) per token.
    // With the unclamped s0 (kUnc) the last two need every token consumed by t (the last one's
    // consumption I_last + max(c, dz) <= t); a lane where some token clamps walks its sub-range
    // with the carry instead (pass 2 for that lane only).
    // (warp-uniform branch: fits32 bounds every sum below 2^32, as for pass 2)
    const uint32_t L1 = max(d1, Is) - Is;
    const uint32_t Ilast = Is + (nn_all ? nn_all - 1u : 0u) * P;
    // (also when the zero-carry lateness is constant, L1 == dz: then A(c) = I + max(c, dz) at
    // every token -- e.g. a request's first sub-range with its later tokens delivered ahead)
    const bool cb = carry >= dz || L1 >= dz;
    const uint32_t Lc = max(carry, dz);
    const bool clampfree = !kUnc || kFinal || Ilast + max(carry, dz) <= tcl;
    const bool ca = !cb && carry <= L1;
    bool need = nn_all != 0u && !cb && !ca && clampfree;
    bool full = kUnc && !kFinal && nn_all != 0u && !cb && !clampfree;
    const bool fw = full;
    uint32_t fix = 0u, sumc = 0u;
    if (__any_sync(0xffffffffu, need)) {
      uint32_t A0 = Is - P, Ic = Is - P + carry, x = (uint32_t)xs;
      while (__any_sync(0xffffffffu, need)) {
        if (need) {
          const uint32_t d = ld_shared_u32(tile_s + (x << 2));
          A0 = max(A0 + P, d);
          Ic += P;
          if (A0 >= Ic) {
            need = false;
          } else {
            fix += cl(Ic) - cl(A0);
            need = ++x < (uint32_t)xe;
          }
        }
      }
    }
    if (kUnc && !kFinal && __any_sync(0xffffffffu, full)) {
      uint32_t Ac = Is - P + carry, x = (uint32_t)xs;
      while (__any_sync(0xffffffffu, full)) {
        if (full) {
          Ac = max(Ac + P, ld_shared_u32(tile_s + (x << 2)));
          sumc += min(Ac, tcl);
          full = ++x < (uint32_t)xe;
        }
      }
    }
    if (nn_all) {
      const uint32_t nn = nn_all;
      unsigned long long dsum;
      if (cb) {
        const uint32_t b0 = Is + Lc;  // consumption time of the first token
        uint32_t k;                      // tokens consumed by t
        if (b0 + (nn - 1u) * P <= tcl) k = nn;
        else if (b0 > tcl) k = 0u;
        else k = min(nn, (tcl - b0) / P + 1u);
        const unsigned long long kk = k, n2 = nn;
        dsum = kk * Lc + (n2 - kk) * (unsigned long long)(tcl - Is) -
               (unsigned long long)P * (((n2 * (n2 - 1ull)) >> 1) - ((kk * (kk - 1ull)) >> 1));
      } else {
        const unsigned long long sumI =
            (unsigned long long)nn * Is + (unsigned long long)P * (((unsigned long long)nn * (nn - 1)) >> 1);
        dsum = (unsigned long long)(uint32_t)((fw ? sumc : s0 + fix) - (uint32_t)sumI);
      }
      if (dsum) atomicAdd(&w.spre[qridx], dsum);
      if (qek && xe == qvend) {
        const uint32_t Il = qA + (uint32_t)(xe - 1) * P;
        const uint32_t A_last = Il + max(carry, dz);
        w.edge[qridx] = (qek == 1u) ? A_last - Il : min(A_last, tcl) - Il;
      }
    }
    return;
  }
#ifndef ANDES_NO_NOCLAMP
  // consumption times are nondecreasing, so the clamp min(A, t) is void for the whole warp when
  // every lane's last one, I_last + max(L_end, carry), is <= t (warp-uniform loop choice)
  const uint32_t A_hi = Is + (uint32_t)max(xe - xs - 1, 0) * P + max(dz, carry);
  const bool noclamp = kFinal || __all_sync(0xffffffffu, !active || A_hi <= tcl);
#else
  const bool noclamp = kFinal;
#endif
  unsigned long long sumT = 0ull;
  uint32_t sum32 = 0u;
  if (kHead && hn) {  // the head group (clamped: min(A, t) = A whenever the clamp is void)
    Ac = max(Ac + P, h0);
    unsigned long long hs = min(Ac, tcl);
    if (hn > 1u) {
      Ac = max(Ac + P, h1);
      hs += min(Ac, tcl);
    }
    if (hn > 2u) {
      Ac = max(Ac + P, h2);
      hs += min(Ac, tcl);
    }
    sumT = hs;
    sum32 = (uint32_t)hs;
  }
  if (fits32) {
    if (noclamp) {
#pragma unroll kTokUnroll
      for (uint32_t gi = 0; gi < nmin; ++gi) {
        const uint4 v = ld_shared_v4(a0 + (gi << 4));
        const uint32_t A0 = max(Ac + P, v.x), A1 = max(A0 + P, v.y), A2 = max(A1 + P, v.z), A3 = max(A2 + P, v.w);
        Ac = A3;
        sum32 += A0 + A1 + A2 + A3;
      }
      for (uint32_t gi = nmin; gi < gmax; ++gi) {
        if (gi < nfull) {
          const uint4 v = ld_shared_v4(a0 + (gi << 4));
          const uint32_t A0 = max(Ac + P, v.x), A1 = max(A0 + P, v.y), A2 = max(A1 + P, v.z), A3 = max(A2 + P, v.w);
          Ac = A3;
          sum32 += A0 + A1 + A2 + A3;
        }
      }
    } else {
#pragma unroll kTokUnroll
      for (uint32_t gi = 0; gi < nmin; ++gi) {
        const uint4 v = ld_shared_v4(a0 + (gi << 4));
        const uint32_t A0 = max(Ac + P, v.x), A1 = max(A0 + P, v.y), A2 = max(A1 + P, v.z), A3 = max(A2 + P, v.w);
        Ac = A3;
        sum32 += min(A0, tcl) + min(A1, tcl) + min(A2, tcl) + min(A3, tcl);
      }
      for (uint32_t gi = nmin; gi < gmax; ++gi) {
        if (gi < nfull) {
          const uint4 v = ld_shared_v4(a0 + (gi << 4));
          const uint32_t A0 = max(Ac + P, v.x), A1 = max(A0 + P, v.y), A2 = max(A1 + P, v.z), A3 = max(A2 + P, v.w);
          Ac = A3;
          sum32 += min(A0, tcl) + min(A1, tcl) + min(A2, tcl) + min(A3, tcl);
        }
      }
    }
  } else if (noclamp) {
#pragma unroll kTokUnroll
    for (uint32_t gi = 0; gi < gmax; ++gi) {
      if (gi < nfull) {
        const uint4 v = ld_shared_v4(a0 + (gi << 4));
        const uint32_t A0 = max(Ac + P, v.x), A1 = max(A0 + P, v.y), A2 = max(A1 + P, v.z), A3 = max(A2 + P, v.w);
        Ac = A3;
        sumT += (unsigned long long)A0 + A1 + A2 + A3;
      }
    }
  } else {
#pragma unroll kTokUnroll
    for (uint32_t gi = 0; gi < gmax; ++gi) {
      if (gi < nfull) {
        const uint4 v = ld_shared_v4(a0 + (gi << 4));
        const uint32_t A0 = max(Ac + P, v.x), A1 = max(A0 + P, v.y), A2 = max(A1 + P, v.z), A3 = max(A2 + P, v.w);
        Ac = A3;
        sumT += (unsigned long long)min(A0, tcl) + min(A1, tcl) + min(A2, tcl) + min(A3, tcl);
      }
    }
  }
  uint32_t A_last = Ac;  // consumption time of the last valid token
  if (ntail) {
    const uint32_t A0 = max(Ac + P, t0), A1 = max(A0 + P, t1), A2 = max(A1 + P, t2);
    const uint32_t c0 = min(A0, tcl), c1 = ntail > 1 ? min(A1, tcl) : 0u, c2 = ntail > 2 ? min(A2, tcl) : 0u;
    sum32 += c0 + c1 + c2;
    sumT += (unsigned long long)c0 + c1 + c2;
    A_last = ntail == 1 ? A0 : ntail == 2 ? A1 : A2;
  }
  const int32_t xl = xe - 1;  // the sub-range's last valid token
  if (active && xe > xs) {
    const uint32_t nn = (uint32_t)(xe - xs);
    const unsigned long long sumI =
        (unsigned long long)nn * Is + (unsigned long long)P * (((unsigned long long)nn * (nn - 1)) >> 1);
    const unsigned long long dsum = fits32 ? (unsigned long long)(sum32 - (uint32_t)sumI) : sumT - sumI;
    if (dsum) atomicAdd(&w.spre[qridx], dsum);
    if (qek && xe == qvend) {
      const uint32_t Il = qA + (uint32_t)xl * P;
      w.edge[qridx] = (qek == 1u) ? A_last - Il : min(A_last, tcl) - Il;
    }
  }
}

template <bool kFinal, bool kEval>
__device__ __noinline__ unsigned long long warp_tile_global(const ScanArgs& A, uint32_t tile_s, unsigned long long p0,
                                                            uint32_t r0, uint32_t dummy, uint32_t wn, uint32_t t,
                                                            uint32_t mode, uint32_t cdirect, uint32_t swz_on) {
  RawWin<kEval, kFinal> win{&A, p0, r0, dummy, wn};
  return warp_tile<kFinal>(A, win, tile_s, wn, t, mode, cdirect, swz_on);
}

}  // namespace

// K1.  Persistent CTAs of independent warps.  A warp's work unit is TW consecutive 1024-token
// warp-tiles (TW = 1: double-buffered TMA prefetch; TW = 2 on large pools: one unit fills both
// 4 KB buffers), claimed in chunks from the pool's end (the first two statically).  Each tile
// arrives by a TMA tensor copy (32 rows x 128 B; 128B swizzle for unaligned pools) on an
// mbarrier; the unit's request records come from global memory one unit ahead; the head
// request's earlier tokens are read directly when it started <= kCarryDirect tokens before the
// unit (else a bounded decoupled look-back on per-tile status words, on the row path); the
// scan itself uses warp shuffles only: no CTA-wide barriers on the hot path.
template <bool kFinal, int TW, bool kEval = false>
__global__ void __launch_bounds__(kScanThreads, 6) k_qoe_scan(const __grid_constant__ ScanArgs A,
                                                           const __grid_constant__ CUtensorMap tmap_swz,
                                                           const __grid_constant__ CUtensorMap tmap_plain) {
  extern __shared__ unsigned char s_dyn_raw[];
  unsigned char* s_base =
      reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(s_dyn_raw) + 1023) & ~uintptr_t(1023));
  __shared__ alignas(8) uint64_t s_bar[kScanThreads / 32][2];

  const ReqView& r = A.r;
  const Work& w = A.w;
  const uint32_t tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const uint32_t n = r.n;
  pdl_wait();
  if (blockIdx.x < 1000) ANDES_TRACE(w, 5000 + 2 * blockIdx.x);
  if (A.sched && blockIdx.x == 0) {
    bounds_block(r, w, A.tau, A.B_cap, A.M, A.cur_latency, A.flags);
    bounds_sync();
    ANDES_TRACE(w, 2300);
  }
  if (n == 0) return;
  const uint32_t ntiles = w.g->ntiles;
  const unsigned long long pool_end = w.g->pool_end;
  const unsigned long long full_rows_end = (r.tl_len / 32ull) * 32ull;  // tokens covered by the TMA view
  // 16-byte aligned timelines (every request): plain tiles and the piece-parallel path; else
  // 128B-swizzled tiles and the row-per-lane event path
  // Unaligned timelines (a request starting inside a 16-byte group): plain tiles and the
  // piece-parallel path with head groups (round 2; before, 128B-swizzled tiles and the row-per-lane
  // event path at about a third of the speed, kept under ANDES_UNAL_ROWPATH).  The row path then
  // serves only the tiles that look back, on plain tiles.
  const uint32_t unal = w.g->unal;  // (L1: one L2 request per SM, not per warp)
#ifdef ANDES_UNAL_ROWPATH
  const uint32_t swz_on = unal ? 1u : 0u;
#else
  const uint32_t swz_on = 0u;
#endif
  const CUtensorMap* pmap = swz_on ? &tmap_swz : &tmap_plain;
  const uint32_t wbase = smem_u32(s_base) + wid * kWarpSmem;  // [2][kWTile*4] tiles (shared address)
  uint64_t* bar = s_bar[wid];
  const uint32_t bar_s = smem_u32(bar);  // bar[0]; bar[1] at + 8

  // Chunks of CH consecutive warp-tiles: a warp's first chunk is static, the rest are claimed
  // from a counter (lane 0 runs the tile sequence two tiles ahead of the processing, for the
  // TMA double buffer, and holds the next chunk's claim one chunk ahead).  Chunks are taken from
  // the pool's end first; inside a chunk the carry passes from tile to tile in registers; a
  // chunk's first tile takes it from the head request's earlier tokens (direct read) or by
  // look-back, whose waits are bounded (see lookback()).
  constexpr uint32_t kNone = 0xFFFFFFFFu, kStart = 0x80000000u;
  const uint32_t KW = gridDim.x * (kScanThreads / 32);
  // work unit: TW consecutive warp-tiles (TW = 2 for large pools: one 2048-token unit fills
  // both tile buffers, which halves the per-unit set-up per token; no TMA prefetch then)
  const uint32_t nunits = (ntiles + TW - 1) / TW;
  const uint32_t CH = min(8u, max(1u, nunits / (8u * KW)));
  const uint32_t nchunks = (nunits + CH - 1) / CH;
  // lane 0's generator state (position, chunk end, claimed chunk) lives in shared memory: it is
  // touched once per tile and would otherwise hold registers across the whole tile body
  __shared__ uint32_t s_gen[kScanThreads / 32][4];
  uint32_t* const gs = s_gen[wid];
  // claims: a warp's first R chunks are static (chunk sw + r KS, r < R; sw: the warp's index
  // among the KS static warps), later ones come from the counter (+ R KS); the counter's result
  // is first needed a whole tile after it is asked.  R = 2 on small pools; on large ones the
  // static rounds cover ~kStaticPct % of the chunks, 95 (the counter's same-address round trips
  // held ~10% of the 2^20 scan's stall samples; the dynamic rest still balances the tail).
  // CTA 0 of a decision computes the bounds first: its warps claim from the counter only
  // (static chunks there would start last and form the tail).
  const uint32_t cta0_dyn = (A.sched && blockIdx.x == 0) ? 1u : 0u;
  const uint32_t KS = KW - (A.sched ? (kScanThreads / 32) : 0u);
  const uint32_t R = max(2u, (uint32_t)(((unsigned long long)nchunks * kStaticPct / 100u) / KS));
  const uint32_t Rw = cta0_dyn ? 0u : R;
  auto gen = [&]() -> uint32_t {
    const uint32_t g_t = gs[0], g_hi = gs[1], g_nxt = gs[2];
    if (g_t + 1 < g_hi) {
      gs[0] = g_t + 1;
      return g_t + 1;
    }
    if (g_nxt >= nchunks) return kNone;
    // chunks from the pool's end first: arrival-ordered pools keep the newest, shortest
    // timelines there (the densest tiles), which then do not form the tail
    const uint32_t t0 = (nchunks - 1u - g_nxt) * CH;
    gs[0] = t0;
    gs[1] = min(t0 + CH, nunits);
    const uint32_t c = gs[3] + 1u;  // chunks this warp has started
    gs[3] = c;
    gs[2] = c < Rw ? g_nxt + KS : atomicAdd(A.tile_ctr, 1u) + R * KS;
    return t0 | kStart;
  };
  uint32_t cur = kNone, s1 = kNone;
  if (lane == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    // static first claims: no start-up burst of KW atomics on one counter ahead of the first
    // two TMA copies
    gs[0] = kNone;
    gs[1] = 0u;
    gs[3] = 0u;
    gs[2] = cta0_dyn ? atomicAdd(A.tile_ctr, 1u) + R * KS
                     : (blockIdx.x - (A.sched ? 1u : 0u)) * (kScanThreads / 32) + wid;
    cur = gen();
    if (cur != kNone) {
      mbar_expect_tx_s(bar_s, TW * kWTile * 4u);
#pragma unroll
      for (int h = 0; h < TW; ++h)
        tma_tile(pmap, wbase + h * kWTile * 4, ((cur & ~kStart) * TW + h) * (kWTile / 32), bar_s);
    }
    s1 = gen();
    if (TW == 1 && s1 != kNone) {
      mbar_expect_tx_s(bar_s + 8u, kWTile * 4u);
      tma_tile(pmap, wbase + kWTile * 4, (s1 & ~kStart) * (kWTile / 32), bar_s + 8u);
    }
  }
  __syncwarp();
  cur = __shfl_sync(0xffffffffu, cur, 0);
  unsigned long long acc_reg = 0ull;  // carry out of the previous tile of the chunk
  uint32_t buf = 0, ph0 = 0, ph1 = 0;
  // the current tile's descriptor (lane 0) and request records (lane k: request r0 + k), loaded
  // one tile ahead: within a chunk the next tile's first request is this tile's last one, so its
  // records are requested before this tile is computed
  struct MetaLite {
    uint32_t r0, flags, hcnt;
  };
  MetaLite tm{0u, 0u, 0u};
  uint32_t r_end = 0;
  using PR = typename PipeRec<kEval>::T;
  PR rec;
  if constexpr (kEval) rec.g = 0u;
  else rec.lim = 0u;
  auto load_meta = [&](uint32_t tt, MetaLite& m, uint32_t& re) {  // tt: unit index
    if (lane == 0) {
      const TileMeta* tmp = w.tile_meta + tt * TW;
      m.r0 = tmp->r0;
      m.flags = tmp->flags;
      m.hcnt = tmp->hcnt;
      re = (tt * TW + TW < ntiles) ? w.tile_meta[tt * TW + TW].r0 : n - 1;
    }
  };
  auto load_rec = [&](uint32_t rr, PR& sr) {
    if constexpr (kEval) {
      sr.g = 0u;
      if (rr + lane < n) sr = raw_of<kFinal>(r, rr + lane);
    } else {
      sr.lim = 0u;
      if (rr + lane < n) sr = w.srec[rr + lane];
    }
  };
  // three-stage pipeline: the descriptor of the tile after next is requested when that tile is
  // generated (end of an iteration), the records of the next tile once the current tile's data
  // has arrived (its descriptor is in by then), both consumed one iteration later
  MetaLite tm1{0u, 0u, 0u};
  uint32_t r_end1 = 0;
  if (cur != kNone) {
    load_meta(cur & ~kStart, tm, r_end);
    load_rec(__shfl_sync(0xffffffffu, tm.r0, 0), rec);
    const uint32_t n1 = __shfl_sync(0xffffffffu, s1, 0);
    if (n1 != kNone) load_meta(n1 & ~kStart, tm1, r_end1);
  }
#ifdef ANDES_SCAN_PHASES
  uint32_t ph_it = 0;
  if (w.trace && blockIdx.x * 4 + wid < 4096 && lane == 0) w.trace[49152 + 4 * (blockIdx.x * 4 + wid)] = gtimer();
#endif
  while (cur != kNone) {
    const uint32_t tcur = cur & ~kStart;
    const bool chunk_start = (cur & kStart) != 0u;
    const unsigned long long p0 = (unsigned long long)tcur * (TW * kWTile);
    const uint32_t r0 = __shfl_sync(0xffffffffu, tm.r0, 0);
    const uint32_t flags = __shfl_sync(0xffffffffu, tm.flags, 0);
#ifdef ANDES_SCAN_PHASES
    const uint32_t gw_ = blockIdx.x * 4 + wid;
    const bool ph_on = w.trace && gw_ < 4096 && ph_it == 0 && lane == 0;
    if (ph_on) w.trace[49152 + 4 * gw_ + 1] = gtimer();
#endif
    const uint32_t re = __shfl_sync(0xffffffffu, r_end, 0);
    // ---- the next tile (its descriptor is in tm1)
    const uint32_t nxt = __shfl_sync(0xffffffffu, s1, 0);
    PR recn;
    if constexpr (kEval) recn.g = 0u;
    else recn.lim = 0u;
    const bool seq = nxt != kNone && (nxt & ~kStart) == tcur + 1u;
    if (seq) load_rec(re, recn);
    const uint32_t dummy = flags & 1u;
    // inside a chunk the carry comes from the previous tile (mode 1 with that value)
    const uint32_t mode = chunk_start ? (flags >> 1) & 3u : 1u;
    const uint32_t wn = re - r0 + 1 + dummy;
    const uint32_t nrec = wn - dummy;
    const uint32_t nbatch = (nrec + 30u) / 31u;
    // the aligned path never looks back: the look-back stays out of the hot loop's code
    const bool fast = !swz_on && mode != 2u;
    // direct head carry
    uint32_t cm = chunk_start ? 0u : (uint32_t)acc_reg;
    if (chunk_start && mode == 1u) {
      const uint32_t hcnt = __shfl_sync(0xffffffffu, tm.hcnt, 0);
      const TileMeta* tmp = w.tile_meta + tcur * TW;  // the head request's parameters (chunk starts only)
      const uint32_t httft = tmp->httft, hP = tmp->hP;
      const unsigned long long hbase = tmp->hbase;
      for (uint32_t k0 = 0; k0 < hcnt; k0 += 8 * 32) {  // 8 independent loads in flight per lane
        uint32_t d[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const uint32_t kk = k0 + u * 32 + lane;
          d[u] = kk < hcnt ? __ldg(&r.tl_pool[hbase + kk]) : 0u;
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const uint32_t kk = k0 + u * 32 + lane;
          const uint32_t I = httft + kk * hP;
          if (kk < hcnt) cm = max(cm, max(d[u], I) - I);
        }
      }
      for (int o = 16; o; o >>= 1) cm = max(cm, __shfl_xor_sync(0xffffffffu, cm, o));
    }
    // this tile's data
#ifdef ANDES_SCAN_PHASES
    if (ph_on) w.trace[49152 + 4 * gw_ + 2] = gtimer();
#endif
    if (buf == 0) { mbar_wait_s(bar_s, ph0); ph0 ^= 1u; }
    else { mbar_wait_s(bar_s + 8u, ph1); ph1 ^= 1u; }  // (TW = 1 only)
#ifdef ANDES_SCAN_PHASES
    if (ph_on) w.trace[49152 + 4 * gw_ + 3] = gtimer();
    ++ph_it;
#endif
    if (nxt != kNone && !seq) load_rec(__shfl_sync(0xffffffffu, tm1.r0, 0), recn);
    const uint32_t tile = wbase + buf * (kWTile * 4);
    {
      const unsigned long long pe = min(p0 + (unsigned long long)(TW * kWTile), pool_end);
      if (pe > full_rows_end) {
        const unsigned long long lo = max(p0, full_rows_end);
        for (unsigned long long p = lo + lane; p < pe; p += 32)
          st_shared_u32(tile + (swz_on ? swz((uint32_t)(p - p0)) : (uint32_t)(p - p0) * 4u), r.tl_pool[p]);
      }
    }
    __syncwarp();
#ifdef ANDES_SCAN_PHASES
    const unsigned long long t_body = (w.trace && tcur < 16384) ? gtimer() : 0ull;
#endif
    if (fast) {
      // piece-parallel path, batches of 31 requests (lane q of batch b = request r0 + 31 b + q)
      unsigned long long pref = 0ull;
      uint32_t mb = mode, cb = cm;
      for (uint32_t b = 0; b < nbatch; ++b) {
        const uint32_t nb_req = min(31u, nrec - 31u * b);
        ScanRec rb;
        if constexpr (kEval) rb = rec_from_raw<kFinal>(A.eval_abs, rec);
        else rb = rec;
        if (b && lane < nb_req) rb = rec_of<kEval, kFinal>(A, r0 + 31u * b + lane);
        const Entry e = lane < nb_req ? entry_of<TW * kWTile>(rb, r0 + 31u * b + lane, p0) : null_entry(true);
        // the status words are read only by look-backs, i.e. from inside a request longer than
        // kCarryDirect: publish when the request crossing the tile's end (the last one) is such
        const bool pub = __shfl_sync(0xffffffffu, rb.lim, nb_req - 1u) > (uint32_t)kCarryDirect;
        if (unal) warp_tile_aligned<kFinal, TW, true>(A, e, tile, tcur * TW, mb, cb, pref, b == 0, b + 1 == nbatch, pub);
        else warp_tile_aligned<kFinal, TW, false>(A, e, tile, tcur * TW, mb, cb, pref, b == 0, b + 1 == nbatch, pub);
        mb = 1u;
        cb = (uint32_t)pref;
      }
      acc_reg = pref;
    } else {
      // row-per-lane event path (unaligned pools, or a dense tile that must look back); the
      // window's records are read from global memory
      if (TW == 1) {
        acc_reg = warp_tile_global<kFinal, kEval>(A, tile, p0, r0, dummy, wn, tcur, mode, cm, swz_on);
      } else {
        // a unit's warp-tiles one by one, each with its own descriptor; the second continues
        // from the first's carry (the in-chunk rule)
        unsigned long long a = cm;
#pragma unroll 1
        for (uint32_t h = 0; h < (uint32_t)TW; ++h) {
          const uint32_t t = tcur * TW + h;
          if (t >= ntiles) break;
          uint32_t r0h = r0, fh = flags, reh = 0;
          if (lane == 0) {
            if (h) {
              r0h = w.tile_meta[t].r0;
              fh = w.tile_meta[t].flags;
            }
            reh = (t + 1 < ntiles) ? w.tile_meta[t + 1].r0 : n - 1;
          }
          r0h = __shfl_sync(0xffffffffu, r0h, 0);
          fh = __shfl_sync(0xffffffffu, fh, 0);
          reh = __shfl_sync(0xffffffffu, reh, 0);
          const uint32_t dh = fh & 1u;
          a = warp_tile_global<kFinal, kEval>(A, tile + h * (kWTile * 4), p0 + h * kWTile, r0h, dh, reh - r0h + 1 + dh, t,
                                       h ? 1u : mode, (uint32_t)a, swz_on);
        }
        acc_reg = a;
      }
    }
    // refill this buffer with the tile two ahead in the warp's sequence
    __syncwarp();
#ifdef ANDES_SCAN_PHASES
    if (t_body && lane == 0) {
      w.trace[16384 + 2 * tcur] = t_body;
      w.trace[16384 + 2 * tcur + 1] = gtimer();
    }
#endif
    uint32_t nx = kNone;
    MetaLite tm2{0u, 0u, 0u};
    uint32_t r_end2 = 0;
    if (lane == 0) {
      const uint32_t s2 = gen();
      if (TW == 1 && s2 != kNone) {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        mbar_expect_tx_s(bar_s + 8u * buf, kWTile * 4u);
        tma_tile(pmap, tile, (s2 & ~kStart) * (kWTile / 32), bar_s + 8u * buf);
      }
      if (TW > 1 && s1 != kNone) {
        // the unit already claimed (s1) now gets the buffers this one has released
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        mbar_expect_tx_s(bar_s, TW * kWTile * 4u);
#pragma unroll
        for (int h = 0; h < TW; ++h)
          tma_tile(pmap, wbase + h * kWTile * 4, ((s1 & ~kStart) * TW + h) * (kWTile / 32), bar_s);
      }
      if (s2 != kNone) load_meta(s2 & ~kStart, tm2, r_end2);
      nx = s1;
      s1 = s2;
    }
    cur = __shfl_sync(0xffffffffu, nx, 0);
    if (TW == 1) buf ^= 1u;
    tm = tm1;
    r_end = r_end1;
    rec = recn;
    tm1 = tm2;
    r_end1 = r_end2;
  }
  if (A.qnow) {
    const int64_t now_abs = A.now_abs + tshift(w);
    // k_qnow's work by the warps that have run out of tiles (chunks of 32 requests from a
    // counter): it overlaps the scan's tail instead of costing a kernel of its own
    unsigned long long best = 0ull;
    const uint32_t nq = (n + 31u) / 32u;
    for (;;) {
      uint32_t c = 0;
      if (lane == 0) c = atomicAdd(&globals2(w)->qnow_ctr, 1u);
      c = __shfl_sync(0xffffffffu, c, 0);
      if (c >= nq) break;
      const uint32_t i = c * 32u + lane;
      if (i < n) best = max(best, qnow_of(r, w, i, now_abs));
    }
    for (int o = 16; o; o >>= 1) best = max(best, __shfl_xor_sync(0xffffffffu, best, o));
    if (lane == 0) qmin_raise(w, best);
  }
  if (w.trace && blockIdx.x < 1000 && lane == 0) atomicMax(&w.trace[5000 + 2 * blockIdx.x + 1], gtimer());
}

// ---------------------------------------------------------------- qoe finalize
// S_delay / S_whole / QoE per request from K1's state (DESIGN.md "Closed forms":
// undelivered due tokens sit at t, Eq. 1-3).
__global__ void k_qoe_final(ReqView r, Work w, int64_t eval_abs, uint32_t final_mode, float* q,
                            double* q64, int64_t* sdo, int64_t* swo, uint32_t* mo) {
  pdl_wait();
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

// ---------------------------------------------------------------- QoE now (Appendix-A objectives)
// Q_now,i from the decision-time scan (eval = now; reading R3) into w.qnow, and min_i Q_now,i
// (max-min objective, reading R22) into g->qmin_bits as the inverted fp64 bit pattern.
__global__ void __launch_bounds__(256) k_qnow(ReqView r, Work w, int64_t now) {
  __shared__ unsigned long long s_best;
  pdl_wait();
  if (threadIdx.x == 0) s_best = 0ull;
  __syncthreads();
  unsigned long long best = 0ull;
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < r.n; i += gridDim.x * blockDim.x)
    best = max(best, qnow_of(r, w, i, now));
  for (int o = 16; o; o >>= 1) best = max(best, __shfl_xor_sync(0xffffffffu, best, o));
  if ((threadIdx.x & 31) == 0 && best) atomicMax(&s_best, best);
  __syncthreads();
  if (threadIdx.x == 0) qmin_raise(w, s_best);
}

void launch_qnow(const LaunchCfg& L, const ReqView& r, const Work& w, int64_t now) {
  if (r.n == 0) return;
  launch_pdl(k_qnow, umin32((r.n + 255) / 256, L.sm_count * 8), 256, 0, L.stream, r, w, now);
}

// ---------------------------------------------------------------- config-5 sweep: scenario means
// One CTA per scenario s: QoE of its requests [off[s], off[s+1]) in FINAL mode (m = g, Eq. 1-3,
// reading R19) and their mean over the requests with g >= 1 ("averaged across all
// requests").  Fixed-order reduction (strided per-thread sums, then a fixed tree): deterministic.
constexpr int kScenThreads = 256;
__global__ void __launch_bounds__(kScenThreads) k_scenario_mean(ReqView r, Work w, const uint32_t* __restrict__ off,
                                                                uint32_t S, double* mean_out, uint32_t* count_out) {
  __shared__ double s_sum[kScenThreads];
  __shared__ uint32_t s_cnt[kScenThreads];
  pdl_wait();
  for (uint32_t sc = blockIdx.x; sc < S; sc += gridDim.x) {
    const uint32_t lo = off[sc], hi = off[sc + 1];
    double acc = 0.0;
    uint32_t cnt = 0;
    for (uint32_t i = lo + threadIdx.x; i < hi; i += kScenThreads) {
      const uint32_t g = r.n_deliv[i];
      if (g == 0) continue;
      const int64_t P = r.period[i];
      const int64_t sw = (int64_t)g * (int64_t)w.edge[i] + P * (((int64_t)g * ((int64_t)g - 1)) >> 1);
      acc = __dadd_rn(acc, qoe_value((int64_t)w.spre[i], sw));
      ++cnt;
    }
    s_sum[threadIdx.x] = acc;
    s_cnt[threadIdx.x] = cnt;
    __syncthreads();
    for (uint32_t h = kScenThreads / 2; h; h >>= 1) {
      if (threadIdx.x < h) {
        s_sum[threadIdx.x] = __dadd_rn(s_sum[threadIdx.x], s_sum[threadIdx.x + h]);
        s_cnt[threadIdx.x] += s_cnt[threadIdx.x + h];
      }
      __syncthreads();
    }
    if (threadIdx.x == 0) {
      mean_out[sc] = s_cnt[0] ? __ddiv_rn(s_sum[0], (double)s_cnt[0]) : 0.0;
      if (count_out) count_out[sc] = s_cnt[0];
    }
    __syncthreads();
  }
}

// ---------------------------------------------------------------- host launchers
void launch_scenario_mean(const LaunchCfg& L, const ReqView& r, const Work& w, const uint32_t* off, uint32_t S,
                          double* mean_out, uint32_t* count_out) {
  if (S == 0) return;
  launch_pdl(k_scenario_mean, umin32(S, L.sm_count * 8), kScenThreads, 0, L.stream, r, w, off, S, mean_out,
             count_out);
}

void launch_prep(const LaunchCfg& L, const ReqView& r, const Work& w, int64_t eval_abs, bool final_mode,
                 bool sched, uint64_t kv_cap, bool debug, uint8_t* serve_mask, int64_t now_abs, bool dual,
                 bool eval) {
  if (r.n == 0) return;
// (CTAs per SM: 8 for a decision's prep, 16 for the other calls' -- the 2^20 andes_qoe_eval's
// prep and final passes measured -4 us with 16 instead of 8: more requests in flight per SM)
#ifndef ANDES_PREP_EVAL_PER_SM
#define ANDES_PREP_EVAL_PER_SM 16
#endif
  const uint32_t blocks =
      umin32((r.n + kPrepThreads - 1) / kPrepThreads, L.sm_count * (sched ? 8 : ANDES_PREP_EVAL_PER_SM));
  launch_pdl(k_prep, blocks, kPrepThreads, 0, L.stream, r, w, eval_abs, final_mode ? 1u : 0u, sched ? 1u : 0u,
             kv_cap, debug ? 1u : 0u, serve_mask, now_abs, dual ? 1u : 0u, eval ? 1u : 0u);
}

void launch_scan(const LaunchCfg& L, const ReqView& r, const Work& w, int64_t eval_abs, bool final_mode,
                 const CUtensorMap* tmap, bool sched, const uint32_t* tau, uint32_t B_cap, uint64_t M,
                 uint32_t cur_latency, uint32_t flags, bool second, bool qnow, int64_t now_abs, bool eval) {
  if (r.n == 0 && !sched) return;
  ScanArgs A{r, w, eval_abs, sched ? 1u : 0u, tau, B_cap, M, cur_latency, flags,
             second ? &globals2(w)->tile_ctr_b : &w.g->tile_ctr, qnow ? 1u : 0u, now_abs};
  // two-tile units for large pools (>= 16 M tokens: enough units per warp for balance);
  // ANDES_SCAN_TW=1|2 forces one (tests)
  static const int tw_env = [] {
    const char* v = getenv("ANDES_SCAN_TW");
    return v ? atoi(v) : 0;
  }();
  const bool tw2 = tw_env ? tw_env == 2 : r.tl_len >= (1ull << 24);
  // small pools (one-tile units, ~2.4 units per warp at 64K requests) run 5 CTAs per SM instead
  // of 6: the scan's tail shortens more than its throughput drops (config-3 decision -0.85 us,
  // means of 600 replays; the 2^20 scan keeps 6: 151.6 vs 154.5 us at 5)
  const uint32_t grid = r.n ? (tw2 ? L.scan_grid : umin32(L.scan_grid, L.sm_count * 5u)) : 1u;
  // eval: records from the request table (prep wrote none); else prep's records
  auto* k = eval ? (final_mode ? (tw2 ? &k_qoe_scan<true, 2, true> : &k_qoe_scan<true, 1, true>)
                               : (tw2 ? &k_qoe_scan<false, 2, true> : &k_qoe_scan<false, 1, true>))
                 : (final_mode ? (tw2 ? &k_qoe_scan<true, 2> : &k_qoe_scan<true, 1>)
                               : (tw2 ? &k_qoe_scan<false, 2> : &k_qoe_scan<false, 1>));
  launch_pdl(k, grid, kScanThreads, kScanDynSmem, L.stream, A, tmap[0], tmap[1]);
}

void launch_qoe_final(const LaunchCfg& L, const ReqView& r, const Work& w, int64_t eval_abs, bool final_mode,
                      float* q, double* q64, int64_t* sd, int64_t* sw, uint32_t* m) {
  if (r.n == 0) return;
#ifndef ANDES_FINAL_PER_SM
#define ANDES_FINAL_PER_SM 16
#endif
  const uint32_t blocks = umin32((r.n + 255) / 256, L.sm_count * ANDES_FINAL_PER_SM);
  launch_pdl(k_qoe_final, blocks, 256, 0, L.stream, r, w, eval_abs, final_mode ? 1u : 0u, q, q64, sd, sw, m);
}

void init_scan_kernels() {
  cudaFuncSetAttribute(k_qoe_scan<false, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, kScanDynSmem);
  cudaFuncSetAttribute(k_qoe_scan<true, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, kScanDynSmem);
  cudaFuncSetAttribute(k_qoe_scan<false, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, kScanDynSmem);
  cudaFuncSetAttribute(k_qoe_scan<true, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, kScanDynSmem);
  cudaFuncSetAttribute(k_qoe_scan<false, 1, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, kScanDynSmem);
  cudaFuncSetAttribute(k_qoe_scan<true, 1, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, kScanDynSmem);
  cudaFuncSetAttribute(k_qoe_scan<false, 2, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, kScanDynSmem);
  cudaFuncSetAttribute(k_qoe_scan<true, 2, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, kScanDynSmem);
}

int scan_blocks_per_sm() {
  int b = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, k_qoe_scan<false, 1>, kScanThreads, kScanDynSmem);
  int b2 = 0, b3 = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b2, k_qoe_scan<true, 2>, kScanThreads, kScanDynSmem);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b3, k_qoe_scan<false, 2, true>, kScanThreads, kScanDynSmem);
  b = b < b2 ? b : b2;
  return b < b3 ? b : b3;
}

}  // namespace andes
