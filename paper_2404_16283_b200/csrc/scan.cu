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
  __syncthreads();
  for (uint32_t off = 1; off < NT; off <<= 1) {
    unsigned long long a = 0, b2 = 0;
    if (tid >= off) { a = s_cnt[tid - off]; b2 = s_sum[tid - off]; }
    __syncthreads();
    s_cnt[tid] += a;
    s_sum[tid] += b2;
    __syncthreads();
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
        for (uint32_t z = 0; z < h; ++z) {
          if (k >= need || W + b > M) { stop = true; break; }
          W += b;
          ++k;
        }
      }
      s_kM = ovf && !stop && k < need ? 0xFFFFFFFEu : (uint32_t)min(k, (unsigned long long)need);
    }
  }
  __syncthreads();
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
      __syncthreads();
      if (tid == 0) {
        unsigned long long b2 = ~0ull;
        for (uint32_t q = 0; q < NT / 32; ++q) b2 = min(b2, s_red[q]);
        s_best = b2;
      }
      __syncthreads();
      const unsigned long long b2 = s_best;
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
  const uint32_t B_hi = min(need, kM);
  // B_min (reading R16) and the tau range of the candidate B
  if (flags & 2u) {
    uint32_t best = 1;
    for (uint32_t B = 1 + tid; B <= B_hi; B += NT)
      if (tau[B - 1] <= minP) best = max(best, B);
    atomicMax(&s_Blo, best);
  }
  __syncthreads();
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
  __syncthreads();
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
__global__ void __launch_bounds__(kPrepThreads) k_prep(ReqView r, Work w, int64_t eval_abs, uint32_t final_mode,
                                                      uint32_t sched, uint64_t kv_cap, uint32_t debug,
                                                      uint8_t* __restrict__ serve_mask) {
  __shared__ uint32_t s_hl[kHistL];
  __shared__ uint32_t s_minP;
  __shared__ unsigned long long s_runl;
  const uint32_t n = r.n;
  uint32_t local_err = 0;
  if (sched) {
    for (uint32_t q = threadIdx.x; q < kHistL; q += blockDim.x) s_hl[q] = 0u;
    if (threadIdx.x == 0) {
      s_minP = 0xFFFFFFFFu;
      s_runl = 0;
    }
    __syncthreads();
  }
  uint32_t my_minP = 0xFFFFFFFFu;
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
    {
      ScanRec sr;
      sr.base = r.tl_base[i];
      sr.lim = min(g, m);
      sr.P = P;
      sr.ttft = r.ttft[i];
      sr.trel = final_mode ? 0u : (uint32_t)(eval_abs - r.arrival[i]);
      sr.ek = (!final_mode && g < m) ? 1u : 2u;
      sr.pad = 0u;
      w.srec[i] = sr;
    }
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
      unsigned long long pe = min(base + g, (unsigned long long)w.tiles_cap * kTile);
      if (pe > r.tl_len) {  // pool shorter than the spans it claims: refuse (flagged), never overread
        pe = r.tl_len;
        local_err |= kErrTokens;
      }
      w.g->ntiles = (uint32_t)((pe + kTile - 1) / kTile);
      w.g->pool_end = pe;
    }
    if (debug) {
      if (P == 0) local_err |= kErrPeriod;
      if (i + 1 < n && next < base + g) local_err |= kErrBase;
      if (!final_mode && m >= (1u << 20)) local_err |= kErrDue;
    }
    if (sched) {
      const uint32_t l = r.ctx_len[i];
      my_minP = min(my_minP, P);
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
  if (local_err) atomicOr(&w.g->err, local_err);
  if (!sched) return;
  for (int o = 16; o; o >>= 1) my_minP = min(my_minP, __shfl_xor_sync(0xffffffffu, my_minP, o));
  if ((threadIdx.x & 31) == 0) atomicMin(&s_minP, my_minP);
  __syncthreads();
  for (uint32_t q = threadIdx.x; q < kHistL; q += blockDim.x)
    if (s_hl[q]) atomicAdd(&w.hist_l[q], s_hl[q]);
  if (threadIdx.x == 0) {
    atomicMax(&w.g->inv_minP, 0xFFFFFFFFu - s_minP);
    if (s_runl) atomicAdd(&w.g->run_l, s_runl);
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
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, 1000000;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(phase)
      : "memory");
}
// TMA: one [128 rows x 32 u32] box of the pool, 128-byte swizzled, completion on bar
__device__ __forceinline__ void tma_tile(const CUtensorMap* tmap, void* dst, uint32_t row0, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::
          "r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(tmap)), "r"(0), "r"(row0), "r"(smem_u32(bar))
      : "memory");
}

// segmented max monoid on (flag, value): combine(a, b) with a earlier than b
__device__ __forceinline__ unsigned long long seg_combine(unsigned long long a, unsigned long long b) {
  if (b & kFlagBit) return b;
  const uint32_t v = max((uint32_t)a, (uint32_t)b);
  return (a & kFlagBit) | v;
}

// byte offset of tile-local token x in a 128B-swizzled [128 x 32] u32 tile
__device__ __forceinline__ uint32_t swz(uint32_t x) {
  const uint32_t row = x >> 5, chunk = (x >> 2) & 7u;
  return (row << 7) | ((chunk ^ (row & 7u)) << 4) | ((x & 3u) << 2);
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
};

// One request of a tile's window in tile-local coordinates (x = position - p0).
struct Entry {
  int32_t ls;     // local start (base - p0), clamped to [-1, kTile + 1]
  int32_t vend;   // local end of the valid tokens (base + lim - p0), clamped to [-1, kTile]
  uint32_t A;     // ideal time of local position 0: ttft + (p0 - base) P (mod 2^32); I(x) = A + x P
  uint32_t U;     // t_rel - A (mod 2^32): t - I(x) = U - x P
  uint32_t P;
  uint32_t ek;    // edge kind: 1 = delta_g (g < m, unclamped), 2 = delta~_m
  uint32_t ridx;  // request index (0xFFFFFFFF: dummy / sentinel)
};

__device__ __forceinline__ Entry make_entry(const ScanRec* __restrict__ srec, unsigned long long p0, uint32_t r0,
                                            uint32_t dummy, uint32_t wn, uint32_t q) {
  Entry e;
  if ((dummy && q == 0) || q >= wn) {
    e.ls = (q >= wn) ? kTile + 1 : -1;
    e.vend = -1;
    e.A = 0; e.U = 0; e.P = 0; e.ek = 0; e.ridx = 0xFFFFFFFFu;
    return e;
  }
  const uint32_t ri = r0 + q - dummy;
  const ScanRec s = srec[ri];
  const long long ls = (long long)s.base - (long long)p0;
  const long long ve = ls + (long long)s.lim;
  e.ls = (int32_t)max(-1ll, min(ls, (long long)kTile + 1));
  e.vend = (int32_t)max(-1ll, min(ve, (long long)kTile));
  e.A = s.ttft + (uint32_t)(unsigned long long)(-ls) * s.P;
  e.U = s.trel - e.A;
  e.P = s.P;
  // the edge token (last valid token) is written only by the tile that contains it
  e.ek = (ve >= 1 && ve <= (long long)kTile) ? s.ek : 0u;
  e.ridx = ri;
  return e;
}

// Window accessors: shared-memory window (hot path) or straight from the scan records when
// the tile overlaps more than kWinCap requests (slow path, separate instantiation).
struct SmemWin {
  const int32_t *ls, *vend;
  const uint32_t *A, *U, *P, *ek, *ridx;
  __device__ __forceinline__ int32_t start(uint32_t q) const { return ls[q]; }
  __device__ __forceinline__ Entry get(uint32_t q) const {
    Entry e;
    e.ls = ls[q]; e.vend = vend[q]; e.A = A[q]; e.U = U[q]; e.P = P[q]; e.ek = ek[q]; e.ridx = ridx[q];
    return e;
  }
};
struct GlobalWin {
  const ScanRec* srec;
  unsigned long long p0;
  uint32_t r0, dummy, wn;
  __device__ __forceinline__ int32_t start(uint32_t q) const {
    if (q >= wn) return kTile + 1;
    if (dummy && q == 0) return -1;
    const long long ls = (long long)srec[r0 + q - dummy].base - (long long)p0;
    return (int32_t)max(-1ll, min(ls, (long long)kTile + 1));
  }
  __device__ __forceinline__ Entry get(uint32_t q) const { return make_entry(srec, p0, r0, dummy, wn, q); }
};

struct TileShared {
  unsigned long long* warp;  // [kScanThreads / 32]
  uint32_t* cm;              // [kScanThreads / 32]
  unsigned long long* carry;
};

// Per-thread cursor over the window: the current request q, the next event position ev
// (end of q's valid tokens, or the start of the next request), and the arithmetic state of
// the valid ("live") or invalid ("null": lat = 0, delta~ = 0) range.
struct Cursor {
  uint32_t q;
  int32_t vend, ns;
  uint32_t P, I, u, Pu;
  uint32_t ek, ridx;
  bool live;
};

template <bool kFinal, class Win>
__device__ __forceinline__ void cursor_enter(Cursor& c, const Win& win, uint32_t q, int32_t x) {
  // enter request q at local position x (q's first position in this thread, or x0)
  const Entry e = win.get(q);
  c.q = q;
  c.vend = e.vend;
  c.ns = win.start(q + 1);
  c.ek = e.ek;
  c.ridx = e.ridx;
  c.live = x < e.vend;
  if (c.live) {
    c.P = e.P;
    c.I = e.A + (uint32_t)x * e.P;
    c.u = kFinal ? 0xFFFFFFFFu : e.U - (uint32_t)x * e.P;
    c.Pu = kFinal ? 0u : e.P;
  } else {
    c.P = 0; c.I = 0xFFFFFFFFu; c.u = 0; c.Pu = 0;
  }
}

template <bool kFinal, class Win>
__device__ __forceinline__ void cursor_next_request(Cursor& c, const Win& win, int32_t x) {
  uint32_t q = c.q;
  do {
    ++q;
  } while (win.start(q + 1) <= x);
  cursor_enter<kFinal>(c, win, q, x);
}

template <bool kFinal, class Win>
__device__ void tile_body(const ScanArgs& A, const Win& win, const unsigned char* tile, uint32_t wn, uint32_t t,
                          uint32_t mode, const TileShared& sh) {
  const Work& w = A.w;
  const uint32_t tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int32_t x0 = (int32_t)(tid * kScanItems);
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
  const uint32_t rowb = tid << 7, rsw = tid & 7u;
  const bool starts_here = win.start(q0) == x0;

  // ---- pass 1: the thread aggregate of the segmented max of lat+
  unsigned long long agg;
  {
    Cursor c;
    cursor_enter<kFinal>(c, win, q0, x0);
    uint32_t flag = starts_here ? 1u : 0u, v = 0;
    int32_t ev = min(c.live ? c.vend : c.ns, c.ns);
#pragma unroll 1
    for (uint32_t g = 0; g < kScanItems / 4; ++g) {
      const uint4 dv = *reinterpret_cast<const uint4*>(tile + (rowb | ((g ^ rsw) << 4)));
      const uint32_t dd[4] = {dv.x, dv.y, dv.z, dv.w};
      const int32_t gx = x0 + (int32_t)(4 * g);
      int32_t rel = ev - gx;  // items until the next event
#pragma unroll
      for (int jj = 0; jj < 4; ++jj) {
        if (rel == jj) {
          const int32_t x = gx + jj;
          if (x == c.ns) {
            cursor_next_request<kFinal>(c, win, x);
            flag = 1u;
            v = 0;
          } else {  // end of the valid tokens: null range until the next request
            c.live = false; c.P = 0; c.I = 0xFFFFFFFFu;
          }
          ev = c.live ? min(c.vend, c.ns) : c.ns;
          rel = ev - gx;
        }
        v = max(v, max(dd[jj], c.I) - c.I);
        c.I += c.P;
      }
    }
    agg = (flag ? kFlagBit : 0ull) | v;
  }
  // ---- block-wide exclusive scan of the thread aggregates
  unsigned long long incl = agg;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const unsigned long long v = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= (uint32_t)o) incl = seg_combine(v, incl);
  }
  if (lane == 31) sh.warp[wid] = incl;
  unsigned long long excl = __shfl_up_sync(0xffffffffu, incl, 1);
  if (lane == 0) excl = 0ull;
  __syncthreads();
  {
    unsigned long long wp = 0ull;
    for (uint32_t k = 0; k < wid; ++k) wp = seg_combine(wp, sh.warp[k]);
    excl = seg_combine(wp, excl);
  }
  if (tid == 0) {
    unsigned long long tile_agg = 0ull;
    for (uint32_t k = 0; k < kScanThreads / 32; ++k) tile_agg = seg_combine(tile_agg, sh.warp[k]);
    unsigned long long acc = 0ull;
    if (mode == 2u) {
      st_release(&w.tile_status[t], kStAgg | tile_agg);
      for (int64_t j = (int64_t)t - 1; j >= 0; --j) {
        unsigned long long s;
        do {
          s = ld_acquire(&w.tile_status[j]);
        } while ((s & kStMask) == 0ull);
        acc = seg_combine(s & ~kStMask, acc);
        if ((s & kStMask) == kStPrefix || (acc & kFlagBit)) break;
      }
    } else if (mode == 1u) {
      uint32_t cm = 0;
      for (uint32_t k = 0; k < kScanThreads / 32; ++k) cm = max(cm, sh.cm[k]);
      acc = kFlagBit | cm;
    }
    st_release(&w.tile_status[t], kStPrefix | seg_combine(acc, tile_agg));
    *sh.carry = acc;
  }
  __syncthreads();
  const unsigned long long carry = seg_combine(*sh.carry, excl);

  // ---- pass 2: clamped delays, per-request sums, edge values
  {
    Cursor c;
    cursor_enter<kFinal>(c, win, q0, x0);
    uint32_t pm = starts_here ? 0u : (uint32_t)carry;
    uint32_t dt = 0;
    unsigned long long sum = 0ull;
    int32_t ev = c.live ? min(c.vend, c.ns) : c.ns;
#pragma unroll 1
    for (uint32_t g = 0; g < kScanItems / 4; ++g) {
      const uint4 dv = *reinterpret_cast<const uint4*>(tile + (rowb | ((g ^ rsw) << 4)));
      const uint32_t dd[4] = {dv.x, dv.y, dv.z, dv.w};
      const int32_t gx = x0 + (int32_t)(4 * g);
      int32_t rel = ev - gx;
#pragma unroll
      for (int jj = 0; jj < 4; ++jj) {
        if (rel == jj) {
          const int32_t x = gx + jj;
          if (c.live && x == c.vend && x > x0 && c.ek) w.edge[c.ridx] = (c.ek == 1u) ? pm : dt;  // last valid token
          if (x == c.ns) {
            if (sum) atomicAdd(&w.spre[c.ridx], sum);
            sum = 0ull;
            cursor_next_request<kFinal>(c, win, x);
            pm = 0;
          } else {
            c.live = false; c.P = 0; c.I = 0xFFFFFFFFu; c.u = 0; c.Pu = 0;
          }
          ev = c.live ? min(c.vend, c.ns) : c.ns;
          rel = ev - gx;
        }
        pm = max(pm, max(dd[jj], c.I) - c.I);
        c.I += c.P;
        dt = min(pm, c.u);
        c.u -= c.Pu;
        sum += dt;
      }
    }
    // the last valid token of the current request is this thread's last token
    if (c.live && c.vend == x0 + kScanItems && c.ek) w.edge[c.ridx] = (c.ek == 1u) ? pm : dt;
    // the last piece may continue into the next lanes: segmented warp reduction by request
    uint32_t key = c.ridx;
    unsigned long long val = sum;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t k2 = __shfl_down_sync(0xffffffffu, key, o);
      const unsigned long long v2 = __shfl_down_sync(0xffffffffu, val, o);
      if (lane + o < 32 && k2 == key) val += v2;
    }
    const uint32_t kprev = __shfl_up_sync(0xffffffffu, key, 1);
    if ((lane == 0 || kprev != key) && val && key != 0xFFFFFFFFu) atomicAdd(&w.spre[key], val);
  }
}

template <bool kFinal>
__device__ __noinline__ void tile_body_global(const ScanArgs& A, const unsigned char* tile, unsigned long long p0,
                                              uint32_t r0, uint32_t dummy, uint32_t wn, uint32_t t, uint32_t mode,
                                              TileShared sh) {
  GlobalWin win{A.w.srec, p0, r0, dummy, wn};
  tile_body<kFinal>(A, win, tile, wn, t, mode, sh);
}

}  // namespace

// K1.  Persistent CTAs claim 4096-token tiles in increasing order; each tile arrives by one
// TMA tensor copy into a double-buffered, 128B-swizzled shared-memory tile; each thread owns
// one 32-token row (conflict-free LDS.128); requests overlapping the tile are staged in a
// shared-memory window; the carry of the head segment is read directly (short segments) or
// obtained by decoupled look-back (long segments).
template <bool kFinal>
__global__ void __launch_bounds__(kScanThreads) k_qoe_scan(const __grid_constant__ ScanArgs A,
                                                           const __grid_constant__ CUtensorMap tmap) {
  extern __shared__ unsigned char s_dyn_raw[];
  unsigned char* s_tiles =
      reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(s_dyn_raw) + 1023) & ~uintptr_t(1023));
  __shared__ alignas(8) uint64_t s_bar[2];
  __shared__ int32_t w_ls[kWinCap + 2], w_vend[kWinCap + 2];
  __shared__ uint32_t w_A[kWinCap + 2], w_U[kWinCap + 2], w_P[kWinCap + 2], w_ek[kWinCap + 2],
      w_ridx[kWinCap + 2];
  __shared__ unsigned long long s_warp[kScanThreads / 32];
  __shared__ uint32_t s_cm[kScanThreads / 32];
  __shared__ unsigned long long s_carry;
  __shared__ uint32_t s_tile_id[2], s_r0, s_wn, s_dummy, s_mode, s_hcnt, s_hP, s_httft;
  __shared__ unsigned long long s_hbase;

  const ReqView& r = A.r;
  const Work& w = A.w;
  const ScanRec* __restrict__ srec = w.srec;
  const uint32_t tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const uint32_t ntiles = w.g->ntiles;
  const unsigned long long pool_end = w.g->pool_end;
  const unsigned long long full_rows_end = (r.tl_len / 32ull) * 32ull;  // tokens covered by the TMA view
  const uint32_t n = r.n;
  const TileShared sh{s_warp, s_cm, &s_carry};
  const SmemWin swin{w_ls, w_vend, w_A, w_U, w_P, w_ek, w_ridx};
  if (A.sched && blockIdx.x == 0) {
    bounds_block(r, w, A.tau, A.B_cap, A.M, A.cur_latency, A.flags);
    __syncthreads();
  }
  if (n == 0) return;

  if (tid == 0) {
    mbar_init(&s_bar[0], 1);
    mbar_init(&s_bar[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmap)) : "memory");
    // claim two tiles (increasing order: a tile waited on in a look-back is owned by a running CTA)
    for (int b = 0; b < 2; ++b) {
      const uint32_t tt = atomicAdd(&w.g->tile_ctr, 1u);
      s_tile_id[b] = tt;
      if (tt < ntiles) {
        mbar_expect_tx(&s_bar[b], kTile * 4u);
        tma_tile(&tmap, s_tiles + b * (kTile * 4), tt * (kTile / 32), &s_bar[b]);
      }
    }
  }
  __syncthreads();
  uint32_t buf = 0, ph0 = 0, ph1 = 0;
  for (uint32_t t = s_tile_id[0]; t < ntiles; buf ^= 1u) {
    const unsigned long long p0 = (unsigned long long)t * kTile;
    if (tid == 0) {
      const uint32_t r0 = w.tile_owner[t];
      const uint32_t r_end = (t + 1 < ntiles) ? w.tile_owner[t + 1] : n - 1;
      const ScanRec h = srec[r0];
      s_dummy = (h.base > p0) ? 1u : 0u;
      s_r0 = r0;
      s_wn = r_end - r0 + 1 + s_dummy;
      uint32_t mode = 0;  // head-segment carry: 0 none needed, 1 direct read, 2 look-back
      if (h.base < p0) {
        const unsigned long long span = p0 - h.base;
        if ((unsigned long long)h.lim > span) {
          s_hbase = h.base;
          s_hcnt = (uint32_t)span;
          s_httft = h.ttft;
          s_hP = h.P;
          mode = (span <= (unsigned long long)kCarryDirect) ? 1u : 2u;
        }
      }
      s_mode = mode;
    }
    __syncthreads();
    const uint32_t r0 = s_r0, wn = s_wn, dummy = s_dummy, mode = s_mode;
    const bool win_ok = wn <= (uint32_t)kWinCap;
    if (win_ok) {
      for (uint32_t q = tid; q <= wn; q += kScanThreads) {
        const Entry e = make_entry(srec, p0, r0, dummy, wn, q);
        w_ls[q] = e.ls; w_vend[q] = e.vend; w_A[q] = e.A; w_U[q] = e.U; w_P[q] = e.P;
        w_ek[q] = e.ek; w_ridx[q] = e.ridx;
      }
    }
    // direct head carry: max lat+ of the head segment's tokens before p0
    uint32_t cmax = 0;
    if (mode == 1u) {
      const unsigned long long hb = s_hbase;
      const uint32_t cnt = s_hcnt, P = s_hP, ttft = s_httft;
      for (uint32_t k = tid; k < cnt; k += kScanThreads) {
        const uint32_t d = r.tl_pool[hb + k];
        const uint32_t I = ttft + k * P;
        cmax = max(cmax, max(d, I) - I);
      }
    }
    for (int o = 16; o; o >>= 1) cmax = max(cmax, __shfl_xor_sync(0xffffffffu, cmax, o));
    if (lane == 0) s_cm[wid] = cmax;
    if (buf == 0) { mbar_wait(&s_bar[0], ph0); ph0 ^= 1u; }
    else { mbar_wait(&s_bar[1], ph1); ph1 ^= 1u; }
    unsigned char* tile = s_tiles + buf * (kTile * 4);
    {
      // tokens past the last full 32-token row of the pool view: read directly
      const unsigned long long pe = min(p0 + (unsigned long long)kTile, pool_end);
      if (pe > full_rows_end) {
        const unsigned long long lo = max(p0, full_rows_end);
        for (unsigned long long p = lo + tid; p < pe; p += kScanThreads)
          *reinterpret_cast<uint32_t*>(tile + swz((uint32_t)(p - p0))) = r.tl_pool[p];
      }
    }
    __syncthreads();
    if (win_ok) tile_body<kFinal>(A, swin, tile, wn, t, mode, sh);
    else tile_body_global<kFinal>(A, tile, p0, r0, dummy, wn, t, mode, sh);
    __syncthreads();  // tile buffer and window are reused below
    // refill this buffer with a newly claimed tile (two tiles ahead)
    if (tid == 0) {
      const uint32_t tt = atomicAdd(&w.g->tile_ctr, 1u);
      s_tile_id[buf] = tt;
      if (tt < ntiles) {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        mbar_expect_tx(&s_bar[buf], kTile * 4u);
        tma_tile(&tmap, s_tiles + buf * (kTile * 4), tt * (kTile / 32), &s_bar[buf]);
      }
    }
    t = s_tile_id[buf ^ 1u];
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
                 bool sched, uint64_t kv_cap, bool debug, uint8_t* serve_mask) {
  if (r.n == 0) return;
  const uint32_t blocks = umin32((r.n + kPrepThreads - 1) / kPrepThreads, L.sm_count * 8);
  k_prep<<<blocks, kPrepThreads, 0, L.stream>>>(r, w, eval_abs, final_mode ? 1u : 0u, sched ? 1u : 0u, kv_cap,
                                                debug ? 1u : 0u, serve_mask);
}

void launch_scan(const LaunchCfg& L, const ReqView& r, const Work& w, int64_t eval_abs, bool final_mode,
                 const CUtensorMap* tmap, bool sched, const uint32_t* tau, uint32_t B_cap, uint64_t M,
                 uint32_t cur_latency, uint32_t flags) {
  if (r.n == 0 && !sched) return;
  ScanArgs A{r, w, eval_abs, sched ? 1u : 0u, tau, B_cap, M, cur_latency, flags};
  const uint32_t grid = r.n ? L.scan_grid : 1u;
  if (final_mode)
    k_qoe_scan<true><<<grid, kScanThreads, kScanDynSmem, L.stream>>>(A, *tmap);
  else
    k_qoe_scan<false><<<grid, kScanThreads, kScanDynSmem, L.stream>>>(A, *tmap);
}

void launch_qoe_final(const LaunchCfg& L, const ReqView& r, const Work& w, int64_t eval_abs, bool final_mode,
                      float* q, double* q64, int64_t* sd, int64_t* sw, uint32_t* m) {
  if (r.n == 0) return;
  const uint32_t blocks = umin32((r.n + 255) / 256, L.sm_count * 8);
  k_qoe_final<<<blocks, 256, 0, L.stream>>>(r, w, eval_abs, final_mode ? 1u : 0u, q, q64, sd, sw, m);
}

void init_scan_kernels() {
  cudaFuncSetAttribute(k_qoe_scan<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, kScanDynSmem);
  cudaFuncSetAttribute(k_qoe_scan<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, kScanDynSmem);
}

int scan_blocks_per_sm() {
  int b = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, k_qoe_scan<false>, kScanThreads, kScanDynSmem);
  int b2 = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b2, k_qoe_scan<true>, kScanThreads, kScanDynSmem);
  return b < b2 ? b : b2;
}

}  // namespace andes
