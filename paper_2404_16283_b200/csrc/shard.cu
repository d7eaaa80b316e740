// shard.cu -- the scheduling decision over a request population sharded across GPUs
// (include/andes.h andes_schedule_shard).
//
// Every rank holds a contiguous range of the population (global index = shard base + local
// index).  S1 (timeline scan) and S3 (gains, key bounds) are per request and stay local.  The
// steps that need global information exchange small integer blocks, gathered by the caller in
// rank order after each step (an all-gather; NCCL over NVLink in bench.py):
//   round 0  trigger inputs + l histogram (S0/S2: B_max counts the shortest contexts globally)
//   round 1  lower-bound key histogram -> the global theta of the bound-and-prune selection
//   round 2  per B, the rank's top-min(B, local survivors) list in Algorithm 1's order: the
//            global top-B is a subset of the union of the ranks' top-B lists, so a merge of the
//            sorted lists gives Algorithm 1's prefix exactly
//   round 3  the rank's preemption victims at B* (reading R18)
// Every rank then derives the identical decision; all payloads are integers, so the result is
// bit-identical to the single-GPU andes_schedule on the concatenated population.
#include "block.cuh"
#include "device.cuh"
#include "launch.h"

namespace andes {

// ---------------------------------------------------------------- step 0: round-0 block
__global__ void __launch_bounds__(kSelThreads) k_shard_summary(ReqView r, Work w, uint32_t B_cap,
                                                               ShardSummary* out) {
  __shared__ unsigned long long s_key[kSortCap];
  __shared__ uint32_t s_idx[kSortCap];
  __shared__ uint32_t s_short[kSelThreads / 32];
  pdl_wait();
  const uint32_t tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  uint32_t sh = 0;
  for (uint32_t b = tid; b < kHistL; b += kSelThreads) {
    const uint32_t v = __ldcg(&w.hist_l[b]);
    out->hist[b] = v;
    w.hist_l[b] = 0u;  // self-clean for the next call
    if (b < kHistL - 1) sh += v;
  }
  for (int o = 16; o; o >>= 1) sh += __shfl_xor_sync(0xffffffffu, sh, o);
  if (lane == 0) s_short[wid] = sh;
  if (tid == 0) {
    out->n = r.n;
    out->n_run = __ldcg(&w.g->n_run);
    out->minP = 0xFFFFFFFFu - __ldcg(&w.g->inv_minP);
    out->run_l = __ldcg(&w.g->run_l);
    out->pad[0] = out->pad[1] = 0u;
  }
  __syncthreads();
  uint32_t n_short = 0;
  for (uint32_t q = 0; q < kSelThreads / 32; ++q) n_short += s_short[q];
  // The global B_max walk can reach contexts >= kHistL - 1 only if fewer than B_cap contexts
  // are shorter on every rank; then this rank lists its smallest long contexts exactly.
  uint32_t k = 0;
  if (n_short < B_cap) {
    const uint32_t n_long = out->hist[kHistL - 1];
    k = min(B_cap - n_short, n_long);
    if (k)
      select_top_k(
          r.n, k,
          [&](uint32_t e, bool) -> unsigned long long {
            const uint32_t l = r.ctx_len[e];
            return l >= kHistL - 1 ? (((unsigned long long)(~l) << 32) | (0xFFFFFFFFu - e)) : 0ull;
          },
          [&](uint32_t e) { return e; }, s_key, s_idx);
  }
  for (uint32_t q = tid; q < kMaxB; q += kSelThreads) out->ovf[q] = q < k ? r.ctx_len[s_idx[q]] : 0xFFFFFFFFu;
  if (tid == 0) out->has_ovf = n_short < B_cap ? 1u : 0u;
}

// ---------------------------------------------------------------- step 1: global S0 / S2
// Sums the gathered round-0 blocks; then the same trigger (R15) and batch-size range
// (R16) as the single-GPU bounds step, on the global histogram.
__global__ void __launch_bounds__(kSelThreads) k_shard_bounds(Work w, const ShardSummary* all, uint32_t G,
                                                              uint32_t rank, const uint32_t* __restrict__ tau,
                                                              uint32_t B_cap, uint64_t M, uint32_t cur_latency,
                                                              uint32_t flags) {
  constexpr uint32_t NT = kSelThreads, kPer = kHistL / NT;
  __shared__ unsigned long long s_run_l, s_ws[NT / 32];
  __shared__ uint32_t s_n, s_base, s_nrun, s_minP, s_kM, s_Blo, s_tlo, s_thi, s_wc[NT / 32];
  pdl_wait();
  const uint32_t tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  if (tid == 0) {
    unsigned long long rl = 0;
    uint32_t n = 0, base = 0, nr = 0, mp = 0xFFFFFFFFu;
    for (uint32_t g = 0; g < G; ++g) {
      if (g == rank) base = n;
      n += all[g].n;
      nr += all[g].n_run;
      rl += all[g].run_l;
      mp = min(mp, all[g].minP);
    }
    s_n = n;
    s_base = base;
    s_nrun = nr;
    s_run_l = rl;
    s_minP = mp;
    s_kM = 0xFFFFFFFFu;
    s_Blo = 1;
    s_tlo = 0xFFFFFFFFu;
    s_thi = 0;
  }
  // this thread's kPer consecutive bins of the global histogram
  uint32_t hv[kPer];
  unsigned long long c = 0, sm = 0;
#pragma unroll
  for (uint32_t q = 0; q < kPer; ++q) {
    const uint32_t b = tid * kPer + q;
    uint32_t v = 0;
    for (uint32_t g = 0; g < G; ++g) v += all[g].hist[b];
    hv[q] = v;
    c += v;
    sm += (unsigned long long)v * b;
  }
  __syncthreads();
  const uint32_t n = s_n;
  const uint32_t need = min(B_cap, n);
  // block-wide inclusive scan of (count, sum of l)
  unsigned long long ic = c, is = sm;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const unsigned long long a = __shfl_up_sync(0xffffffffu, ic, o), b2 = __shfl_up_sync(0xffffffffu, is, o);
    if (lane >= (uint32_t)o) {
      ic += a;
      is += b2;
    }
  }
  if (lane == 31) {
    s_wc[wid] = (uint32_t)ic;
    s_ws[wid] = is;
  }
  __syncthreads();
  unsigned long long wc = 0, ws = 0;
  for (uint32_t q = 0; q < wid; ++q) {
    wc += s_wc[q];
    ws += s_ws[q];
  }
  const unsigned long long c_ex = wc + ic - c, s_ex = ws + is - sm;
  if ((c_ex + c >= need || s_ex + sm > M) && (c_ex < need && s_ex <= M)) {
    unsigned long long k = c_ex, W = s_ex;
    bool stop = false;
    for (uint32_t q = 0; q < kPer && !stop; ++q) {
      const uint32_t b = tid * kPer + q;
      const uint32_t h = hv[q];
      if (b == kHistL - 1) {
        // long contexts: merge the ranks' ascending lists of their smallest ones (exact)
        uint32_t head[kMaxWorld];
        for (uint32_t g = 0; g < G; ++g) head[g] = 0;
        while (k < need) {
          uint32_t best = 0xFFFFFFFFu, bg = 0;
          for (uint32_t g = 0; g < G; ++g) {
            const uint32_t v = head[g] < kMaxB ? all[g].ovf[head[g]] : 0xFFFFFFFFu;
            if (v < best) {
              best = v;
              bg = g;
            }
          }
          if (best == 0xFFFFFFFFu || W + best > M) break;
          W += best;
          ++k;
          ++head[bg];
        }
        stop = true;
        break;
      }
      unsigned long long take = min((unsigned long long)h, need - k);
      if (b > 0) take = min(take, (M - W) / b);
      W += take * b;
      k += take;
      if (take < h) stop = true;
    }
    s_kM = (uint32_t)min(k, (unsigned long long)need);
  }
  __syncthreads();
  const uint32_t kM = s_kM == 0xFFFFFFFFu ? 0u : s_kM;
  const uint32_t B_hi = min(need, kM);
  const uint32_t minP = s_minP;
  const bool trig = (flags & 1u) || (10ull * s_run_l > 9ull * M) || (n > 0 && cur_latency > minP);
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
  __syncthreads();
  if (tid == 0) {
    Globals* g = w.g;
    g->B_hi = B_hi;
    g->B_lo = B_lo;
    g->tau_lo = s_tlo;
    g->tau_hi = s_thi;
    g->triggered = trig ? 1u : 0u;
    g->run_l = s_run_l;
    g->inv_minP = 0xFFFFFFFFu - minP;
    g->shard_base = s_base;
    g->n_global = n;
    g->n_run_global = s_nrun;
  }
}

__global__ void k_shard_copy_lb(Work w, uint32_t* send) {
  pdl_wait();
  for (uint32_t b = blockIdx.x * blockDim.x + threadIdx.x; b < kHistK; b += gridDim.x * blockDim.x)
    send[b] = __ldcg(&w.hist_lb[b]);
}

// ---------------------------------------------------------------- step 3: merge per B
// number of entries > c in a descending list of len composites (padding 0 at the tail)
__device__ __forceinline__ uint32_t count_gt(const unsigned long long* list, uint32_t len, unsigned long long c) {
  uint32_t lo = 0, hi = len;
  while (lo < hi) {
    const uint32_t mid = (lo + hi) >> 1;
    if (list[mid] > c) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}

struct MergeArgs {
  ReqView r;
  Work w;
  const XEntry* recv;  // G blocks of tri(B_cap + 1) entries
  uint32_t G;
  const uint32_t* tau;
  uint32_t B_cap;
  uint64_t M;
  SchedOut o;
  ShardVictims* send;
};

// CTA b handles B = b + 1: rank of every listed entry in the merged order (its own position
// plus the number of larger entries in every other rank's sorted list), Algorithm 1's walk over
// the merged top-B, V(B); the last CTA picks B* (R13) and lists the local victims.
__global__ void __launch_bounds__(kSelThreads) k_shard_merge(MergeArgs A) {
  extern __shared__ unsigned long long s_c[];  // [G * B] composites of the G lists
  __shared__ uint32_t s_m[kSortCap];           // merged position -> entry (g * B + p)
  __shared__ unsigned long long s_l[kSortCap];
  __shared__ uint32_t s_k, s_last, s_Bstar, s_nv;
  __shared__ long long s_red[32];
  __shared__ long long s_bv[kSelThreads / 32];
  __shared__ uint32_t s_bb[kSelThreads / 32];
  const Work& w = A.w;
  const uint32_t tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const uint32_t B = blockIdx.x + 1, G = A.G;
  __shared__ Globals s_g;
  pdl_wait();
  snap_globals(w.g, &s_g);
  const bool trig = s_g.triggered != 0;
  const uint32_t B_lo = s_g.B_lo, B_hi = s_g.B_hi;
  const size_t stride = tri_off(A.B_cap + 1);
  if (!trig || B < B_lo || B > B_hi) {
    if (tid == 0) {
      A.o.V[B - 1] = (long long)0x8000000000000000ull;
      A.o.kstar[B - 1] = 0u;
    }
  } else {
    const XEntry* lists = A.recv + tri_off(B);
    for (uint32_t e = tid; e < G * B; e += kSelThreads) {
      const uint32_t g = e / B, p = e - g * B;
      s_c[e] = __ldcg(&lists[g * stride + p].comp);
    }
    __syncthreads();
    for (uint32_t e = tid; e < G * B; e += kSelThreads) {
      const unsigned long long c = s_c[e];
      if (c == 0ull) continue;
      const uint32_t g = e / B, p = e - g * B;
      uint32_t pos = p;
      for (uint32_t g2 = 0; g2 < G && pos < B; ++g2)
        if (g2 != g) pos += count_gt(s_c + g2 * B, B, c);
      if (pos < B) s_m[pos] = e;
    }
    __syncthreads();
    // Algorithm 1 walk over the merged top-B (>= B listed entries exist: >= B_hi survivors)
    for (uint32_t q = tid; q < B; q += kSelThreads) {
      const uint32_t e = s_m[q], g = e / B, p = e - g * B;
      s_l[q] = __ldcg(&lists[g * stride + p].l);
    }
    __syncthreads();
    if (tid < 32) {
      const uint32_t per = (B + 31) / 32, q0 = tid * per, q1 = min(B, q0 + per);
      unsigned long long part = 0;
      for (uint32_t q = q0; q < q1; ++q) part += s_l[q];
      unsigned long long inc = part;
      for (int o = 1; o < 32; o <<= 1) {
        const unsigned long long v = __shfl_up_sync(0xffffffffu, inc, o);
        if (tid >= (uint32_t)o) inc += v;
      }
      unsigned long long run = inc - part;
      uint32_t mine = 0;
      for (uint32_t q = q0; q < q1; ++q) {
        run += s_l[q];
        mine += (run <= A.M) ? 1u : 0u;
      }
      for (int o = 16; o; o >>= 1) mine += __shfl_xor_sync(0xffffffffu, mine, o);
      if (tid == 0) s_k = mine;
    }
    __syncthreads();
    const uint32_t kstar = s_k;
    long long v = 0;
    XEntry* xm = w.xm + tri_off(B);
    for (uint32_t q = tid; q < kstar; q += kSelThreads) {
      const uint32_t e = s_m[q], g = e / B, p = e - g * B;
      const XEntry x = lists[g * stride + p];
      v += x.gfix;
      xm[q] = x;
    }
    v = block_sum_ll<kSelThreads>(v, s_red);
    if (tid == 0) {
      A.o.V[B - 1] = v;
      A.o.kstar[B - 1] = kstar;
      w.sel_thr[B - 1] = kstar ? s_c[s_m[kstar - 1]] : ~0ull;
    }
  }
  __threadfence();
  __syncthreads();
  if (tid == 0) s_last = (atomicAdd(&w.g->done, 1u) == gridDim.x - 1) ? 1u : 0u;
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  // S5: B* = argmax V, ties to the larger B
  {
    long long bv = (long long)0x8000000000000000ull;
    uint32_t bb = 0;
    if (trig)
      for (uint32_t Bq = B_lo + tid; Bq <= B_hi; Bq += kSelThreads) {
        const long long vq = __ldcg(A.o.V + (Bq - 1));
        if (bb == 0 || vq > bv || (vq == bv && Bq > bb)) {
          bv = vq;
          bb = Bq;
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
      s_nv = 0;
      w.g->shard_Bstar = bb;
    }
    __syncthreads();
  }
  // local victims at B*: running requests whose composite is below the k*-th merged one
  const uint32_t Bs = s_Bstar;
  const uint32_t n_run = min(__ldcg(&w.g->n_run), (uint32_t)kStageRun);
  if (Bs) {
    const uint32_t tB = A.tau[Bs - 1];
    const uint32_t ks = __ldcg(A.o.kstar + (Bs - 1));
    const unsigned long long thr = __ldcg(w.sel_thr + (Bs - 1));
    const uint32_t base = __ldcg(&w.g->shard_base);
    for (uint32_t q = tid; q < n_run; q += kSelThreads) {
      const uint32_t i = __ldcg(w.run_list + q);
      const PackedState st = w.st[i];
      const unsigned long long c = comp_of(st, tB, w.lqsf, w.obj);
      if (ks == 0 || c < thr) {
        const uint32_t slot = atomicAdd(&s_nv, 1u);
        VictimX x;
        x.comp = c;
        x.l = st.l;
        x.gidx = base + i;
        A.send->v[slot] = x;
      }
    }
  }
  __syncthreads();
  if (tid == 0) {
    A.send->count = s_nv;
    A.send->pad[0] = A.send->pad[1] = A.send->pad[2] = 0u;
    if (__ldcg(&w.g->n_run) > (uint32_t)kStageRun) raise_err(w, kErrRunning);
  }
}

// ---------------------------------------------------------------- step 4: cap + outputs
// Reading R18 on the global victims (every rank's list, ordered by composite ascending = key asc,
// rank desc) and the admits S_{B*} \ R in the merged greedy order; writes the replicated
// scalars and global-index admit / preempt lists, and edits this rank's serve mask.
__global__ void __launch_bounds__(kSelThreads) k_shard_cap(ReqView r, Work w, const ShardVictims* recv, uint32_t G,
                                                           uint64_t M, uint32_t preempt_cap, SchedOut o) {
  extern __shared__ unsigned long long s_dyn64[];
  unsigned long long* vkey = s_dyn64;                                    // [kVictCap]
  unsigned long long* vcum = s_dyn64 + kVictCap;                         // [kVictCap]
  uint32_t* vg = reinterpret_cast<uint32_t*>(s_dyn64 + 2 * kVictCap);    // [kVictCap]
  uint32_t* vl = vg + kVictCap;                                          // [kVictCap]
  uint32_t* vtmp = vl + kVictCap;                                        // [kVictCap]
  __shared__ unsigned long long s_acum[kSortCap];
  __shared__ uint32_t s_adm[kSortCap], s_afl[kSortCap];
  __shared__ unsigned long long s_tmp[kSelThreads / 32];
  __shared__ uint32_t s_nv, s_na, s_e, s_a;
  pdl_wait();
  const uint32_t tid = threadIdx.x, lane = tid & 31;
  uint32_t* sc = o.scalars;
  const bool trig = __ldcg(&w.g->triggered) != 0;
  const uint32_t B_lo = __ldcg(&w.g->B_lo), B_hi = __ldcg(&w.g->B_hi);
  const uint32_t n_run = __ldcg(&w.g->n_run_global);
  const uint32_t Bs = trig ? __ldcg(&w.g->shard_Bstar) : 0u;
  if (!trig || Bs == 0) {
    if (tid == 0) {
      for (int q = 0; q < 8; ++q) sc[q] = 0u;  // ANDES_SC_COUNT
      sc[1] = n_run;
      if (trig) {
        sc[4] = B_lo;
        sc[5] = B_hi;
        sc[6] = 1u;
      }
    }
    return;
  }
  const uint32_t base = __ldcg(&w.g->shard_base), n_local = r.n;
  // gather the victims of every rank
  if (tid == 0) {
    uint32_t nv = 0;
    for (uint32_t g = 0; g < G; ++g) nv += __ldcg(&recv[g].count);
    if (nv > (uint32_t)kVictCap) raise_err(w, kErrRunning);
    s_nv = min(nv, (uint32_t)kVictCap);
    s_e = 0;
    s_a = 0;
  }
  __syncthreads();
  const uint32_t nv = s_nv;
  {
    uint32_t off = 0;
    for (uint32_t g = 0; g < G && off < nv; ++g) {
      const uint32_t cg = min(__ldcg(&recv[g].count), nv - off);
      for (uint32_t q = tid; q < cg; q += kSelThreads) {
        const VictimX x = recv[g].v[q];
        vkey[off + q] = x.comp;
        vg[off + q] = x.gidx;
        vl[off + q] = x.l;
      }
      off += cg;
    }
  }
  __syncthreads();
  // victim order: ascending composite (unique), by rank counting; vtmp[pos] = slot
  for (uint32_t q = tid; q < nv; q += kSelThreads) {
    const unsigned long long c = vkey[q];
    uint32_t pos = 0;
    for (uint32_t f = 0; f < nv; ++f) pos += (vkey[f] < c) ? 1u : 0u;
    vtmp[pos] = q;
  }
  // admits: S_{B*} \ R in the merged greedy order
  const uint32_t ks = __ldcg(o.kstar + (Bs - 1));
  const XEntry* xm = w.xm + tri_off(Bs);
  for (uint32_t q = tid; q < ks; q += kSelThreads) {
    const uint32_t gi = __ldcg(&xm[q].gidx);
    s_adm[q] = gi;
    s_acum[q] = (gi & 0x80000000u) ? 0ull : 1ull;
  }
  __syncthreads();
  block_inclusive_scan(s_acum, ks, s_tmp);
  for (uint32_t q = tid; q < ks; q += kSelThreads)
    if (s_acum[q] != (q ? s_acum[q - 1] : 0ull)) s_afl[s_acum[q] - 1] = q;  // admit -> merged slot
  if (tid == 0) s_na = ks ? (uint32_t)s_acum[ks - 1] : 0u;
  __syncthreads();
  const uint32_t na = s_na;
  const bool cap_hit = !(preempt_cap == 0xFFFFFFFFu || nv <= preempt_cap);
  uint32_t n_pre, n_adm, flags = 1u, realized;
  if (!cap_hit) {
    n_pre = nv;
    n_adm = na;
    realized = ks;
  } else {
    flags |= 2u;
    for (uint32_t q = tid; q < nv; q += kSelThreads) vcum[q] = vl[vtmp[q]];
    __syncthreads();
    block_inclusive_scan(vcum, nv, s_tmp);
    const unsigned long long W0a = __ldcg(&w.g->run_l);
    const unsigned long long W0 = W0a - (preempt_cap ? vcum[preempt_cap - 1] : 0ull);
    const uint32_t c0 = n_run - preempt_cap;
    if (W0 > M) {
      flags |= 4u;  // memory beats the cap
      if (tid == 0) s_e = nv;
      __syncthreads();
      for (uint32_t q = preempt_cap + tid; q < nv; q += kSelThreads)
        if (W0a - vcum[q] <= M) atomicMin(&s_e, q + 1);
      __syncthreads();
      n_pre = s_e;
      n_adm = 0;
      realized = n_run - n_pre;
    } else {
      for (uint32_t q = tid; q < na; q += kSelThreads) s_acum[q] = __ldcg(&xm[s_afl[q]].l);
      __syncthreads();
      block_inclusive_scan(s_acum, na, s_tmp);
      uint32_t mine = 0;
      for (uint32_t q = tid; q < na; q += kSelThreads) mine += (W0 + s_acum[q] <= M && c0 + q + 1 <= Bs) ? 1u : 0u;
      for (int off = 16; off; off >>= 1) mine += __shfl_xor_sync(0xffffffffu, mine, off);
      if (lane == 0 && mine) atomicAdd(&s_a, mine);
      __syncthreads();
      n_pre = preempt_cap;
      n_adm = s_a;
      realized = c0 + n_adm;
    }
  }
  for (uint32_t q = tid; q < n_pre; q += kSelThreads) {
    const uint32_t gi = vg[vtmp[q]];
    o.preempt_idx[q] = gi;
    if (gi >= base && gi - base < n_local) o.serve_mask[gi - base] = 0;
  }
  for (uint32_t q = tid; q < n_adm; q += kSelThreads) {
    const uint32_t gi = s_adm[s_afl[q]] & 0x7FFFFFFFu;
    o.admit_idx[q] = gi;
    if (gi >= base && gi - base < n_local) o.serve_mask[gi - base] = 1;
  }
  if (tid == 0) {
    if (__ldcg(&w.g->slow)) flags |= 8u;
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

// ---------------------------------------------------------------- host launchers
void launch_shard_summary(const LaunchCfg& L, const ReqView& r, const Work& w, uint32_t B_cap, ShardSummary* out) {
  launch_pdl(k_shard_summary, 1, kSelThreads, 0, L.stream, r, w, B_cap, out);
}

void launch_shard_bounds(const LaunchCfg& L, const Work& w, const ShardSummary* all, uint32_t G, uint32_t rank,
                         const uint32_t* tau, uint32_t B_cap, uint64_t M, uint32_t cur_latency, uint32_t flags) {
  launch_pdl(k_shard_bounds, 1, kSelThreads, 0, L.stream, w, all, G, rank, tau, B_cap, M, cur_latency, flags);
}

void launch_shard_copy_lb(const LaunchCfg& L, const Work& w, uint32_t* send) {
  launch_pdl(k_shard_copy_lb, 16, 256, 0, L.stream, w, send);
}

static size_t merge_smem(uint32_t G, uint32_t B_cap) { return sizeof(unsigned long long) * G * B_cap; }
static size_t cap_smem() { return (2 * sizeof(unsigned long long) + 3 * sizeof(uint32_t)) * kVictCap; }

void init_shard_kernels() {
  cudaFuncSetAttribute(k_shard_merge, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       (int)merge_smem(kMaxWorld, kMaxB));
  cudaFuncSetAttribute(k_shard_cap, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)cap_smem());
}

void launch_shard_merge(const LaunchCfg& L, const ReqView& r, const Work& w, const XEntry* recv, uint32_t G,
                        const uint32_t* tau, uint32_t B_cap, uint64_t M, const SchedOut& o, ShardVictims* send) {
  MergeArgs A{r, w, recv, G, tau, B_cap, M, o, send};
  launch_pdl(k_shard_merge, B_cap, kSelThreads, merge_smem(G, B_cap), L.stream, A);
}

void launch_shard_cap(const LaunchCfg& L, const ReqView& r, const Work& w, const ShardVictims* recv, uint32_t G,
                      uint32_t B_cap, uint64_t M, uint32_t preempt_cap, const SchedOut& o) {
  (void)B_cap;
  launch_pdl(k_shard_cap, 1, kSelThreads, cap_smem(), L.stream, r, w, recv, G, M, preempt_cap, o);
}

}  // namespace andes
