// tracker.cu -- device-resident Request Tracker update (the tracker "keeps track of"
// every request's delivered tokens and their times; the decision reads its state).  One call per
// serving iteration appends the tokens the engine delivered to their requests' timelines in
// place, so the decision's inputs stay in HBM and only the per-iteration deltas cross PCIe.
//
//   for every delivered token k: i = idx[k]; its timestamp (t_abs[k] - a_i, us since arrival)
//   goes to tl_pool[tl_base[i] + n_deliv[i]], then n_deliv[i] += 1 and ctx_len[i] += 1 (a
//   generated token extends the context, Eq. 5's l_i); optionally running := serve_mask.
// Tokens of one request within a call are appended in k order (stable), by one thread each after
// a per-request rank among the call's tokens; a timeline without room (the next request's
// tl_base, or tl_len for the last one) rejects the token and raises the capacity bit.
#include "device.cuh"
#include "launch.h"

namespace andes {

constexpr int kTrackThreads = 256;

// count = number of tokens; they must be grouped so that a request's tokens are consecutive in
// k with nondecreasing times (the engine reports them in order).  Thread k appends token k at
// offset (k - first k of its request) past the current n_deliv; the last token of each request
// then bumps the counters.
// count_dev (optional): the count is read on the device (at most count, the slots), so that a
// serving loop can capture the whole iteration -- append and decision -- in one graph; idx,
// t_abs and count_dev may sit in mapped host memory: every slot's loads are issued before the
// count is known (one PCIe round trip, not three), and the count is read once per CTA.
// serve_mask (optional): running := serve_mask, by the same grid (grid-stride over n).
__global__ void __launch_bounds__(kTrackThreads) k_tracker_append(TrackerView t, const uint32_t* __restrict__ idx,
                                                                 const int64_t* __restrict__ t_abs, uint32_t count,
                                                                 const uint32_t* __restrict__ count_dev,
                                                                 const uint8_t* __restrict__ serve_mask, Work w) {
  const uint32_t k = blockIdx.x * blockDim.x + threadIdx.x;
  // this slot's inputs, requested up front (k < count: the slots the call provides)
  uint32_t i = 0xFFFFFFFFu, ip = 0xFFFFFFFFu, in = 0xFFFFFFFFu;
  long long ta = 0;
  if (k < count) {
    i = idx[k];
    ta = t_abs[k];
    if (k > 0) ip = idx[k - 1];
    if (k + 1 < count) in = idx[k + 1];
  }
  if (serve_mask)
    for (uint32_t q = k; q < t.n; q += gridDim.x * blockDim.x) t.running[q] = serve_mask[q];
  // CTAs past the provided slots only copy the running set (no count read: same-address PCIe
  // reads from hundreds of CTAs serialise at the host, ~1 us each)
  if (blockIdx.x * blockDim.x >= count) return;
  if (count_dev) {
    // one read per CTA (same-address PCIe reads serialise at the host)
    __shared__ uint32_t s_c;
    if (threadIdx.x == 0) s_c = *reinterpret_cast<const volatile uint32_t*>(count_dev);
    __syncthreads();
    const uint32_t c = s_c;
    if (c > count) {  // more deliveries than the call allows: flagged, none appended
      if (k == 0) raise_err(w, kErrTokens);
      return;
    }
    count = c;
  }
  if (k >= count) return;
  if (i >= t.n) {
    raise_err(w, kErrTokens);
    return;
  }
  // first token of this request's run of tokens (runs are consecutive in k)
  uint32_t k0 = k;
  if (k > 0 && ip == i) {
    --k0;
    while (k0 > 0 && idx[k0 - 1] == i) --k0;
  }
  const bool last = (k + 1 == count) || in != i;
  const uint32_t g = t.n_deliv[i];
  const unsigned long long base = t.tl_base[i];
  const unsigned long long limit = (i + 1 < t.n) ? t.tl_base[i + 1] : t.tl_len;
  const unsigned long long slot = base + g + (k - k0);
  const unsigned long long runlen = (unsigned long long)(k - k0) + 1ull;
  if (base + g + runlen > limit) {  // no room for this run's tokens: reject the whole run
    if (last) raise_err(w, kErrTokens);
    return;
  }
  const long long d = ta - t.arrival[i];
  t.tl_pool[slot] = (uint32_t)(d < 0 ? 0 : d);
  if (last) {
    t.n_deliv[i] = g + (uint32_t)runlen;
    t.ctx_len[i] += (uint32_t)runlen;
  }
}

void launch_tracker_append(const LaunchCfg& L, const TrackerView& t, const uint32_t* idx, const int64_t* t_abs,
                           uint32_t count, const uint8_t* serve_mask, const Work& w, const uint32_t* count_dev) {
  const uint32_t ba = (count + kTrackThreads - 1) / kTrackThreads;
  const uint32_t br = (serve_mask && t.n) ? umin32((t.n + kTrackThreads - 1) / kTrackThreads, L.sm_count * 4) : 0u;
  const uint32_t blocks = ba > br ? ba : br;
  if (blocks)
    k_tracker_append<<<blocks, kTrackThreads, 0, L.stream>>>(t, idx, t_abs, count, count_dev, serve_mask, w);
}

// The per-call reset of a decision (instead of a memset node, which no programmatic launch can
// overlap): zero both lines of the call's globals; with now_dev, then read the decision time ONCE -- it may sit in mapped host memory, where every
// read is a PCIe round trip serialised at the host -- and publish the shift for every kernel.
__global__ void k_reset_now(Work w, const long long* now_dev, long long now_ref) {
  uint32_t* g = reinterpret_cast<uint32_t*>(w.g);
  for (uint32_t q = threadIdx.x; q < 2 * sizeof(Globals) / 4; q += blockDim.x) g[q] = 0u;
  __syncthreads();
  if (threadIdx.x == 0 && now_dev)
    globals2(w)->tshift = *reinterpret_cast<const volatile long long*>(now_dev) - now_ref;
}

void launch_reset_now(const LaunchCfg& L, const Work& w) {
  k_reset_now<<<1, 64, 0, L.stream>>>(w, w.now_dev, w.now_ref);
}

// The decision's head to mapped host memory (AndesDecision.export_host): one CTA, zero-copy writes
// over PCIe; the host reads it after its stream sync.
__global__ void k_decision_export(const uint32_t* __restrict__ scalars, const int64_t* __restrict__ V,
                                  const uint32_t* __restrict__ admit, const uint32_t* __restrict__ preempt,
                                  const uint8_t* __restrict__ serve_mask, Work w, uint32_t B_cap, uint32_t pmax,
                                  uint32_t smax, unsigned char* host) {
  __shared__ uint32_t s_n;
  uint32_t* h_sc = reinterpret_cast<uint32_t*>(host);
  long long* h_V = reinterpret_cast<long long*>(host + 32);
  uint32_t* h_adm = reinterpret_cast<uint32_t*>(host + 32 + 8 * (size_t)B_cap);
  uint32_t* h_pre = reinterpret_cast<uint32_t*>(host + 32 + 12 * (size_t)B_cap);
  const uint32_t tid = threadIdx.x;
  const uint32_t n_adm = min(__ldcg(scalars + 2), B_cap);
  const uint32_t n_pre = min(__ldcg(scalars + 3), pmax);
  if (tid < 8u) h_sc[tid] = __ldcg(scalars + tid);
  for (uint32_t b = tid; b < B_cap; b += blockDim.x) h_V[b] = __ldcg(V + b);
  for (uint32_t q = tid; q < n_adm; q += blockDim.x) h_adm[q] = __ldcg(admit + q);
  for (uint32_t q = tid; q < n_pre; q += blockDim.x) h_pre[q] = __ldcg(preempt + q);
  if (smax == 0) return;
  // the next batch: the running requests the decision kept (prep's run_list, serve mask still 1),
  // block-compacted, then the admits
  uint32_t* h_srv = reinterpret_cast<uint32_t*>(host + 32 + 12 * (size_t)B_cap + 4 * (size_t)pmax);
  if (tid == 0) s_n = 0u;
  __syncthreads();
  const uint32_t n_run = min(__ldcg(&w.g->n_run), (uint32_t)kMaxRunning);
  for (uint32_t q0 = 0; q0 < n_run; q0 += blockDim.x) {
    const uint32_t q = q0 + tid;
    const uint32_t i = q < n_run ? __ldcg(w.run_list + q) : 0u;
    const bool keep = q < n_run && serve_mask[i] != 0;
    const uint32_t bal = __ballot_sync(0xffffffffu, keep);
    uint32_t base = 0;
    if ((tid & 31) == 0 && bal) base = atomicAdd(&s_n, (uint32_t)__popc(bal));
    base = __shfl_sync(0xffffffffu, base, 0);
    const uint32_t slot = base + __popc(bal & ((1u << (tid & 31)) - 1u));
    if (keep && slot < smax) h_srv[slot] = i;
  }
  __syncthreads();
  const uint32_t nk = s_n;
  for (uint32_t q = tid; q < n_adm; q += blockDim.x)
    if (nk + q < smax) h_srv[nk + q] = __ldcg(admit + q);
}

// the export's completion word (after every section): the kernel's last store, behind a
// system-scope fence, so a host that polls it may read the block without a stream sync
__global__ void k_decision_export_done(unsigned long long* flag, unsigned long long v) {
  __threadfence_system();
  *reinterpret_cast<volatile unsigned long long*>(flag) = v;
}

void launch_decision_export(const LaunchCfg& L, const SchedOut& o, const Work& w, uint32_t B_cap, uint32_t pmax,
                            uint32_t smax, void* host) {
  k_decision_export<<<1, 256, 0, L.stream>>>(o.scalars, o.V, o.admit_idx, o.preempt_idx, o.serve_mask, w, B_cap, pmax,
                                             smax, static_cast<unsigned char*>(host));
  const size_t off = 32 + 12 * (size_t)B_cap + 4 * (size_t)pmax + 4 * (size_t)smax;
  k_decision_export_done<<<1, 1, 0, L.stream>>>(
      reinterpret_cast<unsigned long long*>(static_cast<unsigned char*>(host) + ((off + 7) & ~size_t(7))), 1ull);
}

}  // namespace andes
