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
__global__ void __launch_bounds__(kTrackThreads) k_tracker_append(TrackerView t, const uint32_t* __restrict__ idx,
                                                                 const int64_t* __restrict__ t_abs, uint32_t count,
                                                                 Work w) {
  const uint32_t k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= count) return;
  const uint32_t i = idx[k];
  if (i >= t.n) {
    raise_err(w, kErrTokens);
    return;
  }
  // first token of this request's run of tokens (runs are consecutive in k)
  uint32_t k0 = k;
  while (k0 > 0 && idx[k0 - 1] == i) --k0;
  const bool last = (k + 1 == count) || idx[k + 1] != i;
  const uint32_t g = t.n_deliv[i];
  const unsigned long long base = t.tl_base[i];
  const unsigned long long limit = (i + 1 < t.n) ? t.tl_base[i + 1] : t.tl_len;
  const unsigned long long slot = base + g + (k - k0);
  const unsigned long long runlen = (unsigned long long)(k - k0) + 1ull;
  if (base + g + runlen > limit) {  // no room for this run's tokens: reject the whole run
    if (last) raise_err(w, kErrTokens);
    return;
  }
  const long long d = t_abs[k] - t.arrival[i];
  t.tl_pool[slot] = (uint32_t)(d < 0 ? 0 : d);
  if (last) {
    t.n_deliv[i] = g + (uint32_t)runlen;
    t.ctx_len[i] += (uint32_t)runlen;
  }
}

__global__ void k_tracker_running(TrackerView t, const uint8_t* __restrict__ serve_mask) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < t.n; i += gridDim.x * blockDim.x)
    t.running[i] = serve_mask[i];
}

void launch_tracker_append(const LaunchCfg& L, const TrackerView& t, const uint32_t* idx, const int64_t* t_abs,
                           uint32_t count, const uint8_t* serve_mask, const Work& w) {
  if (count) {
    k_tracker_append<<<(count + kTrackThreads - 1) / kTrackThreads, kTrackThreads, 0, L.stream>>>(t, idx, t_abs,
                                                                                                  count, w);
  }
  if (serve_mask && t.n) {
    const uint32_t blocks = umin32((t.n + 255) / 256, L.sm_count * 4);
    k_tracker_running<<<blocks, 256, 0, L.stream>>>(t, serve_mask);
  }
}

}  // namespace andes
