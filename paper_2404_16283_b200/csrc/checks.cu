// checks.cu -- device-side data-precondition checks of a decision (ANDES_DEBUG_CHECKS only;
// include/andes.h "Conventions").  Off the hot path: launched only when the flag is set.
//
//   timestamps  every request's delivery times are nondecreasing and each is <= now - a_i (a
//               token cannot have been delivered after the decision time; P:L337 tracks
//               delivered tokens) -> kErrTimes
//   ranks       the rank field is unique over the population (the deterministic tie-break of
//               reading R10 needs a total order) -> kErrRank; exact, by an open-addressing set of
//               rank + 1 (u64 slots, 0 = empty) in the workspace, cleared before every check
// The context-length, period, tl_base-order and due-count checks run inside k_prep.
#include "device.cuh"
#include "launch.h"

namespace andes {

constexpr int kCheckThreads = 256;

__global__ void __launch_bounds__(kCheckThreads) k_debug_checks(ReqView r, Work w, int64_t now) {
  now += tshift(w);  // (AndesSchedParams.now_dev)
  const uint32_t n = r.n;
  const uint32_t lane = threadIdx.x & 31;
  uint32_t err = 0;
  // timestamps: one warp per request
  const uint32_t warps = gridDim.x * (blockDim.x / 32);
  for (uint32_t i = (blockIdx.x * blockDim.x + threadIdx.x) / 32; i < n; i += warps) {
    const uint64_t base = r.tl_base[i];
    const uint32_t g = r.n_deliv[i];
    const int64_t age = now - r.arrival[i];
    if (base + g > r.tl_len) {
      err |= kErrTimes;
      continue;
    }
    for (uint32_t j = lane; j < g; j += 32) {
      const uint32_t d = r.tl_pool[base + j];
      if ((int64_t)d > age) err |= kErrTimes;
      if (j > 0 && r.tl_pool[base + j - 1] > d) err |= kErrTimes;
    }
  }
  // rank uniqueness: insert rank + 1 into the open-addressing set (2 N_cap slots)
  const uint64_t S = 2ull * w.N_cap;
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const unsigned long long key = (unsigned long long)r.rank[i] + 1ull;
    uint64_t slot = (key * 0x9E3779B97F4A7C15ull) % S;
    for (uint64_t probe = 0; probe < S; ++probe) {
      const unsigned long long old = atomicCAS(reinterpret_cast<unsigned long long*>(w.rank_set) + slot, 0ull, key);
      if (old == 0ull) break;
      if (old == key) {
        err |= kErrRank;
        break;
      }
      slot = slot + 1 == S ? 0 : slot + 1;
    }
  }
  err = __reduce_or_sync(0xffffffffu, err);
  if (lane == 0 && err) raise_err(w, err);
}

void launch_debug_checks(const LaunchCfg& L, const ReqView& r, const Work& w, int64_t now) {
  if (r.n == 0) return;
  cudaMemsetAsync(w.rank_set, 0, sizeof(unsigned long long) * 2ull * w.N_cap, L.stream);
  const uint32_t blocks = umin32((r.n + kCheckThreads / 32 - 1) / (kCheckThreads / 32), L.sm_count * 8);
  k_debug_checks<<<blocks, kCheckThreads, 0, L.stream>>>(r, w, now);
}

}  // namespace andes
