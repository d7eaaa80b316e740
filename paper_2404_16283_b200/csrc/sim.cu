// sim.cu -- NEXT-3: an on-device serving-loop simulator.  A trace of requests
// (arrival order) is served iteration by iteration with the library's own decision in the loop,
// the delivered tokens appended on the device, so that average end-of-trace QoE can be
// compared across policies (Andes' priority gain / l vs LQSF, reading R21) and loads -- the
// fig:e2e-intensity / fig:e2e-duration analogs of P:L989-1022, without models (the iteration
// latency is the tau(B) table; zero preemption overhead, as config 1's driver).
//
// One iteration at time `now`:
//   k_sim_live  the live table: arrived (a_i <= now) and unfinished (g_i < out_i) requests, a
//               stable compaction of the trace prefix (rank = trace index, running = served in
//               the previous iteration, l = prompt + g, output length unknown to the scheduler:
//               max_total = UINT32_MAX, reading R7); counts into the control block
//   andes_schedule over the live table (S0-S6, forced)
//   k_sim_step  every served request receives one token at now' = now + tau(min(realized, B_cap))
//               (realized >= 1), appended to its timeline; the served set becomes the running set
// The host loop (api.cu, andes_simulate) reads the 32-byte control block once per iteration.
#include "device.cuh"
#include "launch.h"

namespace andes {

constexpr int kSimThreads = 1024;

// now_in: the iteration's time, or INT64_MIN to take the one k_sim_step left in the control block
__global__ void __launch_bounds__(kSimThreads) k_sim_live(SimView v, int64_t now_in) {
  __shared__ uint32_t s_w[kSimThreads / 32];
  __shared__ uint32_t s_hi, s_done, s_base;
  const uint32_t tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int64_t now = now_in == (int64_t)0x8000000000000000ll ? v.ctl->now : now_in;
  if (tid == 0) {
    // arrived prefix: arrivals are nondecreasing (binary search)
    uint32_t lo = 0, hi = v.n;
    while (lo < hi) {
      const uint32_t mid = (lo + hi) >> 1;
      if (v.arrival[mid] <= now) lo = mid + 1;
      else hi = mid;
    }
    s_hi = lo;
    s_done = 0;
    s_base = 0;
  }
  __syncthreads();
  const uint32_t hi = s_hi;
  uint32_t done = 0;
  for (uint32_t c0 = 0; c0 < hi; c0 += kSimThreads) {
    const uint32_t i = c0 + tid;
    const bool in = i < hi;
    const uint32_t g = in ? v.g[i] : 0u;
    const bool live = in && g < v.out_len[i];
    done += (in && !live) ? 1u : 0u;
    const uint32_t bal = __ballot_sync(0xffffffffu, live);
    if (lane == 0) s_w[wid] = __popc(bal);
    __syncthreads();
    uint32_t off = s_base;
    for (uint32_t k = 0; k < wid; ++k) off += s_w[k];
    if (live) {
      const uint32_t s = off + __popc(bal & ((1u << lane) - 1u));
      v.l_arr[s] = v.arrival[i];
      v.l_ttft[s] = v.ttft[i];
      v.l_period[s] = v.period[i];
      v.l_ctx[s] = v.prompt[i] + g;
      v.l_g[s] = g;
      v.l_rank[s] = i;
      v.l_run[s] = v.served[i];
      v.l_base[s] = v.tl_base[i];
      v.l_idx[s] = i;
      v.l_maxtot[s] = 0xFFFFFFFFu;
    }
    __syncthreads();
    if (tid == 0) {
      uint32_t t = 0;
      for (uint32_t k = 0; k < kSimThreads / 32; ++k) t += s_w[k];
      s_base += t;
    }
    __syncthreads();
  }
  for (int o = 16; o; o >>= 1) done += __shfl_xor_sync(0xffffffffu, done, o);
  if (lane == 0 && done) atomicAdd(&s_done, done);
  __syncthreads();
  if (tid == 0) {
    SimCtl* c = v.ctl;
    c->now = now;
    c->n_live = s_base;
    c->finished = s_done;
    c->next_arrival = hi < v.n ? v.arrival[hi] : (int64_t)0x7FFFFFFFFFFFFFFFll;
  }
}

__global__ void k_sim_step(SimView v, uint32_t n_live, int64_t now, const uint32_t* __restrict__ tau, uint32_t B_cap,
                           const uint8_t* __restrict__ serve_mask, const uint32_t* __restrict__ scalars) {
  const uint32_t realized = max(1u, min(scalars[1], B_cap));
  const int64_t t_new = now + (int64_t)tau[realized - 1];
  for (uint32_t s = blockIdx.x * blockDim.x + threadIdx.x; s < n_live; s += gridDim.x * blockDim.x) {
    const uint32_t i = v.l_idx[s];
    const uint8_t on = serve_mask[s];
    v.served[i] = on;
    if (on) {
      const uint32_t g = v.l_g[s];
      const unsigned long long slot = v.tl_base[i] + g;
      const unsigned long long limit = (i + 1 < v.n) ? v.tl_base[i + 1] : v.tl_len;
      if (slot < limit) {
        v.tl_pool[slot] = (uint32_t)(t_new - v.arrival[i]);
        v.g[i] = g + 1;
      }
    }
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) v.ctl->now = t_new;
}

void launch_sim_live(cudaStream_t s, const SimView& v, int64_t now) { k_sim_live<<<1, kSimThreads, 0, s>>>(v, now); }

void launch_sim_step(cudaStream_t s, uint32_t sm_count, const SimView& v, uint32_t n_live, int64_t now,
                     const uint32_t* tau, uint32_t B_cap, const uint8_t* serve_mask, const uint32_t* scalars) {
  const uint32_t blocks = umin32((n_live + 255) / 256, sm_count * 4);
  k_sim_step<<<blocks ? blocks : 1u, 256, 0, s>>>(v, n_live, now, tau, B_cap, serve_mask, scalars);
}

}  // namespace andes
