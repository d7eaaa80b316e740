// launch.h -- internal host-side launchers of libandes (not part of the C ABI).
#pragma once
#include <cstdint>
#include <utility>
#include <cuda_runtime.h>
#include "device.cuh"

namespace andes {

// Programmatic dependent launch: off unless the environment sets ANDES_PDL=1 (see api.cu).
bool pdl_enabled();

// Launch with programmatic stream serialization (PDL): the kernel may begin while its stream
// predecessor finishes; it must call pdl_wait() before touching the predecessor's results.
template <class... KArgs, class... Args>
inline cudaError_t launch_pdl(void (*k)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                              Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, k, std::forward<Args>(args)...);
}

struct LaunchCfg {
  cudaStream_t stream;
  uint32_t sm_count;
  uint32_t scan_grid;  // persistent grid of the timeline scan (all CTAs co-resident)
};

void launch_prep(const LaunchCfg& L, const ReqView& r, const Work& w, int64_t eval_abs, bool final_mode,
                 bool sched, uint64_t kv_cap, bool debug, uint8_t* serve_mask = nullptr, int64_t now_abs = 0,
                 bool dual = false, bool eval = false);
void launch_scan(const LaunchCfg& L, const ReqView& r, const Work& w, int64_t eval_abs, bool final_mode,
                 const CUtensorMap* tmap, bool sched = false, const uint32_t* tau = nullptr, uint32_t B_cap = 0,
                 uint64_t M = 0, uint32_t cur_latency = 0, uint32_t flags = 0, bool second = false,
                 bool qnow = false, int64_t now_abs = 0, bool eval = false);
void launch_qoe_final(const LaunchCfg& L, const ReqView& r, const Work& w, int64_t eval_abs, bool final_mode,
                      float* q, double* q64, int64_t* sd, int64_t* sw, uint32_t* m);
void launch_scenario_mean(const LaunchCfg& L, const ReqView& r, const Work& w, const uint32_t* off, uint32_t S,
                          double* mean_out, uint32_t* count_out);
void launch_qnow(const LaunchCfg& L, const ReqView& r, const Work& w, int64_t now);
int scan_blocks_per_sm();
void init_scan_kernels();

struct SchedOut {
  uint8_t* serve_mask;
  uint32_t* admit_idx;
  uint32_t* preempt_idx;
  uint32_t* scalars;
  int64_t* V;
  uint32_t* kstar;
};

void launch_reset_now(const LaunchCfg& L, const Work& w);
struct CommView;
void launch_comm_allgather(cudaStream_t s, const CommView& v, const void* send, void* recv, uint64_t bytes,
                           uint32_t sm_count);
void launch_decision_export(const LaunchCfg& L, const SchedOut& o, const Work& w, uint32_t B_cap, uint32_t pmax,
                            uint32_t smax, void* host);
void launch_gain_estimate(const LaunchCfg& L, const ReqView& r, const Work& w, int64_t now, uint32_t horizon,
                          const uint32_t* tau, const uint32_t* B_list_dev, uint32_t nB, double* gain_out,
                          float* key_out, double* qwait_out);
void launch_state(const LaunchCfg& L, const ReqView& r, const Work& w, int64_t now, uint32_t horizon);
void launch_select(const LaunchCfg& L, const ReqView& r, const Work& w, int64_t now, uint32_t horizon,
                   const uint32_t* tau, uint32_t B_cap, uint64_t M, uint32_t preempt_cap, const SchedOut& o,
                   XEntry* xsend = nullptr);
void launch_compact(const LaunchCfg& L, const ReqView& r, const Work& w, const uint32_t* lb_src, uint32_t G);
bool launch_decide(const LaunchCfg& L, const ReqView& r, const Work& w, int64_t now, uint32_t horizon,
                   const uint32_t* tau, uint32_t B_cap, uint64_t M, uint32_t preempt_cap, const SchedOut& o);
// multi-GPU decision steps (shard.cu)
constexpr uint32_t kMaxWorld = 8;
void launch_shard_summary(const LaunchCfg& L, const ReqView& r, const Work& w, uint32_t B_cap, ShardSummary* out);
void launch_shard_bounds(const LaunchCfg& L, const Work& w, const ShardSummary* all, uint32_t G, uint32_t rank,
                         const uint32_t* tau, uint32_t B_cap, uint64_t M, uint32_t cur_latency, uint32_t flags);
void launch_shard_copy_lb(const LaunchCfg& L, const Work& w, uint32_t* send);
void launch_shard_merge(const LaunchCfg& L, const ReqView& r, const Work& w, const XEntry* recv, uint32_t G,
                        const uint32_t* tau, uint32_t B_cap, uint64_t M, const SchedOut& o, ShardVictims* send);
void launch_shard_cap(const LaunchCfg& L, const ReqView& r, const Work& w, const ShardVictims* recv, uint32_t G,
                      uint32_t B_cap, uint64_t M, uint32_t preempt_cap, const SchedOut& o);
void init_shard_kernels();
void init_refine_kernels();
size_t knapsack_dp_workspace(uint32_t n, uint32_t B, uint64_t M);
void launch_knapsack_dp(cudaStream_t s, const long long* q, const uint32_t* l, uint32_t n, uint32_t B, uint32_t M,
                        void* ws, uint8_t* x, long long* best, long long* Vb);
void launch_refine(const LaunchCfg& L, const ReqView& r, const Work& w, const SchedOut& o, int64_t now,
                   const uint32_t* tau, uint64_t M, uint32_t prefill, uint32_t swap);
void init_kernels();
void launch_tracker_append(const LaunchCfg& L, const TrackerView& t, const uint32_t* idx, const int64_t* t_abs,
                           uint32_t count, const uint8_t* serve_mask, const Work& w, const uint32_t* count_dev = nullptr);
void launch_sim_live(cudaStream_t s, const SimView& v, int64_t now);
void launch_sim_step(cudaStream_t s, uint32_t sm_count, const SimView& v, uint32_t n_live, int64_t now,
                     const uint32_t* tau, uint32_t B_cap, const uint8_t* serve_mask, const uint32_t* scalars);
void launch_debug_checks(const LaunchCfg& L, const ReqView& r, const Work& w, int64_t now);

}  // namespace andes
