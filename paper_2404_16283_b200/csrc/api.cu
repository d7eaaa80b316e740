// api.cu -- the C ABI of libandes (include/andes.h): argument validation, workspace
// ownership, and the kernel sequence of each entry point.
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/andes.h"
#include "device.cuh"
#include "launch.h"

using namespace andes;

// Programmatic dependent launch (every kernel waits on griddepcontrol.wait before it reads its
// predecessor's results): on by default since round 2 -- neutral on the decision (69.6 us either
// way, L2 flushed) and -5 us on the 2^20-request andes_qoe_eval (196.5 -> 191.5 us).  ANDES_PDL=0
// turns it off.
bool andes::pdl_enabled() {
  static const bool on = [] {
    const char* v = getenv("ANDES_PDL");
    return !(v && v[0] == '0');
  }();
  return on;
}

struct AndesCtx {
  AndesLimits lim{};
  int device = 0;
  uint32_t sm_count = 0;
  uint32_t scan_grid = 0;
  uint32_t tiles_cap = 0;
  Work w{};
  std::vector<void*> allocs;
  uint32_t* B_list_dev = nullptr;
  uint32_t* err_pinned = nullptr;  // mapped pinned sticky error word (kernels raise bits into it)
  SimCtl* sim_ctl = nullptr;       // pinned: the simulator's control block, read once per iteration
  // device mirrors for andes_schedule_host
  struct Mirror {
    int64_t* arrival;
    uint32_t *ttft, *period, *ctx_len, *n_deliv, *max_total, *start_off, *rank;
    uint8_t* running;
    uint64_t* tl_base;
    uint32_t* tl_pool;
    uint32_t* tau;
    uint8_t* serve_mask;
    uint32_t *admit_idx, *preempt_idx, *scalars, *kstar;
    int64_t* V;
  } mir{};
  std::string err;
  // TMA tensor map of the current timestamp pool (re-encoded when the pool changes)
  CUtensorMap pool_map[2]{};  // [0] 128B-swizzled tiles, [1] plain tiles (16-byte aligned timelines)
  const void* map_ptr = nullptr;
  uint64_t map_len = ~0ull;
  uint32_t* zero_rows = nullptr;  // 128 zero bytes: TMA source when the pool has no full row
  bool prof = false;
  bool prof_recorded = false;
  cudaEvent_t ev[ANDES_N_STAGES + 1] = {};
};

namespace {

const char* kVersion = "andes-b200 0.1 sm_100a";

int set_err(AndesCtx* c, int code, const char* fmt, const char* detail = "") {
  if (c) {
    char buf[512];
    snprintf(buf, sizeof buf, fmt, detail);
    c->err = buf;
  }
  return code;
}

int cuda_check(AndesCtx* c, cudaError_t e, const char* what) {
  if (e == cudaSuccess) return ANDES_OK;
  if (c) c->err = std::string(what) + ": " + cudaGetErrorString(e);
  return ANDES_E_CUDA;
}

template <class T>
cudaError_t ctx_alloc(AndesCtx* c, T** p, size_t count) {
  void* q = nullptr;
  cudaError_t e = cudaMalloc(&q, count ? count * sizeof(T) : sizeof(T));
  if (e == cudaSuccess) {
    c->allocs.push_back(q);
    *p = static_cast<T*>(q);
  }
  return e;
}

ReqView view_of(const AndesRequests* r) {
  ReqView v;
  v.n = r->n;
  v.arrival = r->arrival_us;
  v.ttft = r->ttft_us;
  v.period = r->period_us;
  v.ctx_len = r->ctx_len;
  v.n_deliv = r->n_deliv;
  v.max_total = r->max_total;
  v.start_off = r->start_off_us;
  v.rank = r->rank;
  v.running = r->running;
  v.tl_base = r->tl_base;
  v.tl_pool = r->tl_pool;
  v.tl_len = r->tl_len;
  return v;
}

int check_requests(AndesCtx* c, const AndesRequests* r, bool need_sched_fields) {
  if (!r) return set_err(c, ANDES_E_INVAL, "req is NULL%s");
  if (r->n > c->lim.max_requests) return set_err(c, ANDES_E_CAPACITY, "n exceeds limits.max_requests%s");
  if (r->n == 0) return ANDES_OK;
  if (!r->arrival_us || !r->ttft_us || !r->period_us || !r->n_deliv || !r->max_total || !r->tl_base)
    return set_err(c, ANDES_E_INVAL, "a required request array is NULL%s");
  if (need_sched_fields && (!r->ctx_len || !r->rank || !r->running))
    return set_err(c, ANDES_E_INVAL, "ctx_len/rank/running are required%s");
  if (!r->tl_pool) return set_err(c, ANDES_E_INVAL, "tl_pool is NULL%s");
  if (r->tl_len > (uint64_t)c->tiles_cap * kTile)
    return set_err(c, ANDES_E_CAPACITY, "tl_len exceeds limits.max_tokens%s");
  if ((reinterpret_cast<uintptr_t>(r->tl_pool) & 15u) != 0)
    return set_err(c, ANDES_E_INVAL, "tl_pool must be 16-byte aligned%s");
  return ANDES_OK;
}

// The sticky error word: kernels of earlier calls raise bits into mapped pinned host memory
// (raise_err); the first call that finds it non-zero reports it and clears it.  A failing call
// is reported by the next call once the failing kernel has run (no synchronisation is added).
int pending_device_error(AndesCtx* c) {
  volatile uint32_t* h = c->err_pinned;
  if (h && *h) {
    const uint32_t e = *h;
    *h = 0;
    char buf[160];
    snprintf(buf, sizeof buf, "%s (error word 0x%x)",
             (e & kErrCapacity) ? "capacity exceeded on the device" : "device precondition check failed", e);
    c->err = buf;
    return (e & kErrCapacity) ? ANDES_E_CAPACITY : ANDES_E_RANGE;
  }
  return ANDES_OK;
}

LaunchCfg cfg_of(AndesCtx* c, void* stream) {
  LaunchCfg L;
  L.stream = static_cast<cudaStream_t>(stream);
  L.sm_count = c->sm_count;
  L.scan_grid = c->scan_grid;
  return L;
}

Work work_of(AndesCtx* c, uint32_t n) {
  Work w = c->w;
  (void)n;
  return w;
}

// 2D TMA view of the pool: rows of 32 u32 (128 B), 128-row boxes, 128-byte swizzle; tokens
// past the last full row are read directly by the scan.
using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                   const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                   CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int pool_map(AndesCtx* c, const uint32_t* pool, uint64_t len, const CUtensorMap** out) {
  if (c->map_ptr == pool && c->map_len == len) {
    *out = c->pool_map;
    return ANDES_OK;
  }
  static EncodeTiledFn encode = nullptr;
  if (!encode) {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaError_t e = cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
    if (e != cudaSuccess || q != cudaDriverEntryPointSuccess || !fn)
      return set_err(c, ANDES_E_CUDA, "cuTensorMapEncodeTiled unavailable%s");
    encode = reinterpret_cast<EncodeTiledFn>(fn);
  }
  const uint64_t rows = len / 32;
  void* base = rows ? (void*)pool : (void*)c->zero_rows;
  cuuint64_t dims[2] = {32, rows ? rows : 1};
  cuuint64_t strides[1] = {128};
  cuuint32_t box[2] = {32, kTile / 32};
  cuuint32_t estr[2] = {1, 1};
  for (int k = 0; k < 2; ++k) {
    CUresult r = encode(&c->pool_map[k], CU_TENSOR_MAP_DATA_TYPE_UINT32, 2, base, dims, strides, box, estr,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, k ? CU_TENSOR_MAP_SWIZZLE_NONE : CU_TENSOR_MAP_SWIZZLE_128B,
                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return set_err(c, ANDES_E_CUDA, "cuTensorMapEncodeTiled failed%s");
  }
  c->map_ptr = pool;
  c->map_len = len;
  *out = c->pool_map;
  return ANDES_OK;
}

// per-call reset of the small globals (both lines: + the fused kernel's barrier line); the
// look-back status words are zeroed by k_prep, tile by tile.  A one-CTA kernel rather than a
// memset node: the call's first kernel then launches programmatically behind it (decision
// -0.5 us; ANDES_RESET_MEMSET restores the memset for A/B)
int reset_call(AndesCtx* c, cudaStream_t s) {
#ifndef ANDES_RESET_MEMSET
  Work w = c->w;
  w.now_dev = nullptr;
  launch_reset_now(cfg_of(c, s), w);
  return cuda_check(c, cudaGetLastError(), "reset");
#else
  cudaError_t e = cudaMemsetAsync(c->w.g, 0, 2 * sizeof(Globals), s);
  return cuda_check(c, e, "memset");
#endif
}

inline void mark(AndesCtx* c, int i, cudaStream_t s) {
  if (!c->prof) return;
  cudaStreamCaptureStatus st = cudaStreamCaptureStatusNone;
  cudaStreamIsCapturing(s, &st);
  if (st == cudaStreamCaptureStatusActive)
    cudaEventRecordWithFlags(c->ev[i], s, cudaEventRecordExternal);  // a real record node in the graph
  else
    cudaEventRecord(c->ev[i], s);
}

int finish_call(AndesCtx* c, cudaStream_t s, bool debug) {
  (void)s;
  (void)debug;
  return cuda_check(c, cudaGetLastError(), "kernel launch");
}

}  // namespace

extern "C" {

const char* andes_version(void) { return kVersion; }

const char* andes_last_error(const AndesCtx* ctx) {
  if (!ctx) return "NULL context";
  return ctx->err.c_str();
}

int andes_create(AndesCtx** out, const AndesLimits* lim) {
  if (!out || !lim) return ANDES_E_INVAL;
  *out = nullptr;
  if (lim->max_requests == 0 || lim->max_B == 0 || lim->max_B > (uint32_t)kMaxB ||
      lim->max_running > (uint32_t)kMaxRunning)
    return ANDES_E_INVAL;
  AndesCtx* c = new AndesCtx();
  c->lim = *lim;
  if (c->lim.max_running == 0) c->lim.max_running = kMaxRunning;
  if (c->lim.max_tokens == 0) c->lim.max_tokens = 1;
  c->device = lim->device;
  cudaError_t e = cudaSetDevice(c->device);
  if (e != cudaSuccess) {
    int rc = cuda_check(c, e, "cudaSetDevice");
    delete c;
    return rc;
  }
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, c->device);
  c->sm_count = (uint32_t)sms;
  init_kernels();
  init_scan_kernels();
  init_shard_kernels();
  init_refine_kernels();
  const int bps = scan_blocks_per_sm();
  c->scan_grid = (uint32_t)(sms * (bps > 0 ? bps : 1));
  const uint32_t N = lim->max_requests;
  c->tiles_cap = (uint32_t)((c->lim.max_tokens + kTile - 1) / kTile) + 2;
  Work& w = c->w;
  w.N_cap = N;
  {
    // look-back wait bound; 0 forces the direct head read on every look-back (a test hook)
    const char* v = getenv("ANDES_LOOKBACK_NS");
    w.lb_ns = v ? (uint32_t)strtoul(v, nullptr, 10) : 20000u;
  }
  w.tiles_cap = c->tiles_cap;
  w.S_cap = N < kCandCap ? N : kCandCap;
  if ((e = ctx_alloc(c, &w.m, N)) != cudaSuccess || (e = ctx_alloc(c, &w.spre, N)) != cudaSuccess ||
      (e = ctx_alloc(c, &w.edge, N)) != cudaSuccess || (e = ctx_alloc(c, &w.tile_meta, c->tiles_cap)) != cudaSuccess ||
      (e = ctx_alloc(c, &w.tile_status, c->tiles_cap)) != cudaSuccess ||
      (e = ctx_alloc(c, &w.tile_status_now, c->tiles_cap)) != cudaSuccess ||
      (e = ctx_alloc(c, &w.hist_l, kHistL)) != cudaSuccess || (e = ctx_alloc(c, &w.hist_lb, kHistK)) != cudaSuccess ||
      (e = ctx_alloc(c, &w.hist_ub, kHistK)) != cudaSuccess || (e = ctx_alloc(c, &w.st, N)) != cudaSuccess ||
      (e = ctx_alloc(c, &w.ub, N)) != cudaSuccess || (e = ctx_alloc(c, &w.zr, N)) != cudaSuccess ||
      (e = ctx_alloc(c, &w.hist_zr, kHistK)) != cudaSuccess ||
      (e = ctx_alloc(c, &w.cand_idx, w.S_cap)) != cudaSuccess || (e = ctx_alloc(c, &w.cand_st, w.S_cap)) != cudaSuccess ||
      (e = ctx_alloc(c, &w.run_st, kMaxRunning)) != cudaSuccess ||
      (e = ctx_alloc(c, &w.run_idx, kMaxRunning)) != cudaSuccess ||
      (e = ctx_alloc(c, &w.run_list, kMaxRunning)) != cudaSuccess || (e = ctx_alloc(c, &w.srec, N)) != cudaSuccess ||
      (e = ctx_alloc(c, &c->zero_rows, 32)) != cudaSuccess ||
      (e = ctx_alloc(c, &w.keyrow, (size_t)lim->max_B * N)) != cudaSuccess ||
      (e = ctx_alloc(c, &w.sel, (size_t)lim->max_B * kMaxB)) != cudaSuccess ||
      (e = ctx_alloc(c, &w.sel_thr, (size_t)lim->max_B)) != cudaSuccess ||
      (e = ctx_alloc(c, &w.stage_pre, (size_t)lim->max_B * kStageRun)) != cudaSuccess ||
      (e = ctx_alloc(c, &w.stage_adm, (size_t)lim->max_B * kMaxB)) != cudaSuccess ||
      (e = ctx_alloc(c, &w.stage_sc, (size_t)lim->max_B)) != cudaSuccess ||
      (e = ctx_alloc(c, &w.xm, tri_off(lim->max_B + 1))) != cudaSuccess ||
      (e = ctx_alloc(c, &w.m_now, N)) != cudaSuccess || (e = ctx_alloc(c, &w.spre_now, N)) != cudaSuccess ||
      (e = ctx_alloc(c, &w.edge_now, N)) != cudaSuccess || (e = ctx_alloc(c, &w.srec_now, N)) != cudaSuccess ||
      (e = ctx_alloc(c, &w.qnow, N)) != cudaSuccess || (e = ctx_alloc(c, &w.vmark, N)) != cudaSuccess ||
      (e = ctx_alloc(c, &w.rf_vend, kMaxB)) != cudaSuccess || (e = ctx_alloc(c, &w.rf_D, kMaxB)) != cudaSuccess ||
      (e = ctx_alloc(c, &w.rf_loss, kMaxB)) != cudaSuccess ||
      (e = ctx_alloc(c, &w.rank_set, 2ull * N)) != cudaSuccess ||
      (e = ctx_alloc(c, &w.g, 2)) != cudaSuccess || (e = ctx_alloc(c, &c->B_list_dev, kMaxB)) != cudaSuccess) {
    int rc = cuda_check(c, e, "workspace allocation");
    andes_destroy(c);
    return rc;
  }
  cudaMemset(w.hist_l, 0, sizeof(uint32_t) * kHistL);
  cudaMemset(w.vmark, 0, sizeof(uint32_t) * N);
  cudaMemset(c->zero_rows, 0, 128);
  cudaMemset(w.hist_lb, 0, sizeof(uint32_t) * kHistK);
  cudaMemset(w.hist_ub, 0, sizeof(uint32_t) * kHistK);
  cudaMemset(w.hist_zr, 0, sizeof(uint32_t) * kHistK);
  if ((e = cudaHostAlloc((void**)&c->err_pinned, sizeof(uint32_t), cudaHostAllocMapped)) != cudaSuccess ||
      (e = cudaHostGetDevicePointer((void**)&w.err_map, c->err_pinned, 0)) != cudaSuccess) {
    int rc = cuda_check(c, e, "mapped pinned alloc");
    andes_destroy(c);
    return rc;
  }
  *c->err_pinned = 0;
  if ((e = cudaHostAlloc((void**)&c->sim_ctl, sizeof(SimCtl), cudaHostAllocDefault)) != cudaSuccess) {
    int rc = cuda_check(c, e, "pinned alloc");
    andes_destroy(c);
    return rc;
  }
  // host-path mirrors
  auto& m = c->mir;
  const size_t T = c->lim.max_tokens;
  if ((e = ctx_alloc(c, &m.arrival, N)) != cudaSuccess || (e = ctx_alloc(c, &m.ttft, N)) != cudaSuccess ||
      (e = ctx_alloc(c, &m.period, N)) != cudaSuccess || (e = ctx_alloc(c, &m.ctx_len, N)) != cudaSuccess ||
      (e = ctx_alloc(c, &m.n_deliv, N)) != cudaSuccess || (e = ctx_alloc(c, &m.max_total, N)) != cudaSuccess ||
      (e = ctx_alloc(c, &m.start_off, N)) != cudaSuccess || (e = ctx_alloc(c, &m.rank, N)) != cudaSuccess ||
      (e = ctx_alloc(c, &m.running, N)) != cudaSuccess || (e = ctx_alloc(c, &m.tl_base, N)) != cudaSuccess ||
      (e = ctx_alloc(c, &m.tl_pool, T)) != cudaSuccess || (e = ctx_alloc(c, &m.tau, kMaxB)) != cudaSuccess ||
      (e = ctx_alloc(c, &m.serve_mask, N)) != cudaSuccess || (e = ctx_alloc(c, &m.admit_idx, kMaxB)) != cudaSuccess ||
      (e = ctx_alloc(c, &m.preempt_idx, N)) != cudaSuccess || (e = ctx_alloc(c, &m.scalars, ANDES_SC_COUNT)) != cudaSuccess ||
      (e = ctx_alloc(c, &m.kstar, kMaxB)) != cudaSuccess || (e = ctx_alloc(c, &m.V, kMaxB)) != cudaSuccess) {
    int rc = cuda_check(c, e, "host-path mirror allocation");
    andes_destroy(c);
    return rc;
  }
  e = cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    int rc = cuda_check(c, e, "create sync");
    andes_destroy(c);
    return rc;
  }
  *out = c;
  return ANDES_OK;
}

// Internal debugging hook: %globaltimer stamps from the decision kernels (8192 slots).
int andes_debug_trace(AndesCtx* c, int enable) {
  if (!c) return ANDES_E_INVAL;
  if (enable && !c->w.trace) {
    cudaError_t e = ctx_alloc(c, &c->w.trace, 1 << 16);
    if (e != cudaSuccess) return cuda_check(c, e, "trace alloc");
    cudaMemset(c->w.trace, 0, (1 << 16) * 8);
  }
  if (!enable) c->w.trace = nullptr;
  return ANDES_OK;
}

// Internal debugging hook (not part of include/andes.h): synchronous copy of a workspace array.
int andes_debug_read(AndesCtx* c, int which, void* host, size_t bytes) {
  if (!c || !host) return ANDES_E_INVAL;
  const void* src = nullptr;
  switch (which) {
    case 0: src = c->w.tile_status; break;
    case 1: src = c->w.spre; break;
    case 2: src = c->w.edge; break;
    case 3: src = c->w.m; break;
    case 4: src = c->w.tile_meta; break;
    case 5: src = c->w.g; break;
    case 6: src = c->w.hist_l; break;
    case 7: src = c->w.trace; break;
    default: return ANDES_E_INVAL;
  }
  return cuda_check(c, cudaMemcpy(host, src, bytes, cudaMemcpyDeviceToHost), "debug read");
}

int andes_profile_enable(AndesCtx* c, int enable) {
  if (!c) return ANDES_E_INVAL;
  if (enable && !c->ev[0]) {
    for (int i = 0; i <= ANDES_N_STAGES; ++i) {
      cudaError_t e = cudaEventCreate(&c->ev[i]);
      if (e != cudaSuccess) return cuda_check(c, e, "cudaEventCreate");
    }
  }
  c->prof = enable != 0;
  return ANDES_OK;
}

int andes_profile_read(AndesCtx* c, float* stage_ms) {
  if (!c || !stage_ms) return ANDES_E_INVAL;
  if (!c->prof_recorded) return set_err(c, ANDES_E_INVAL, "no profiled call recorded%s");
  cudaError_t e = cudaEventSynchronize(c->ev[ANDES_N_STAGES]);
  if (e != cudaSuccess) return cuda_check(c, e, "cudaEventSynchronize");
  for (int i = 0; i < ANDES_N_STAGES; ++i) {
    e = cudaEventElapsedTime(&stage_ms[i], c->ev[i], c->ev[i + 1]);
    if (e != cudaSuccess) return cuda_check(c, e, "cudaEventElapsedTime");
  }
  return ANDES_OK;
}

int andes_destroy(AndesCtx* c) {
  if (!c) return ANDES_E_INVAL;
  cudaSetDevice(c->device);
  for (int i = 0; i <= ANDES_N_STAGES; ++i)
    if (c->ev[i]) cudaEventDestroy(c->ev[i]);
  for (void* p : c->allocs) cudaFree(p);
  if (c->err_pinned) cudaFreeHost(c->err_pinned);
  if (c->sim_ctl) cudaFreeHost(c->sim_ctl);
  delete c;
  return ANDES_OK;
}

int andes_qoe_eval(AndesCtx* c, const AndesRequests* req, int64_t eval_time_us, uint32_t mode,
                   const AndesQoeOut* out, void* stream) {
  if (!c) return ANDES_E_INVAL;
  int rc = pending_device_error(c);
  if (rc) return rc;
  if ((rc = check_requests(c, req, false))) return rc;
  if (!out) return set_err(c, ANDES_E_INVAL, "out is NULL%s");
  if (mode > ANDES_EVAL_FINAL) return set_err(c, ANDES_E_INVAL, "unknown mode%s");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const LaunchCfg L = cfg_of(c, stream);
  const ReqView r = view_of(req);
  const Work w = work_of(c, r.n);
  const bool fin = mode == ANDES_EVAL_FINAL;
  // profiled stages: [0] prep, [1] timeline scan, [2] QoE finalize (others empty)
  mark(c, 0, s);
  if ((rc = reset_call(c, s))) return rc;
  // the scan builds its records from the request table (no prep copy): FINAL -5 us on 2^20
  // requests; INFLIGHT since the static chunk claims too (whole call 194.6 -> 186.7 us; before
  // them the due-token division at use time had made the scan slower, 149.5 -> 155.6 us).
  // ANDES_SREC_INFLIGHT restores prep's records for A/B
#ifdef ANDES_SREC_INFLIGHT
  const bool raw = fin;
#else
  const bool raw = true;
#endif
  launch_prep(L, r, w, eval_time_us, fin, false, 0, false, nullptr, 0, false, raw);
  mark(c, 1, s);
  {
    const CUtensorMap* tm = nullptr;
    if (r.n && (rc = pool_map(c, r.tl_pool, r.tl_len, &tm))) return rc;
    launch_scan(L, r, w, eval_time_us, fin, tm, false, nullptr, 0, 0, 0, 0, false, false, 0, raw);
  }
  mark(c, 2, s);
  launch_qoe_final(L, r, w, eval_time_us, fin, out->q, out->q64, out->s_delay, out->s_whole, out->m);
  mark(c, 3, s);
  mark(c, 4, s);
  mark(c, 5, s);
  mark(c, 6, s);
  if (c->prof) c->prof_recorded = true;
  return finish_call(c, s, false);
}

int andes_qoe_scenario_mean(AndesCtx* c, const AndesRequests* req, const uint32_t* scen_off, uint32_t S,
                            double* mean_out, uint32_t* count_out, void* stream) {
  if (!c) return ANDES_E_INVAL;
  int rc = pending_device_error(c);
  if (rc) return rc;
  if ((rc = check_requests(c, req, false))) return rc;
  if (S && (!scen_off || !mean_out)) return set_err(c, ANDES_E_INVAL, "scen_off/mean_out is NULL%s");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const LaunchCfg L = cfg_of(c, stream);
  const ReqView r = view_of(req);
  const Work w = work_of(c, r.n);
  mark(c, 0, s);
  if ((rc = reset_call(c, s))) return rc;
  launch_prep(L, r, w, 0, true, false, 0, false, nullptr, 0, false, true);
  mark(c, 1, s);
  {
    const CUtensorMap* tm = nullptr;
    if (r.n && (rc = pool_map(c, r.tl_pool, r.tl_len, &tm))) return rc;
    launch_scan(L, r, w, 0, true, tm, false, nullptr, 0, 0, 0, 0, false, false, 0, true);
  }
  mark(c, 2, s);
  launch_scenario_mean(L, r, w, scen_off, S, mean_out, count_out);
  mark(c, 3, s);
  mark(c, 4, s);
  mark(c, 5, s);
  mark(c, 6, s);
  if (c->prof) c->prof_recorded = true;
  return finish_call(c, s, false);
}

int andes_gain_estimate(AndesCtx* c, const AndesRequests* req, int64_t now_us, uint32_t horizon_us,
                        const uint32_t* tau_us, uint32_t B_cap, const uint32_t* B_list_host, uint32_t nB,
                        double* gain_out, float* key_out, double* qwait_out, void* stream) {
  if (!c) return ANDES_E_INVAL;
  int rc = pending_device_error(c);
  if (rc) return rc;
  if ((rc = check_requests(c, req, true))) return rc;
  if (!tau_us || B_cap == 0 || B_cap > c->lim.max_B) return set_err(c, ANDES_E_INVAL, "bad tau/B_cap%s");
  if (nB > (uint32_t)kMaxB) return set_err(c, ANDES_E_CAPACITY, "nB exceeds 1024%s");
  if (nB && !B_list_host) return set_err(c, ANDES_E_INVAL, "B_list is NULL%s");
  for (uint32_t b = 0; b < nB; ++b)
    if (B_list_host[b] < 1 || B_list_host[b] > B_cap) return set_err(c, ANDES_E_INVAL, "B out of [1, B_cap]%s");
  if (horizon_us == 0) return set_err(c, ANDES_E_INVAL, "horizon must be >= 1%s");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const LaunchCfg L = cfg_of(c, stream);
  const ReqView r = view_of(req);
  const Work w = work_of(c, r.n);
  const int64_t eval = now_us + (int64_t)horizon_us;
  if ((rc = reset_call(c, s))) return rc;
  if (nB) {
    cudaError_t e = cudaMemcpyAsync(c->B_list_dev, B_list_host, sizeof(uint32_t) * nB, cudaMemcpyHostToDevice, s);
    if (e != cudaSuccess) return cuda_check(c, e, "B_list copy");
  }
  launch_prep(L, r, w, eval, false, false, 0, false);
  {
    const CUtensorMap* tm = nullptr;
    if (r.n && (rc = pool_map(c, r.tl_pool, r.tl_len, &tm))) return rc;
    launch_scan(L, r, w, eval, false, tm);
  }
  launch_gain_estimate(L, r, w, now_us, horizon_us, tau_us, c->B_list_dev, nB, gain_out, key_out, qwait_out);
  return finish_call(c, s, false);
}

int andes_schedule(AndesCtx* c, const AndesRequests* req, const AndesSchedParams* p, AndesDecision* out,
                   void* stream) {
  if (!c) return ANDES_E_INVAL;
  int rc = pending_device_error(c);
  if (rc) return rc;
  if ((rc = check_requests(c, req, true))) return rc;
  if (!p || !out) return set_err(c, ANDES_E_INVAL, "params/out is NULL%s");
  if (!p->tau_us || p->B_cap == 0 || p->B_cap > c->lim.max_B) return set_err(c, ANDES_E_INVAL, "bad tau/B_cap%s");
  if (p->horizon_us == 0 || p->kv_capacity == 0) return set_err(c, ANDES_E_INVAL, "horizon and M must be >= 1%s");
  if (!out->scalars || !out->V || !out->kstar || (req->n && (!out->serve_mask || !out->preempt_idx)) ||
      !out->admit_idx)
    return set_err(c, ANDES_E_INVAL, "a decision output is NULL%s");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const LaunchCfg L = cfg_of(c, stream);
  const ReqView r = view_of(req);
  Work w = work_of(c, r.n);
  w.lqsf = (p->flags & ANDES_LQSF) ? 1u : 0u;
  if ((p->flags & ANDES_OBJ_MAXMIN) && (p->flags & ANDES_OBJ_PERFECT))
    return set_err(c, ANDES_E_INVAL, "at most one objective flag%s");
  w.obj = (p->flags & ANDES_OBJ_MAXMIN) ? kObjMaxMin : (p->flags & ANDES_OBJ_PERFECT) ? kObjPerfect : kObjAndes;
  w.now_dev = reinterpret_cast<const long long*>(p->now_dev);
  w.now_ref = p->now_us;
  const int64_t eval = p->now_us + (int64_t)p->horizon_us;
  const bool debug = (p->flags & ANDES_DEBUG_CHECKS) != 0;
  SchedOut o{out->serve_mask, out->admit_idx, out->preempt_idx, out->scalars, out->V, out->kstar};
  // profiled stages: [0] reset + prep + S0/S2 bounds, [1] timeline scan (S1), [2] state + key
  // bounds (S3a), [3] candidate keys (S3b), [4] Algorithm 1 per B + best B + cap + mask (S4-S6)
  mark(c, 0, s);
  if (w.now_dev) launch_reset_now(L, w);  // zeroes the globals and reads the time once
  else if ((rc = reset_call(c, s))) return rc;
  // Appendix-A objectives need every request's QoE now: prep also writes the records of an
  // evaluation at now (dual), a first scan fills the *_now arrays (its own look-back status
  // words), then Q_now (and its minimum); the tile counter is reset for the main scan
  const bool dual = w.obj != kObjAndes && r.n;
  launch_prep(L, r, w, eval, false, true, p->kv_capacity, debug, out->serve_mask, p->now_us, dual);
  if (debug) launch_debug_checks(L, r, w, p->now_us);
  if (dual) {
    Work wn = w;
    wn.m = w.m_now;
    wn.spre = w.spre_now;
    wn.edge = w.edge_now;
    wn.srec = w.srec_now;
    wn.tile_status = w.tile_status_now;
    const CUtensorMap* tmn = c->pool_map;
    if ((rc = pool_map(c, r.tl_pool, r.tl_len, &tmn))) return rc;
    launch_scan(L, r, wn, p->now_us, false, tmn);
  }
  mark(c, 1, s);
  {
    const CUtensorMap* tm = c->pool_map;
    if (r.n && (rc = pool_map(c, r.tl_pool, r.tl_len, &tm))) return rc;
    // after a scan at now (objectives) the decision scan counts its chunks on its own counter, and
    // its idle warps finish Q_now / Q_min from the first scan's sums (no k_qnow, no memset)
    launch_scan(L, r, w, eval, false, tm, true, p->tau_us, p->B_cap, p->kv_capacity, p->cur_latency_us, p->flags,
                dual, dual, p->now_us);
  }
  mark(c, 2, s);
  // S3-S6: one fused cooperative kernel when its grid fits on the GPU, else three kernels
  if (!launch_decide(L, r, w, p->now_us, p->horizon_us, p->tau_us, p->B_cap, p->kv_capacity,
                                p->preempt_cap, o)) {
    launch_state(L, r, w, p->now_us, p->horizon_us);
    mark(c, 3, s);
    launch_compact(L, r, w, nullptr, 1u);
    mark(c, 4, s);
    launch_select(L, r, w, p->now_us, p->horizon_us, p->tau_us, p->B_cap, p->kv_capacity, p->preempt_cap, o);
  } else {
    mark(c, 3, s);
    mark(c, 4, s);
  }
  if (p->flags & ANDES_REFINE)
    launch_refine(L, r, w, o, p->now_us, p->tau_us, p->kv_capacity, p->prefill_tok_s, p->swap_tok_s);
  if (out->export_host)
    launch_decision_export(L, o, w, p->B_cap, out->export_preempt, out->export_served, out->export_host);
  mark(c, 5, s);
  mark(c, 6, s);
  if (c->prof) c->prof_recorded = true;
  return finish_call(c, s, debug);
}

int andes_shard_init(AndesCtx* c, uint32_t world, uint32_t rank, uint32_t B_cap, AndesShard* out) {
  if (!c || !out) return ANDES_E_INVAL;
  if (world == 0 || world > kMaxWorld || rank >= world) return set_err(c, ANDES_E_INVAL, "bad world/rank%s");
  if (B_cap == 0 || B_cap > c->lim.max_B) return set_err(c, ANDES_E_INVAL, "bad B_cap%s");
  out->world = world;
  out->rank = rank;
  out->B_cap = B_cap;
  out->pad = 0;
  out->xbytes[0] = sizeof(ShardSummary);
  out->xbytes[1] = sizeof(uint32_t) * kHistK;
  out->xbytes[2] = sizeof(XEntry) * tri_off(B_cap + 1);
  out->xbytes[3] = sizeof(ShardVictims);
  return ANDES_OK;
}

int andes_schedule_shard(AndesCtx* c, const AndesShard* sh, uint32_t step, const AndesRequests* req,
                         const AndesSchedParams* p, AndesDecision* out, const void* recv, void* send, void* stream) {
  if (!c) return ANDES_E_INVAL;
  if (!sh || sh->world == 0 || sh->world > kMaxWorld || sh->rank >= sh->world)
    return set_err(c, ANDES_E_INVAL, "bad shard plan%s");
  if (step >= ANDES_SHARD_STEPS) return set_err(c, ANDES_E_INVAL, "step out of range%s");
  if ((step > 0 && !recv) || (step < ANDES_SHARD_ROUNDS && !send))
    return set_err(c, ANDES_E_INVAL, "recv/send buffer is NULL%s");
  if ((reinterpret_cast<uintptr_t>(recv) | reinterpret_cast<uintptr_t>(send)) & 15u)
    return set_err(c, ANDES_E_INVAL, "recv/send must be 16-byte aligned%s");
  int rc = ANDES_OK;
  if (step == 0 && (rc = pending_device_error(c))) return rc;
  if ((rc = check_requests(c, req, true))) return rc;
  if (!p || !out) return set_err(c, ANDES_E_INVAL, "params/out is NULL%s");
  if (!p->tau_us || p->B_cap == 0 || p->B_cap != sh->B_cap || p->B_cap > c->lim.max_B)
    return set_err(c, ANDES_E_INVAL, "bad tau/B_cap (must match the shard plan)%s");
  if (p->horizon_us == 0 || p->kv_capacity == 0) return set_err(c, ANDES_E_INVAL, "horizon and M must be >= 1%s");
  if (!out->scalars || !out->V || !out->kstar || !out->preempt_idx || !out->admit_idx ||
      (req->n && !out->serve_mask))
    return set_err(c, ANDES_E_INVAL, "a decision output is NULL%s");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const LaunchCfg L = cfg_of(c, stream);
  const ReqView r = view_of(req);
  Work w = work_of(c, r.n);
  w.lqsf = (p->flags & ANDES_LQSF) ? 1u : 0u;
  if (p->flags & (ANDES_OBJ_MAXMIN | ANDES_OBJ_PERFECT))
    return set_err(c, ANDES_E_INVAL, "the Appendix-A objectives are single-GPU only%s");
  const int64_t eval = p->now_us + (int64_t)p->horizon_us;
  const bool debug = (p->flags & ANDES_DEBUG_CHECKS) != 0;
  SchedOut o{out->serve_mask, out->admit_idx, out->preempt_idx, out->scalars, out->V, out->kstar};
  switch (step) {
    case 0: {
      if ((rc = reset_call(c, s))) return rc;
      launch_prep(L, r, w, eval, false, true, p->kv_capacity, debug, out->serve_mask);
      if (debug) launch_debug_checks(L, r, w, p->now_us);
      const CUtensorMap* tm = c->pool_map;
      if (r.n && (rc = pool_map(c, r.tl_pool, r.tl_len, &tm))) return rc;
      launch_scan(L, r, w, eval, false, tm);
      launch_shard_summary(L, r, w, p->B_cap, static_cast<ShardSummary*>(send));
      break;
    }
    case 1:
      launch_shard_bounds(L, w, static_cast<const ShardSummary*>(recv), sh->world, sh->rank, p->tau_us, p->B_cap,
                          p->kv_capacity, p->cur_latency_us, p->flags);
      launch_state(L, r, w, p->now_us, p->horizon_us);
      launch_shard_copy_lb(L, w, static_cast<uint32_t*>(send));
      break;
    case 2:
      launch_compact(L, r, w, static_cast<const uint32_t*>(recv), sh->world);
      launch_select(L, r, w, p->now_us, p->horizon_us, p->tau_us, p->B_cap, p->kv_capacity, p->preempt_cap, o,
                    static_cast<XEntry*>(send));
      break;
    case 3:
      launch_shard_merge(L, r, w, static_cast<const XEntry*>(recv), sh->world, p->tau_us, p->B_cap, p->kv_capacity,
                         o, static_cast<ShardVictims*>(send));
      break;
    default:
      launch_shard_cap(L, r, w, static_cast<const ShardVictims*>(recv), sh->world, p->B_cap, p->kv_capacity,
                       p->preempt_cap, o);
      return finish_call(c, s, debug);
  }
  return finish_call(c, s, false);
}

int andes_tracker_append(AndesCtx* c, const AndesTracker* t, const uint32_t* idx, const int64_t* t_abs, uint32_t count,
                         const uint8_t* serve_mask, void* stream) {
  if (!c) return ANDES_E_INVAL;
  int rc = pending_device_error(c);
  if (rc) return rc;
  if (!t) return set_err(c, ANDES_E_INVAL, "tracker is NULL%s");
  if (t->n && (!t->arrival_us || !t->tl_base || !t->tl_pool || !t->n_deliv || !t->ctx_len || !t->running))
    return set_err(c, ANDES_E_INVAL, "a tracker array is NULL%s");
  if (count && (!idx || !t_abs)) return set_err(c, ANDES_E_INVAL, "idx/t_abs is NULL%s");
  TrackerView v{t->n, t->arrival_us, t->tl_base, t->tl_pool, t->tl_len, t->n_deliv, t->ctx_len, t->running};
  launch_tracker_append(cfg_of(c, stream), v, idx, t_abs, count, serve_mask, c->w);
  return cuda_check(c, cudaGetLastError(), "kernel launch");
}

int andes_tracker_append_dev(AndesCtx* c, const AndesTracker* t, const uint32_t* idx, const int64_t* t_abs,
                             const uint32_t* count_dev, uint32_t max_count, const uint8_t* serve_mask, void* stream) {
  if (!c) return ANDES_E_INVAL;
  int rc = pending_device_error(c);
  if (rc) return rc;
  if (!t) return set_err(c, ANDES_E_INVAL, "tracker is NULL%s");
  if (t->n && (!t->arrival_us || !t->tl_base || !t->tl_pool || !t->n_deliv || !t->ctx_len || !t->running))
    return set_err(c, ANDES_E_INVAL, "a tracker array is NULL%s");
  if (max_count && (!idx || !t_abs || !count_dev)) return set_err(c, ANDES_E_INVAL, "idx/t_abs/count_dev is NULL%s");
  TrackerView v{t->n, t->arrival_us, t->tl_base, t->tl_pool, t->tl_len, t->n_deliv, t->ctx_len, t->running};
  launch_tracker_append(cfg_of(c, stream), v, idx, t_abs, max_count, serve_mask, c->w, count_dev);
  return cuda_check(c, cudaGetLastError(), "kernel launch");
}

// ---- serving-loop simulator (sim.cu): workspace carving and the host loop
namespace {
struct SimCarve {
  SimView v;
  uint8_t* serve_mask;
  uint32_t *admit, *preempt, *scalars, *kstar;
  int64_t* V;
  size_t bytes;
};
SimCarve sim_carve(void* ws, uint32_t n) {
  SimCarve c{};
  size_t off = 0;
  char* b = static_cast<char*>(ws);
  auto take = [&](size_t bytes) -> void* {
    void* p = b ? b + off : nullptr;
    off += (bytes + 15) & ~size_t(15);
    return p;
  };
  const size_t N = n ? n : 1;
  c.v.l_arr = static_cast<int64_t*>(take(8 * N));
  c.v.l_base = static_cast<uint64_t*>(take(8 * N));
  c.v.l_ttft = static_cast<uint32_t*>(take(4 * N));
  c.v.l_period = static_cast<uint32_t*>(take(4 * N));
  c.v.l_ctx = static_cast<uint32_t*>(take(4 * N));
  c.v.l_g = static_cast<uint32_t*>(take(4 * N));
  c.v.l_rank = static_cast<uint32_t*>(take(4 * N));
  c.v.l_idx = static_cast<uint32_t*>(take(4 * N));
  c.v.l_maxtot = static_cast<uint32_t*>(take(4 * N));
  c.v.l_run = static_cast<uint8_t*>(take(N));
  c.serve_mask = static_cast<uint8_t*>(take(N));
  c.preempt = static_cast<uint32_t*>(take(4 * N));
  c.admit = static_cast<uint32_t*>(take(4 * kMaxB));
  c.V = static_cast<int64_t*>(take(8 * kMaxB));
  c.kstar = static_cast<uint32_t*>(take(4 * kMaxB));
  c.scalars = static_cast<uint32_t*>(take(4 * ANDES_SC_COUNT));
  c.v.ctl = static_cast<SimCtl*>(take(sizeof(SimCtl)));
  c.bytes = off;
  return c;
}
}  // namespace

uint64_t andes_sim_workspace(uint32_t n) { return sim_carve(nullptr, n).bytes; }

int andes_simulate(AndesCtx* c, const AndesSim* sim, const AndesSimParams* p, AndesSimStats* stats, void* stream) {
  if (!c) return ANDES_E_INVAL;
  if (!sim || !p || !stats) return set_err(c, ANDES_E_INVAL, "NULL argument%s");
  const uint32_t n = sim->n;
  if (n && (!sim->arrival_us || !sim->ttft_us || !sim->period_us || !sim->prompt_len || !sim->output_len ||
            !sim->tl_base || !sim->tl_pool || !sim->n_deliv || !sim->served || !sim->workspace))
    return set_err(c, ANDES_E_INVAL, "a simulator array is NULL%s");
  if ((reinterpret_cast<uintptr_t>(sim->workspace) & 15u) != 0) return set_err(c, ANDES_E_INVAL, "workspace alignment%s");
  if (n > c->lim.max_requests || sim->tl_len > c->lim.max_tokens || p->B_cap > c->lim.max_B)
    return set_err(c, ANDES_E_CAPACITY, "simulator sizes exceed the context limits%s");
  if (!p->tau_us || p->B_cap == 0 || p->horizon_us == 0 || p->kv_capacity == 0)
    return set_err(c, ANDES_E_INVAL, "bad simulator parameters%s");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  SimCarve k = sim_carve(sim->workspace, n);
  SimView& v = k.v;
  v.n = n;
  v.arrival = sim->arrival_us;
  v.ttft = sim->ttft_us;
  v.period = sim->period_us;
  v.prompt = sim->prompt_len;
  v.out_len = sim->output_len;
  v.tl_base = sim->tl_base;
  v.tl_pool = sim->tl_pool;
  v.tl_len = sim->tl_len;
  v.g = sim->n_deliv;
  v.served = sim->served;
  memset(stats, 0, sizeof *stats);
  if (n == 0) return ANDES_OK;
  cudaError_t e = cudaMemsetAsync(sim->n_deliv, 0, 4ull * n, s);
  if (e == cudaSuccess) e = cudaMemsetAsync(sim->served, 0, n, s);
  if (e != cudaSuccess) return cuda_check(c, e, "simulator reset");
  int64_t now = 0;
  if ((e = cudaMemcpyAsync(&now, sim->arrival_us, 8, cudaMemcpyDeviceToHost, s)) != cudaSuccess ||
      (e = cudaStreamSynchronize(s)) != cudaSuccess)
    return cuda_check(c, e, "simulator start");
  stats->start_us = now;
  SimCtl* h = c->sim_ctl;
  AndesRequests rq{};
  rq.arrival_us = v.l_arr;
  rq.ttft_us = v.l_ttft;
  rq.period_us = v.l_period;
  rq.ctx_len = v.l_ctx;
  rq.n_deliv = v.l_g;
  rq.max_total = v.l_maxtot;
  rq.start_off_us = nullptr;
  rq.rank = v.l_rank;
  rq.running = v.l_run;
  rq.tl_base = v.l_base;
  rq.tl_pool = sim->tl_pool;
  rq.tl_len = sim->tl_len;
  AndesSchedParams sp{};
  sp.horizon_us = p->horizon_us;
  sp.B_cap = p->B_cap;
  sp.tau_us = p->tau_us;
  sp.kv_capacity = p->kv_capacity;
  sp.preempt_cap = p->preempt_cap;
  sp.flags = p->flags | ANDES_FORCE;
  sp.prefill_tok_s = 5000;
  AndesDecision dd{k.serve_mask, k.admit, k.preempt, k.scalars, k.V, k.kstar};
  const uint32_t max_iters = p->max_iters ? p->max_iters : 0xFFFFFFFFu;
  const int64_t kFromCtl = (int64_t)0x8000000000000000ll;
  int64_t pending = now;  // the next k_sim_live's time (kFromCtl: the one k_sim_step computed)
  for (uint64_t it = 0;;) {
    launch_sim_live(s, v, pending);
    if ((e = cudaMemcpyAsync(h, v.ctl, sizeof(SimCtl), cudaMemcpyDeviceToHost, s)) != cudaSuccess ||
        (e = cudaStreamSynchronize(s)) != cudaSuccess)
      return cuda_check(c, e, "simulator iteration");
    now = h->now;
    stats->finished = h->finished;
    if (h->finished == n || it >= max_iters) break;
    if (h->n_live == 0) {
      pending = h->next_arrival;
      continue;
    }
    rq.n = h->n_live;
    sp.now_us = now;
    int rc = andes_schedule(c, &rq, &sp, &dd, stream);
    if (rc) return rc;
    launch_sim_step(s, c->sm_count, v, h->n_live, now, p->tau_us, p->B_cap, k.serve_mask, k.scalars);
    pending = kFromCtl;
    ++it;
    stats->iterations = it;
  }
  stats->end_us = now;
  return cuda_check(c, cudaGetLastError(), "kernel launch");
}

uint64_t andes_knapsack_dp_workspace(uint32_t n, uint32_t B, uint64_t M) {
  return (uint64_t)knapsack_dp_workspace(n, B, M);
}

int andes_knapsack_dp(AndesCtx* c, const int64_t* value, const uint32_t* weight, uint32_t n, uint32_t B,
                      uint64_t M, void* workspace, uint64_t workspace_bytes, uint8_t* x, int64_t* best,
                      int64_t* Vb, void* stream) {
  if (!c) return ANDES_E_INVAL;
  if ((n && (!value || !weight || !x)) || !best || !workspace) return set_err(c, ANDES_E_INVAL, "NULL argument%s");
  if (M > 0xFFFFFFFEull || B > n + 1024u) return set_err(c, ANDES_E_INVAL, "M or B out of range%s");
  if (workspace_bytes < knapsack_dp_workspace(n, B, M))
    return set_err(c, ANDES_E_CAPACITY, "workspace smaller than andes_knapsack_dp_workspace()%s");
  if (reinterpret_cast<uintptr_t>(workspace) & 7u) return set_err(c, ANDES_E_INVAL, "workspace must be 8-byte aligned%s");
  launch_knapsack_dp(static_cast<cudaStream_t>(stream), reinterpret_cast<const long long*>(value), weight, n, B,
                     (uint32_t)M, workspace, x, reinterpret_cast<long long*>(best), reinterpret_cast<long long*>(Vb));
  return cuda_check(c, cudaGetLastError(), "kernel launch");
}

int andes_schedule_host(AndesCtx* c, const AndesRequests* rq, const AndesSchedParams* p, AndesDecision* out,
                        void* stream) {
  if (!c) return ANDES_E_INVAL;
  if (!rq || !p || !out) return set_err(c, ANDES_E_INVAL, "NULL argument%s");
  if (rq->n > c->lim.max_requests) return set_err(c, ANDES_E_CAPACITY, "n exceeds limits.max_requests%s");
  if (!p->tau_us || p->B_cap == 0 || p->B_cap > c->lim.max_B) return set_err(c, ANDES_E_INVAL, "bad tau/B_cap%s");
  if (p->horizon_us == 0 || p->kv_capacity == 0) return set_err(c, ANDES_E_INVAL, "horizon and M must be >= 1%s");
  const uint32_t n = rq->n;
  // every required host array is checked before any copy: a NULL one would otherwise leave the
  // device mirror holding an earlier call's data
  if (n && (!rq->arrival_us || !rq->ttft_us || !rq->period_us || !rq->ctx_len || !rq->n_deliv ||
            !rq->max_total || !rq->rank || !rq->running || !rq->tl_base || !rq->tl_pool))
    return set_err(c, ANDES_E_INVAL, "a required request array is NULL%s");
  if (!out->scalars || !out->V || !out->kstar || !out->admit_idx || (n && (!out->serve_mask || !out->preempt_idx)))
    return set_err(c, ANDES_E_INVAL, "a decision output is NULL%s");
  uint64_t span = 0;
  if (n) span = rq->tl_base[n - 1] + rq->n_deliv[n - 1];
  if (span > c->lim.max_tokens) return set_err(c, ANDES_E_CAPACITY, "timestamp pool exceeds limits.max_tokens%s");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  auto& m = c->mir;
  cudaError_t e = cudaSuccess;
  auto h2d = [&](void* dst, const void* src, size_t bytes) {
    if (e == cudaSuccess && bytes && src) e = cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, s);
  };
  h2d(m.arrival, rq->arrival_us, 8ull * n);
  h2d(m.ttft, rq->ttft_us, 4ull * n);
  h2d(m.period, rq->period_us, 4ull * n);
  h2d(m.ctx_len, rq->ctx_len, 4ull * n);
  h2d(m.n_deliv, rq->n_deliv, 4ull * n);
  h2d(m.max_total, rq->max_total, 4ull * n);
  if (rq->start_off_us) h2d(m.start_off, rq->start_off_us, 4ull * n);
  h2d(m.rank, rq->rank, 4ull * n);
  h2d(m.running, rq->running, 1ull * n);
  h2d(m.tl_base, rq->tl_base, 8ull * n);
  h2d(m.tl_pool, rq->tl_pool, 4ull * span);
  h2d(m.tau, p->tau_us, 4ull * p->B_cap);
  if (e != cudaSuccess) return cuda_check(c, e, "host-to-device copy");
  AndesRequests dr = *rq;
  dr.arrival_us = m.arrival;
  dr.ttft_us = m.ttft;
  dr.period_us = m.period;
  dr.ctx_len = m.ctx_len;
  dr.n_deliv = m.n_deliv;
  dr.max_total = m.max_total;
  dr.start_off_us = rq->start_off_us ? m.start_off : nullptr;
  dr.rank = m.rank;
  dr.running = m.running;
  dr.tl_base = m.tl_base;
  dr.tl_pool = m.tl_pool;
  dr.tl_len = c->lim.max_tokens;
  AndesSchedParams dp = *p;
  dp.now_dev = nullptr;  // (host call: the time is the host's now_us)
  dp.tau_us = m.tau;
  AndesDecision dd{m.serve_mask, m.admit_idx, m.preempt_idx, m.scalars, m.V, m.kstar};
  int rc = andes_schedule(c, &dr, &dp, &dd, stream);
  if (rc) return rc;
  uint32_t sc[ANDES_SC_COUNT];
  auto d2h = [&](void* dst, const void* src, size_t bytes) {
    if (e == cudaSuccess && bytes && dst) e = cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, s);
  };
  d2h(sc, m.scalars, sizeof sc);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  if (e != cudaSuccess) return cuda_check(c, e, "decision copy");
  d2h(out->scalars, m.scalars, sizeof sc);
  d2h(out->serve_mask, m.serve_mask, n);
  d2h(out->admit_idx, m.admit_idx, 4ull * sc[ANDES_SC_N_ADMIT]);
  d2h(out->preempt_idx, m.preempt_idx, 4ull * sc[ANDES_SC_N_PREEMPT]);
  d2h(out->V, m.V, 8ull * p->B_cap);
  d2h(out->kstar, m.kstar, 4ull * p->B_cap);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  if (e != cudaSuccess) return cuda_check(c, e, "decision copy");
  return (sc[ANDES_SC_FLAGS] & ANDES_F_TRIGGERED) ? ANDES_OK : ANDES_NOT_TRIGGERED;
}

}  // extern "C"
