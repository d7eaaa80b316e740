// comm.cu -- the sharded decision's all-gathers over peer memory (CUDA IPC), without NCCL.
//
// SURVEY 8(e) / include/andes.h andes_comm_*: every rank owns an arena in its device memory --
// G flags (u64) and two parities of G slots of max_block bytes -- exported once as an IPC handle
// and opened by every peer (P2P mappings over NVLink between GPUs of a node; on one GPU, plain
// device memory of another process).  One all-gather of `bytes` <= max_block at sequence number q
// (q counts this communicator's all-gathers, the same on every rank: all ranks issue them in the
// same order):
//   k_comm_push   every CTA copies this rank's block into slot `rank` of parity q & 1 of every
//                 arena (own included), fences at system scope and counts itself; the last CTA
//                 publishes q into flag `rank` of every arena (volatile stores);
//   k_comm_pull   every CTA waits until its arena's G flags reach q (bounded spin, %globaltimer),
//                 then copies its part of the G slots of parity q & 1 into recv (rank order).
// Two parities suffice: a rank can start all-gather q + 1 (writing parity (q+1) & 1) only after
// every peer published q, i.e. after every peer finished all-gather q - 1, whose slots (parity
// (q-1) & 1) are the ones it overwrites.  A wait that exceeds the bound (a peer that never
// arrives) raises the communicator's error word; the next all-gather returns ANDES_E_NCCL.
#include <cuda_runtime.h>

#include <cstdint>

#include "device.cuh"
#include "launch.h"

namespace andes {

constexpr int kCommThreads = 256;
constexpr uint32_t kCommMaxWorld = 8;

struct CommView {
  uint8_t* arena[kCommMaxWorld];  // every rank's arena base (own included), this process's mapping
  uint32_t world, rank;
  uint64_t slot;                  // bytes per slot (max_block rounded up to 256)
  unsigned long long* seq;        // this rank's all-gather counter (device, local)
  uint32_t* ctr;                  // push CTAs finished (last-block pattern, self-cleaning)
  uint32_t* err;                  // sticky error word (device, local)
  unsigned long long wait_ns;     // spin bound
};

__device__ __forceinline__ unsigned long long* flags_of(uint8_t* arena) {
  return reinterpret_cast<unsigned long long*>(arena);
}
__device__ __forceinline__ uint8_t* slot_of(const CommView& v, uint8_t* arena, uint32_t par, uint32_t g) {
  return arena + 256 + ((size_t)par * v.world + g) * v.slot;
}

__global__ void __launch_bounds__(kCommThreads) k_comm_push(CommView v, const uint8_t* __restrict__ send,
                                                            uint64_t bytes) {
  const unsigned long long q = *reinterpret_cast<volatile unsigned long long*>(v.seq) + 1ull;
  const uint32_t par = (uint32_t)(q & 1ull);
  const uint64_t n16 = bytes / 16;
  const uint4* src = reinterpret_cast<const uint4*>(send);
  for (uint64_t e = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n16 * v.world;
       e += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t g = (uint32_t)(e / n16);
    const uint64_t k = e - (uint64_t)g * n16;
    reinterpret_cast<uint4*>(slot_of(v, v.arena[g], par, v.rank))[k] = src[k];
  }
  // the tail bytes (bytes not a multiple of 16)
  if (blockIdx.x == 0)
    for (uint64_t b = n16 * 16 + threadIdx.x; b < bytes; b += blockDim.x)
      for (uint32_t g = 0; g < v.world; ++g) slot_of(v, v.arena[g], par, v.rank)[b] = send[b];
  __threadfence_system();
  __syncthreads();
  __shared__ uint32_t s_last;
  if (threadIdx.x == 0) s_last = (atomicAdd(v.ctr, 1u) == gridDim.x - 1) ? 1u : 0u;
  __syncthreads();
  if (!s_last) return;
  __threadfence_system();
  if (threadIdx.x < v.world)
    reinterpret_cast<volatile unsigned long long*>(flags_of(v.arena[threadIdx.x]))[v.rank] = q;
  if (threadIdx.x == 0) {
    *v.ctr = 0u;
    *reinterpret_cast<volatile unsigned long long*>(v.seq) = q;  // read by k_comm_pull (next in stream)
  }
}

__global__ void __launch_bounds__(kCommThreads) k_comm_pull(CommView v, uint8_t* __restrict__ recv, uint64_t bytes) {
  const unsigned long long q = *reinterpret_cast<volatile unsigned long long*>(v.seq);
  const uint32_t par = (uint32_t)(q & 1ull);
  uint8_t* own = v.arena[v.rank];
  if (threadIdx.x == 0) {
    const volatile unsigned long long* f = flags_of(own);
    const unsigned long long t0 = gtimer();
    uint32_t ok = 1u;
    for (uint32_t g = 0; g < v.world; ++g) {
      while (f[g] < q) {
        if (gtimer() - t0 > v.wait_ns) {
          ok = 0u;
          break;
        }
        __nanosleep(256);
      }
    }
    if (!ok) atomicOr(v.err, 1u);
  }
  __syncthreads();
  __threadfence_system();
  const uint64_t n16 = bytes / 16;
  for (uint64_t e = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n16 * v.world;
       e += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t g = (uint32_t)(e / n16);
    const uint64_t k = e - (uint64_t)g * n16;
    reinterpret_cast<uint4*>(recv + (size_t)g * bytes)[k] =
        __ldcv(reinterpret_cast<const uint4*>(slot_of(v, own, par, g)) + k);  // (not cached in L1)
  }
  if (blockIdx.x == 0)
    for (uint64_t b = n16 * 16 + threadIdx.x; b < bytes; b += blockDim.x)
      for (uint32_t g = 0; g < v.world; ++g)
        recv[(size_t)g * bytes + b] = *reinterpret_cast<const volatile uint8_t*>(slot_of(v, own, par, g) + b);
}

void launch_comm_allgather(cudaStream_t s, const CommView& v, const void* send, void* recv, uint64_t bytes,
                           uint32_t sm_count) {
  const uint64_t n16 = bytes / 16 * v.world;
  uint32_t blocks = (uint32_t)((n16 + kCommThreads - 1) / kCommThreads);
  if (blocks < 1) blocks = 1;
  if (blocks > sm_count) blocks = sm_count;
  k_comm_push<<<blocks, kCommThreads, 0, s>>>(v, static_cast<const uint8_t*>(send), bytes);
  k_comm_pull<<<blocks, kCommThreads, 0, s>>>(v, static_cast<uint8_t*>(recv), bytes);
}

}  // namespace andes

// ---------------------------------------------------------------- host side (include/andes.h)
#include <cstring>

#include "../../include/andes.h"

struct AndesComm {
  int device = 0;
  uint32_t world = 0, rank = 0, sm_count = 1;
  uint64_t max_block = 0, slot = 0;
  uint8_t* arena = nullptr;
  uint8_t* peer[andes::kCommMaxWorld] = {};
  unsigned long long* seq = nullptr;
  uint32_t* ctr = nullptr;
  uint32_t* err = nullptr;  // mapped pinned host word (device writes, host reads)
  bool connected = false;
};

namespace {
size_t arena_bytes(uint32_t world, uint64_t slot) { return 256 + 2ull * world * slot; }
}  // namespace

extern "C" int andes_comm_create(AndesComm** out, int device, uint32_t world, uint32_t rank, uint64_t max_block,
                                 void* handle_out) {
  if (!out || !handle_out || world == 0 || world > andes::kCommMaxWorld || rank >= world || max_block == 0)
    return ANDES_E_INVAL;
  *out = nullptr;
  if (cudaSetDevice(device) != cudaSuccess) return ANDES_E_CUDA;
  AndesComm* c = new AndesComm();
  c->device = device;
  c->world = world;
  c->rank = rank;
  c->max_block = max_block;
  c->slot = (max_block + 255) / 256 * 256;
  int sms = 1;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
  c->sm_count = (uint32_t)sms;
  const size_t ab = arena_bytes(world, c->slot);
  if (cudaMalloc(&c->arena, ab) != cudaSuccess || cudaMalloc(&c->seq, 64) != cudaSuccess ||
      cudaHostAlloc(reinterpret_cast<void**>(&c->err), 4, cudaHostAllocMapped) != cudaSuccess) {
    andes_comm_destroy(c);
    return ANDES_E_CUDA;
  }
  c->ctr = reinterpret_cast<uint32_t*>(reinterpret_cast<uint8_t*>(c->seq) + 8);
  cudaMemset(c->arena, 0, ab);
  cudaMemset(c->seq, 0, 64);
  *c->err = 0u;
  cudaIpcMemHandle_t h;
  if (cudaIpcGetMemHandle(&h, c->arena) != cudaSuccess || cudaDeviceSynchronize() != cudaSuccess) {
    andes_comm_destroy(c);
    return ANDES_E_CUDA;
  }
  static_assert(sizeof(cudaIpcMemHandle_t) == ANDES_COMM_HANDLE_BYTES, "IPC handle size");
  std::memcpy(handle_out, &h, sizeof h);
  c->peer[rank] = c->arena;
  *out = c;
  return ANDES_OK;
}

extern "C" int andes_comm_connect(AndesComm* c, const void* handles) {
  if (!c || !handles) return ANDES_E_INVAL;
  if (cudaSetDevice(c->device) != cudaSuccess) return ANDES_E_CUDA;
  for (uint32_t g = 0; g < c->world; ++g) {
    if (g == c->rank) continue;
    cudaIpcMemHandle_t h;
    std::memcpy(&h, static_cast<const uint8_t*>(handles) + (size_t)g * ANDES_COMM_HANDLE_BYTES, sizeof h);
    void* p = nullptr;
    if (cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess) != cudaSuccess) return ANDES_E_CUDA;
    c->peer[g] = static_cast<uint8_t*>(p);
  }
  c->connected = true;
  return ANDES_OK;
}

extern "C" int andes_comm_allgather(AndesComm* c, const void* send, void* recv, uint64_t bytes, void* stream) {
  if (!c || !c->connected || !send || !recv || bytes > c->max_block) return ANDES_E_INVAL;
  // 16-byte vector copies: blocks, send and recv 16-byte aligned
  if ((bytes & 15u) || ((reinterpret_cast<uintptr_t>(send) | reinterpret_cast<uintptr_t>(recv)) & 15u))
    return ANDES_E_INVAL;
  if (c->err && *reinterpret_cast<volatile uint32_t*>(c->err)) {
    *c->err = 0u;
    return ANDES_E_NCCL;  // an earlier all-gather waited past its bound for a peer
  }
  andes::CommView v{};
  for (uint32_t g = 0; g < c->world; ++g) v.arena[g] = c->peer[g];
  v.world = c->world;
  v.rank = c->rank;
  v.slot = c->slot;
  v.seq = c->seq;
  v.ctr = c->ctr;
  uint32_t* derr = nullptr;
  cudaHostGetDevicePointer(reinterpret_cast<void**>(&derr), c->err, 0);
  v.err = derr;
  v.wait_ns = 10ull * 1000 * 1000 * 1000;  // 10 s: processes sharing one GPU are time-sliced
  andes::launch_comm_allgather(static_cast<cudaStream_t>(stream), v, send, recv, bytes, c->sm_count);
  return cudaGetLastError() == cudaSuccess ? ANDES_OK : ANDES_E_CUDA;
}

extern "C" int andes_comm_destroy(AndesComm* c) {
  if (!c) return ANDES_OK;
  cudaSetDevice(c->device);
  for (uint32_t g = 0; g < c->world; ++g)
    if (g != c->rank && c->peer[g]) cudaIpcCloseMemHandle(c->peer[g]);
  if (c->arena) cudaFree(c->arena);
  if (c->seq) cudaFree(c->seq);
  if (c->err) cudaFreeHost(c->err);
  delete c;
  return ANDES_OK;
}
