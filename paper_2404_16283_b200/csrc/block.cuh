// block.cuh -- CTA-wide helpers shared by the selection kernels (select.cu, shard.cu):
// ordered keys of the closed-form gain, block reductions and scans, bitonic sort and an exact
// radix top-k select in shared memory.  Internal to libandes.
#pragma once
#include "device.cuh"

namespace andes {

constexpr int kSelThreads = 512;
constexpr int kSortCap = kMaxB;
constexpr int kVictCap = kMaxRunning;


// ---------------------------------------------------------------- block helpers
__device__ __forceinline__ double gain_of(const PackedState& p, uint32_t tau, uint32_t obj) {
  return gain_obj(unpack_state(p), p.qx, tau, obj);
}

__device__ __forceinline__ uint32_t okey_of(const PackedState& p, uint32_t tau, uint32_t lqsf, uint32_t obj) {
  return ordered_key(prio_key(gain_of(p, tau, obj), p.l, lqsf));
}

__device__ __forceinline__ unsigned long long comp_of(const PackedState& p, uint32_t tau, uint32_t lqsf,
                                                     uint32_t obj) {
  return composite(okey_of(p, tau, lqsf, obj), p.rank);
}

template <int NT>
__device__ __forceinline__ long long block_sum_ll(long long v, long long* red) {
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  __syncthreads();
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  long long t = 0;
  if (threadIdx.x < 32) {
    t = (threadIdx.x < NT / 32) ? red[threadIdx.x] : 0;
    for (int o = 16; o; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
    if (threadIdx.x == 0) red[0] = t;
  }
  __syncthreads();
  t = red[0];
  __syncthreads();
  return t;
}

// In-place bitonic sort of (key, idx) pairs in shared memory, size = power of two.
template <int NT>
__device__ void bitonic_sort(unsigned long long* key, uint32_t* idx, uint32_t size, bool descending) {
  for (uint32_t k = 2; k <= size; k <<= 1) {
    for (uint32_t j = k >> 1; j > 0; j >>= 1) {
      for (uint32_t t = threadIdx.x; t < size; t += NT) {
        const uint32_t p = t ^ j;
        if (p > t) {
          const bool up = ((t & k) == 0) == descending;
          const unsigned long long a = key[t], b = key[p];
          if ((a < b) == up) {
            key[t] = b;
            key[p] = a;
            const uint32_t x = idx[t];
            idx[t] = idx[p];
            idx[p] = x;
          }
        }
      }
      __syncthreads();
    }
  }
}

// Exact MSB-first radix select (8-bit digits) of the k-th largest of ne unique 64-bit
// composites, then collection of the k largest into (s_key, s_idx), sorted descending.
// comp(e, low) returns element e's composite (its low 32 bits are needed only when low is
// true); id(e) the request index stored with it.
template <class Comp, class Id>
__device__ uint32_t select_top_k(uint32_t ne, uint32_t k, Comp comp, Id id, unsigned long long* s_key,
                                 uint32_t* s_idx) {
  __shared__ uint32_t s_hist[256];
  __shared__ unsigned long long s_prefix;
  __shared__ uint32_t s_need, s_cnt;
  __shared__ int s_stop;
  const uint32_t tid = threadIdx.x;
  unsigned long long prefix = 0ull, mask = 0ull;
  uint32_t need = k;
  for (int shift = 56; shift >= 0; shift -= 8) {
    for (uint32_t q = tid; q < 256; q += kSelThreads) s_hist[q] = 0u;
    __syncthreads();
    for (uint32_t e = tid; e < ne; e += kSelThreads) {
      const unsigned long long c = comp(e, shift < 32);
      if ((c & mask) == prefix) atomicAdd(&s_hist[(uint32_t)(c >> shift) & 255u], 1u);
    }
    __syncthreads();
    if (tid < 32) {
      uint32_t cnt[8], tot = 0;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        cnt[j] = s_hist[255 - 8 * tid - j];
        tot += cnt[j];
      }
      uint32_t inc = tot;
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t v = __shfl_up_sync(0xffffffffu, inc, o);
        if (tid >= (uint32_t)o) inc += v;
      }
      const uint32_t exc = inc - tot;
      if (exc < need && inc >= need) {
        uint32_t above = exc;
        for (int j = 0; j < 8; ++j) {
          if (above + cnt[j] >= need) {
            s_prefix = prefix | ((unsigned long long)(255 - 8 * tid - j) << shift);
            s_need = need - above;
            s_stop = (cnt[j] == need - above) ? 1 : 0;
            break;
          }
          above += cnt[j];
        }
      }
    }
    __syncthreads();
    prefix = s_prefix;
    need = s_need;
    mask |= 255ull << shift;
    if (s_stop) break;
  }
  const unsigned long long theta = prefix;
  if (tid == 0) s_cnt = 0;
  __syncthreads();
  for (uint32_t e = tid; e < ne; e += kSelThreads) {
    const unsigned long long hi = comp(e, false) | 0xFFFFFFFFull;
    if (hi < theta) continue;
    const unsigned long long c = comp(e, true);
    if (c >= theta) {
      const uint32_t slot = atomicAdd(&s_cnt, 1u);
      if (slot < (uint32_t)kSortCap) {
        s_key[slot] = c;
        s_idx[slot] = id(e);
      }
    }
  }
  __syncthreads();
  const uint32_t cnt = min(s_cnt, (uint32_t)kSortCap);
  uint32_t size = 1;
  while (size < cnt) size <<= 1;
  for (uint32_t q = cnt + tid; q < size; q += kSelThreads) {
    s_key[q] = 0ull;
    s_idx[q] = 0xFFFFFFFFu;
  }
  __syncthreads();
  bitonic_sort<kSelThreads>(s_key, s_idx, size, true);
  return cnt;
}

// In-place inclusive prefix sums of v[0..cnt) (cnt <= 8 * kSelThreads) by the whole CTA.
__device__ __forceinline__ void block_inclusive_scan(unsigned long long* v, uint32_t cnt, unsigned long long* s_tmp) {
  const uint32_t tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const uint32_t per = (cnt + kSelThreads - 1) / kSelThreads;
  const uint32_t lo = min(cnt, tid * per), hi = min(cnt, lo + per);
  unsigned long long part = 0;
  for (uint32_t q = lo; q < hi; ++q) part += v[q];
  unsigned long long inc = part;
  for (int o = 1; o < 32; o <<= 1) {
    const unsigned long long x = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= (uint32_t)o) inc += x;
  }
  if (lane == 31) s_tmp[wid] = inc;
  __syncthreads();
  unsigned long long wpre = lane < wid ? s_tmp[lane] : 0ull;  // kSelThreads / 32 <= 32 warps
  for (int o = 16; o; o >>= 1) wpre += __shfl_xor_sync(0xffffffffu, wpre, o);
  unsigned long long run = wpre + inc - part;
  for (uint32_t q = lo; q < hi; ++q) {
    run += v[q];
    v[q] = run;
  }
  __syncthreads();
}

}  // namespace andes
