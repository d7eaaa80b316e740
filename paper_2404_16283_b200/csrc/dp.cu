// dp.cu -- Algorithm 2: the exact 3D dynamic program for Eq. 5 at a target batch
// size B (NEXT-4: a decision-quality reference for small N * M; the paper's point is that it is
// too slow for real-time use).  Values are int64 (e.g. llrint(gain 2^32), reading
// R9) so that the table is exact and the comparisons match the oracle's transcription.
//   dp[i][b][m] = max(dp[i-1][b][m], dp[i-1][b-1][m-l_i] + q_i), the line order of Algorithm 2:
//   "not served" when strictly better than the current cell, then "served" when strictly better;
//   Q_max = the first maximum of dp[N][B][:]; backtracking over the choice table.
// One CTA sweeps the items; every (b, m) cell of a layer is updated in parallel from the previous
// layer (double-buffered in the caller's workspace); the choice table is one byte per cell.
#include <cstdint>

#include "device.cuh"
#include "launch.h"

namespace andes {

constexpr uint32_t kDpThreads = 1024;
constexpr long long kNeg = (long long)0x8000000000000000ull;  // -infinity

__global__ void __launch_bounds__(kDpThreads) k_knapsack_dp(const long long* __restrict__ q,
                                                            const uint32_t* __restrict__ l, uint32_t n, uint32_t B,
                                                            uint32_t M, long long* lay0, long long* lay1,
                                                            uint8_t* choice, uint8_t* x, long long* best,
                                                            long long* Vb) {
  __shared__ long long s_v[32];
  __shared__ uint32_t s_m[32];
  __shared__ uint32_t s_mcur;
  __shared__ long long s_best;
  const uint32_t tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const size_t W = (size_t)M + 1, cells = (size_t)(B + 1) * W;
  for (size_t c = tid; c < cells; c += kDpThreads) lay0[c] = (c == 0) ? 0ll : kNeg;
  __syncthreads();
  long long* prev = lay0;
  long long* cur = lay1;
  for (uint32_t i = 1; i <= n; ++i) {
    const uint32_t li = l[i - 1];
    const long long qi = q[i - 1];
    const uint32_t bmax = min(i, B);
    uint8_t* ch = choice + (size_t)(i - 1) * cells;
    for (size_t c = tid; c < cells; c += kDpThreads) {
      const uint32_t b = (uint32_t)(c / W), m = (uint32_t)(c - (size_t)b * W);
      long long v = kNeg;
      uint8_t cc = 0;
      if (b <= bmax) {
        const long long o = prev[c];
        if (o != kNeg) v = o;  // -inf < dp[i-1][b][m]: not served
        if (b >= 1 && m >= li) {
          const long long p = prev[c - W - li];
          if (p != kNeg && (v == kNeg || p + qi > v)) {  // served
            v = p + qi;
            cc = 1;
          }
        }
      }
      cur[c] = v;
      ch[c] = cc;
    }
    __syncthreads();
    long long* t = prev;
    prev = cur;
    cur = t;
  }
  // per-b optimum (max over m of dp[N][b][:]) and the first argmax of dp[N][B][:]
  for (uint32_t b = 0; b <= B; ++b) {
    long long bv = kNeg;
    uint32_t bm = 0xFFFFFFFFu;
    for (uint32_t m = tid; m <= M; m += kDpThreads) {
      const long long v = prev[(size_t)b * W + m];
      if (v != kNeg && (bv == kNeg || v > bv)) {  // strictly greater keeps the smallest m
        bv = v;
        bm = m;
      }
    }
    for (int o = 16; o; o >>= 1) {
      const long long v2 = __shfl_xor_sync(0xffffffffu, bv, o);
      const uint32_t m2 = __shfl_xor_sync(0xffffffffu, bm, o);
      if (v2 != kNeg && (bv == kNeg || v2 > bv || (v2 == bv && m2 < bm))) {
        bv = v2;
        bm = m2;
      }
    }
    if (lane == 0) {
      s_v[wid] = bv;
      s_m[wid] = bm;
    }
    __syncthreads();
    if (tid == 0) {
      long long v = kNeg;
      uint32_t mm = 0xFFFFFFFFu;
      for (uint32_t k = 0; k < kDpThreads / 32; ++k)
        if (s_v[k] != kNeg && (v == kNeg || s_v[k] > v || (s_v[k] == v && s_m[k] < mm))) {
          v = s_v[k];
          mm = s_m[k];
        }
      if (Vb) Vb[b] = v;
      if (b == B) {
        s_best = v;
        s_mcur = mm;
      }
    }
    __syncthreads();
  }
  for (uint32_t k = tid; k < n; k += kDpThreads) x[k] = 0;
  __syncthreads();
  if (tid == 0) {
    *best = s_best;
    if (s_best != kNeg) {
      uint32_t b = B, m = s_mcur;
      for (uint32_t i = n; i >= 1; --i) {
        const uint8_t c = choice[(size_t)(i - 1) * cells + (size_t)b * W + m];
        x[i - 1] = c;
        if (c) {
          m -= l[i - 1];
          b -= 1;
        }
      }
    }
  }
}

size_t knapsack_dp_workspace(uint32_t n, uint32_t B, uint64_t M) {
  const size_t cells = (size_t)(B + 1) * (size_t)(M + 1);
  return 2 * cells * sizeof(long long) + (size_t)n * cells;
}

void launch_knapsack_dp(cudaStream_t s, const long long* q, const uint32_t* l, uint32_t n, uint32_t B, uint32_t M,
                        void* ws, uint8_t* x, long long* best, long long* Vb) {
  const size_t cells = (size_t)(B + 1) * (size_t)(M + 1);
  long long* lay0 = static_cast<long long*>(ws);
  long long* lay1 = lay0 + cells;
  uint8_t* choice = reinterpret_cast<uint8_t*>(lay1 + cells);
  k_knapsack_dp<<<1, kDpThreads, 0, s>>>(q, l, n, B, M, lay0, lay1, choice, x, best, Vb);
}

}  // namespace andes
