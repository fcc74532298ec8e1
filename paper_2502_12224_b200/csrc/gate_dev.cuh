// Device building blocks of K1 (router + cross-layer predictor), shared by
// the standalone gate kernel and the engine's fused decode/prefill kernels.
#pragma once

#include "fate_internal.cuh"

namespace fate {

// fp64 dot product of one row with h, by one warp; h and row are [H].
// Fixed per-lane stride order and a fixed butterfly, so the result is
// deterministic run to run.
__device__ __forceinline__ double warp_dot64(const double *__restrict__ row, const double *__restrict__ h, int H) {
  const int lane = threadIdx.x & 31;
  double acc = 0.0;
  if ((H & 1) == 0 && ((reinterpret_cast<uintptr_t>(row) | reinterpret_cast<uintptr_t>(h)) & 15) == 0) {
    const double2 *r2 = reinterpret_cast<const double2 *>(row);
    const double2 *h2 = reinterpret_cast<const double2 *>(h);
#pragma unroll 4
    for (int i = lane; i < H / 2; i += 32) {
      const double2 a = __ldg(r2 + i);
      const double2 b = h2[i];
      acc = fma(a.x, b.x, acc);
      acc = fma(a.y, b.y, acc);
    }
  } else {
    for (int i = lane; i < H; i += 32) acc = fma(__ldg(row + i), h[i], acc);
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  return acc;
}

// Softmax over z[E] (shared memory, already divided by tau) into w[E], then
// the rank order by (-w, id) into order[E].  Executed by ONE full warp.
// Returns the prediction-prefix length for the policy (predict.py:92-107):
// policy 0 -> top_k, policy 1 -> max(top_k, #{w > nearest-rank-q threshold}).
__device__ inline int warp_softmax_rank(const double *z, double *w, int32_t *order, int E, int top_k, int policy,
                                        double q) {
  const int lane = threadIdx.x & 31;
  double mx = -INFINITY;
  for (int e = lane; e < E; e += 32) mx = fmax(mx, z[e]);
#pragma unroll
  for (int o = 16; o; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  double sum = 0.0;
  for (int e = lane; e < E; e += 32) {
    const double v = exp(__dsub_rn(z[e], mx));
    w[e] = v;
    sum += v;
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
  __syncwarp();
  for (int e = lane; e < E; e += 32) w[e] = __ddiv_rn(w[e], sum);
  __syncwarp();
  for (int e = lane; e < E; e += 32) {
    const double we = w[e];
    int r = 0;
#pragma unroll 8
    for (int j = 0; j < E; ++j) {
      const double wj = w[j];
      r += (wj > we) || (wj == we && j < e);
    }
    order[r] = e;
  }
  __syncwarp();
  if (policy == 0) return top_k < E ? top_k : E;
  // nearest-rank percentile: ascending rank ceil(q*E) -> descending index E - rank
  int rank = (int)ceil(q * (double)E);
  rank = rank < 1 ? 1 : (rank > E ? E : rank);
  const double thr = w[order[E - rank]];
  int cnt = 0;
  for (int e = lane; e < E; e += 32) cnt += (w[e] > thr);
#pragma unroll
  for (int o = 16; o; o >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
  return cnt > top_k ? cnt : (top_k < E ? top_k : E);
}

// The pieces of warp_softmax_rank, for callers that spread the work: the
// softmax (same per-lane order and butterfly as above, so w is bit-identical),
// the rank by (-w, id) over any set of threads (pure comparisons: exact in any
// order), and the policy's prediction-prefix length from w and order.
__device__ inline void warp_softmax(const double *z, double *w, int E) {
  const int lane = threadIdx.x & 31;
  double mx = -INFINITY;
  for (int e = lane; e < E; e += 32) mx = fmax(mx, z[e]);
#pragma unroll
  for (int o = 16; o; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  double sum = 0.0;
  for (int e = lane; e < E; e += 32) {
    const double v = exp(__dsub_rn(z[e], mx));
    w[e] = v;
    sum += v;
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
  __syncwarp();
  for (int e = lane; e < E; e += 32) w[e] = __ddiv_rn(w[e], sum);
  __syncwarp();
}

__device__ inline void rank_by_weight(const double *w, int32_t *order, int E, int t0, int nthreads) {
  for (int e = t0; e < E; e += nthreads) {
    const double we = w[e];
    int r = 0;
#pragma unroll 8
    for (int j = 0; j < E; ++j) {
      const double wj = w[j];
      r += (wj > we) || (wj == we && j < e);
    }
    order[r] = e;
  }
}

__device__ inline int warp_pred_len(const double *w, const int32_t *order, int E, int top_k, int policy, double q) {
  const int lane = threadIdx.x & 31;
  if (policy == 0) return top_k < E ? top_k : E;
  int rank = (int)ceil(q * (double)E);
  rank = rank < 1 ? 1 : (rank > E ? E : rank);
  const double thr = w[order[E - rank]];
  int cnt = 0;
  for (int e = lane; e < E; e += 32) cnt += (w[e] > thr);
#pragma unroll
  for (int o = 16; o; o >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
  return cnt > top_k ? cnt : (top_k < E ? top_k : E);
}

}  // namespace fate
