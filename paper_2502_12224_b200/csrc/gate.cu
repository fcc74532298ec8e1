// K1 (standalone form): batched fp64 router + softmax + rank order + policy
// prefix, for the API mirrors gate_forward / cross_layer_predict
// (gatesim.py:113-123, predict.py:84-107).  The engine uses the fused
// decode/prefill variants in engine.cu built from the same device blocks.
#include "gate_dev.cuh"

namespace fate {
namespace {

constexpr int kGateThreads = 256;

// One block per hidden vector: warps split the E router rows, then warp 0
// ranks.  Shared: z[E], w[E] (fp64), order[E].
__global__ void __launch_bounds__(kGateThreads) gate_batch_kernel(
    const double *__restrict__ W, double tau, const double *__restrict__ h, int64_t h_stride, int E, int H,
    double *__restrict__ routing, int32_t *__restrict__ order, int32_t *__restrict__ list_len, int top_k,
    int policy, double q) {
  extern __shared__ double sm[];
  double *z = sm;
  double *w = sm + E;
  int32_t *ord = reinterpret_cast<int32_t *>(sm + 2 * E);
  const int t = blockIdx.x;
  const double *ht = h + (int64_t)t * h_stride;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  for (int e = warp; e < E; e += nw) {
    const double d = warp_dot64(W + (int64_t)e * H, ht, H);
    if (lane == 0) z[e] = __ddiv_rn(d, tau);
  }
  __syncthreads();
  if (warp == 0) {
    const int len = warp_softmax_rank(z, w, ord, E, top_k, policy, q);
    for (int e = lane; e < E; e += 32) {
      if (routing) routing[(int64_t)t * E + e] = w[e];
      if (order) order[(int64_t)t * E + e] = ord[e];
    }
    if (lane == 0 && list_len) list_len[t] = len;
  }
}

}  // namespace

cudaError_t launch_gate_batch(const double *W, double tau, const double *h, int64_t h_stride, int T, int E, int H, double *routing,
                              int32_t *order, int32_t *list_len, int top_k, int policy, double q, cudaStream_t s) {
  const size_t smem = (size_t)E * (2 * sizeof(double) + sizeof(int32_t));
  gate_batch_kernel<<<T, kGateThreads, smem, s>>>(W, tau, h, h_stride, E, H, routing, order, list_len, top_k, policy, q);
  return cudaGetLastError();
}

cudaError_t gate_preload() {
  cudaFuncAttributes a;
  return cudaFuncGetAttributes(&a, gate_batch_kernel);
}

}  // namespace fate

extern "C" int fate_gate_forward(const double *W_dev, double tau, const double *h_dev, int T, int E, int H,
                                 double *routing_dev, int32_t *order_dev, int32_t *list_len_dev, int top_k,
                                 int policy, double q, void *stream) {
  if (T < 0 || E < 1 || E > FATE_MAX_EXPERTS || H < 1 || top_k < 1 || top_k > E || !(tau > 0.0) ||
      (policy != 0 && policy != 1) || !(q > 0.0 && q < 1.0)) {
    fate::set_error("fate_gate_forward: bad arguments");
    return FATE_EINVAL;
  }
  if (T == 0) return FATE_OK;
  FATE_CUDA(fate::launch_gate_batch(W_dev, tau, h_dev, H, T, E, H, routing_dev, order_dev, list_len_dev, top_k,
                                    policy, q, (cudaStream_t)stream));
  return FATE_OK;
}
