// K4: grouped expert FFN for prefill (replaces the per-expert chunk model of
// pipeline.py:733-750).  Per active expert e with token list t_e:
//   A_e = silu(X[t_e] W1_e^T) * (X[t_e] W3_e^T)      (up phase, [n_e, I])
//   Z[zrow] = A_e W2_e^T                              (down phase, [n_e, H])
// then a combine kernel sums each token's k routed rows (weighted by the
// full-softmax routing weight) plus the shared-expert row, in ascending
// expert order, so Y is deterministic (no atomics).
//
// The expert GEMMs run on the tensor cores (prefill_tc.cu, tcgen05 + TMEM,
// bf16 operands, fp32 accumulation); this file holds the combine and the
// standalone entry point.
#include <algorithm>
#include <vector>

#include "fate_internal.cuh"

namespace fate {

// Y[t] = sum_j w[t][j] * Z[t*(k+1)+j] (+ Z[t*(k+1)+k] when has_shared), j in ascending expert order.
__global__ void k4_combine_kernel(const float *__restrict__ Z, const float *__restrict__ w, int T, int k, int H,
                                  int has_shared, float *__restrict__ Y) {
  const int64_t total = (int64_t)T * H;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int t = (int)(i / H), h = (int)(i % H);
    const float *zt = Z + (int64_t)t * (k + 1) * H + h;
    float acc = 0.f;
    for (int j = 0; j < k; ++j) acc = fmaf(w[t * k + j], zt[(int64_t)j * H], acc);
    if (has_shared) acc += zt[(int64_t)k * H];
    Y[i] = acc;
  }
}

cudaError_t launch_k4_combine(const float *Z, const float *w, int T, int k, int H, int has_shared, float *Y,
                              cudaStream_t s) {
  const int64_t total = (int64_t)T * H;
  int blocks = (int)std::min<int64_t>((total + 255) / 256, 148 * 16);
  k4_combine_kernel<<<blocks, 256, 0, s>>>(Z, w, T, k, H, has_shared, Y);
  return cudaGetLastError();
}

__global__ void to_bf16_rows_kernel(const float *__restrict__ x, int64_t n, __nv_bfloat16 *__restrict__ y) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    y[i] = __float2bfloat16_rn(x[i]);
}

cudaError_t k4_preload() {
  cudaFuncAttributes a;
  return cudaFuncGetAttributes(&a, k4_combine_kernel);
}

}  // namespace fate

// Standalone K4 (fate_ffn_prefill): Y[t] += w * FFN_e(X[t]) over token lists.
extern "C" int fate_ffn_prefill(const float *X_dev, int T, int H, int n, const uint8_t *const *bufs,
                                const int32_t *tok_idx_dev, const float *tok_w_dev, const int32_t *off_host,
                                float *Y_dev, void *stream) {
  using namespace fate;
  if (T < 0 || n < 0 || H < 128 || H % 128) {
    set_error("fate_ffn_prefill: bad arguments");
    return FATE_EINVAL;
  }
  if (n == 0 || T == 0) return FATE_OK;
  cudaStream_t s = (cudaStream_t)stream;
  std::vector<PrefillExpert> ex(n);
  std::vector<int> a_off(n);
  int64_t a_total = 0;
  int tiles_up = 0, tiles_down = 0;
  const int m = off_host[n];
  for (int j = 0; j < n; ++j) {
    ExpertHeader h;
    FATE_CUDA(cudaMemcpy(&h, bufs[j], sizeof(h), cudaMemcpyDeviceToHost));
    if (h.magic != kMagic || h.H != H) {
      set_error("fate_ffn_prefill: buffer header does not describe a packed expert of this hidden size");
      return FATE_EINVAL;
    }
    ex[j] = PrefillExpert{bufs[j], h.I, h.bits, off_host[j], off_host[j + 1] - off_host[j]};
    a_off[j] = (int)a_total;
    a_total += (int64_t)ex[j].n_tok * h.I;
    if (h.I % 128) {
      set_error("fate_ffn_prefill: expert intermediate size must be a multiple of 128");
      return FATE_EINVAL;
    }
    tiles_up += k4_tc_items(ex[j].n_tok, h.I, H, false);
    tiles_down += k4_tc_items(ex[j].n_tok, h.I, H, true);
  }
  PrefillExpert *ex_dev = nullptr;
  int *aoff_dev = nullptr;
  int32_t *zrow = nullptr;
  float *A = nullptr, *Z = nullptr;
  FATE_CUDA(cudaMallocAsync(&ex_dev, sizeof(PrefillExpert) * n, s));
  FATE_CUDA(cudaMallocAsync(&aoff_dev, sizeof(int) * n, s));
  FATE_CUDA(cudaMallocAsync(&zrow, sizeof(int32_t) * std::max(m, 1), s));
  FATE_CUDA(cudaMallocAsync(&A, sizeof(float) * std::max<int64_t>(a_total, 1), s));
  FATE_CUDA(cudaMallocAsync(&Z, sizeof(float) * (int64_t)std::max(m, 1) * H, s));
  FATE_CUDA(cudaMemcpyAsync(ex_dev, ex.data(), sizeof(PrefillExpert) * n, cudaMemcpyHostToDevice, s));
  FATE_CUDA(cudaMemcpyAsync(aoff_dev, a_off.data(), sizeof(int) * n, cudaMemcpyHostToDevice, s));
  std::vector<int32_t> zr(m);
  for (int i = 0; i < m; ++i) zr[i] = i;  // one Z row per (expert, token) entry
  FATE_CUDA(cudaMemcpyAsync(zrow, zr.data(), sizeof(int32_t) * m, cudaMemcpyHostToDevice, s));
  __nv_bfloat16 *Xb = nullptr;
  FATE_CUDA(cudaMallocAsync(&Xb, sizeof(__nv_bfloat16) * (int64_t)T * H, s));
  to_bf16_rows_kernel<<<148 * 4, 256, 0, s>>>(X_dev, (int64_t)T * H, Xb);
  FATE_CUDA(cudaGetLastError());
  FATE_CUDA(launch_k4_tc(Xb, H, ex_dev, n, tok_idx_dev, zrow, aoff_dev, A, Z, tiles_up, tiles_down, s));
  cudaFreeAsync(Xb, s);
  // accumulate into Y in entry order (host-side order = caller's order)
  std::vector<int32_t> idx(m);
  std::vector<float> w(m);
  FATE_CUDA(cudaMemcpyAsync(idx.data(), tok_idx_dev, sizeof(int32_t) * m, cudaMemcpyDeviceToHost, s));
  FATE_CUDA(cudaMemcpyAsync(w.data(), tok_w_dev, sizeof(float) * m, cudaMemcpyDeviceToHost, s));
  FATE_CUDA(cudaStreamSynchronize(s));
  extern cudaError_t fate_axpy_rows(float *Y, const float *Z, const int32_t *dst, const float *w, int m, int H,
                                    cudaStream_t s);
  int32_t *dst = nullptr;
  float *wd = nullptr;
  FATE_CUDA(cudaMallocAsync(&dst, sizeof(int32_t) * m, s));
  FATE_CUDA(cudaMallocAsync(&wd, sizeof(float) * m, s));
  FATE_CUDA(cudaMemcpyAsync(dst, idx.data(), sizeof(int32_t) * m, cudaMemcpyHostToDevice, s));
  FATE_CUDA(cudaMemcpyAsync(wd, w.data(), sizeof(float) * m, cudaMemcpyHostToDevice, s));
  FATE_CUDA(fate_axpy_rows(Y_dev, Z, dst, wd, m, H, s));
  for (void *p : {(void *)ex_dev, (void *)aoff_dev, (void *)zrow, (void *)A, (void *)Z, (void *)dst, (void *)wd})
    cudaFreeAsync(p, s);
  FATE_CUDA(cudaStreamSynchronize(s));
  return FATE_OK;
}

// Y[dst[i]] += w[i] * Z[i], applied sequentially over i for determinism.
__global__ void axpy_rows_kernel(float *Y, const float *Z, const int32_t *dst, const float *w, int m, int H) {
  for (int h = blockIdx.x * blockDim.x + threadIdx.x; h < H; h += gridDim.x * blockDim.x)
    for (int i = 0; i < m; ++i) Y[(int64_t)dst[i] * H + h] = fmaf(w[i], Z[(int64_t)i * H + h], Y[(int64_t)dst[i] * H + h]);
}

cudaError_t fate_axpy_rows(float *Y, const float *Z, const int32_t *dst, const float *w, int m, int H, cudaStream_t s) {
  axpy_rows_kernel<<<(H + 255) / 256, 256, 0, s>>>(Y, Z, dst, w, m, H);
  return cudaGetLastError();
}
