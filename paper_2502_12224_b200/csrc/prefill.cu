// K4: grouped expert FFN for prefill (replaces the per-expert chunk model of
// pipeline.py:733-750).  Per active expert e with token list t_e:
//   A_e = silu(X[t_e] W1_e^T) * (X[t_e] W3_e^T)      (up phase, [n_e, I])
//   Z[zrow] = A_e W2_e^T                              (down phase, [n_e, H])
// then a combine kernel sums each token's k routed rows (weighted by the
// full-softmax routing weight) plus the shared-expert row, in ascending
// expert order, so Y is deterministic (no atomics).
//
// This file holds the portable SIMT tiles (fp32 FMA on dequantized smem
// tiles); the tcgen05 path is in prefill_tc.cu.  Both share the descriptor
// format and the combine kernel.
#include <algorithm>
#include <vector>

#include "fate_internal.cuh"

namespace fate {
namespace {

constexpr int TM = 64;   // tokens per tile
constexpr int TN = 64;   // weight rows per tile
constexpr int TK = 32;   // half a quantization group per k step (static smem < 48 KB)
constexpr int kThreads = 256;

// Dequantize a TN x TK tile (rows r0.., group g) of a packed projection into
// smem fp32 (row-major [TN][TK+1] to avoid bank conflicts on the column reads).
__device__ __forceinline__ void load_w_tile(const uint8_t *codes, const float2 *sz, int bits, int64_t row_elems,
                                            int r0, int nrows, int k0, float (*Ws)[TK + 1]) {
  const int gpr = (int)(row_elems / kGroup);
  for (int i = threadIdx.x; i < TN * TK; i += blockDim.x) {
    const int r = i / TK, c = i % TK;
    float v = 0.f;
    if (r < nrows) {
      const int64_t idx = (int64_t)(r0 + r) * row_elems + k0 + c;
      if (bits == 16) {
        v = __uint_as_float((uint32_t)reinterpret_cast<const uint16_t *>(codes)[idx] << 16);
      } else {
        const int per = 8 / bits;
        const uint32_t q = (codes[idx / per] >> ((idx % per) * bits)) & ((1u << bits) - 1u);
        const float2 p = sz[(int64_t)(r0 + r) * gpr + k0 / kGroup];
        v = __fadd_rn(p.y, __fmul_rn((float)q, p.x));
      }
    }
    Ws[r][c] = v;
  }
}

struct TileRef {
  int e, tt, rr;
};

// Map a linear tile id onto (expert, token tile, row tile).
__device__ __forceinline__ bool find_tile(const PrefillExpert *ex, int n, int rows_per_expert_fn_down, int tile,
                                          int H, TileRef &out) {
  for (int e = 0; e < n; ++e) {
    const int nt = (ex[e].n_tok + TM - 1) / TM;
    const int nr = rows_per_expert_fn_down ? (H + TN - 1) / TN : (ex[e].I + TN - 1) / TN;
    const int cnt = nt * nr;
    if (tile < cnt) {
      out.e = e;
      out.tt = tile / nr;
      out.rr = tile % nr;
      return true;
    }
    tile -= cnt;
  }
  return false;
}

__device__ __forceinline__ int header_bits(const uint8_t *buf) { return reinterpret_cast<const ExpertHeader *>(buf)->bits; }

__global__ void __launch_bounds__(kThreads) k4_up_kernel(const float *__restrict__ X, int H,
                                                          const PrefillExpert *__restrict__ ex, int n,
                                                          const int32_t *__restrict__ tok_idx, const int *a_off,
                                                          float *__restrict__ A, int n_tiles) {
  __shared__ float Xs[TM][TK + 1];
  __shared__ float W1s[TN][TK + 1];
  __shared__ float W3s[TN][TK + 1];
  const int tx = threadIdx.x % 16, ty = threadIdx.x / 16;  // 16 x 16 threads, 4 x 4 outputs each
  for (int tile = blockIdx.x; tile < n_tiles; tile += gridDim.x) {
    TileRef tr;
    if (!find_tile(ex, n, 0, tile, H, tr)) return;
    const PrefillExpert E = ex[tr.e];
    const int bits = header_bits(E.buf);
    const Layout Lo = make_layout(H, E.I, bits);
    const uint8_t *p = E.buf + FATE_HEADER_BYTES;
    const int t0 = tr.tt * TM, r0 = tr.rr * TN;
    const int ntok = min(TM, E.n_tok - t0), nrows = min(TN, E.I - r0);
    float u[4][4] = {}, v[4][4] = {};
    for (int k0 = 0; k0 < H; k0 += TK) {
      for (int i = threadIdx.x; i < TM * TK; i += blockDim.x) {
        const int t = i / TK, c = i % TK;
        Xs[t][c] = t < ntok ? X[(int64_t)tok_idx[E.tok_off + t0 + t] * H + k0 + c] : 0.f;
      }
      load_w_tile(p + Lo.c1, reinterpret_cast<const float2 *>(p + Lo.s1), bits, H, r0, nrows, k0, W1s);
      load_w_tile(p + Lo.c3, reinterpret_cast<const float2 *>(p + Lo.s3), bits, H, r0, nrows, k0, W3s);
      __syncthreads();
#pragma unroll 8
      for (int kk = 0; kk < TK; ++kk) {
        float xa[4], w1[4], w3[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) xa[i] = Xs[ty * 4 + i][kk];
#pragma unroll
        for (int j = 0; j < 4; ++j) w1[j] = W1s[tx * 4 + j][kk], w3[j] = W3s[tx * 4 + j][kk];
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            u[i][j] = fmaf(xa[i], w1[j], u[i][j]);
            v[i][j] = fmaf(xa[i], w3[j], v[i][j]);
          }
      }
      __syncthreads();
    }
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int t = ty * 4 + i, r = tx * 4 + j;
        if (t < ntok && r < nrows) {
          const float a = u[i][j] / (1.0f + expf(-u[i][j])) * v[i][j];
          A[(int64_t)a_off[tr.e] + (int64_t)(t0 + t) * E.I + r0 + r] = a;
        }
      }
  }
}

__global__ void __launch_bounds__(kThreads) k4_down_kernel(int H, const PrefillExpert *__restrict__ ex, int n,
                                                            const int32_t *__restrict__ zrow, const int *a_off,
                                                            const float *__restrict__ A, float *__restrict__ Z,
                                                            int n_tiles) {
  __shared__ float As[TM][TK + 1];
  __shared__ float W2s[TN][TK + 1];
  const int tx = threadIdx.x % 16, ty = threadIdx.x / 16;
  for (int tile = blockIdx.x; tile < n_tiles; tile += gridDim.x) {
    TileRef tr;
    if (!find_tile(ex, n, 1, tile, H, tr)) return;
    const PrefillExpert E = ex[tr.e];
    const int bits = header_bits(E.buf);
    const Layout Lo = make_layout(H, E.I, bits);
    const uint8_t *p = E.buf + FATE_HEADER_BYTES;
    const int t0 = tr.tt * TM, r0 = tr.rr * TN;
    const int ntok = min(TM, E.n_tok - t0), nrows = min(TN, H - r0);
    const float *Ae = A + a_off[tr.e];
    float acc[4][4] = {};
    for (int k0 = 0; k0 < E.I; k0 += TK) {
      for (int i = threadIdx.x; i < TM * TK; i += blockDim.x) {
        const int t = i / TK, c = i % TK;
        As[t][c] = t < ntok ? Ae[(int64_t)(t0 + t) * E.I + k0 + c] : 0.f;
      }
      load_w_tile(p + Lo.c2, reinterpret_cast<const float2 *>(p + Lo.s2), bits, E.I, r0, nrows, k0, W2s);
      __syncthreads();
#pragma unroll 8
      for (int kk = 0; kk < TK; ++kk) {
        float aa[4], w2[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) aa[i] = As[ty * 4 + i][kk];
#pragma unroll
        for (int j = 0; j < 4; ++j) w2[j] = W2s[tx * 4 + j][kk];
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(aa[i], w2[j], acc[i][j]);
      }
      __syncthreads();
    }
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int t = ty * 4 + i, r = tx * 4 + j;
        if (t < ntok && r < nrows) Z[(int64_t)zrow[E.tok_off + t0 + t] * H + r0 + r] = acc[i][j];
      }
  }
}

}  // namespace

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

// Host-side launcher: the expert table is in DEVICE memory; n_tiles bounds
// are computed on the host from host copies of the counts.
cudaError_t launch_k4_simt(const float *X, int H, const PrefillExpert *ex_dev, int n, const int32_t *tok_idx,
                           const int32_t *zrow, const int *a_off_dev, float *A, float *Z, int tiles_up,
                           int tiles_down, cudaStream_t s) {
  if (tiles_up > 0) k4_up_kernel<<<min(tiles_up, 148 * 8), kThreads, 0, s>>>(X, H, ex_dev, n, tok_idx, a_off_dev, A,
                                                                           tiles_up);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  if (tiles_down > 0)
    k4_down_kernel<<<min(tiles_down, 148 * 8), kThreads, 0, s>>>(H, ex_dev, n, zrow, a_off_dev, A, Z, tiles_down);
  return cudaGetLastError();
}

cudaError_t launch_k4_combine(const float *Z, const float *w, int T, int k, int H, int has_shared, float *Y,
                              cudaStream_t s) {
  const int64_t total = (int64_t)T * H;
  int blocks = (int)std::min<int64_t>((total + 255) / 256, 148 * 16);
  k4_combine_kernel<<<blocks, 256, 0, s>>>(Z, w, T, k, H, has_shared, Y);
  return cudaGetLastError();
}

cudaError_t k4_preload() {
  cudaFuncAttributes a;
  cudaError_t e = cudaFuncGetAttributes(&a, k4_up_kernel);
  if (e == cudaSuccess) e = cudaFuncGetAttributes(&a, k4_down_kernel);
  if (e == cudaSuccess) e = cudaFuncGetAttributes(&a, k4_combine_kernel);
  return e;
}

int k4_tiles(int n_tok, int I, int H, bool down) {
  const int nt = (n_tok + TM - 1) / TM;
  return nt * (down ? (H + TN - 1) / TN : (I + TN - 1) / TN);
}

}  // namespace fate

// Standalone K4 (fate_ffn_prefill): Y[t] += w * FFN_e(X[t]) over token lists.
extern "C" int fate_ffn_prefill(const float *X_dev, int T, int H, int n, const uint8_t *const *bufs,
                                const int32_t *tok_idx_dev, const float *tok_w_dev, const int32_t *off_host,
                                float *Y_dev, void *stream) {
  using namespace fate;
  if (T < 0 || n < 0 || H < 64 || H % 64) {
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
    tiles_up += k4_tiles(ex[j].n_tok, h.I, H, false);
    tiles_down += k4_tiles(ex[j].n_tok, h.I, H, true);
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
  FATE_CUDA(launch_k4_simt(X_dev, H, ex_dev, n, tok_idx_dev, zrow, aoff_dev, A, Z, tiles_up, tiles_down, s));
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
