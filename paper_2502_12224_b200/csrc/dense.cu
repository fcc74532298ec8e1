// The dense part of a decode step: the attention block and
// the shared-expert gate that the reference charges as the constants t_attn /
// t_gate (core.py:79-83, pipeline.py:418, 484), executed for one token (bs = 1)
// on sm_100a.  Per layer l of token t:
//   h   = residual stream (fp32 [H]; layer 0: the token's embedding stand-in)
//   xn  = RMSNorm(h) * g_l
//   qkv = Wqkv_l xn + b_l                       (D1: bf16 GEMV, HBM bound)
//   q, k <- RoPE(pos); K/V cache[l][pos] <- k, v (bf16)
//   o   = softmax(q K^T / sqrt(d)) V            (D2: split-context decode attention, GQA)
//   a   = h + Wo_l o                            (D3: bf16 GEMV + residual)
// and, when the layer has a gated shared expert, s_l = sigmoid(w_l . x) with x
// the MoE input (Qwen1.5-MoE's shared_expert_gate), which K1 uses as the shared
// expert's routing weight.  The MoE output y of the step is added by the next
// step's D1 (h = a + y).  Routing stays trace-driven, so the attention output
// feeds the residual stream and the timing, not the router.
#include <cuda_bf16.h>

#include "fate_internal.cuh"

namespace fate {
namespace {

constexpr int kGemvWarps = 8;

__device__ __forceinline__ float warp_sum_d(float v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// y[n] = W[n, :] . v (+ bias[n]) (+ res[n]), W bf16 row-major [N, K], v fp32 in
// shared memory.  MODE 0: v = RMSNorm(h_prev + y_prev) * g (and h is written),
// MODE 1: v = the given vector.  One warp per row, 16-byte loads, fixed-order
// reductions (deterministic).
template <int MODE>
__global__ void __launch_bounds__(32 * kGemvWarps) gemv_kernel(const __nv_bfloat16 *__restrict__ W,
                                                               const float *__restrict__ bias, int N, int K,
                                                               const float *__restrict__ vin, const float *__restrict__ vadd,
                                                               const float *__restrict__ g, float eps,
                                                               float *__restrict__ hout, const float *__restrict__ res,
                                                               float *__restrict__ y) {
  extern __shared__ float vs[];
  __shared__ float red[kGemvWarps];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (MODE == 0) {
    // K <= 4096 = 16 * blockDim.x: every load of the prologue in flight at once
    float hv[16], av[16], gv[16];
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      const int i = tid + u * 32 * kGemvWarps;
      hv[u] = i < K ? vin[i] : 0.f;
      av[u] = i < K && vadd ? vadd[i] : 0.f;
      gv[u] = i < K ? g[i] : 0.f;
    }
    float ss = 0.f;
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      const int i = tid + u * 32 * kGemvWarps;
      const float h = hv[u] + av[u];
      if (i < K) vs[i] = h;
      ss += h * h;
    }
    ss = warp_sum_d(ss);
    if (lane == 0) red[warp] = ss;
    __syncthreads();
    float tot = 0.f;
    for (int w = 0; w < kGemvWarps; ++w) tot += red[w];
    const float inv = rsqrtf(tot / K + eps);
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      const int i = tid + u * 32 * kGemvWarps;
      if (i < K) {
        const float h = hv[u] + av[u];
        if (blockIdx.x == 0) hout[i] = h;
        vs[i] = h * inv * gv[u];
      }
    }
  } else {
    for (int i = tid; i < K; i += blockDim.x) vs[i] = vin[i];
  }
  __syncthreads();
  for (int n = blockIdx.x * kGemvWarps + warp; n < N; n += gridDim.x * kGemvWarps) {
    const uint4 *w = reinterpret_cast<const uint4 *>(W + (int64_t)n * K);
    const float add = (bias ? bias[n] : 0.f) + (res ? res[n] : 0.f);  // issued with the row's loads
    float a0 = 0.f, a1 = 0.f;
    // eight 16-byte loads per lane in flight before the first FMA (latency bound otherwise)
    constexpr int kL = 8;
    for (int c0 = lane; c0 < K / 8; c0 += 32 * kL) {
      uint4 qv[kL];
#pragma unroll
      for (int u = 0; u < kL; ++u) {
        const int c = c0 + 32 * u;
        qv[u] = c < K / 8 ? __ldg(w + c) : make_uint4(0u, 0u, 0u, 0u);
      }
#pragma unroll
      for (int u = 0; u < kL; ++u) {
        const int c = c0 + 32 * u;
        if (c < K / 8) {
          const uint4 q = qv[u];
          const float4 x0 = reinterpret_cast<const float4 *>(vs)[2 * c], x1 = reinterpret_cast<const float4 *>(vs)[2 * c + 1];
          a0 = fmaf(__uint_as_float(q.x << 16), x0.x, a0);
          a1 = fmaf(__uint_as_float(q.x & 0xFFFF0000u), x0.y, a1);
          a0 = fmaf(__uint_as_float(q.y << 16), x0.z, a0);
          a1 = fmaf(__uint_as_float(q.y & 0xFFFF0000u), x0.w, a1);
          a0 = fmaf(__uint_as_float(q.z << 16), x1.x, a0);
          a1 = fmaf(__uint_as_float(q.z & 0xFFFF0000u), x1.y, a1);
          a0 = fmaf(__uint_as_float(q.w << 16), x1.z, a0);
          a1 = fmaf(__uint_as_float(q.w & 0xFFFF0000u), x1.w, a1);
        }
      }
    }
    const float s = warp_sum_d(a0 + a1);
    if (lane == 0) y[n] = s + add;
  }
}

// RoPE (rotate-half, theta) on q and k of position pos, K/V appended to the
// bf16 cache [ctx][2][nkv*hd], then split-context decode attention: block (head
// group, split) with one warp per query head of the kv group; each warp walks
// its split's positions, lanes own hd/32 dims.  Partials (m, l, o) per split
// are combined in attn_combine_kernel in split order (deterministic).

__global__ void rope_append_kernel(const float *__restrict__ qkv, int nh, int nkv, int hd, int pos, float theta,
                                   __nv_bfloat16 *__restrict__ kv_pos, float *__restrict__ q_out,
                                   const float *__restrict__ gate_w, const double *__restrict__ gate_in, int H,
                                   float *__restrict__ gate_out) {
  if (gate_w && blockIdx.x == gridDim.x - 1) {
    // the last block: shared-expert gate s = sigmoid(w . x), x = sqrt(H) * gate_in
    __shared__ float red[32];
    const double sH = sqrt((double)H);
    float acc = 0.f;
    for (int i = threadIdx.x; i < H; i += blockDim.x) acc = fmaf(gate_w[i], (float)(sH * gate_in[i]), acc);
    acc = warp_sum_d(acc);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
    __syncthreads();
    if (threadIdx.x == 0) {
      float t = 0.f;
      for (int i = 0; i < (int)(blockDim.x >> 5); ++i) t += red[i];
      *gate_out = 1.0f / (1.0f + expf(-t));
    }
    return;
  }
  // one thread per rotation pair of q and k heads, plus the v copy
  const int half = hd / 2;
  const int nq = nh * half, nk = nkv * half;
  const int nblk = gate_w ? gridDim.x - 1 : gridDim.x;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < nq + nk + nkv * hd; i += nblk * blockDim.x) {
    if (i < nq + nk) {
      const bool isq = i < nq;
      const int j = isq ? i : i - nq, head = j / half, d = j % half;
      const float *src = qkv + (isq ? 0 : nh * hd) + head * hd;
      const float inv = powf(theta, -2.0f * d / hd);
      float sn, cs;
      sincosf(pos * inv, &sn, &cs);
      const float x0 = src[d], x1 = src[d + half];
      const float r0 = x0 * cs - x1 * sn, r1 = x1 * cs + x0 * sn;
      if (isq) {
        q_out[head * hd + d] = r0;
        q_out[head * hd + d + half] = r1;
      } else {
        kv_pos[head * hd + d] = __float2bfloat16_rn(r0);
        kv_pos[head * hd + d + half] = __float2bfloat16_rn(r1);
      }
    } else {
      const int j = i - nq - nk;
      kv_pos[nkv * hd + j] = __float2bfloat16_rn(qkv[(nh + nkv) * hd + j]);
    }
  }
}

// Split-context decode attention: block (query head, split of kAttnPos
// positions), 128 threads.  Phase 1: thread p scores position p (its key row
// in 16-byte loads against q in shared memory).  Phase 2: block max / sum of
// the exponentials.  Phase 3: thread d accumulates output dim d over the
// split's positions (coalesced value rows).  The last split block of a head to
// finish (counter) combines the head's splits in split order, so the result is
// deterministic and no separate combine launch is needed.
constexpr int kAttnPos = 32;
constexpr int kAttnThreads = 128;

__global__ void __launch_bounds__(kAttnThreads) attn_kernel(const float *__restrict__ q,
                                                             const __nv_bfloat16 *__restrict__ kv, int nh, int nkv,
                                                             int hd, int ctx, float scale, float *__restrict__ part_o,
                                                             float2 *__restrict__ part_ml, unsigned *__restrict__ cnt,
                                                             float *__restrict__ o) {
  __shared__ __align__(16) float qs[128];
  __shared__ float ps[kAttnPos];
  __shared__ float red[kAttnThreads / 32];
  __shared__ unsigned last;
  const int head = blockIdx.x, split = blockIdx.y, splits = gridDim.y, tid = threadIdx.x;
  const int kvh = head / (nh / nkv), rowlen = 2 * nkv * hd;
  if (tid < hd) qs[tid] = q[head * hd + tid] * scale;
  __syncthreads();
  const int p0 = split * kAttnPos, np = min(kAttnPos, ctx - p0);
  // phase 1: scores
  if (tid < np) {
    const uint4 *kp = reinterpret_cast<const uint4 *>(kv + (int64_t)(p0 + tid) * rowlen + kvh * hd);
    float s = 0.f;
    uint4 kw[16];  // the key row (hd <= 128) in flight at once
#pragma unroll
    for (int c = 0; c < 16; ++c) kw[c] = c < hd / 8 ? __ldg(kp + c) : make_uint4(0u, 0u, 0u, 0u);
#pragma unroll
    for (int c = 0; c < 16; ++c) {
      if (c >= hd / 8) break;
      const uint4 w = kw[c];
      const float4 a = reinterpret_cast<const float4 *>(qs)[2 * c], b = reinterpret_cast<const float4 *>(qs)[2 * c + 1];
      s = fmaf(__uint_as_float(w.x << 16), a.x, s);
      s = fmaf(__uint_as_float(w.x & 0xFFFF0000u), a.y, s);
      s = fmaf(__uint_as_float(w.y << 16), a.z, s);
      s = fmaf(__uint_as_float(w.y & 0xFFFF0000u), a.w, s);
      s = fmaf(__uint_as_float(w.z << 16), b.x, s);
      s = fmaf(__uint_as_float(w.z & 0xFFFF0000u), b.y, s);
      s = fmaf(__uint_as_float(w.w << 16), b.z, s);
      s = fmaf(__uint_as_float(w.w & 0xFFFF0000u), b.w, s);
    }
    ps[tid] = s;
  }
  __syncthreads();
  // phase 2: max and sum over the split (one warp)
  float m = -INFINITY, l = 0.f;
  if (tid < 32) {
    float v = tid < np ? ps[tid] : -INFINITY;
    m = v;
#pragma unroll
    for (int off = 16; off; off >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, off));
    const float e = tid < np ? expf(v - m) : 0.f;
    if (tid < np) ps[tid] = e;
    l = warp_sum_d(e);
    if (tid == 0) red[0] = m, red[1] = l;
  }
  __syncthreads();
  m = red[0], l = red[1];
  // phase 3: weighted values, thread = output dim
  if (tid < hd) {
    const __nv_bfloat16 *vp = kv + (int64_t)p0 * rowlen + nkv * hd + kvh * hd + tid;
    float acc = 0.f;
    __nv_bfloat16 vv[kAttnPos];  // every value of the split in flight at once
#pragma unroll
    for (int p = 0; p < kAttnPos; ++p) vv[p] = p < np ? vp[(int64_t)p * rowlen] : __float2bfloat16_rn(0.f);
#pragma unroll
    for (int p = 0; p < kAttnPos; ++p)
      if (p < np) acc = fmaf(ps[p], __bfloat162float(vv[p]), acc);
    part_o[((int64_t)split * nh + head) * hd + tid] = acc;
  }
  if (tid == 0) part_ml[split * nh + head] = make_float2(m, l);
  // the last split of this head combines all splits in order
  __threadfence();
  __syncthreads();
  if (tid == 0) last = atomicAdd(&cnt[head], 1u) == (unsigned)splits - 1u;
  __syncthreads();
  if (!last) return;
  __threadfence();
  if (tid < hd) {
    float M = -INFINITY;
    for (int sp = 0; sp < splits; ++sp) M = fmaxf(M, __ldcg(&part_ml[sp * nh + head].x));
    float L = 0.f, acc = 0.f;
    for (int sp = 0; sp < splits; ++sp) {
      const float2 ml = __ldcg(&part_ml[sp * nh + head]);
      const float c = ml.y > 0.f ? expf(ml.x - M) : 0.f;
      L = fmaf(ml.y, c, L);
      acc = fmaf(__ldcg(&part_o[((int64_t)sp * nh + head) * hd + tid]), c, acc);
    }
    o[head * hd + tid] = acc / L;
  }
  if (tid == 0) cnt[head] = 0;  // ready for the next step
}

// the token's embedding stand-in: h = sqrt(H) * gate_in (the layer-0 MoE input)
__global__ void embed_kernel(const double *__restrict__ gate_in, int H, float *__restrict__ h) {
  const double sH = sqrt((double)H);
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < H; i += gridDim.x * blockDim.x) h[i] = (float)(sH * gate_in[i]);
}

// synthetic prompt K/V (deterministic hash -> bf16 in [-0.5, 0.5))
__global__ void fill_kv_kernel(__nv_bfloat16 *__restrict__ kv, int64_t n, uint32_t seed) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    uint32_t x = (uint32_t)i * 2654435761u ^ seed;
    x ^= x >> 16;
    x *= 0x7feb352du;
    x ^= x >> 15;
    kv[i] = __float2bfloat16_rn((x >> 8) * (1.0f / 16777216.0f) - 0.5f);
  }
}

int gemv_grid(int N) {
  // up to four blocks per SM (32 warps): the RMSNorm prologue is paid per block
  int g = (N + kGemvWarps - 1) / kGemvWarps;
  return g > 148 * 4 ? 148 * 4 : g;
}

}  // namespace

cudaError_t launch_embed(const double *gate_in, int H, float *h, cudaStream_t s) {
  embed_kernel<<<(H + 255) / 256, 256, 0, s>>>(gate_in, H, h);
  return cudaGetLastError();
}

cudaError_t launch_fill_kv(__nv_bfloat16 *kv, int64_t n, uint32_t seed, cudaStream_t s) {
  fill_kv_kernel<<<592, 256, 0, s>>>(kv, n, seed);
  return cudaGetLastError();
}

// Launch the dense part of one decode step on stream s (see the header comment).
cudaError_t launch_dense_step(const DenseLayer &Ly, const DenseDims &D, const float *h_prev, const float *y_prev,
                              const double *gate_in, int pos, DenseScratch &S, cudaStream_t s) {
  const int H = D.H, hd = D.head_dim, nh = D.n_heads, nkv = D.n_kv_heads;
  const int nqkv = (nh + 2 * nkv) * hd;
  const size_t vsm = (size_t)H * sizeof(float);
  gemv_kernel<0><<<gemv_grid(nqkv), 32 * kGemvWarps, vsm, s>>>(Ly.wqkv, Ly.bqkv, nqkv, H, h_prev, y_prev, Ly.norm,
                                                                 D.eps, S.h, nullptr, S.qkv);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  __nv_bfloat16 *kv_pos = Ly.kv + (int64_t)pos * 2 * nkv * hd;
  rope_append_kernel<<<Ly.shared_gate ? 33 : 32, 256, 0, s>>>(S.qkv, nh, nkv, hd, pos, D.rope_theta, kv_pos, S.q,
                                                             Ly.shared_gate, gate_in, H, Ly.shared_gate_out);
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  const int ctx = pos + 1;
  const int splits = (ctx + kAttnPos - 1) / kAttnPos;
  if (splits > D.max_splits) return cudaErrorInvalidValue;
  attn_kernel<<<dim3(nh, splits), kAttnThreads, 0, s>>>(S.q, Ly.kv, nh, nkv, hd, ctx, rsqrtf((float)hd), S.part_o,
                                                        S.part_ml, S.cnt, S.o);
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  gemv_kernel<1><<<gemv_grid(H), 32 * kGemvWarps, (size_t)nh * hd * sizeof(float), s>>>(
      Ly.wo, nullptr, H, nh * hd, S.o, nullptr, nullptr, 0.f, nullptr, S.h, S.a);
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  return cudaSuccess;
}

}  // namespace fate

using namespace fate;

// Standalone dense step (numerics tests; the engine calls launch_dense_step):
// every pointer is a device buffer; outputs land in the scratch buffers
// h (= h_prev + y_prev), qkv, q (roped), o (attention), a (= h + Wo o), and the
// shared gate in *gate_out when gate_w is given.  Synchronous.
extern "C" int fate_dense_step(int H, int n_heads, int n_kv_heads, int head_dim, float eps, float rope_theta,
                               const void *wqkv, const float *bqkv, const float *norm, const void *wo, void *kv,
                               const float *gate_w, float *gate_out, const float *h_prev, const float *y_prev,
                               const double *gate_in, int pos, float *h, float *qkv, float *q, float *o, float *a,
                               float *part_o, float *part_ml, void *stream) {
  if (H % 256 || head_dim % 32 || head_dim > 128 || n_heads % n_kv_heads || n_heads / n_kv_heads > 32 || pos < 0 ||
      pos >= 32 * kDenseMaxSplits) {
    set_error("fate_dense_step: unsupported geometry (H % 256, head_dim in {32..128} step 32, GQA group <= 32)");
    return FATE_EINVAL;
  }
  DenseDims D{H, n_heads, n_kv_heads, head_dim, eps, rope_theta, kDenseMaxSplits};
  DenseLayer Ly{reinterpret_cast<const __nv_bfloat16 *>(wqkv), bqkv, norm, reinterpret_cast<const __nv_bfloat16 *>(wo),
                reinterpret_cast<__nv_bfloat16 *>(kv), gate_w, gate_out};
  cudaStream_t s = (cudaStream_t)stream;
  unsigned *cnt = nullptr;
  FATE_CUDA(cudaMallocAsync(&cnt, (size_t)n_heads * 4, s));
  FATE_CUDA(cudaMemsetAsync(cnt, 0, (size_t)n_heads * 4, s));
  DenseScratch S{h, qkv, q, o, part_o, a, reinterpret_cast<float2 *>(part_ml), cnt};
  const cudaError_t e = launch_dense_step(Ly, D, h_prev, y_prev, gate_in, pos, S, s);
  cudaFreeAsync(cnt, s);
  FATE_CUDA(e);
  FATE_CUDA(cudaStreamSynchronize(s));
  return FATE_OK;
}
