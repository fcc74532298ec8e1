// K5: group-wise affine quantization and packing (quant.py:30-120), sm_100a.
//
// One warp per group of 64 elements.  The arithmetic is the reference's
// fp64 sequence exactly: mn/mx over the group, scale = (mx - mn) / levels,
// code = clip(rint((x - mn) / scale), 0, levels), with IEEE division and
// round-half-even (no fast-math, no contraction), so packed bytes are
// bit-identical to quant.quantize on the same fp32 inputs.
#include <cuda_bf16.h>

#include "fate_internal.cuh"

namespace fate {
namespace {

template <typename T>
__global__ void quant_pack_kernel(const T *__restrict__ w, int64_t n, int bits, int group,
                                  uint8_t *__restrict__ codes, float2 *__restrict__ sz,
                                  double *__restrict__ s64, double *__restrict__ z64) {
  extern __shared__ uint8_t smem_codes[];  // [warps][group]
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  const int warps = blockDim.x >> 5;
  uint8_t *my = smem_codes + warp * group;
  const int64_t n_groups = (n + group - 1) / group;
  const int levels = (1 << bits) - 1;
  const int per_byte = 8 / bits;
  for (int64_t g = (int64_t)blockIdx.x * warps + warp; g < n_groups; g += (int64_t)gridDim.x * warps) {
    const int64_t lo = g * group;
    const int m = (int)(n - lo < (int64_t)group ? n - lo : (int64_t)group);
    double mn = INFINITY, mx = -INFINITY;
    for (int i = lane; i < m; i += 32) {
      const double v = (double)w[lo + i];
      mn = fmin(mn, v);
      mx = fmax(mx, v);
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      mn = fmin(mn, __shfl_xor_sync(0xffffffffu, mn, o));
      mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    }
    const double scale = (mx == mn) ? 0.0 : __ddiv_rn(__dsub_rn(mx, mn), (double)levels);
    for (int i = lane; i < group; i += 32) {
      int c = 0;
      if (i < m && scale != 0.0) {
        const double q = rint(__ddiv_rn(__dsub_rn((double)w[lo + i], mn), scale));
        c = (int)fmin(fmax(q, 0.0), (double)levels);
      }
      my[i] = (uint8_t)c;
    }
    __syncwarp();
    // Byte j packs elements j*per_byte .. +per_byte-1, element i at bit i*bits (quant.py:30-39).
    const int nbytes = (m * bits + 7) / 8;
    const int64_t byte0 = lo * bits / 8;  // groups of 64 start on byte boundaries for bits in {2,4,8}
    for (int j = lane; j < nbytes; j += 32) {
      uint32_t b = 0;
      for (int t = 0; t < per_byte; ++t) b |= (uint32_t)my[j * per_byte + t] << (t * bits);
      codes[byte0 + j] = (uint8_t)b;
    }
    if (lane == 0) {
      if (sz) sz[g] = make_float2((float)scale, (float)mn);
      if (s64) s64[g] = scale;
      if (z64) z64[g] = mn;
    }
    __syncwarp();
  }
}

__global__ void to_bf16_kernel(const float *__restrict__ w, int64_t n, __nv_bfloat16 *__restrict__ out) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = __float2bfloat16_rn(w[i]);
}

__global__ void dequant_kernel(const uint8_t *__restrict__ codes, const float2 *__restrict__ sz, int64_t n,
                               int bits, int group, float *__restrict__ out) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    if (bits == 16) {
      out[i] = __bfloat162float(reinterpret_cast<const __nv_bfloat16 *>(codes)[i]);
      continue;
    }
    const int per_byte = 8 / bits;
    const uint32_t c = (codes[i / per_byte] >> ((i % per_byte) * bits)) & ((1u << bits) - 1);
    const float2 p = sz[i / group];
    out[i] = __fadd_rn(p.y, __fmul_rn((float)c, p.x));
  }
}

// fp64 dequantization with the reference's rounding: zero + (code * scale),
// two roundings, no contraction (quant.py:119).
__global__ void dequant64_kernel(const uint8_t *__restrict__ codes, const double *__restrict__ s64,
                                 const double *__restrict__ z64, int64_t n, int bits, int group,
                                 double *__restrict__ out) {
  const int per_byte = 8 / bits;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t c = (codes[i / per_byte] >> ((i % per_byte) * bits)) & ((1u << bits) - 1);
    out[i] = __dadd_rn(z64[i / group], __dmul_rn((double)c, s64[i / group]));
  }
}

__global__ void write_header_kernel(uint8_t *dst, int bits, int layer, int expert, int H, int I) {
  ExpertHeader *h = reinterpret_cast<ExpertHeader *>(dst);
  const int t = threadIdx.x;
  if (t < (int)(sizeof(ExpertHeader) / 4)) reinterpret_cast<int32_t *>(h)[t] = 0;
  __syncthreads();
  if (t == 0) {
    h->magic = kMagic;
    h->bits = bits;
    h->layer = layer;
    h->expert = expert;
    h->H = H;
    h->I = I;
  }
}

// W2 [H, I] row-major -> slab-major (fate_internal.cuh): element (h, c) to
// ((c / C) * H + h) * C + c % C.  With C = 64 every 64-element group of the
// permuted array is one row segment of one original group.
__global__ void w2_slab_kernel(const float *__restrict__ w2, int H, int I, int C, float *__restrict__ out) {
  const int64_t n = (int64_t)H * I;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t h = i / I, c = i % I;
    out[((c / C) * H + h) * C + c % C] = w2[i];
  }
}

int grid_for(int64_t work, int per_block) {
  int64_t g = (work + per_block - 1) / per_block;
  if (g > 148 * 32) g = 148 * 32;
  return (int)(g < 1 ? 1 : g);
}

template <typename T>
cudaError_t quant_pack_launch(const T *w, int64_t n, int bits, int group, uint8_t *codes, float *sz,
                              double *s64, double *z64, cudaStream_t s) {
  if constexpr (sizeof(T) == 4) if (bits == 16) {
    to_bf16_kernel<<<grid_for(n, 256), 256, 0, s>>>(w, n, reinterpret_cast<__nv_bfloat16 *>(codes));
    return cudaGetLastError();
  }
  const int warps = 8;
  const int64_t n_groups = (n + group - 1) / group;
  quant_pack_kernel<T><<<grid_for(n_groups, warps), warps * 32, warps * group, s>>>(
      w, n, bits, group, codes, reinterpret_cast<float2 *>(sz), s64, z64);
  return cudaGetLastError();
}

}  // namespace
}  // namespace fate

using namespace fate;

extern "C" int fate_quant_pack(const float *w_dev, int64_t n, int bits, int group, uint8_t *codes_dev,
                               float *sz_dev, double *scale64_dev, double *zero64_dev, void *stream) {
  if (n < 0 || group < 1 || group > 1024 || !(bits == 2 || bits == 4 || bits == 8 || bits == 16)) {
    set_error("fate_quant_pack: bad arguments");
    return FATE_EINVAL;
  }
  if (bits != 16 && group % 8 != 0) {
    set_error("fate_quant_pack: group must be a multiple of 8 so groups start on byte boundaries");
    return FATE_EINVAL;
  }
  if (n == 0) return FATE_OK;
  FATE_CUDA(quant_pack_launch(w_dev, n, bits, group, codes_dev, sz_dev, scale64_dev, zero64_dev,
                              (cudaStream_t)stream));
  return FATE_OK;
}

extern "C" int fate_quant_pack64(const double *w_dev, int64_t n, int bits, int group, uint8_t *codes_dev,
                                 float *sz_dev, double *scale64_dev, double *zero64_dev, void *stream) {
  if (n < 0 || group < 1 || group > 1024 || !(bits == 2 || bits == 4 || bits == 8) || group % 8 != 0) {
    set_error("fate_quant_pack64: bad arguments");
    return FATE_EINVAL;
  }
  if (n == 0) return FATE_OK;
  FATE_CUDA(quant_pack_launch(w_dev, n, bits, group, codes_dev, sz_dev, scale64_dev, zero64_dev,
                              (cudaStream_t)stream));
  return FATE_OK;
}

extern "C" int fate_dequant(const uint8_t *codes_dev, const float *sz_dev, int64_t n, int bits, int group,
                            float *out_dev, void *stream) {
  if (n < 0 || group < 1 || !(bits == 2 || bits == 4 || bits == 8 || bits == 16)) {
    set_error("fate_dequant: bad arguments");
    return FATE_EINVAL;
  }
  if (n == 0) return FATE_OK;
  dequant_kernel<<<grid_for(n, 256), 256, 0, (cudaStream_t)stream>>>(
      codes_dev, reinterpret_cast<const float2 *>(sz_dev), n, bits, group, out_dev);
  FATE_CHECK_LAUNCH("dequant_kernel");
  return FATE_OK;
}

extern "C" int fate_dequant64(const uint8_t *codes_dev, const double *scale64_dev, const double *zero64_dev,
                              int64_t n, int bits, int group, double *out_dev, void *stream) {
  if (n < 0 || group < 1 || !(bits == 2 || bits == 4 || bits == 8)) {
    set_error("fate_dequant64: bad arguments");
    return FATE_EINVAL;
  }
  if (n == 0) return FATE_OK;
  dequant64_kernel<<<grid_for(n, 256), 256, 0, (cudaStream_t)stream>>>(codes_dev, scale64_dev, zero64_dev, n, bits,
                                                                        group, out_dev);
  FATE_CHECK_LAUNCH("dequant64_kernel");
  return FATE_OK;
}

extern "C" int64_t fate_expert_buffer_bytes(int H, int I, int bits) {
  if (H <= 0 || I <= 0 || H % kGroup || I % kGroup) return -1;
  if (!(bits == 2 || bits == 4 || bits == 8 || bits == 16)) return -1;
  return buffer_bytes(H, I, bits);
}

extern "C" int fate_pack_expert(const float *w1_dev, const float *w3_dev, const float *w2_dev, int H, int I,
                                int bits, int layer, int expert, uint8_t *dst_dev, void *stream) {
  if (fate_expert_buffer_bytes(H, I, bits) < 0) {
    set_error("fate_pack_expert: H and I must be positive multiples of 64; bits in {2,4,8,16}");
    return FATE_EINVAL;
  }
  cudaStream_t s = (cudaStream_t)stream;
  const Layout L = make_layout(H, I, bits);
  uint8_t *p = dst_dev + FATE_HEADER_BYTES;
  const int64_t n = (int64_t)H * I;
  write_header_kernel<<<1, 64, 0, s>>>(dst_dev, bits, layer, expert, H, I);
  FATE_CHECK_LAUNCH("write_header_kernel");
  // W2 goes into the slab-major order first (64-column slabs = whole groups; bf16: 8 columns)
  float *w2s = nullptr;
  FATE_CUDA(cudaMallocAsync(&w2s, (size_t)n * sizeof(float), s));
  w2_slab_kernel<<<grid_for(n, 256), 256, 0, s>>>(w2_dev, H, I, bits == 16 ? kW2SlabBf16 : kW2SlabQuant, w2s);
  cudaError_t le = cudaGetLastError();
  const float *src[3] = {w1_dev, w3_dev, w2s};
  const int64_t co[3] = {L.c1, L.c3, L.c2};
  const int64_t so[3] = {L.s1, L.s3, L.s2};
  for (int j = 0; j < 3 && le == cudaSuccess; ++j)
    le = quant_pack_launch(src[j], n, bits, kGroup, p + co[j],
                           bits == 16 ? nullptr : reinterpret_cast<float *>(p + so[j]), nullptr, nullptr, s);
  cudaFreeAsync(w2s, s);
  FATE_CUDA(le);
  return FATE_OK;
}
