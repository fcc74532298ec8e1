// K3: dequant-fused SwiGLU expert FFN for one decode token (bs = 1), sm_100a.
//
// y = sum_j w_j * W2_j (silu(W1_j x) * (W3_j x))  over the routed experts of
// the step (+ the shared expert with weight 1), reading each expert's packed
// buffer straight from HBM (cache slot or freshly landed staging slot).
//
// The op is a chain of GEMVs: pure HBM streaming.  Design for B200:
//  * every weight byte is read exactly once with 128-bit streaming loads
//    (ld.global.nc.L1::no_allocate), 32 lanes covering 512 contiguous bytes;
//  * the activation vector is staged once per CTA in shared memory in a
//    chunk-transposed layout (xt[quad][chunk]) so the 32 lanes of a warp read
//    32 consecutive float4s: conflict-free LDS.128 at the 4-wavefront floor;
//  * dequant folds the affine map per chunk: sum_i (z + s c_i) x_i
//    = s * sum_i c_i x_i + z * sum_i x_i, with the chunk sums precomputed,
//    so the inner loop is one FFMA per element (plus code extraction);
//  * phase A computes gate+up rows in pairs sharing the x loads and writes
//    the activation a = silu(u) * v; phase B reduces every expert's row r of
//    W2 into y[r] inside one warp (deterministic, no atomics);
//  * grids are multiples of the 148 SMs and persistent over rows, so the
//    launch shape is independent of which experts were chosen (graph-stable).
#include <cuda_bf16.h>

#include "fate_internal.cuh"

namespace fate {
namespace {

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;

__device__ __forceinline__ uint4 ld_stream(const void *p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}

__device__ __forceinline__ float2 ld_sz(const float2 *p) {
  float2 r;
  asm volatile("ld.global.nc.L1::no_allocate.v2.f32 {%0,%1}, [%2];" : "=f"(r.x), "=f"(r.y) : "l"(p));
  return r;
}

// Exact small-integer to float: 2^23 + c has c in the low mantissa bits.
__device__ __forceinline__ float code_f(uint32_t word, int sh, uint32_t mask) {
  return __int_as_float(0x4B000000u | ((word >> sh) & mask)) - 8388608.0f;
}

__device__ __forceinline__ float bf_lo(uint32_t w) { return __uint_as_float(w << 16); }
__device__ __forceinline__ float bf_hi(uint32_t w) { return __uint_as_float(w & 0xFFFF0000u); }

// Columns covered by one 16-byte chunk for a storage width.
template <int BITS>
struct Fmt {
  static constexpr int kCols = 128 / BITS;
  static constexpr int kQuads = kCols / 4;
};

// NR chunk dot products against the same activation chunk c.
// xt: chunk-transposed activation, ld = chunks per row.
template <int BITS, int NR>
__device__ __forceinline__ void chunk_dots(const uint4 (&q)[NR], const float4 *__restrict__ xt, int ld, int c,
                                           float (&p)[NR]) {
#pragma unroll
  for (int r = 0; r < NR; ++r) p[r] = 0.f;
  if constexpr (BITS == 16) {
    const float4 x0 = xt[c], x1 = xt[ld + c];
#pragma unroll
    for (int r = 0; r < NR; ++r) {
      float a = p[r];
      a = fmaf(bf_lo(q[r].x), x0.x, a);
      a = fmaf(bf_hi(q[r].x), x0.y, a);
      a = fmaf(bf_lo(q[r].y), x0.z, a);
      a = fmaf(bf_hi(q[r].y), x0.w, a);
      a = fmaf(bf_lo(q[r].z), x1.x, a);
      a = fmaf(bf_hi(q[r].z), x1.y, a);
      a = fmaf(bf_lo(q[r].w), x1.z, a);
      a = fmaf(bf_hi(q[r].w), x1.w, a);
      p[r] = a;
    }
  } else {
    constexpr int per_word = 32 / BITS;
    constexpr uint32_t mask = (1u << BITS) - 1u;
#pragma unroll
    for (int m = 0; m < Fmt<BITS>::kQuads; ++m) {
      const float4 xv = xt[m * ld + c];
      constexpr int dummy = 0;
      (void)dummy;
      const int wi = (4 * m) / per_word;
      const int sh = ((4 * m) % per_word) * BITS;
#pragma unroll
      for (int r = 0; r < NR; ++r) {
        const uint32_t word = wi == 0 ? q[r].x : wi == 1 ? q[r].y : wi == 2 ? q[r].z : q[r].w;
        float a = p[r];
        a = fmaf(code_f(word, sh, mask), xv.x, a);
        a = fmaf(code_f(word, sh + BITS, mask), xv.y, a);
        a = fmaf(code_f(word, sh + 2 * BITS, mask), xv.z, a);
        a = fmaf(code_f(word, sh + 3 * BITS, mask), xv.w, a);
        p[r] = a;
      }
    }
  }
}

// Build the chunk-transposed layout of v[n] for storage width BITS into
// smem: xt[m * nch + c] = v[c*cols + 4m .. +4], xs[c] = sum of the chunk.
template <int BITS>
__device__ void build_layout(const float *__restrict__ v, int n, float4 *xt, float *xs) {
  constexpr int cols = Fmt<BITS>::kCols;
  const int nch = n / cols;
  for (int i = threadIdx.x; i < nch * Fmt<BITS>::kQuads; i += blockDim.x) {
    const int c = i % nch, m = i / nch;
    xt[m * nch + c] = *reinterpret_cast<const float4 *>(v + c * cols + 4 * m);
  }
  for (int c = threadIdx.x; c < nch; c += blockDim.x) {
    float s = 0.f;
    for (int i = 0; i < cols; ++i) s += v[c * cols + i];
    xs[c] = s;
  }
}

// Copy the batch into shared memory; experts with bits == 0 take their
// storage width from the packed buffer's header (the copy that landed in a
// staging slot carries its own format).
__device__ __forceinline__ void load_batch(FfnBatch &b, const FfnBatch *src) {
  b = *src;
  for (int j = 0; j < b.n; ++j)
    if (b.e[j].bits == 0) b.e[j].bits = reinterpret_cast<const ExpertHeader *>(b.e[j].buf)->bits;
}

__device__ __forceinline__ int bits_slot(int bits) { return bits == 16 ? 0 : bits == 8 ? 1 : bits == 4 ? 2 : 3; }

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// ----------------------------------------------------------------- phase A
// Two rows of W1 and the same two rows of W3 per warp iteration.
template <int BITS>
__device__ __forceinline__ void up_pair(const FfnExpert &ex, int H, int r0, const float4 *xt, const float *xs,
                                        float *a_out) {
  const int lane = threadIdx.x & 31;
  const Layout L = make_layout(H, ex.I, BITS);
  const uint8_t *base = ex.buf + FATE_HEADER_BYTES;
  const int64_t rb = L.row_bytes_up;
  const int nch = (int)(rb / 16);
  const uint8_t *w1 = base + L.c1 + r0 * rb;
  const uint8_t *w3 = base + L.c3 + r0 * rb;
  const int gpr = H / kGroup;
  const float2 *s1 = reinterpret_cast<const float2 *>(base + L.s1) + (int64_t)r0 * gpr;
  const float2 *s3 = reinterpret_cast<const float2 *>(base + L.s3) + (int64_t)r0 * gpr;
  float acc[4] = {0.f, 0.f, 0.f, 0.f};  // w1 r0, w1 r1, w3 r0, w3 r1
  for (int c = lane; c < nch; c += 32) {
    uint4 q[4];
    q[0] = ld_stream(w1 + (int64_t)c * 16);
    q[1] = ld_stream(w1 + rb + (int64_t)c * 16);
    q[2] = ld_stream(w3 + (int64_t)c * 16);
    q[3] = ld_stream(w3 + rb + (int64_t)c * 16);
    float p[4];
    if constexpr (BITS == 16) {
      chunk_dots<BITS, 4>(q, xt, nch, c, p);
#pragma unroll
      for (int r = 0; r < 4; ++r) acc[r] += p[r];
    } else {
      const int g = c * Fmt<BITS>::kCols / kGroup;
      const float2 z0 = ld_sz(s1 + g), z1 = ld_sz(s1 + gpr + g);
      const float2 z2 = ld_sz(s3 + g), z3 = ld_sz(s3 + gpr + g);
      chunk_dots<BITS, 4>(q, xt, nch, c, p);
      const float sx = xs[c];
      acc[0] = fmaf(z0.x, p[0], fmaf(z0.y, sx, acc[0]));
      acc[1] = fmaf(z1.x, p[1], fmaf(z1.y, sx, acc[1]));
      acc[2] = fmaf(z2.x, p[2], fmaf(z2.y, sx, acc[2]));
      acc[3] = fmaf(z3.x, p[3], fmaf(z3.y, sx, acc[3]));
    }
  }
#pragma unroll
  for (int r = 0; r < 4; ++r) acc[r] = warp_sum(acc[r]);
  if (lane < 2) {
    const float u = lane == 0 ? acc[0] : acc[1];
    const float v = lane == 0 ? acc[2] : acc[3];
    a_out[ex.a_off + r0 + lane] = u / (1.0f + expf(-u)) * v;
  }
}

__global__ void __launch_bounds__(kThreads) ffn_up_kernel(const FfnBatch *__restrict__ batch_p,
                                                          const float *__restrict__ x, float *__restrict__ a) {
  extern __shared__ float4 smx[];
  __shared__ FfnBatch batch;
  if (threadIdx.x == 0) load_batch(batch, batch_p);
  __syncthreads();
  const int H = batch.H;
  // Layouts for the widths present: slot s at smx + s * (H/4) float4 + sums.
  int present = 0;
  for (int j = 0; j < batch.n; ++j) present |= 1 << bits_slot(batch.e[j].bits);
  float4 *xt[4];
  float *xs[4];
  for (int s = 0; s < 4; ++s) {
    xt[s] = smx + s * (H / 4 + H / 32);
    xs[s] = reinterpret_cast<float *>(xt[s] + H / 4);
  }
  if (present & 1) build_layout<16>(x, H, xt[0], xs[0]);
  if (present & 2) build_layout<8>(x, H, xt[1], xs[1]);
  if (present & 4) build_layout<4>(x, H, xt[2], xs[2]);
  if (present & 8) build_layout<2>(x, H, xt[3], xs[3]);
  __syncthreads();
  int n_tiles = 0;
  for (int j = 0; j < batch.n; ++j) n_tiles += batch.e[j].I / 2;
  const int gw = blockIdx.x * kWarps + (threadIdx.x >> 5);
  for (int t = gw; t < n_tiles; t += gridDim.x * kWarps) {
    int j = 0, off = t;
    while (off >= batch.e[j].I / 2) off -= batch.e[j].I / 2, ++j;
    const FfnExpert &ex = batch.e[j];
    const int r0 = 2 * off;
    switch (ex.bits) {
      case 16: up_pair<16>(ex, H, r0, xt[0], xs[0], a); break;
      case 8: up_pair<8>(ex, H, r0, xt[1], xs[1], a); break;
      case 4: up_pair<4>(ex, H, r0, xt[2], xs[2], a); break;
      default: up_pair<2>(ex, H, r0, xt[3], xs[3], a); break;
    }
  }
}

// ----------------------------------------------------------------- phase B
template <int BITS>
__device__ __forceinline__ float down_row(const FfnExpert &ex, int H, int r, const float4 *at, const float *as) {
  const int lane = threadIdx.x & 31;
  const Layout L = make_layout(H, ex.I, BITS);
  const uint8_t *base = ex.buf + FATE_HEADER_BYTES;
  const int64_t rb = L.row_bytes_down;
  const int nch = (int)(rb / 16);
  const uint8_t *w2 = base + L.c2 + (int64_t)r * rb;
  const int gpr = ex.I / kGroup;
  const float2 *s2 = reinterpret_cast<const float2 *>(base + L.s2) + (int64_t)r * gpr;
  float acc = 0.f;
  int c = lane;
  // two chunks in flight per lane per iteration
  for (; c + 32 < nch; c += 64) {
    uint4 q[2];
    q[0] = ld_stream(w2 + (int64_t)c * 16);
    q[1] = ld_stream(w2 + (int64_t)(c + 32) * 16);
    if constexpr (BITS == 16) {
      float p0[1], p1[1];
      uint4 qa[1] = {q[0]}, qb[1] = {q[1]};
      chunk_dots<BITS, 1>(qa, at, nch, c, p0);
      chunk_dots<BITS, 1>(qb, at, nch, c + 32, p1);
      acc += p0[0] + p1[0];
    } else {
      const float2 z0 = ld_sz(s2 + c * Fmt<BITS>::kCols / kGroup);
      const float2 z1 = ld_sz(s2 + (c + 32) * Fmt<BITS>::kCols / kGroup);
      float p0[1], p1[1];
      uint4 qa[1] = {q[0]}, qb[1] = {q[1]};
      chunk_dots<BITS, 1>(qa, at, nch, c, p0);
      chunk_dots<BITS, 1>(qb, at, nch, c + 32, p1);
      acc = fmaf(z0.x, p0[0], fmaf(z0.y, as[c], acc));
      acc = fmaf(z1.x, p1[0], fmaf(z1.y, as[c + 32], acc));
    }
  }
  for (; c < nch; c += 32) {
    uint4 qa[1] = {ld_stream(w2 + (int64_t)c * 16)};
    float p0[1];
    chunk_dots<BITS, 1>(qa, at, nch, c, p0);
    if constexpr (BITS == 16) {
      acc += p0[0];
    } else {
      const float2 z0 = ld_sz(s2 + c * Fmt<BITS>::kCols / kGroup);
      acc = fmaf(z0.x, p0[0], fmaf(z0.y, as[c], acc));
    }
  }
  return acc;
}

__device__ __forceinline__ int layout_floats(int I, int bits) {
  const int cols = 128 / bits;
  return I + I / cols;  // xt (I floats) + chunk sums
}

__global__ void __launch_bounds__(kThreads) ffn_down_kernel(const FfnBatch *__restrict__ batch_p,
                                                            const float *__restrict__ a, float *__restrict__ y,
                                                            unsigned long long *bytes_stat) {
  extern __shared__ float4 sma[];
  __shared__ FfnBatch batch;
  __shared__ int lay_off[kMaxFfnExperts];
  if (threadIdx.x == 0) {
    load_batch(batch, batch_p);
    if (bytes_stat && blockIdx.x == 0) {
      unsigned long long bytes = 0;
      for (int j = 0; j < batch.n; ++j) bytes += make_layout(batch.H, batch.e[j].I, batch.e[j].bits).payload;
      atomicAdd(bytes_stat, bytes);
    }
    int off = 0;
    for (int j = 0; j < batch.n; ++j) {
      lay_off[j] = off;
      off += (layout_floats(batch.e[j].I, batch.e[j].bits) + 3) / 4 * 4;
    }
  }
  __syncthreads();
  float *base = reinterpret_cast<float *>(sma);
  for (int j = 0; j < batch.n; ++j) {
    const FfnExpert &ex = batch.e[j];
    float4 *at = reinterpret_cast<float4 *>(base + lay_off[j]);
    float *as = base + lay_off[j] + ex.I;
    switch (ex.bits) {
      case 16: build_layout<16>(a + ex.a_off, ex.I, at, as); break;
      case 8: build_layout<8>(a + ex.a_off, ex.I, at, as); break;
      case 4: build_layout<4>(a + ex.a_off, ex.I, at, as); break;
      default: build_layout<2>(a + ex.a_off, ex.I, at, as); break;
    }
  }
  __syncthreads();
  const int H = batch.H;
  const int gw = blockIdx.x * kWarps + (threadIdx.x >> 5);
  for (int r = gw; r < H; r += gridDim.x * kWarps) {
    float acc = 0.f;
    for (int j = 0; j < batch.n; ++j) {
      const FfnExpert &ex = batch.e[j];
      const float4 *at = reinterpret_cast<const float4 *>(base + lay_off[j]);
      const float *as = base + lay_off[j] + ex.I;
      float part;
      switch (ex.bits) {
        case 16: part = down_row<16>(ex, H, r, at, as); break;
        case 8: part = down_row<8>(ex, H, r, at, as); break;
        case 4: part = down_row<4>(ex, H, r, at, as); break;
        default: part = down_row<2>(ex, H, r, at, as); break;
      }
      acc = fmaf(ex.weight, part, acc);
    }
    acc = warp_sum(acc);
    if ((threadIdx.x & 31) == 0) y[r] = acc;
  }
}

int g_num_sms = 0;

int num_sms() {
  if (!g_num_sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, dev);
    if (!g_num_sms) g_num_sms = 148;
  }
  return g_num_sms;
}

}  // namespace

size_t ffn_up_smem(int H) { return (size_t)4 * (H + H / 8) * sizeof(float); }

size_t ffn_down_smem(int max_total_I) {
  // worst case: every expert in bf16 (one chunk sum per 8 columns) + alignment padding
  return ((size_t)max_total_I + max_total_I / 8 + 4 * kMaxFfnExperts) * sizeof(float);
}

// Force module loading of the K3 kernels (CUDA lazy loading would otherwise
// load them at first launch, which deadlocks behind a stream parked on a
// cuStreamWaitValue32 flag).  Also sets the dynamic shared memory limits.
cudaError_t ffn_preload() {
  cudaFuncAttributes a;
  cudaError_t e = cudaFuncGetAttributes(&a, ffn_up_kernel);
  if (e == cudaSuccess) e = cudaFuncGetAttributes(&a, ffn_down_kernel);
  if (e == cudaSuccess) e = cudaFuncSetAttribute(ffn_up_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  if (e == cudaSuccess) e = cudaFuncSetAttribute(ffn_down_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  return e;
}

cudaError_t launch_ffn_decode(const FfnBatch *batch_dev, const float *x_dev, float *a_dev, float *y_dev, int H,
                              int max_total_I, cudaStream_t s) {
  return launch_ffn_decode_engine(batch_dev, x_dev, a_dev, y_dev, H, max_total_I, nullptr, s);
}

cudaError_t launch_ffn_decode_engine(const FfnBatch *batch_dev, const float *x_dev, float *a_dev, float *y_dev, int H,
                                     int max_total_I, unsigned long long *bytes_stat, cudaStream_t s) {
  static bool configured = false;
  const size_t su = ffn_up_smem(H), sd = ffn_down_smem(max_total_I);
  if (!configured) {
    cudaError_t e = ffn_preload();
    if (e != cudaSuccess) return e;
    configured = true;
  }
  const int sms = num_sms();
  ffn_up_kernel<<<sms * 4, kThreads, su, s>>>(batch_dev, x_dev, a_dev);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  const int blocks_b = sd > 100 * 1024 ? sms : sms * 2;
  ffn_down_kernel<<<blocks_b, kThreads, sd, s>>>(batch_dev, a_dev, y_dev, bytes_stat);
  return cudaGetLastError();
}

}  // namespace fate

extern "C" int fate_ffn_decode(const float *x_dev, int H, int n, const uint8_t *const *bufs, const float *weights,
                               float *scratch_dev, float *y_dev, void *stream) {
  using namespace fate;
  if (n < 1 || n > kMaxFfnExperts || H < 64 || H % 64) {
    set_error("fate_ffn_decode: bad arguments");
    return FATE_EINVAL;
  }
  cudaStream_t s = (cudaStream_t)stream;
  FfnBatch b{};
  b.n = n;
  b.H = H;
  int off = 0;
  for (int j = 0; j < n; ++j) {
    ExpertHeader h;
    FATE_CUDA(cudaMemcpyAsync(&h, bufs[j], sizeof(h), cudaMemcpyDeviceToHost, s));
    FATE_CUDA(cudaStreamSynchronize(s));
    if (h.magic != kMagic || h.H != H || h.I % 64) {
      set_error("fate_ffn_decode: buffer header does not describe a packed expert of this hidden size");
      return FATE_EINVAL;
    }
    b.e[j] = FfnExpert{bufs[j], weights[j], h.I, h.bits, off};
    off += h.I;
  }
  b.total_I = off;
  FfnBatch *bd = nullptr;
  FATE_CUDA(cudaMallocAsync(&bd, sizeof(FfnBatch), s));
  FATE_CUDA(cudaMemcpyAsync(bd, &b, sizeof(b), cudaMemcpyHostToDevice, s));
  cudaError_t e = launch_ffn_decode(bd, x_dev, scratch_dev, y_dev, H, off, s);
  cudaFreeAsync(bd, s);
  FATE_CUDA(e);
  FATE_CUDA(cudaStreamSynchronize(s));  // b lives on this stack frame
  return FATE_OK;
}
