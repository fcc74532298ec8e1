// Microbenchmark of K3's phase-A row-pair dot (up_pair) on shared-memory data
// only (no TMA, no barriers): cycles per row pair vs warps per CTA.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 --expt-relaxed-constexpr
//        -I include tools/bench/k3_dotbench.cu -o gpurun_out/k3_dotbench -L paper_2502_12224_b200 -lfate_b200
#include "../../paper_2502_12224_b200/csrc/ffn.cu"
#include <cstdio>

namespace fate {
namespace {
template <int BITS>
__global__ void dot_bench(int iters, long long *out, float *sink) {
  extern __shared__ __align__(128) uint8_t sm[];
  const int H = 2048, lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int rb = H * BITS / 8, szb = BITS == 16 ? 0 : H / 8;
  const int R = BITS == 16 ? 4 : BITS == 4 ? 12 : 20;
  uint8_t *tile = sm;
  float4 *xl = reinterpret_cast<float4 *>(sm + 32768);
  for (int i = threadIdx.x; i < 32768 / 4; i += blockDim.x) reinterpret_cast<uint32_t *>(tile)[i] = 0x3C003C00u ^ (i * 2654435761u & 0x0F0F0F0Fu);
  for (int i = threadIdx.x; i < 4 * (H / 4 + H / 32) * 4; i += blockDim.x) reinterpret_cast<float *>(xl)[i] = 1e-3f * (i % 97);
  if (BITS != 16)
    for (int r = threadIdx.x; r < 2 * R * H / 64; r += blockDim.x)
      reinterpret_cast<float2 *>(tile + 2 * R * rb)[r] = make_float2(1e-3f, -7e-3f);
  __syncthreads();
  const int sl = BITS == 16 ? 0 : BITS == 8 ? 1 : BITS == 4 ? 2 : 3;
  const int lay_stride = H / 4 + H / 32;
  const float4 *xt = xl + sl * lay_stride;
  const float *xs = reinterpret_cast<const float *>(xl + sl * lay_stride + H / 4);
  float acc = 0.f;
  const long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    float u, v;
    up_pair<BITS, 2048>(tile, R, (warp + it) % R, H, xt, xs, lane, u, v);
    acc += warp_sum(u) + warp_sum(v);
  }
  const long long t1 = clock64();
  if (lane == 0) out[blockIdx.x * 64 + warp] = t1 - t0;
  if (acc == 12345.f) sink[0] = acc;
}
}  // namespace
}  // namespace fate

int main() {
  using namespace fate;
  long long *out;
  float *sink;
  cudaMalloc(&out, 148 * 64 * sizeof(long long));
  cudaMalloc(&sink, 4);
  const int smem = 32768 + 4 * (2048 / 4 + 2048 / 32) * 16;
  cudaFuncSetAttribute(dot_bench<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(dot_bench<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(dot_bench<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int iters = 200;
  for (int bits : {16, 4, 2}) {
    for (int w : {1, 4, 8, 12, 16, 24, 32}) {
      cudaMemset(out, 0, 148 * 64 * sizeof(long long));
      if (bits == 4) dot_bench<4><<<148, 32 * w, smem>>>(iters, out, sink);
      else if (bits == 16) dot_bench<16><<<148, 32 * w, smem>>>(iters, out, sink);
      else dot_bench<2><<<148, 32 * w, smem>>>(iters, out, sink);
      cudaError_t e = cudaDeviceSynchronize();
      long long h[64];
      cudaMemcpy(h, out, sizeof(h), cudaMemcpyDeviceToHost);
      double avg = 0;
      for (int i = 0; i < w; ++i) avg += h[i];
      avg /= w;
      const double elems = 2.0 * 2048;  // per row pair
      const double bytes = elems * bits / 8 + (bits == 16 ? 0 : 2 * 2048 / 64 * 8);
      // per SM: w warps each doing iters row pairs in avg cycles
      const double bpc = bytes * iters * w / avg;  // bytes per cycle per SM
      printf("bits %2d warps %2d: %8.0f cycles/rowpair/warp, SM throughput %6.1f B/cycle = %6.1f GB/s/SM (x148 = %5.2f TB/s) %s\n",
             bits, w, avg / iters, bpc, bpc * 1.965, bpc * 1.965 * 148 / 1000, e == cudaSuccess ? "" : cudaGetErrorString(e));
    }
  }
  return 0;
}
