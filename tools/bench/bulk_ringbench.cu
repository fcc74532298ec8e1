// Microbenchmark of the TMA-bulk streaming ring K3 is built on: one producer
// warp per CTA issues cp.async.bulk copies (global -> shared) into an S-stage
// ring of B-byte stages, NC copies per stage (issued by NC lanes); C consumer
// warps read every byte of a stage with LDS.128 and release it.  One CTA per
// SM, each streaming its own contiguous share of a 2 GB buffer (larger than
// L2).  Reports whole-GPU GB/s per (S, B, NC, C).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17
//        tools/bench/bulk_ringbench.cu -o gpurun_out/bulk_ringbench
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t sa(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void bar_init(uint64_t *b, uint32_t n) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(sa(b)), "r"(n));
}
__device__ __forceinline__ void bar_tx(uint64_t *b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bar_arrive(uint64_t *b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(sa(b)) : "memory");
}
__device__ __forceinline__ void bar_wait(uint64_t *b, uint32_t par) {
  asm volatile(
      "{\n .reg .pred p;\n W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra W;\n}" ::"r"(sa(b)),
      "r"(par)
      : "memory");
}
__device__ __forceinline__ void g2s(void *dst, const void *src, uint32_t bytes, uint64_t *b) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(sa(dst)),
               "l"(src), "r"(bytes), "r"(sa(b))
               : "memory");
}

__global__ void ring(const uint8_t *src, size_t per_cta, int S, int B, int NC, int C, unsigned *sink) {
  extern __shared__ __align__(128) uint8_t sm[];
  __shared__ __align__(8) uint64_t full[8], empty[8];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) bar_init(&full[s], 1), bar_init(&empty[s], C);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const uint8_t *base = src + (size_t)blockIdx.x * per_cta;
  const int tiles = (int)(per_cta / B);
  if (warp == 0) {
    int st = 0;
    uint32_t ph = 0;
    const uint32_t cb = B / NC;
    for (int t = 0; t < tiles; ++t) {
      bar_wait(&empty[st], ph ^ 1);
      if (lane == 0) bar_tx(&full[st], B);
      __syncwarp();
      if (lane < NC) g2s(sm + (size_t)st * B + lane * cb, base + (size_t)t * B + lane * cb, cb, &full[st]);
      if (++st == S) st = 0, ph ^= 1;
    }
    return;
  }
  const int cw = warp - 1;
  int st = 0;
  uint32_t ph = 0, acc = 0;
  for (int t = 0; t < tiles; ++t) {
    bar_wait(&full[st], ph);
    const uint4 *p = reinterpret_cast<const uint4 *>(sm + (size_t)st * B);
    for (int i = cw * 32 + lane; i < B / 16; i += C * 32) {
      const uint4 v = p[i];
      acc ^= v.x ^ v.y ^ v.z ^ v.w;
    }
    __syncwarp();
    if (lane == 0) bar_arrive(&empty[st]);
    if (++st == S) st = 0, ph ^= 1;
  }
  if (acc == 0x12345678u) sink[0] = acc;
}

int main() {
  const size_t total = (size_t)2 << 30;
  uint8_t *buf;
  unsigned *sink;
  cudaMalloc(&buf, total);
  cudaMalloc(&sink, 4);
  cudaMemset(buf, 1, total);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaFuncSetAttribute(ring, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  struct Cfg { int S, B, NC, C; } cfgs[] = {
      {2, 32768, 1, 12}, {3, 32768, 1, 12}, {4, 32768, 1, 12}, {5, 32768, 1, 12}, {6, 32768, 1, 12},
      {5, 32768, 2, 12}, {5, 32768, 4, 12}, {5, 32768, 16, 12}, {5, 32768, 32, 12},
      {10, 16384, 1, 12}, {12, 16384, 1, 12}, {12, 16384, 4, 12}, {8, 24576, 2, 12},
      {4, 49152, 1, 12}, {4, 49152, 4, 12}, {3, 65536, 4, 12}, {5, 32768, 1, 4}, {5, 32768, 1, 1},
  };
  const size_t per_cta = total / sms / 196608 * 196608;  // multiple of every B
  for (const Cfg &c : cfgs) {
    const int threads = 32 * (c.C + 1);
    float best = 1e30f;
    for (int rep = 0; rep < 5; ++rep) {
      cudaEventRecord(e0);
      ring<<<sms, threads, (size_t)c.S * c.B>>>(buf, per_cta, c.S, c.B, c.NC, c.C, sink);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms = 0;
      cudaEventElapsedTime(&ms, e0, e1);
      if (ms < best) best = ms;
    }
    cudaError_t err = cudaGetLastError();
    printf("S=%2d B=%6d NC=%2d C=%2d  in-flight=%4d KB  %7.1f GB/s  %s\n", c.S, c.B, c.NC, c.C, c.S * c.B / 1024,
           (double)per_cta * sms / best / 1e6, err == cudaSuccess ? "" : cudaGetErrorString(err));
  }
  return 0;
}
