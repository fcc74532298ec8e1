// IMMA (mma.sync m16n8k32 u8 x s8) latency / throughput on sm_100a, and HMMA
// m16n8k16 bf16 for comparison.  nvcc -gencode arch=compute_100a,code=sm_100a -O3 imma_bench.cu
#include <cstdio>
#include <cstdint>
__device__ __forceinline__ void imma(int (&d)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  asm volatile("mma.sync.aligned.m16n8k32.row.col.s32.u8.s8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
      : "+r"(d[0]), "+r"(d[1]), "+r"(d[2]), "+r"(d[3]) : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
__device__ __forceinline__ void hmma(float (&d)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3]) : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
template <int CHAINS, bool INT>
__global__ void k(int iters, long long *out, int *sink) {
  uint32_t a[4] = {threadIdx.x, threadIdx.x * 3u, 7u, 9u};
  int d[CHAINS][4] = {};
  float f[CHAINS][4] = {};
  __syncthreads();
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) {
      if (INT) imma(d[c], a, i, c); else hmma(f[c], a, i, c);
    }
  }
  long long t1 = clock64();
  int s = 0;
  for (int c = 0; c < CHAINS; ++c) s += d[c][0] + d[c][3] + (int)f[c][0];
  sink[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
}
template <int CHAINS, bool INT>
void run(int warps) {
  long long *o; int *s; cudaMalloc(&o, 8 * 148); cudaMalloc(&s, 4 * 148 * 1024);
  const int iters = 4096;
  k<CHAINS, INT><<<148, 32 * warps>>>(iters, o, s);
  k<CHAINS, INT><<<148, 32 * warps>>>(iters, o, s);
  cudaDeviceSynchronize();
  long long h; cudaMemcpy(&h, o, 8, cudaMemcpyDeviceToHost);
  const double per = (double)h / (iters * CHAINS);
  printf("%s chains %d warps/SM %2d: %.2f cycles per mma per warp, SM rate %.3f mma/cycle\n", INT ? "IMMA.16832" : "HMMA.16816",
         CHAINS, warps, per, warps / per);
  cudaFree(o); cudaFree(s);
}
int main() {
  run<1, true>(1); run<4, true>(1); run<8, true>(1); run<4, true>(4); run<4, true>(8); run<4, true>(16); run<8, true>(16);
  run<1, false>(1); run<4, false>(1); run<4, false>(4); run<4, false>(16);
  return 0;
}
