// Kernel-to-kernel hand-off microbenchmark: a full-GPU K3-shaped kernel (one
// CTA per SM, 512 threads, large dynamic smem, optionally cooperative) followed
// by a K1-shaped kernel (122 CTAs x 256 threads, ~24 KB static smem), repeated
// on one stream.  Reports the mean gap (globaltimer) last-CTA end of one ->
// first-CTA start of the next, both directions.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o gap_bench gap_bench.cu
#include <cstdio>
#include <cstdlib>
#include <vector>
__device__ __forceinline__ unsigned long long gt() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
struct Stamps { unsigned long long a_start, a_end, b_start, b_end; };
__global__ void __launch_bounds__(512, 1) kA(Stamps *s, int i, int spin_ns) {
  extern __shared__ unsigned char sm[];
  if (threadIdx.x == 0) {
    unsigned long long t = gt();
    atomicMin(&s[i].a_start, t);
    while (gt() - t < (unsigned long long)spin_ns) {}
    sm[0] = 1;
    atomicMax(&s[i].a_end, gt());
  }
}
__global__ void __launch_bounds__(256) kB(Stamps *s, int i, int spin_ns) {
  __shared__ float big[6000];
  if (threadIdx.x == 0) {
    unsigned long long t = gt();
    atomicMin(&s[i].b_start, t);
    while (gt() - t < (unsigned long long)spin_ns) {}
    big[0] = 1.f;
    atomicMax(&s[i].b_end, gt() + (unsigned long long)big[threadIdx.x + 1]);
  }
}
int main(int argc, char **argv) {
  const int coop = argc > 1 ? atoi(argv[1]) : 1;
  const int smemA = argc > 2 ? atoi(argv[2]) : 200 * 1024;
  const int pdl = argc > 3 ? atoi(argv[3]) : 0;
  const int nev = argc > 4 ? atoi(argv[4]) : 0;  // timing-event records between A and B
  std::vector<cudaEvent_t> evs(2 * 200 * 4);
  for (auto &e : evs) cudaEventCreate(&e);
  const int N = 200;
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaFuncSetAttribute(kA, cudaFuncAttributeMaxDynamicSharedMemorySize, smemA);
  cudaFuncSetAttribute(kA, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
  cudaFuncSetAttribute(kB, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
  Stamps *s;
  cudaMalloc(&s, N * sizeof(Stamps));
  std::vector<Stamps> h(N);
  for (auto &x : h) x = Stamps{~0ull, 0, ~0ull, 0};
  cudaMemcpy(s, h.data(), N * sizeof(Stamps), cudaMemcpyHostToDevice);
  cudaStream_t st;
  cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
  for (int i = 0; i < N; ++i) {
    cudaLaunchConfig_t c = {};
    c.gridDim = dim3(sms); c.blockDim = dim3(512); c.dynamicSmemBytes = smemA; c.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeCooperative; at[0].val.cooperative = 1;
    c.attrs = at; c.numAttrs = coop ? 1 : 0;
    cudaLaunchKernelEx(&c, kA, s, i, 20000);
    for (int j = 0; j < nev; ++j) cudaEventRecord(evs[4 * i + j], st);
    cudaLaunchConfig_t cb = {};
    cb.gridDim = dim3(122); cb.blockDim = dim3(256); cb.stream = st;
    cudaLaunchAttribute ab[1];
    ab[0].id = cudaLaunchAttributeProgrammaticStreamSerialization; ab[0].val.programmaticStreamSerializationAllowed = 1;
    cb.attrs = ab; cb.numAttrs = pdl ? 1 : 0;
    cudaLaunchKernelEx(&cb, kB, s, i, 10000);
  }
  cudaError_t e = cudaStreamSynchronize(st);
  cudaMemcpy(h.data(), s, N * sizeof(Stamps), cudaMemcpyDeviceToHost);
  double ab = 0, ba = 0; int n = 0;
  for (int i = 20; i < N - 1; ++i, ++n) {
    ab += (double)(h[i].b_start - h[i].a_end);
    ba += (double)(h[i + 1].a_start - h[i].b_end);
  }
  printf("nev=%d coop=%d smemA=%d pdl=%d err=%s: A end -> B start %.2f us, B end -> A start %.2f us\n", nev, coop, smemA, pdl,
         cudaGetErrorString(e), ab / n * 1e-3, ba / n * 1e-3);
  return 0;
}
