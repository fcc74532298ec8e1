// NOTE: exercises up_mma / w2_mma of the K3 integer tensor-core experiment; apply
// profiles/r02_k3_imma_experiment.patch first (the shipped K3 is the SIMT path).
// Per-item cost of K3's quantized A-piece path (up_mma) and W-piece path
// (w2_mma) in isolation: 12 consumer warps loop over the work items of one
// shared-memory tile.  Build from the repo root:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 --expt-relaxed-constexpr \
//        -I include -o tools/bench/k3_mma_bench tools/bench/k3_mma_bench.cu
#include "../../paper_2502_12224_b200/csrc/ffn.cu"
#include <cstdio>

namespace fate {
void set_error(const std::string &) {}
int cuda_status(cudaError_t, const char *) { return 1; }
}  // namespace fate

using namespace fate;

template <int BITS>
__global__ void up_bench(int reps, long long *cyc, float *sink) {
  extern __shared__ __align__(128) uint8_t sm[];
  const int H = 2048, NG = H / 64;
  const int rb = H * BITS / 8, szb = NG * 8;
  const int nr = BITS == 2 ? 16 : 8;
  uint8_t *tile = sm;
  const int tbytes = 2 * nr * (rb + szb);
  uint8_t *xl = sm + ((tbytes + 127) / 128) * 128;
  for (int i = threadIdx.x; i < tbytes / 4; i += blockDim.x) reinterpret_cast<uint32_t *>(tile)[i] = i * 2654435761u;
  // sz: small sane floats
  for (int i = threadIdx.x; i < 2 * nr * NG; i += blockDim.x)
    reinterpret_cast<float2 *>(tile + 2 * nr * rb)[i] = make_float2(0.01f, -0.02f);
  for (int i = threadIdx.x; i < xlay_total_bytes(H) / 4; i += blockDim.x) reinterpret_cast<uint32_t *>(xl)[i] = i * 97u;
  __syncthreads();
  const int w = BITS == 8 ? 0 : BITS == 4 ? 1 : 2;
  const uint8_t *xtab = xl + xlay_tab_off(H, w);
  const float *gsc = reinterpret_cast<const float *>(xl + xlay_gsc_off(H));
  const float *gsum = reinterpret_cast<const float *>(xl + xlay_gsum_off(H));
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int np = n_parts_g(NG, kParts), nit = ((nr + 7) / 8) * np;
  float acc = 0.f;
  long long t0 = clock64();
  for (int r = 0; r < reps; ++r) {
    const int it = (warp + r) % nit;
    float u, v;
    up_mma<BITS>(tile, nr, NG, 0, it / np, it % np, np, NG, xtab, gsc, gsum, lane, u, v);
    acc += u + v;
  }
  long long t1 = clock64();
  sink[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  if (lane == 0) cyc[blockIdx.x * 32 + warp] = t1 - t0;
}

template <int BITS>
__global__ void w_bench(int reps, long long *cyc, float *sink) {
  extern __shared__ __align__(128) uint8_t sm[];
  __shared__ QUnit U;
  const int WRB = 64 * BITS / 8;
  const int nh = 32768 / (WRB + 8) / 96 * 96;
  uint8_t *tile = sm;
  for (int i = threadIdx.x; i < nh * WRB / 4; i += blockDim.x) reinterpret_cast<uint32_t *>(tile)[i] = i * 2654435761u;
  for (int i = threadIdx.x; i < nh; i += blockDim.x) reinterpret_cast<float2 *>(tile + nh * WRB)[i] = make_float2(0.01f, 0.f);
  float *ysm = reinterpret_cast<float *>(sm + 40000);
  for (int i = threadIdx.x; i < 2048; i += blockDim.x) ysm[i] = 0.f;
  for (int i = threadIdx.x; i < 256; i += blockDim.x) reinterpret_cast<uint8_t *>(&U.wtab[0][0][0][0])[i] = i;
  if (threadIdx.x == 0) U.asc = 1e-6f, U.asum = 1.f;
  __syncthreads();
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  long long t0 = clock64();
  for (int r = 0; r < reps; ++r) w2_mma<BITS>(tile, 0, nh, U, warp, lane, ysm);
  long long t1 = clock64();
  __syncthreads();
  sink[blockIdx.x * blockDim.x + threadIdx.x] = ysm[threadIdx.x];
  if (lane == 0) cyc[blockIdx.x * 32 + warp] = t1 - t0;
}

template <int BITS>
void run(int warps) {
  long long *c; float *s;
  cudaMalloc(&c, 8 * 148 * 32);
  cudaMalloc(&s, 4 * 148 * 1024);
  const int reps = 64;
  cudaFuncSetAttribute(up_bench<BITS>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200000);
  cudaFuncSetAttribute(w_bench<BITS>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200000);
  for (int k = 0; k < 2; ++k) up_bench<BITS><<<148, 32 * warps, 100000>>>(reps, c, s);
  cudaDeviceSynchronize();
  long long h[32];
  cudaMemcpy(h, c, 8 * 32, cudaMemcpyDeviceToHost);
  double m = 0;
  for (int i = 0; i < warps; ++i) m += h[i];
  m /= warps * reps;
  const int nr = BITS == 2 ? 16 : 8;
  const double item_bytes = 2.0 * 8 * 2048 * BITS / 8 / n_parts_g(32, kParts) * 1.0;  // codes of one item (16 rows x H/4)
  printf("up_mma<%d> warps %2d: %7.0f cycles per item per warp, SM %.1f B/cycle (codes) err=%s\n", BITS, warps, m,
         warps * item_bytes / m, cudaGetErrorString(cudaGetLastError()));
  for (int k = 0; k < 2; ++k) w_bench<BITS><<<148, 32 * warps, 100000>>>(reps, c, s);
  cudaDeviceSynchronize();
  cudaMemcpy(h, c, 8 * 32, cudaMemcpyDeviceToHost);
  m = 0;
  for (int i = 0; i < warps; ++i) m += h[i];
  m /= warps * reps;
  const int WRB = 64 * BITS / 8, nh = 32768 / (WRB + 8) / 96 * 96;
  printf("w2_mma<%d> warps %2d: %7.0f cycles per piece (%d rows) per warp, SM %.1f B/cycle err=%s\n", BITS, warps, m,
         nh, nh * (WRB + 8) / m, cudaGetErrorString(cudaGetLastError()));
  (void)nr;
  cudaFree(c); cudaFree(s);
}

int main() {
  run<2>(12); run<4>(12); run<8>(12); run<2>(1); run<4>(1);
  return 0;
}
