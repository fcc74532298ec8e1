// K3: dequant-fused SwiGLU expert FFN for one decode token (bs = 1), sm_100a.
//
// y = sum_j w_j * W2_j (silu(W1_j x) * (W3_j x))  over the routed experts of
// the step (+ the shared expert with weight 1), reading each expert's packed
// buffer straight from HBM (cache slot or freshly landed staging slot).
//
// The op is a chain of GEMVs: pure HBM streaming, and the B200 design is a
// TMA-bulk pipeline per SM:
//  * one persistent CTA per SM: warp 0 is the producer, warps 1..16 consume;
//  * weights move global -> shared with cp.async.bulk (the TMA engine; SASS
//    UBLKCP) into a ring of 32 KB stages completed on mbarriers, so ~100 KB
//    per SM are in flight independently of register pressure, and every
//    weight byte crosses HBM exactly once;
//  * a tile is a block of contiguous rows of one projection (plus their fp32
//    scale/zero pairs); rows of W1 and W3 with the same index share a tile so
//    silu(u)*v is formed on chip (phase A); phase B tiles are rows of W2 of
//    every expert, reduced over experts inside the CTA (deterministic, no atomics);
//  * the activation vector is staged once per CTA and laid out
//    chunk-transposed, xt[quad][chunk], so 32 lanes read 32 consecutive float4s;
//  * dequant folds the affine map per 16-byte chunk: sum_i (z + s c_i) x_i
//    = s * sum_i c_i x_i + z * sum_i x_i with chunk sums precomputed, i.e. one
//    FFMA per weight element plus code extraction.
#include <cuda_bf16.h>

#include "fate_internal.cuh"

namespace fate {
namespace {

constexpr int kConsumers = 16;
constexpr int kThreads = 32 * (1 + kConsumers);
constexpr int kStageBytes = 32 * 1024;
constexpr int kMaxStages = 4;
constexpr int kSmemLimit = 227 * 1024;
constexpr int kMaxUpRows = 64;

// ---------------------------------------------------------------------------
// PTX helpers: mbarrier + bulk async copy (TMA, non-tensor form)

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ void consumer_sync() {  // named barrier over the consumer warps
  asm volatile("bar.sync 1, %0;" ::"n"(32 * kConsumers) : "memory");
}

// ---------------------------------------------------------------------------
// arithmetic on one 16-byte chunk

// Exact small-integer to float: 2^23 + c has c in the low mantissa bits.
__device__ __forceinline__ float code_f(uint32_t word, int sh, uint32_t mask) {
  return __int_as_float(0x4B000000u | ((word >> sh) & mask)) - 8388608.0f;
}

__device__ __forceinline__ float bf_lo(uint32_t w) { return __uint_as_float(w << 16); }
__device__ __forceinline__ float bf_hi(uint32_t w) { return __uint_as_float(w & 0xFFFF0000u); }

template <int BITS>
struct Fmt {
  static constexpr int kCols = 128 / BITS;  // columns per 16-byte chunk
};

// Packed fp32x2 arithmetic (sm_100a FFMA2 / FADD2): two weight elements per
// instruction.  The activation quads are consumed as (x, y) and (z, w) pairs.
__device__ __forceinline__ float2 ffma2(float2 a, float2 b, float2 c) {
  unsigned long long d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;"
      : "=l"(d)
      : "l"(*reinterpret_cast<unsigned long long *>(&a)), "l"(*reinterpret_cast<unsigned long long *>(&b)),
        "l"(*reinterpret_cast<unsigned long long *>(&c)));
  return *reinterpret_cast<float2 *>(&d);
}

__device__ __forceinline__ float2 fsub2(float2 a, float2 b) {
  unsigned long long d;
  asm("sub.rn.f32x2 %0, %1, %2;"
      : "=l"(d)
      : "l"(*reinterpret_cast<unsigned long long *>(&a)), "l"(*reinterpret_cast<unsigned long long *>(&b)));
  return *reinterpret_cast<float2 *>(&d);
}

// two codes (bit offsets sh, sh + BITS) of a word as an exact float pair
template <int BITS>
__device__ __forceinline__ float2 codes2(uint32_t w, int sh) {
  constexpr uint32_t mask = (1u << BITS) - 1u;
  const float2 m = make_float2(__int_as_float(0x4B000000u | ((w >> sh) & mask)),
                               __int_as_float(0x4B000000u | ((w >> (sh + BITS)) & mask)));
  return fsub2(m, make_float2(8388608.0f, 8388608.0f));
}

__device__ __forceinline__ float2 lo2(const float4 &v) { return make_float2(v.x, v.y); }
__device__ __forceinline__ float2 hi2(const float4 &v) { return make_float2(v.z, v.w); }

// Dot of NR rows' 16-byte code chunks (same column chunk c) with the shared
// activation chunk: each activation quad is loaded once for all NR rows.
// acc[r] holds two independent FFMA2 chains per row.
template <int BITS, int NR>
__device__ __forceinline__ void chunk_dot_rows(const uint4 (&q)[NR], const float4 *__restrict__ xt, int ld, int c,
                                               float2 (&acc)[NR][2]) {
  if constexpr (BITS == 16) {
    const float4 x0 = xt[c], x1 = xt[ld + c];
#pragma unroll
    for (int r = 0; r < NR; ++r) {
      acc[r][0] = ffma2(make_float2(bf_lo(q[r].x), bf_hi(q[r].x)), lo2(x0), acc[r][0]);
      acc[r][1] = ffma2(make_float2(bf_lo(q[r].y), bf_hi(q[r].y)), hi2(x0), acc[r][1]);
      acc[r][0] = ffma2(make_float2(bf_lo(q[r].z), bf_hi(q[r].z)), lo2(x1), acc[r][0]);
      acc[r][1] = ffma2(make_float2(bf_lo(q[r].w), bf_hi(q[r].w)), hi2(x1), acc[r][1]);
    }
  } else {
    constexpr int qpw = 32 / BITS / 4;  // activation quads per 32-bit code word
#pragma unroll
    for (int wi = 0; wi < 4; ++wi)
#pragma unroll
      for (int qi = 0; qi < qpw; ++qi) {
        const float4 xv = xt[(wi * qpw + qi) * ld + c];
        const int sh = qi * 4 * BITS;
#pragma unroll
        for (int r = 0; r < NR; ++r) {
          const uint32_t w = wi == 0 ? q[r].x : wi == 1 ? q[r].y : wi == 2 ? q[r].z : q[r].w;
          acc[r][0] = ffma2(codes2<BITS>(w, sh), lo2(xv), acc[r][0]);
          acc[r][1] = ffma2(codes2<BITS>(w, sh + 2 * BITS), hi2(xv), acc[r][1]);
        }
      }
  }
}

// Partial dots of NR rows held in shared memory (rows at codes[r], scale/zero
// pairs at sz[r]): chunks c = c_begin + stride*i.  Returns per-row sums.
template <int BITS, int NR>
__device__ __forceinline__ void rows_dot_smem(const uint8_t *const (&codes)[NR], const float2 *const (&sz)[NR],
                                              const float4 *xt, const float *xs, int nch, int c_begin, int c_stride,
                                              float (&out)[NR]) {
  float acc_s[NR];
#pragma unroll
  for (int r = 0; r < NR; ++r) acc_s[r] = 0.f;
  for (int c = c_begin; c < nch; c += c_stride) {
    uint4 q[NR];
#pragma unroll
    for (int r = 0; r < NR; ++r) q[r] = reinterpret_cast<const uint4 *>(codes[r])[c];
    float2 acc[NR][2];
#pragma unroll
    for (int r = 0; r < NR; ++r) acc[r][0] = acc[r][1] = make_float2(0.f, 0.f);
    chunk_dot_rows<BITS, NR>(q, xt, nch, c, acc);
#pragma unroll
    for (int r = 0; r < NR; ++r) {
      const float p = (acc[r][0].x + acc[r][0].y) + (acc[r][1].x + acc[r][1].y);
      if constexpr (BITS == 16) {
        acc_s[r] += p;
      } else {
        const float2 z = sz[r][c * Fmt<BITS>::kCols / kGroup];
        acc_s[r] = fmaf(z.x, p, fmaf(z.y, xs[c], acc_s[r]));
      }
    }
  }
#pragma unroll
  for (int r = 0; r < NR; ++r) out[r] = acc_s[r];
}

// single-row convenience wrapper
template <int BITS>
__device__ __forceinline__ float row_dot_smem(const uint8_t *codes, const float2 *sz, const float4 *xt,
                                              const float *xs, int nch, int c_begin, int c_stride) {
  const uint8_t *const cs[1] = {codes};
  const float2 *const zs[1] = {sz};
  float out[1];
  rows_dot_smem<BITS, 1>(cs, zs, xt, xs, nch, c_begin, c_stride, out);
  return out[0];
}

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__device__ __forceinline__ int bits_slot(int bits) { return bits == 16 ? 0 : bits == 8 ? 1 : bits == 4 ? 2 : 3; }
__device__ __forceinline__ int slot_cols(int slot) { return slot == 0 ? 8 : slot == 1 ? 16 : slot == 2 ? 32 : 64; }
__host__ __device__ __forceinline__ int64_t sz_row_bytes(int K, int bits) {
  return bits == 16 ? 0 : (int64_t)K / kGroup * 8;
}

// Copy the batch; experts with bits == 0 take their storage width from the
// packed buffer's header (a copy that landed in a staging slot carries its
// own format).
__device__ __forceinline__ void load_batch(FfnBatch &b, const FfnBatch *src) {
  b = *src;
  for (int j = 0; j < b.n; ++j)
    if (b.e[j].bits == 0) b.e[j].bits = reinterpret_cast<const ExpertHeader *>(b.e[j].buf)->bits;
}

struct Ring {
  uint64_t full[kMaxStages], empty[kMaxStages];
};

__device__ __forceinline__ void ring_init(Ring &r, int stages) {
  for (int s = 0; s < stages; ++s) {
    mbar_init(&r.full[s], 1);
    mbar_init(&r.empty[s], kConsumers);
  }
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

// ----------------------------------------------------------------- tiles
// Phase A tile = rows [r0, r0+R) of W1_j and W3_j of one expert; smem layout
// [W1 codes R*rb][W3 codes R*rb][W1 sz R*szb][W3 sz R*szb].
// Phase B tile = rows [r0, r0+RB) of W2 of every expert; per expert j
// [codes RB*rb_j][sz RB*szb_j].

__device__ __forceinline__ int up_rows_per_tile(int64_t rb, int64_t szb) {
  int R = (int)(kStageBytes / (2 * (rb + szb)));
  R = R > kMaxUpRows ? kMaxUpRows : R;
  return R >= 4 ? R / 4 * 4 : (R >= 1 ? R : 1);
}

struct Plan {
  int n_a;                                  // phase A tiles
  int RBB, n_blk;                           // phase B: rows per CTA row block, number of row blocks
  int tile_off[kMaxFfnExperts + 1], rows_pt[kMaxFfnExperts];
  int lay_off[kMaxFfnExperts + 1];          // activation layout offsets (floats)
  int rows_b[kMaxFfnExperts];               // phase B rows per tile, per expert
  int tiles_b[kMaxFfnExperts + 1];          // phase B tiles per row block, prefix over experts
};

__device__ void make_plan(const FfnBatch &b, Plan &p, int grid) {
  const int H = b.H;
  int t = 0, off = 0, tb = 0;
  // phase B row block: ~H / grid rows so every CTA owns one block
  int RBB = (H + grid - 1) / grid;
  RBB = RBB < 1 ? 1 : RBB;
  p.RBB = RBB;
  p.n_blk = (H + RBB - 1) / RBB;
  for (int j = 0; j < b.n; ++j) {
    const int bits = b.e[j].bits, I = b.e[j].I;
    const int R = up_rows_per_tile((int64_t)H * bits / 8, sz_row_bytes(H, bits));
    p.rows_pt[j] = R;
    p.tile_off[j] = t;
    t += (I + R - 1) / R;
    p.lay_off[j] = off;
    off += (I + I / slot_cols(bits_slot(bits)) + 3) / 4 * 4;
    const int64_t rowb = (int64_t)I * bits / 8 + sz_row_bytes(I, bits);
    int rb = (int)(kStageBytes / rowb);
    rb = rb < 1 ? 1 : (rb > RBB ? RBB : rb);
    p.rows_b[j] = rb;
    p.tiles_b[j] = tb;
    tb += (RBB + rb - 1) / rb;
  }
  p.tile_off[b.n] = t;
  p.lay_off[b.n] = off;
  p.tiles_b[b.n] = tb;
  p.n_a = t;
}

__device__ unsigned int g_grid_barrier = 0;

// per-CTA phase timestamps of the last launch (globaltimer ns), diagnostics only
__device__ unsigned long long g_k3_prof[160][8];
// CTA 0 per-tile timeline of the last launch: [tile][issue, full seen by warp 1, released by warp 1]
__device__ unsigned long long g_k3_tiles[64][3];

__device__ __forceinline__ unsigned long long gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// All CTAs are co-resident (grid = #SMs, one CTA per SM); the counter is never
// reset: each launch waits for the next multiple of gridDim.x.
__device__ __forceinline__ void grid_barrier() {
  __threadfence();
  const unsigned int old = atomicAdd(&g_grid_barrier, 1u);
  const unsigned int target = (old / gridDim.x + 1u) * gridDim.x;
  while ((int)(*(volatile unsigned int *)&g_grid_barrier - target) < 0) {
  }
  __threadfence();
}

// x laid out for every width: slot s (chunk width cols = 8, 16, 32, 64
// columns) at xlay + s * (H/4 + H/32) float4: xt[m * nch + c] = x[c*cols + 4m
// .. +4], then the nch chunk sums.  Built by K1's tail (engine) or by this
// kernel (standalone entry point); K3 bulk-copies it into shared memory.
__global__ void build_xlay_kernel(const float *__restrict__ x, int H, float4 *__restrict__ xlay) {
  extern __shared__ float xs_raw[];
  for (int i = threadIdx.x; i < H; i += blockDim.x) xs_raw[i] = x[i];
  __syncthreads();
  const int stride = H / 4 + H / 32;
  for (int sl = 0; sl < 4; ++sl) {
    const int cols = 8 << sl, nch = H / cols, nq = cols / 4;
    float4 *xt = xlay + sl * stride;
    float *sums = reinterpret_cast<float *>(xt + H / 4);
    for (int i = threadIdx.x; i < H / 4; i += blockDim.x) {
      const int c = (4 * i) / cols, m = ((4 * i) % cols) / 4;
      xt[m * nch + c] = reinterpret_cast<const float4 *>(xs_raw)[i];
    }
    for (int c = threadIdx.x; c < nch; c += blockDim.x) {
      float acc = 0.f;
      for (int m = 0; m < nq; ++m) {
        const float4 q = reinterpret_cast<const float4 *>(xs_raw)[(c * cols) / 4 + m];
        acc += (q.x + q.y) + (q.z + q.w);
      }
      sums[c] = acc;
    }
  }
}

template <int BITS>
__device__ __forceinline__ void up_pair_dots(const uint8_t *c1, const uint8_t *c3, const float2 *z1, const float2 *z3,
                                             const float4 *xt, const float *xs, int nch, int lane, float &u, float &v) {
  const uint8_t *const cs[2] = {c1, c3};
  const float2 *const zs[2] = {z1, z3};
  float out[2];
  rows_dot_smem<BITS, 2>(cs, zs, xt, xs, nch, lane, 32, out);
  u = out[0];
  v = out[1];
}

// One launch per decode step:
//   phase A  gate+up rows: a = silu(W1 x) * (W3 x), written straight into the
//            chunk-transposed activation layout of its expert (alay, global);
//   barrier  grid-wide (all CTAs resident) so every activation is visible;
//   phase B  each CTA owns a block of output rows and streams those rows of W2
//            of every expert, per-expert tiles; partials are combined in a
//            fixed order, so y is deterministic.
// The producer never waits for the barrier: W2 tiles are in flight while
// phase A drains.
__global__ void __launch_bounds__(kThreads, 1) ffn_kernel(const FfnBatch *__restrict__ batch_p,
                                                          const float4 *__restrict__ xlay, float *__restrict__ alay,
                                                          float *__restrict__ y, unsigned long long *bytes_stat,
                                                          int stages) {
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ FfnBatch batch;
  __shared__ Plan plan;
  __shared__ Ring ring;
  __shared__ __align__(8) uint64_t aux_bar[2];
  __shared__ float red[kMaxStages][kConsumers];
  __shared__ int cnt[kMaxStages][kConsumers];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  unsigned long long *prof = g_k3_prof[blockIdx.x < 160 ? blockIdx.x : 159];
  if (tid < 32) {
    // warp 0: batch copy with 16-byte loads, then the plan (lane 0)
    const int4 *src = reinterpret_cast<const int4 *>(batch_p);
    int4 *dst = reinterpret_cast<int4 *>(&batch);
    for (int i = tid; i < (int)(sizeof(FfnBatch) / 16); i += 32) dst[i] = __ldg(src + i);
    __syncwarp();
    if (tid == 0) {
      prof[0] = gtime();
      for (int j = 0; j < batch.n; ++j)
        if (batch.e[j].bits == 0) batch.e[j].bits = reinterpret_cast<const ExpertHeader *>(batch.e[j].buf)->bits;
      make_plan(batch, plan, gridDim.x);
      if (bytes_stat && blockIdx.x == 0) {
        unsigned long long bytes = 0;
        for (int j = 0; j < batch.n; ++j) bytes += make_layout(batch.H, batch.e[j].I, batch.e[j].bits).payload;
        atomicAdd(bytes_stat, bytes);
      }
      ring_init(ring, stages);
      mbar_init(&aux_bar[0], 1);
      mbar_init(&aux_bar[1], 1);
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
  }
  for (int q = tid; q < kMaxStages * kConsumers; q += kThreads) (&cnt[0][0])[q] = 0;
  __syncthreads();
  const int H = batch.H;
  const int lay_stride = H / 4 + H / 32;
  uint8_t *ring_buf = smem;
  float4 *xl = reinterpret_cast<float4 *>(smem + (size_t)stages * kStageBytes);  // x layouts (phase A)
  float *al = reinterpret_cast<float *>(xl);                                      // activation layouts (phase B)
  float *psum = reinterpret_cast<float *>(smem + (size_t)stages * kStageBytes) + plan.lay_off[batch.n] +
                plan.lay_off[batch.n] / 8 + 64;  // [n][RBB] weighted partials (after the activation region)
  if (warp == 0) {
    // ================= producer (one elected lane)
    if (lane == 0) {
      const uint32_t xbytes = (uint32_t)(4 * lay_stride * 16);
      mbar_expect_tx(&aux_bar[0], xbytes);
      bulk_g2s(xl, xlay, xbytes, &aux_bar[0]);
      int stage = 0, ti = 0;
      uint32_t phase = 0;
      for (int t = blockIdx.x; t < plan.n_a; t += gridDim.x) {
        int j = 0;
        while (t >= plan.tile_off[j + 1]) ++j;
        const FfnExpert &ex = batch.e[j];
        const Layout L = make_layout(H, ex.I, ex.bits);
        if (blockIdx.x == 0 && ti < 64) g_k3_tiles[ti][0] = 0;
        const int R = plan.rows_pt[j];
        const int r0 = (t - plan.tile_off[j]) * R, nr = min(R, ex.I - r0);
        const int64_t rb = L.row_bytes_up, szb = sz_row_bytes(H, ex.bits);
        const uint8_t *p = ex.buf + FATE_HEADER_BYTES;
        mbar_wait(&ring.empty[stage], phase ^ 1);
        if (blockIdx.x == 0 && ti < 64) g_k3_tiles[ti][0] = gtime();
        ++ti;
        uint8_t *dst = ring_buf + (size_t)stage * kStageBytes;
        const uint32_t cb = (uint32_t)(nr * rb), sb = (uint32_t)(nr * szb);
        mbar_expect_tx(&ring.full[stage], 2 * (cb + sb));
        bulk_g2s(dst, p + L.c1 + r0 * rb, cb, &ring.full[stage]);
        bulk_g2s(dst + R * rb, p + L.c3 + r0 * rb, cb, &ring.full[stage]);
        if (sb) {
          bulk_g2s(dst + 2 * R * rb, p + L.s1 + r0 * szb, sb, &ring.full[stage]);
          bulk_g2s(dst + 2 * R * rb + R * szb, p + L.s3 + r0 * szb, sb, &ring.full[stage]);
        }
        if (++stage == stages) stage = 0, phase ^= 1;
      }
      for (int blk = blockIdx.x; blk < plan.n_blk; blk += gridDim.x) {
        const int R0 = blk * plan.RBB, nrb = min(plan.RBB, H - R0);
        for (int j = 0; j < batch.n; ++j) {
          const FfnExpert &ex = batch.e[j];
          const Layout L = make_layout(H, ex.I, ex.bits);
          const int64_t rb = L.row_bytes_down, szb = sz_row_bytes(ex.I, ex.bits);
          const uint8_t *p = ex.buf + FATE_HEADER_BYTES;
          const int rt = plan.rows_b[j];
          for (int q0 = 0; q0 < nrb; q0 += rt) {
            const int nr = min(rt, nrb - q0), r0 = R0 + q0;
            mbar_wait(&ring.empty[stage], phase ^ 1);
            if (blockIdx.x == 0 && ti < 64) g_k3_tiles[ti][0] = gtime();
            ++ti;
            uint8_t *dst = ring_buf + (size_t)stage * kStageBytes;
            mbar_expect_tx(&ring.full[stage], (uint32_t)(nr * (rb + szb)));
            bulk_g2s(dst, p + L.c2 + r0 * rb, (uint32_t)(nr * rb), &ring.full[stage]);
            if (szb) bulk_g2s(dst + rt * rb, p + L.s2 + r0 * szb, (uint32_t)(nr * szb), &ring.full[stage]);
            if (++stage == stages) stage = 0, phase ^= 1;
          }
        }
      }
      prof[7] = gtime();
    }
    return;
  }
  // ================= consumers
  const int ctid = tid - 32, cthr = 32 * kConsumers, cw = warp - 1;
  if (ctid == 0) prof[1] = gtime();
  mbar_wait(&aux_bar[0], 0);  // x layouts landed
  if (ctid == 0) prof[2] = gtime();
  // ---- phase A: each warp walks the ring on its own; in tile t it takes
  // rows with (row + k) % kConsumers == warp, both W1 and W3 of the row
  int stage = 0;
  uint32_t phase = 0;
  int k = 0;
  for (int t = blockIdx.x; t < plan.n_a; t += gridDim.x, ++k) {
    int j = 0;
    while (t >= plan.tile_off[j + 1]) ++j;
    const FfnExpert &ex = batch.e[j];
    const int bits = ex.bits, sl = bits_slot(bits), cols = slot_cols(sl);
    const int R = plan.rows_pt[j];
    const int r0 = (t - plan.tile_off[j]) * R, nr = min(R, ex.I - r0);
    const int64_t rb = (int64_t)H * bits / 8, szb = sz_row_bytes(H, bits);
    const int nch = (int)(rb / 16);
    const float4 *xt = xl + sl * lay_stride;
    const float *xs = reinterpret_cast<const float *>(xl + sl * lay_stride + H / 4);
    float *aj = alay + plan.lay_off[j];
    const int nch_a = ex.I / cols;
    mbar_wait(&ring.full[stage], phase);
    if (blockIdx.x == 0 && cw == 0 && lane == 0 && k < 64) g_k3_tiles[k][1] = gtime();
    const uint8_t *tile = ring_buf + (size_t)stage * kStageBytes;
    for (int row = (cw - k % kConsumers + kConsumers) % kConsumers; row < nr; row += kConsumers) {
      const uint8_t *c1 = tile + row * rb, *c3 = tile + (R + row) * rb;
      const float2 *z1 = reinterpret_cast<const float2 *>(tile + 2 * R * rb + row * szb);
      const float2 *z3 = reinterpret_cast<const float2 *>(tile + 2 * R * rb + (R + row) * szb);
      float u, v;
      switch (bits) {
        case 16: up_pair_dots<16>(c1, c3, z1, z3, xt, xs, nch, lane, u, v); break;
        case 8: up_pair_dots<8>(c1, c3, z1, z3, xt, xs, nch, lane, u, v); break;
        case 4: up_pair_dots<4>(c1, c3, z1, z3, xt, xs, nch, lane, u, v); break;
        default: up_pair_dots<2>(c1, c3, z1, z3, xt, xs, nch, lane, u, v); break;
      }
      u = warp_sum(u);
      v = warp_sum(v);
      if (lane == 0) {
        // straight into the chunk-transposed activation layout of phase B
        const int r = r0 + row, c = r / cols, m = (r % cols) / 4;
        aj[(m * nch_a + c) * 4 + (r & 3)] = u / (1.0f + expf(-u)) * v;
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&ring.empty[stage]);
    if (blockIdx.x == 0 && cw == 0 && lane == 0 && k < 64) g_k3_tiles[k][2] = gtime();
    if (++stage == stages) stage = 0, phase ^= 1;
  }
  // ---- every CTA's activations are complete and visible
  consumer_sync();
  if (ctid == 0) {
    prof[3] = gtime();
    grid_barrier();
    prof[4] = gtime();
    // one bulk copy of every expert's activation layout (chunk sums are local)
    const uint32_t abytes = (uint32_t)(plan.lay_off[batch.n] * 4);
    mbar_expect_tx(&aux_bar[1], abytes);
    asm volatile("fence.proxy.async.global;" ::: "memory");
    bulk_g2s(al, alay, abytes, &aux_bar[1]);
  }
  mbar_wait(&aux_bar[1], 0);
  for (int j = 0; j < batch.n; ++j) {
    const int I = batch.e[j].I, cols = slot_cols(bits_slot(batch.e[j].bits));
    const int nch = I / cols, nq = cols / 4;
    const float4 *xt = reinterpret_cast<const float4 *>(al + plan.lay_off[j]);
    float *sums = al + plan.lay_off[j] + I;
    for (int c = ctid; c < nch; c += cthr) {
      float acc = 0.f;
      for (int m = 0; m < nq; ++m) {
        const float4 q = xt[m * nch + c];
        acc += (q.x + q.y) + (q.z + q.w);
      }
      sums[c] = acc;
    }
  }
  consumer_sync();
  if (ctid == 0) prof[5] = gtime();
  // ---- phase B: per row block, per expert tiles; task (row, part) with
  // P = kConsumers / rows parts per row; the last part to finish a row writes
  // the expert's weighted partial; rows are summed over experts in order.
  for (int blk = blockIdx.x; blk < plan.n_blk; blk += gridDim.x) {
    const int R0 = blk * plan.RBB, nrb = min(plan.RBB, H - R0);
    for (int j = 0; j < batch.n; ++j) {
      const FfnExpert &ex = batch.e[j];
      const int bits = ex.bits;
      const int64_t rb = (int64_t)ex.I * bits / 8, szb = sz_row_bytes(ex.I, bits);
      const int nch = (int)(rb / 16);
      const float4 *at = reinterpret_cast<const float4 *>(al + plan.lay_off[j]);
      const float *as = al + plan.lay_off[j] + ex.I;
      const int rt = plan.rows_b[j];
      for (int q0 = 0; q0 < nrb; q0 += rt) {
        const int nr = min(rt, nrb - q0);
        const int P = nr >= kConsumers ? 1 : kConsumers / nr;
        mbar_wait(&ring.full[stage], phase);
        if (blockIdx.x == 0 && cw == 0 && lane == 0 && k < 64) g_k3_tiles[k][1] = gtime();
        const uint8_t *tile = ring_buf + (size_t)stage * kStageBytes;
        for (int task = cw; task < (nr >= kConsumers ? nr : nr * P); task += kConsumers) {
          const int row = nr >= kConsumers ? task : task / P, part = nr >= kConsumers ? 0 : task % P;
          const uint8_t *codes = tile + row * rb;
          const float2 *sz = reinterpret_cast<const float2 *>(tile + rt * rb + row * szb);
          float pj;
          switch (bits) {
            case 16: pj = row_dot_smem<16>(codes, sz, at, as, nch, lane + 32 * part, 32 * P); break;
            case 8: pj = row_dot_smem<8>(codes, sz, at, as, nch, lane + 32 * part, 32 * P); break;
            case 4: pj = row_dot_smem<4>(codes, sz, at, as, nch, lane + 32 * part, 32 * P); break;
            default: pj = row_dot_smem<2>(codes, sz, at, as, nch, lane + 32 * part, 32 * P); break;
          }
          pj = warp_sum(pj);
          if (lane == 0) {
            float *ps = psum + j * plan.RBB + q0 + row;
            if (P == 1) {
              *ps = ex.weight * pj;
            } else {
              red[stage][task] = pj;
              __threadfence_block();
              if (atomicAdd(&cnt[stage][row], 1) == P - 1) {
                __threadfence_block();
                float sum = 0.f;
                for (int q = 0; q < P; ++q) sum += ((volatile float *)red[stage])[row * P + q];
                *ps = ex.weight * sum;
                cnt[stage][row] = 0;
              }
            }
          }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&ring.empty[stage]);
        if (blockIdx.x == 0 && cw == 0 && lane == 0 && k < 64) g_k3_tiles[k][2] = gtime();
        ++k;
        if (++stage == stages) stage = 0, phase ^= 1;
      }
    }
    consumer_sync();
    for (int r = ctid; r < nrb; r += cthr) {
      float acc = 0.f;
      for (int j = 0; j < batch.n; ++j) acc += ((volatile float *)psum)[j * plan.RBB + r];  // fixed order
      y[R0 + r] = acc;
    }
    consumer_sync();
  }
  if (ctid == 0) prof[6] = gtime();
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

// dynamic smem beyond the ring: max(x layouts of every width, activation
// layouts of every expert with bf16-size chunk sums + the partial-sum table)
size_t region_bytes(int H, int max_total_I, int max_experts, int grid) {
  const size_t xb = (size_t)4 * (H / 4 + H / 32) * 16;
  const int RBB = (H + grid - 1) / grid;
  const size_t ab = ((size_t)max_total_I + max_total_I / 8 + 4 * max_experts + max_total_I / 8 + 64 +
                     (size_t)max_experts * RBB) * 4;
  return xb > ab ? xb : ab;
}

int stages_for(size_t extra) {
  int s = kMaxStages;
  while (s > 2 && (size_t)s * kStageBytes + extra + 8192 > (size_t)kSmemLimit) --s;
  return s;
}

}  // namespace

cudaError_t ffn_preload() {
  cudaFuncAttributes a;
  cudaError_t e = cudaFuncGetAttributes(&a, ffn_kernel);
  if (e == cudaSuccess) e = cudaFuncGetAttributes(&a, build_xlay_kernel);
  if (e == cudaSuccess) e = cudaFuncSetAttribute(ffn_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
  return e;
}

size_t ffn_xlay_floats(int H) { return (size_t)4 * (H / 4 + H / 32) * 4; }

size_t ffn_alay_floats(int max_total_I) { return (size_t)max_total_I + max_total_I / 8 + 4 * kMaxFfnExperts; }

cudaError_t launch_build_xlay(const float *x, int H, float *xlay, cudaStream_t s) {
  build_xlay_kernel<<<1, 512, H * sizeof(float), s>>>(x, H, reinterpret_cast<float4 *>(xlay));
  return cudaGetLastError();
}

cudaError_t launch_ffn_decode(const FfnBatch *batch_dev, const float *xlay, float *alay, float *y_dev, int H,
                              int max_total_I, cudaStream_t s) {
  return launch_ffn_decode_engine(batch_dev, xlay, alay, y_dev, H, max_total_I, nullptr, s);
}

cudaError_t launch_ffn_decode_engine(const FfnBatch *batch_dev, const float *xlay, float *alay, float *y_dev, int H,
                                     int max_total_I, unsigned long long *bytes_stat, cudaStream_t s) {
  static bool configured = false;
  if (!configured) {
    cudaError_t e = ffn_preload();
    if (e != cudaSuccess) return e;
    configured = true;
  }
  const int sms = num_sms();
  const size_t extra = region_bytes(H, max_total_I, kMaxFfnExperts, sms);
  const int st = stages_for(extra);
  const size_t smem = (size_t)st * kStageBytes + extra;
  if (smem > 220 * 1024) return cudaErrorInvalidConfiguration;
  // the grid barrier needs every CTA resident: one CTA per SM, grid = #SMs
  ffn_kernel<<<sms, kThreads, smem, s>>>(batch_dev, reinterpret_cast<const float4 *>(xlay), alay, y_dev, bytes_stat,
                                         st);
  return cudaGetLastError();
}

}  // namespace fate

// Diagnostics: per-CTA phase timestamps of the last K3 launch, [160][8] ns.
extern "C" int fate_k3_profile(uint64_t *out_host) {
  if (cudaMemcpyFromSymbol(out_host + 160 * 8, fate::g_k3_tiles, sizeof(unsigned long long) * 64 * 3) != cudaSuccess)
    return FATE_ECUDA;
  if (cudaMemcpyFromSymbol(out_host, fate::g_k3_prof, sizeof(unsigned long long) * 160 * 8) != cudaSuccess) {
    fate::set_error("fate_k3_profile: copy failed");
    return FATE_ECUDA;
  }
  return FATE_OK;
}

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
  float *xl = nullptr, *al = nullptr;
  FATE_CUDA(cudaMallocAsync(&bd, sizeof(FfnBatch), s));
  FATE_CUDA(cudaMallocAsync(&xl, ffn_xlay_floats(H) * sizeof(float), s));
  FATE_CUDA(cudaMallocAsync(&al, ffn_alay_floats(off) * sizeof(float), s));
  FATE_CUDA(cudaMemcpyAsync(bd, &b, sizeof(b), cudaMemcpyHostToDevice, s));
  FATE_CUDA(launch_build_xlay(x_dev, H, xl, s));
  cudaError_t e = launch_ffn_decode(bd, xl, al, y_dev, H, off, s);
  cudaFreeAsync(bd, s);
  cudaFreeAsync(xl, s);
  cudaFreeAsync(al, s);
  FATE_CUDA(e);
  (void)scratch_dev;
  FATE_CUDA(cudaStreamSynchronize(s));  // b lives on this stack frame
  return FATE_OK;
}
