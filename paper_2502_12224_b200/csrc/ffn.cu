// K3: dequant-fused SwiGLU expert FFN for one decode token (bs = 1), sm_100a.
//
// y = sum_j w_j * W2_j (silu(W1_j x) * (W3_j x))  over the routed experts of
// the step (+ the shared expert with weight 1), reading each expert's packed
// buffer straight from HBM (cache slot or freshly landed staging slot).
//
// The op is a chain of GEMVs: pure HBM streaming, and the B200 design is a
// TMA-bulk pipeline per SM:
//  * one persistent CTA per SM: warps 0-3 produce (tile g of the stage
//    sequence on warp g mod 4), warps 4-15 consume;
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

#include <cstdlib>
#include <vector>

#include "fate_internal.cuh"

namespace fate {
namespace {

constexpr int kConsumers = 12;  // consumer warps
constexpr int kProducers = 4;   // producer warps (tile g of the stage sequence -> warp g % kProducers);
                                // 16 warps -> 128 registers per thread (allocation in 4-warp units)
constexpr int kThreads = 32 * (kProducers + kConsumers);
constexpr int kStageBytes = 32 * 1024;
constexpr int kMaxStages = 6;
constexpr int kSubRows = 16;     // phase B rows per sub-block (r = 4m + warp%4, m < 4)
constexpr int kMaxBChunks = 96;  // phase B 16-byte chunks per row per tile (3 groups of 32 lanes)
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

// ---------------------------------------------------------------------------
// code extraction: exact small integers as floats through the 2^23 magic
// number.  PRMT places one byte of v under the exponent byte 0x4B, so the
// float is 2^23 + byte exactly; one FSUB2 removes the offset for two codes.

constexpr uint32_t kMagic23 = 0x4B000000u;
__constant__ float kInt4Prescale[4] = {1.0f, 0.0625f, 0.00390625f, 0.000244140625f};
__constant__ float kInt2Prescale[8] = {1.0f, 0.25f, 0.0625f, 0.015625f, 0.00390625f, 0.0009765625f, 0.000244140625f,
                                       6.103515625e-05f};

template <int K>
__device__ __forceinline__ float mag(uint32_t v) {
  return __uint_as_float(__byte_perm(v, kMagic23, 0x7650 + K));
}

// nibble J of v kept in place under the 2^23 magic: 2^23 + c * 2^4J (one LOP3; the magic
// comes in a register so the AND and the OR fuse)
template <int J>
__device__ __forceinline__ float nib(uint32_t v) {
  uint32_t r;
  asm("lop3.b32 %0, %1, %2, %3, 0xEA;" : "=r"(r) : "r"(v), "n"(0xFu << (4 * J)), "r"(kMagic23));
  return __uint_as_float(r);
}

// 2-bit field J of v in place under the 2^23 magic: 2^23 + c * 4^J (one LOP3)
template <int J>
__device__ __forceinline__ float crumb(uint32_t v) {
  uint32_t r;
  asm("lop3.b32 %0, %1, %2, %3, 0xEA;" : "=r"(r) : "r"(v), "n"(0x3u << (2 * J)), "r"(kMagic23));
  return __uint_as_float(r);
}

__device__ __forceinline__ float bf_lo(uint32_t w) { return __uint_as_float(w << 16); }
__device__ __forceinline__ float bf_hi(uint32_t w) { return __uint_as_float(w & 0xFFFF0000u); }

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

__device__ __forceinline__ float2 fadd2(float2 a, float2 b) {
  unsigned long long d;
  asm("add.rn.f32x2 %0, %1, %2;"
      : "=l"(d)
      : "l"(*reinterpret_cast<unsigned long long *>(&a)), "l"(*reinterpret_cast<unsigned long long *>(&b)));
  return *reinterpret_cast<float2 *>(&d);
}

__device__ __forceinline__ float2 lo2(const float4 &v) { return make_float2(v.x, v.y); }
// (x0 + x2, x1 + x3) of a prescaled INT2 activation quad (odd quads carry another 4^-4)
__device__ __forceinline__ float2 unscale2(const float4 &v, int odd) {
  const float b = odd ? 256.0f : 1.0f;
  return ffma2(make_float2(v.z, v.w), make_float2(16.0f * b, 64.0f * b), make_float2(v.x * b, 4.0f * b * v.y));
}
// (x0 + x2, x1 + x3) of a prescaled INT4 activation quad, exactly as from the unscaled one
__device__ __forceinline__ float2 unscale4(const float4 &v) {
  return ffma2(make_float2(v.z, v.w), make_float2(256.0f, 4096.0f), make_float2(v.x, 16.0f * v.y));
}
__device__ __forceinline__ float2 hi2(const float4 &v) { return make_float2(v.z, v.w); }

template <int WI>
__device__ __forceinline__ uint32_t word(const uint4 &q) {
  return WI == 0 ? q.x : WI == 1 ? q.y : WI == 2 ? q.z : q.w;
}

// One 32-bit code word against its activations xv[0 .. 32/BITS/4): two
// independent FFMA2 chains.  Element i of a byte sits at bit i*BITS (quant.py:30-39).
template <int BITS>
__device__ __forceinline__ void word_dot(uint32_t w, const float4 (&xv)[4], float2 &a0, float2 &a1) {
  const float2 m = make_float2(8388608.0f, 8388608.0f);
  if constexpr (BITS == 8) {
    a0 = ffma2(fsub2(make_float2(mag<0>(w), mag<1>(w)), m), lo2(xv[0]), a0);
    a1 = ffma2(fsub2(make_float2(mag<2>(w), mag<3>(w)), m), hi2(xv[0]), a1);
  } else if constexpr (BITS == 4) {
    // element p of the word is nibble p.  Nibbles 0-3 of w and of w >> 16 (IMAD.HI, FMA
    // pipe) are masked in place under the 2^23 magic: one LOP3 each gives 2^23 + c * 2^4j
    // exactly (j = p mod 4); the x layout is prescaled by 2^-4j, so every product is c * x
    // rounded as before.  8 ALU ops per word instead of 2 LOP3 + 8 PRMT.
    const uint32_t hw = __umulhi(w, 1u << 16);
    a0 = ffma2(fsub2(make_float2(nib<0>(w), nib<1>(w)), m), lo2(xv[0]), a0);
    a1 = ffma2(fsub2(make_float2(nib<2>(w), nib<3>(w)), m), hi2(xv[0]), a1);
    a0 = ffma2(fsub2(make_float2(nib<0>(hw), nib<1>(hw)), m), lo2(xv[1]), a0);
    a1 = ffma2(fsub2(make_float2(nib<2>(hw), nib<3>(hw)), m), hi2(xv[1]), a1);
  } else {
    static_assert(BITS == 2, "2/4/8-bit codes");
    // element p = 2-bit field p; fields 0-7 of w and of w >> 16 masked in place
    // (2^23 + c * 4^q exactly, q = p mod 8) against x prescaled by 4^-q
    const uint32_t hw = __umulhi(w, 1u << 16);
    a0 = ffma2(fsub2(make_float2(crumb<0>(w), crumb<1>(w)), m), lo2(xv[0]), a0);
    a1 = ffma2(fsub2(make_float2(crumb<2>(w), crumb<3>(w)), m), hi2(xv[0]), a1);
    a0 = ffma2(fsub2(make_float2(crumb<4>(w), crumb<5>(w)), m), lo2(xv[1]), a0);
    a1 = ffma2(fsub2(make_float2(crumb<6>(w), crumb<7>(w)), m), hi2(xv[1]), a1);
    a0 = ffma2(fsub2(make_float2(crumb<0>(hw), crumb<1>(hw)), m), lo2(xv[2]), a0);
    a1 = ffma2(fsub2(make_float2(crumb<2>(hw), crumb<3>(hw)), m), hi2(xv[2]), a1);
    a0 = ffma2(fsub2(make_float2(crumb<4>(hw), crumb<5>(hw)), m), lo2(xv[3]), a0);
    a1 = ffma2(fsub2(make_float2(crumb<6>(hw), crumb<7>(hw)), m), hi2(xv[3]), a1);
  }
}

// bf16 word pair (elements 2u, 2u+1 of a chunk) against an activation pair
__device__ __forceinline__ float2 bf_dot(uint32_t w, float2 x, float2 acc) {
  return ffma2(make_float2(bf_lo(w), bf_hi(w)), x, acc);
}

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__device__ __forceinline__ int bits_slot(int bits) { return bits == 16 ? 0 : bits == 8 ? 1 : bits == 4 ? 2 : 3; }
__host__ __device__ __forceinline__ int64_t sz_row_bytes(int K, int bits) {
  return bits == 16 ? 0 : (int64_t)K / kGroup * 8;
}

struct Ring {
  uint64_t full[kMaxStages], empty[kMaxStages];
};

// ----------------------------------------------------------------- tiles
// Phase A tile = rows [r0, r0+nr) of W1_j and W3_j of one expert (contiguous
// in the buffer); smem [W1 codes R*rb][W3 codes R*rb][W1 sz R*szb][W3 sz R*szb]
// with R = rows_pt[j].  Phase B tile = columns [k0, k0+nc) of nr (<= 16)
// consecutive rows of W2_j; smem [codes nr * nc*b/8][sz nr * nc/8] (one bulk
// copy per row and region).  The producer publishes each stage's tile in
// meta[stage] before arming its barrier, so consumers never search or divide.

__device__ __forceinline__ int up_rows_per_tile(int64_t rb, int64_t szb) {
  int R = (int)(kStageBytes / (2 * (rb + szb)));
  R = R > kMaxUpRows ? kMaxUpRows : R;
  return R >= 4 ? R / 4 * 4 : (R >= 1 ? R : 1);
}

struct Plan {
  int n_a;                                  // phase A tiles (grabbed dynamically)
  int RBB, n_blk;                           // phase B: rows per CTA row block, number of row blocks
  int tile_off[kMaxFfnExperts + 1], rows_pt[kMaxFfnExperts];
  int lay_off[kMaxFfnExperts + 1];          // activation layout offsets (floats)
  int colsB[kMaxFfnExperts], ktiles[kMaxFfnExperts];  // phase B: W2 columns per tile, tiles per row set
};

struct TileMeta {
  int j;      // expert; -1 = end of phase A, -2 = end of phase B
  int r0;     // phase A: first row of W1/W3; phase B: first output row
  int nr;     // rows in the tile
  int k0;     // phase B: first column of W2
  int nc;     // phase B: columns
  int flush;  // phase B: last tile of its row sub-block
  int pad[2];
};

// Warp 0 builds the plan: lane j fills expert j, offsets by shuffle scans.
__device__ __forceinline__ void make_plan_warp(const FfnBatch &b, Plan &p, int grid, int lane) {
  const int H = b.H;
  int tiles = 0, I = 0, R = 1, colsB = 1, kt = 0;
  if (lane < b.n) {
    const int bits = b.e[lane].bits;
    I = b.e[lane].I;
    R = up_rows_per_tile((int64_t)H * bits / 8, sz_row_bytes(H, bits));
    tiles = (I + R - 1) / R;
    // W2 columns per tile: kSubRows rows must fit one stage and a row's 16-byte
    // chunks must fit 3 chunk groups of 32 lanes (kMaxBChunks)
    const int per128 = 16 * bits + (bits == 16 ? 0 : 16);  // bytes per 128 columns of one row
    int cols = kStageBytes / (kSubRows * per128) * 128;
    const int by_chunks = kMaxBChunks * (bits == 16 ? 8 : 128 / bits);
    cols = cols < by_chunks ? cols : by_chunks;
    colsB = cols < I ? cols : I;
    kt = (I + colsB - 1) / colsB;
  }
  int ts = tiles, is = I;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int a = __shfl_up_sync(0xffffffffu, ts, o), c = __shfl_up_sync(0xffffffffu, is, o);
    if (lane >= o) ts += a, is += c;
  }
  if (lane < b.n) {
    p.tile_off[lane] = ts - tiles;
    p.rows_pt[lane] = R;
    p.lay_off[lane] = is - I;
    p.colsB[lane] = colsB;
    p.ktiles[lane] = kt;
  }
  if (lane == b.n - 1) {
    p.tile_off[b.n] = ts;
    p.lay_off[b.n] = is;
    p.n_a = ts;
  }
  if (lane == 0) {
    int RBB = (H + grid - 1) / grid;
    RBB = RBB < 1 ? 1 : RBB;
    p.RBB = RBB;
    p.n_blk = (H + RBB - 1) / RBB;
  }
}

__device__ unsigned int g_grid_barrier = 0;

// per-CTA phase timestamps of the last launch (globaltimer ns), diagnostics only
__device__ unsigned long long g_k3_prof[160][8];
// CTA 0 per-warp tile timeline of the last launch (clock64 cycles):
//   producer (warp 0): [tile][empty-wait start, empty passed, copies issued]
//   consumer warp w:   [tile][full-wait start, full passed, stage released]
constexpr int kTraceTiles = 48;
__device__ long long g_k3_trace[17][kTraceTiles][3];
// CTA 0, consumer warp 1, first 8 phase-A rows: [row][after dots, after warp sums, after store]
__device__ long long g_k3_sub[8][4];
#define K3_TRACE(w, t, slot) \
  do { if (blockIdx.x == 0 && lane == 0 && (t) < kTraceTiles) g_k3_trace[w][t][slot] = clock64(); } while (0)

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
  unsigned int v;
  do {
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(&g_grid_barrier) : "memory");
  } while ((int)(v - target) < 0);
}

// x laid out for every width: slot s (chunk width cols = 8, 16, 32, 64
// columns) at xlay + s * (H/4 + H/32) float4: xt[m * nch + c] = x[c*cols + 4m
// .. +4], then the nch chunk sums.  Built by K1's tail (engine) or by this
// kernel (standalone entry point); K3 bulk-copies it into shared memory.
__global__ void build_xlay_kernel(const float *__restrict__ x, int H, float4 *__restrict__ xlay) {
  extern __shared__ float xs_raw[];
  for (int i = threadIdx.x; i < H; i += blockDim.x) xs_raw[i] = x[i];
  __syncthreads();
  write_xlay(xs_raw, H, xlay, threadIdx.x, blockDim.x);
}

// Phase A: this lane's partial dots of row `row` of W1 and W3 in a tile.
// HT = compile-time hidden size (0: runtime H), so the chunk loop is fully
// unrolled and every shared-memory offset is an immediate.
template <int BITS, int HT>
__device__ __forceinline__ void up_pair(const uint8_t *__restrict__ tile, int R, int row, int H_rt,
                                        const float4 *__restrict__ xt, const float *__restrict__ xs, int lane,
                                        float &u, float &v) {
  const int H = HT ? HT : H_rt;
  const int rb = H * BITS / 8;
  const int nch = rb / 16;  // 16-byte chunks per row = stride of the x layout for this width
  const uint4 *q1 = reinterpret_cast<const uint4 *>(tile + row * rb);
  const uint4 *q3 = reinterpret_cast<const uint4 *>(tile + (R + row) * rb);
  const int iters = (nch + 31) / 32;
  if constexpr (BITS == 16) {
    float2 a0 = make_float2(0.f, 0.f), a1 = a0, b0 = a0, b1 = a0;
    constexpr int kU = 2;
#pragma unroll kU
    for (int i = 0; i < iters; ++i) {
      const int c = lane + 32 * i;
      if ((HT && (HT * BITS / 8 / 16) % 32 == 0) || c < nch) {
        const uint4 w1 = q1[c], w3 = q3[c];
        const float4 x0 = xt[c], x1 = xt[nch + c];
        a0 = bf_dot(w1.x, lo2(x0), a0);
        a1 = bf_dot(w1.y, hi2(x0), a1);
        b0 = bf_dot(w3.x, lo2(x0), b0);
        b1 = bf_dot(w3.y, hi2(x0), b1);
        a0 = bf_dot(w1.z, lo2(x1), a0);
        a1 = bf_dot(w1.w, hi2(x1), a1);
        b0 = bf_dot(w3.z, lo2(x1), b0);
        b1 = bf_dot(w3.w, hi2(x1), b1);
      }
    }
    u = (a0.x + a0.y) + (a1.x + a1.y);
    v = (b0.x + b0.y) + (b1.x + b1.y);
  } else {
    constexpr int qpw = 32 / BITS / 4;               // activation quads per 32-bit code word
    constexpr int cpg = kGroup / (128 / BITS);       // chunks per quantization group
    const int szb = H / 8;                           // (scale, zero) bytes per row
    const float2 *z1 = reinterpret_cast<const float2 *>(tile + 2 * R * rb + row * szb);
    const float2 *z3 = reinterpret_cast<const float2 *>(tile + 2 * R * rb + (R + row) * szb);
    float s1 = 0.f, s3 = 0.f;
    constexpr int kUq = 1;
#pragma unroll kUq
    for (int i = 0; i < iters; ++i) {
      const int c = lane + 32 * i;
      if ((HT && (HT * BITS / 8 / 16) % 32 == 0) || c < nch) {
        const uint4 w1 = q1[c], w3 = q3[c];
        float2 p0 = make_float2(0.f, 0.f), p1 = p0, r0 = p0, r1 = p0;
        float4 xv[4];
#define FATE_WORD(WI)                                                                          \
  _Pragma("unroll") for (int qi = 0; qi < qpw; ++qi) xv[qi] = xt[((WI) * qpw + qi) * nch + c]; \
  word_dot<BITS>(word<WI>(w1), xv, p0, p1);                                                    \
  word_dot<BITS>(word<WI>(w3), xv, r0, r1);
        FATE_WORD(0) FATE_WORD(1) FATE_WORD(2) FATE_WORD(3)
#undef FATE_WORD
        const float xsum = xs[c];
        const float2 g1 = z1[c / cpg], g3 = z3[c / cpg];
        s1 = fmaf(g1.x, (p0.x + p0.y) + (p1.x + p1.y), fmaf(g1.y, xsum, s1));
        s3 = fmaf(g3.x, (r0.x + r0.y) + (r1.x + r1.y), fmaf(g3.y, xsum, s3));
      }
    }
    u = s1;
    v = s3;
  }
}

// Phase B: unit (c, h) of a tile -- words [h*U, h*U+U) of 16-byte chunk c
// (global chunk cg of expert j's activation layout `at`, nchI chunks per
// activation quad row) -- for MR rows of the tile, row[i] = 4 m_i + w4,
// valid[i] = row exists; out[i] = w_j * dot(row[i]).  Quantized tiles with few
// chunks per row use U = 2 or 1 so that the units still cover all 3 chunk groups.
template <int BITS, int MR, int U>
__device__ __forceinline__ void down_chunk(const uint8_t *tile, int nr, int nc, int c, int h,
                                           const float4 *__restrict__ at, int nchI, int cg, const int (&row)[MR],
                                           int valid, float wj, float (&out)[MR]) {
  const int rowb = nc * BITS / 8;
  uint4 q[MR];
#pragma unroll
  for (int i = 0; i < MR; ++i) {
    const uint8_t *src = tile + row[i] * rowb + c * 16 + h * 4 * U;
    if (!(valid >> i & 1)) q[i] = make_uint4(0, 0, 0, 0);
    else if constexpr (U == 4) q[i] = *reinterpret_cast<const uint4 *>(src);
    else if constexpr (U == 2) {
      const uint2 t = *reinterpret_cast<const uint2 *>(src);
      q[i] = make_uint4(t.x, t.y, 0, 0);
    } else q[i] = make_uint4(*reinterpret_cast<const uint32_t *>(src), 0, 0, 0);
  }
  float2 p[MR][2];
#pragma unroll
  for (int i = 0; i < MR; ++i) p[i][0] = p[i][1] = make_float2(0.f, 0.f);
  if constexpr (BITS == 16) {
    static_assert(U == 4, "bf16 tiles use whole chunks");
    const float4 x0 = at[cg], x1 = at[nchI + cg];
#pragma unroll
    for (int i = 0; i < MR; ++i) {
      p[i][0] = bf_dot(q[i].x, lo2(x0), p[i][0]);
      p[i][1] = bf_dot(q[i].y, hi2(x0), p[i][1]);
      p[i][0] = bf_dot(q[i].z, lo2(x1), p[i][0]);
      p[i][1] = bf_dot(q[i].w, hi2(x1), p[i][1]);
    }
#pragma unroll
    for (int i = 0; i < MR; ++i) out[i] = wj * ((p[i][0].x + p[i][0].y) + (p[i][1].x + p[i][1].y));
  } else {
    constexpr int qpw = 32 / BITS / 4;
    float2 sa = make_float2(0.f, 0.f);
    float4 xv[4];
#define FATE_WORD(WI)                                                      \
  if constexpr ((WI) < U) {                                                \
    _Pragma("unroll") for (int qi = 0; qi < qpw; ++qi) {                   \
      xv[qi] = at[((h * U + (WI)) * qpw + qi) * nchI + cg];                \
      sa = fadd2(sa, BITS == 4 ? unscale4(xv[qi]) : BITS == 2 ? unscale2(xv[qi], qi & 1)  \
                                                   : fadd2(lo2(xv[qi]), hi2(xv[qi])));               \
    }                                                                      \
    _Pragma("unroll") for (int i = 0; i < MR; ++i) word_dot<BITS>(word<WI>(q[i]), xv, p[i][0], p[i][1]); \
  }
    FATE_WORD(0) FATE_WORD(1) FATE_WORD(2) FATE_WORD(3)
#undef FATE_WORD
    const float xsum = sa.x + sa.y;
    const int szr = nc / 8;  // bytes of (scale, zero) pairs per row
    const int grp = c / (kGroup / (128 / BITS));
#pragma unroll
    for (int i = 0; i < MR; ++i) {
      const float2 z = (valid >> i & 1) ? reinterpret_cast<const float2 *>(tile + nr * rowb + row[i] * szr)[grp]
                                        : make_float2(0.f, 0.f);
      const float s = (p[i][0].x + p[i][0].y) + (p[i][1].x + p[i][1].y);
      out[i] = wj * fmaf(z.x, s, z.y * xsum);
    }
  }
}

// Rows of a phase B tile owned by consumer warp cw (12 warps): with 3 chunk
// groups (G = 3) warp cw takes chunk group cw / 4 and rows r = 4m + cw % 4
// (m = 0..3); with one group (G = 1, at most 32 units per row) it takes rows
// cw and cw + 12.  Either way r = 4m + (cw & 3), so every thread's rows stay in
// acc[m] for the whole sub-block whatever the tile's chunk-group count.
template <int BITS, int MR, int U>
__device__ __forceinline__ void down_tile(const uint8_t *tile, int nr, int nc, int c, int h,
                                          const float4 *__restrict__ at, int nchI, int cg, int cw, float wj,
                                          float (&acc)[4]) {
  int m[MR], row[MR], valid = 0;
#pragma unroll
  for (int i = 0; i < MR; ++i) {
    m[i] = MR == 4 ? i : (cw >> 2) + 3 * i;
    row[i] = 4 * m[i] + (cw & 3);
    if (row[i] < nr) valid |= 1 << i;
  }
  float out[MR];
  down_chunk<BITS, MR, U>(tile, nr, nc, c, h, at, nchI, cg, row, valid, wj, out);
#pragma unroll
  for (int i = 0; i < MR; ++i) {
    if constexpr (MR == 4) {
      acc[i] += out[i];
    } else {
#pragma unroll
      for (int mm = 0; mm < 4; ++mm) acc[mm] += (m[i] == mm && (valid >> i & 1)) ? out[i] : 0.f;
    }
  }
}

template <int BITS, int U>
__device__ __forceinline__ void down_tile_units(const TileMeta &tm, const uint8_t *tile, const FfnExpert &ex,
                                                const float *al_j, int cw, int lane, int nch, float (&acc)[4]) {
  constexpr int cols = BITS == 16 ? 8 : 128 / BITS;  // columns per 16-byte chunk
  const int nunits = nch * (4 / U);
  const bool g3 = nunits > 32;
  const int u = lane + (g3 ? 32 * (cw >> 2) : 0);
  if (u >= nunits) return;
  const int c = u / (4 / U), h = u % (4 / U);
  const float4 *at = reinterpret_cast<const float4 *>(al_j);
  const int nchI = ex.I / cols, cg = tm.k0 / cols + c;
  if (g3) down_tile<BITS, 4, U>(tile, tm.nr, tm.nc, c, h, at, nchI, cg, cw, ex.weight, acc);
  else down_tile<BITS, 2, U>(tile, tm.nr, tm.nc, c, h, at, nchI, cg, cw, ex.weight, acc);
}

// One phase B tile: the 12 consumer warps split the tile's units (chunks, or
// half / quarter chunks of quantized rows with <= 48 / 24 chunks) into G groups
// of 32 lanes (G = 1 or 3) and its rows into 12 / G residue classes.
template <int BITS>
__device__ __forceinline__ void down_tile_bits(const TileMeta &tm, const uint8_t *tile, const FfnExpert &ex,
                                               const float *al_j, int cw, int lane, float (&acc)[4]) {
  constexpr int cols = BITS == 16 ? 8 : 128 / BITS;
  const int nch = tm.nc / cols;
  if constexpr (BITS == 16) {
    down_tile_units<16, 4>(tm, tile, ex, al_j, cw, lane, nch, acc);
  } else {
    if (nch > 48) down_tile_units<BITS, 4>(tm, tile, ex, al_j, cw, lane, nch, acc);
    else if (nch > 24) down_tile_units<BITS, 2>(tm, tile, ex, al_j, cw, lane, nch, acc);
    else down_tile_units<BITS, 1>(tm, tile, ex, al_j, cw, lane, nch, acc);
  }
}

// One launch per decode step:
//   phase A  gate+up rows: a = silu(W1 x) * (W3 x).  Tiles go round-robin
//            over the CTAs; consumer warp w takes the rows of tile k whose
//            running index is w mod 12, so the rows of consecutive tiles land
//            on different warps; a goes straight into the chunk-transposed layout of its
//            expert (alay, global);
//   barrier  grid-wide (all CTAs resident) so every activation is visible;
//   phase B  each CTA owns a block of output rows (sub-blocks of <= 16) and
//            streams column ranges of those rows of W2 of every expert; the
//            12 consumer warps split the columns (chunk groups) and rows
//            (r = 4m + w%4), accumulating w_j * dot in registers across all
//            tiles, then one fixed-order reduction per row: y is deterministic.
// The producers never wait for the barrier: W2 tiles are in flight while
// phase A drains.
template <int HT>
__global__ void __launch_bounds__(kThreads, 1) ffn_kernel(const FfnBatch *__restrict__ batch_p,
                                                          const float4 *__restrict__ xlay, float *__restrict__ alay,
                                                          float *__restrict__ y, unsigned long long *bytes_stat,
                                                          int stages, int nprod) {
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ FfnBatch batch;
  __shared__ Plan plan;
  __shared__ Ring ring;
  __shared__ TileMeta meta[kMaxStages];
  __shared__ __align__(8) uint64_t x_bar, act_bar[kMaxFfnExperts];
  __shared__ float part[kSubRows][3];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  unsigned long long *prof = g_k3_prof[blockIdx.x < 160 ? blockIdx.x : 159];
  if (blockIdx.x == 0)
    for (int i = tid; i < 17 * kTraceTiles * 3; i += kThreads) (&g_k3_trace[0][0][0])[i] = 0;
  if (warp == 0) {
    // warp 0: batch copy with 16-byte loads, the plan, the barriers
    const int4 *src = reinterpret_cast<const int4 *>(batch_p);
    int4 *dst = reinterpret_cast<int4 *>(&batch);
    for (int i = lane; i < (int)(sizeof(FfnBatch) / 16); i += 32) dst[i] = __ldg(src + i);
    __syncwarp();
    if (lane < batch.n && batch.e[lane].bits == 0)
      batch.e[lane].bits = reinterpret_cast<const ExpertHeader *>(batch.e[lane].buf)->bits;
    __syncwarp();
    make_plan_warp(batch, plan, gridDim.x, lane);
    if (lane == 0) {
      prof[0] = gtime();
      for (int s = 0; s < stages; ++s) {
        mbar_init(&ring.full[s], 1);
        mbar_init(&ring.empty[s], kConsumers);
      }
      mbar_init(&x_bar, 1);
      for (int j = 0; j < batch.n; ++j) mbar_init(&act_bar[j], 1);
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
  }
  __syncthreads();
  const int H = HT ? HT : batch.H;
  const int lay_stride = H / 4 + H / 32;
  uint8_t *ring_buf = smem;
  float4 *xl = reinterpret_cast<float4 *>(smem + (size_t)stages * kStageBytes);  // x layouts (phase A)
  float *al = reinterpret_cast<float *>(xl);                                      // activation layouts (phase B)
  if (warp < kProducers) {
    // ================= producer warps: tile g of the stage sequence (phase A
    // tiles, end marker, phase B tiles) belongs to producer g % kProducers, so
    // the ~0.1 us issue latency of each bulk copy overlaps across warps.  The
    // ring has more stages than producers, so an empty-barrier parity never aliases.
    const int pw = warp;
    if (pw == 0 && lane == 0) {
      const uint32_t xbytes = (uint32_t)(4 * lay_stride * 16);
      mbar_expect_tx(&x_bar, xbytes);
      bulk_g2s(xl, xlay, xbytes, &x_bar);
      if (blockIdx.x == 0 && bytes_stat) {
        unsigned long long bytes = 0;
        for (int j = 0; j < batch.n; ++j) bytes += make_layout(H, batch.e[j].I, batch.e[j].bits).payload;
        atomicAdd(bytes_stat, bytes);
      }
    }
    // active producers: fewer than the ring's stages (parity safety)
    const int np = nprod < stages - 1 ? nprod : stages - 1;
    if (pw >= np) return;
    int stage = 0, ti = 0;  // ti = position in the stage sequence
    uint32_t phase = 0;
    auto mine = [&]() -> bool {
      stage = ti % stages;
      phase = (uint32_t)(ti / stages) & 1u;
      return ti % np == pw;
    };
    // one phase A tile (or the end marker); returns true at the end
    auto step_a = [&](int t) -> bool {
      if (!mine()) {
        ++ti;
        return t >= plan.n_a;
      }
      K3_TRACE(0, ti, 0);
      mbar_wait(&ring.empty[stage], phase ^ 1);
      const bool end = t >= plan.n_a;
      if (end) {
        if (lane == 0) {
          meta[stage].j = -1;
          mbar_arrive(&ring.full[stage]);
        }
      } else {
        int j = 0;
        while (t >= plan.tile_off[j + 1]) ++j;
        const FfnExpert &ex = batch.e[j];
        const int bits = ex.bits;
        const int R = plan.rows_pt[j];
        const int r0 = (t - plan.tile_off[j]) * R, nr = min(R, ex.I - r0);
        const uint32_t rb = (uint32_t)H * bits / 8, szb = bits == 16 ? 0u : (uint32_t)H / 8;
        const uint32_t cb = nr * rb, sb = nr * szb;
        uint8_t *dst = ring_buf + (size_t)stage * kStageBytes;
        if (lane == 0) {
          meta[stage].j = j;
          meta[stage].r0 = r0;
          meta[stage].nr = nr;
          mbar_expect_tx(&ring.full[stage], 2 * (cb + sb));
        }
        __syncwarp();
        K3_TRACE(0, ti, 1);
        if (lane < (sb ? 4 : 2)) {
          // lanes 0..3: W1 codes, W3 codes, W1 (scale, zero), W3 (scale, zero)
          const int64_t n = (int64_t)H * ex.I, cbytes = bits == 16 ? 2 * n : n * bits / 8;
          const int64_t sbytes = n / kGroup * 8;
          const int64_t src = lane == 0 ? (int64_t)r0 * rb
                            : lane == 1 ? cbytes + (int64_t)r0 * rb
                            : lane == 2 ? 3 * cbytes + (int64_t)r0 * szb
                                        : 3 * cbytes + sbytes + (int64_t)r0 * szb;
          const uint32_t off = lane == 0 ? 0u : lane == 1 ? R * rb : lane == 2 ? 2 * R * rb : 2 * R * rb + R * szb;
          bulk_g2s(dst + off, ex.buf + FATE_HEADER_BYTES + src, lane < 2 ? cb : sb, &ring.full[stage]);
        }
      }
      K3_TRACE(0, ti, 2);
      ++ti;
      return end;
    };
    // static round-robin over the tile list (expert-major, so every CTA gets a
    // proportional mix of each expert's format), walked alternately from both
    // ends so compute-heavy quantized tiles interleave with bf16 streaming
    // tiles; then the end marker
    {
      const int K = plan.n_a > (int)blockIdx.x ? (plan.n_a - (int)blockIdx.x + (int)gridDim.x - 1) / (int)gridDim.x : 0;
      for (int i = 0; i < K; ++i) {
        const int kk = (i & 1) ? K - 1 - (i >> 1) : (i >> 1);
        step_a((int)blockIdx.x + kk * (int)gridDim.x);
      }
      step_a(plan.n_a);  // end marker
    }
    for (int blk = blockIdx.x; blk < plan.n_blk; blk += gridDim.x) {
      const int R0 = blk * plan.RBB, rows = min(plan.RBB, H - R0);
      for (int s0 = 0; s0 < rows; s0 += kSubRows) {
        const int nr = min(kSubRows, rows - s0), rs0 = R0 + s0;
        // the sub-block's tiles (expert j, K-range kt), walked alternately from
        // both ends of the expert-major list (routed quantized tiles interleave
        // with the shared expert's bf16 tiles); the last one carries the flush
        int total = 0;
        for (int j = 0; j < batch.n; ++j) total += plan.ktiles[j];
        for (int i = 0; i < total; ++i) {
          int pos = (i & 1) ? total - 1 - (i >> 1) : (i >> 1), j = 0;
          while (pos >= plan.ktiles[j]) pos -= plan.ktiles[j], ++j;
          const int kt = pos;
          const FfnExpert &ex = batch.e[j];
          const int bits = ex.bits;
          const Layout L = make_layout(H, ex.I, bits);
          const int64_t rb = L.row_bytes_down, szb = sz_row_bytes(ex.I, bits);
          const uint8_t *p = ex.buf + FATE_HEADER_BYTES;
          if (!mine()) {
            ++ti;
          } else {
            const int k0 = kt * plan.colsB[j], nc = min(plan.colsB[j], ex.I - k0);
            const uint32_t cb = (uint32_t)nc * bits / 8, sb = bits == 16 ? 0u : (uint32_t)nc / 8;
            K3_TRACE(0, ti, 0);
            mbar_wait(&ring.empty[stage], phase ^ 1);
            uint8_t *dst = ring_buf + (size_t)stage * kStageBytes;
            if (lane == 0) {
              TileMeta &m = meta[stage];
              m.j = j;
              m.r0 = rs0;
              m.nr = nr;
              m.k0 = k0;
              m.nc = nc;
              m.flush = i == total - 1;
              mbar_expect_tx(&ring.full[stage], (uint32_t)nr * (cb + sb));
            }
            __syncwarp();
            K3_TRACE(0, ti, 1);
            if (ex.layout == 1) {
              // bf16 W2 in column slabs (kSlabCols == this K-range): the tile's rows are contiguous
              if (lane == 0) bulk_g2s(dst, p + L.c2 + (int64_t)H * k0 * 2 + (int64_t)rs0 * nc * 2,
                                      nr * cb, &ring.full[stage]);
            } else if (nc == ex.I) {
              // whole rows: the tile's rows are contiguous in the buffer, one copy
              // for the codes and one for the (scale, zero) pairs
              if (lane == 0) bulk_g2s(dst, p + L.c2 + (int64_t)rs0 * rb, nr * cb, &ring.full[stage]);
              if (lane == 1 && sb) bulk_g2s(dst + nr * cb, p + L.s2 + (int64_t)rs0 * szb, nr * sb, &ring.full[stage]);
            } else if (lane < nr) {
              const int64_t r = rs0 + lane;
              bulk_g2s(dst + lane * cb, p + L.c2 + r * rb + (int64_t)k0 * bits / 8, cb, &ring.full[stage]);
              if (sb) bulk_g2s(dst + nr * cb + lane * sb, p + L.s2 + r * szb + k0 / 8, sb, &ring.full[stage]);
            }
            K3_TRACE(0, ti, 2);
            ++ti;
          }
        }
      }
    }
    if (lane == 0 && pw == 0) prof[7] = gtime();
    return;
  }
  // ================= consumers
  const int ctid = tid - 32 * kProducers, cw = warp - kProducers;
  if (ctid == 0) prof[1] = gtime();
  mbar_wait(&x_bar, 0);  // x layouts landed
  if (ctid == 0) prof[2] = gtime();
  int stage = 0, k = 0, rot = 0;
  uint32_t phase = 0;
  for (;; ++k) {
    K3_TRACE(cw + 1, k, 0);
    mbar_wait(&ring.full[stage], phase);
    K3_TRACE(cw + 1, k, 1);
    const int j = meta[stage].j;
    if (j < 0) {
      __syncwarp();
      if (lane == 0) mbar_arrive(&ring.empty[stage]);
      if (++stage == stages) stage = 0, phase ^= 1;
      ++k;
      break;
    }
    const int r0 = meta[stage].r0, nr = meta[stage].nr;
    const FfnExpert &ex = batch.e[j];
    const int bits = ex.bits, sl = bits_slot(bits);
    const int R = plan.rows_pt[j];
    const float4 *xt = xl + sl * lay_stride;
    const float *xs = reinterpret_cast<const float *>(xl + sl * lay_stride + H / 4);
    const uint8_t *tile = ring_buf + (size_t)stage * kStageBytes;
    // W2 chunk width of this expert (power of two): a[r] -> (r/cols, (r%cols)/4, r&3)
    const int lc = bits == 16 ? 3 : bits == 8 ? 4 : bits == 4 ? 5 : 6;
    float *aj = alay + plan.lay_off[j];
    const int nch_a = ex.I >> lc;
    int row0 = cw - rot;
    if (row0 < 0) row0 += kConsumers;
    for (int row = row0; row < nr; row += kConsumers) {
      float u, v;
      switch (bits) {
        case 16: up_pair<16, HT>(tile, R, row, H, xt, xs, lane, u, v); break;
        case 8: up_pair<8, HT>(tile, R, row, H, xt, xs, lane, u, v); break;
        case 4: up_pair<4, HT>(tile, R, row, H, xt, xs, lane, u, v); break;
        default: up_pair<2, HT>(tile, R, row, H, xt, xs, lane, u, v); break;
      }
      const long long c0 = clock64();
      u = warp_sum(u);
      v = warp_sum(v);
      const long long c1 = clock64();
      if (lane == 0) {
        // straight into the chunk-transposed activation layout of phase B
        const int r = r0 + row, c = r >> lc, m = (r & ((1 << lc) - 1)) >> 2;
        float a = u / (1.0f + expf(-u)) * v;
        if (bits == 4) a *= kInt4Prescale[r & 3];  // the INT4 / INT2 activation layouts are prescaled like x
        else if (bits == 2) a *= kInt2Prescale[r & 7];
        aj[(m * nch_a + c) * 4 + (r & 3)] = a;
      }
      if (blockIdx.x == 0 && cw == 0 && lane == 0 && k < 8) {
        g_k3_sub[k][0] = c0;
        g_k3_sub[k][1] = c1;
        g_k3_sub[k][2] = clock64();
      }
    }
    rot = (rot + nr) % kConsumers;
    __syncwarp();
    if (lane == 0) mbar_arrive(&ring.empty[stage]);
    K3_TRACE(cw + 1, k, 2);
    if (++stage == stages) stage = 0, phase ^= 1;
  }
  // ---- every CTA's activations are complete and visible
  consumer_sync();
  if (ctid == 0) {
    prof[3] = gtime();
    grid_barrier();
    prof[4] = gtime();
    // per-expert bulk copies of the activation layouts, in phase-B order
    asm volatile("fence.proxy.async.global;" ::: "memory");
    for (int j = 0; j < batch.n; ++j) {
      const uint32_t abytes = (uint32_t)(batch.e[j].I * 4);
      mbar_expect_tx(&act_bar[j], abytes);
      bulk_g2s(al + plan.lay_off[j], alay + plan.lay_off[j], abytes, &act_bar[j]);
    }
  }
  // ---- phase B: tiles in producer order; flush = last tile of a row sub-block
  const int w4 = cw & 3;  // this warp's rows are r = 4m + w4
  float acc[4] = {0.f, 0.f, 0.f, 0.f};
  bool first = true;
  int subs_left = 0;  // row sub-blocks this CTA reduces (one flush each)
  for (int blk = blockIdx.x; blk < plan.n_blk; blk += gridDim.x)
    subs_left += (min(plan.RBB, H - blk * plan.RBB) + kSubRows - 1) / kSubRows;
  while (subs_left > 0) {
    K3_TRACE(cw + 1, k, 0);
    mbar_wait(&ring.full[stage], phase);
    K3_TRACE(cw + 1, k, 1);
    const TileMeta tm = meta[stage];
    const FfnExpert &ex = batch.e[tm.j];
    mbar_wait(&act_bar[tm.j], 0);
    if (first && ctid == 0) prof[5] = gtime();
    first = false;
    const uint8_t *tile = ring_buf + (size_t)stage * kStageBytes;
    const float *al_j = al + plan.lay_off[tm.j];
    switch (ex.bits) {
      case 16: down_tile_bits<16>(tm, tile, ex, al_j, cw, lane, acc); break;
      case 8: down_tile_bits<8>(tm, tile, ex, al_j, cw, lane, acc); break;
      case 4: down_tile_bits<4>(tm, tile, ex, al_j, cw, lane, acc); break;
      default: down_tile_bits<2>(tm, tile, ex, al_j, cw, lane, acc); break;
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&ring.empty[stage]);
    K3_TRACE(cw + 1, k, 2);
    ++k;
    if (++stage == stages) stage = 0, phase ^= 1;
    if (tm.flush) {
      // fixed-order reduction: row r = 4m + w4 collects warps w4, w4 + 4, w4 + 8
#pragma unroll
      for (int m = 0; m < 4; ++m) {
        const float v = warp_sum(acc[m]);
        if (lane == 0 && 4 * m + w4 < tm.nr) part[4 * m + w4][cw >> 2] = v;
        acc[m] = 0.f;
      }
      consumer_sync();
      if (ctid < tm.nr) y[tm.r0 + ctid] = (part[ctid][0] + part[ctid][1]) + part[ctid][2];
      consumer_sync();
      --subs_left;
    }
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
size_t region_bytes(int H, int max_total_I) {
  const size_t xb = (size_t)4 * (H / 4 + H / 32) * 16;  // x layouts of the four widths (phase A)
  const size_t ab = (size_t)max_total_I * 4;             // activation layouts of every expert (phase B)
  return xb > ab ? xb : ab;
}

constexpr size_t kStaticReserve = 4096;  // static shared memory (batch, plan, barriers, partials)

int stages_for(size_t extra) {
  int s = kMaxStages;
  while (s > 2 && (size_t)s * kStageBytes + extra + kStaticReserve > (size_t)kSmemLimit) --s;
  return s;
}

}  // namespace

cudaError_t ffn_preload() {
  cudaFuncAttributes a;
  cudaError_t e = cudaFuncGetAttributes(&a, build_xlay_kernel);
  const int dyn = (int)(kSmemLimit - kStaticReserve);
  if (e == cudaSuccess) e = cudaFuncSetAttribute(ffn_kernel<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, dyn);
  if (e == cudaSuccess) e = cudaFuncSetAttribute(ffn_kernel<2048>, cudaFuncAttributeMaxDynamicSharedMemorySize, dyn);
  if (e == cudaSuccess) e = cudaFuncSetAttribute(ffn_kernel<4096>, cudaFuncAttributeMaxDynamicSharedMemorySize, dyn);
  for (const void *f : {(const void *)ffn_kernel<0>, (const void *)ffn_kernel<2048>, (const void *)ffn_kernel<4096>,
                        (const void *)build_xlay_kernel})
    if (e == cudaSuccess) e = cudaFuncSetAttribute(f, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
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
  const size_t extra = region_bytes(H, max_total_I);
  const int st = stages_for(extra);
  static const int nprod = [] {
    const char *e = getenv("FATE_K3_PRODUCERS");  // tuning knob: producer warps actually issuing (1..4)
    const int v = e ? atoi(e) : kProducers;
    return v < 1 ? 1 : v > kProducers ? kProducers : v;
  }();
  const size_t smem = (size_t)st * kStageBytes + extra;
  if (smem + kStaticReserve > (size_t)kSmemLimit) return cudaErrorInvalidConfiguration;
  // the grid barrier needs every CTA resident: one CTA per SM, grid = #SMs
  const float4 *xl = reinterpret_cast<const float4 *>(xlay);
  if (H == 2048)
    ffn_kernel<2048><<<sms, kThreads, smem, s>>>(batch_dev, xl, alay, y_dev, bytes_stat, st, nprod);
  else if (H == 4096)
    ffn_kernel<4096><<<sms, kThreads, smem, s>>>(batch_dev, xl, alay, y_dev, bytes_stat, st, nprod);
  else
    ffn_kernel<0><<<sms, kThreads, smem, s>>>(batch_dev, xl, alay, y_dev, bytes_stat, st, nprod);
  return cudaGetLastError();
}

}  // namespace fate

// Diagnostics: per-CTA phase timestamps of the last K3 launch, [160][8] ns.
extern "C" int fate_k3_profile(uint64_t *out_host) {
  if (cudaMemcpyFromSymbol(out_host + 160 * 8 + 17 * fate::kTraceTiles * 3, fate::g_k3_sub, sizeof(long long) * 32) !=
      cudaSuccess)
    return FATE_ECUDA;
  if (cudaMemcpyFromSymbol(out_host + 160 * 8, fate::g_k3_trace, sizeof(long long) * 17 * fate::kTraceTiles * 3) !=
      cudaSuccess)
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
  if (n < 1 || n > kMaxFfnExperts || H < 128 || H % 128) {
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
    if (h.magic != kMagic || h.H != H || h.I < 128 || h.I % 128) {
      set_error("fate_ffn_decode: buffer header does not describe a packed expert of this hidden size");
      return FATE_EINVAL;
    }
    b.e[j] = FfnExpert{bufs[j], weights[j], h.I, h.bits, off, 0};
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

extern "C" int fate_ffn_decode_timed(const float *x_dev, int H, int n, int nsets, const uint8_t *const *bufs,
                                     const float *weights, float *y_dev, int iters, void *stream, float *ms_out) {
  using namespace fate;
  if (n < 1 || n > kMaxFfnExperts || nsets < 1 || nsets > 64 || H < 128 || H % 128 || iters < 1 || !ms_out) {
    set_error("fate_ffn_decode_timed: bad arguments");
    return FATE_EINVAL;
  }
  cudaStream_t s = (cudaStream_t)stream;
  std::vector<FfnBatch> bs(nsets);
  int max_off = 0;
  for (int q = 0; q < nsets; ++q) {
    FfnBatch &b = bs[q];
    b = FfnBatch{};
    b.n = n;
    b.H = H;
    int off = 0;
    for (int j = 0; j < n; ++j) {
      const uint8_t *buf = bufs[q * n + j];
      ExpertHeader h;
      FATE_CUDA(cudaMemcpy(&h, buf, sizeof(h), cudaMemcpyDeviceToHost));
      if (h.magic != kMagic || h.H != H || h.I < 128 || h.I % 128) {
        set_error("fate_ffn_decode_timed: buffer header does not describe a packed expert of this hidden size");
        return FATE_EINVAL;
      }
      b.e[j] = FfnExpert{buf, weights[j], h.I, h.bits, off, 0};
      off += h.I;
    }
    b.total_I = off;
    max_off = off > max_off ? off : max_off;
  }
  FfnBatch *bd = nullptr;
  float *xl = nullptr, *al = nullptr;
  FATE_CUDA(cudaMalloc(&bd, sizeof(FfnBatch) * nsets));
  FATE_CUDA(cudaMalloc(&xl, ffn_xlay_floats(H) * sizeof(float)));
  FATE_CUDA(cudaMalloc(&al, ffn_alay_floats(max_off) * sizeof(float)));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaError_t e = cudaMemcpyAsync(bd, bs.data(), sizeof(FfnBatch) * nsets, cudaMemcpyHostToDevice, s);
  if (e == cudaSuccess) e = launch_build_xlay(x_dev, H, xl, s);
  for (int i = 0; i < nsets && e == cudaSuccess; ++i) e = launch_ffn_decode(bd + i, xl, al, y_dev, H, max_off, s);
  if (e == cudaSuccess) e = cudaEventRecord(e0, s);
  for (int i = 0; i < iters && e == cudaSuccess; ++i)
    e = launch_ffn_decode(bd + (i % nsets), xl, al, y_dev, H, max_off, s);
  if (e == cudaSuccess) e = cudaEventRecord(e1, s);
  if (e == cudaSuccess) e = cudaEventSynchronize(e1);
  float ms = 0.f;
  if (e == cudaSuccess) e = cudaEventElapsedTime(&ms, e0, e1);
  *ms_out = ms / iters;
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(bd);
  cudaFree(xl);
  cudaFree(al);
  FATE_CUDA(e);
  return FATE_OK;
}
