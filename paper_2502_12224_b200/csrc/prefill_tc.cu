// K4 on the 5th-generation tensor cores (tcgen05 + TMEM), sm_100a.
//
// Grouped expert FFN for prefill: per active expert e with token list t_e
//   up:   A_e[t, i]   = silu(X[t] . W1_e[i]) * (X[t] . W3_e[i])   (bf16 out)
//   down: Z[zrow[t], h] = A_e[t] . W2_e[h]                         (fp32 out)
// followed by the deterministic combine of prefill.cu.
//
// One persistent CTA per SM walks work items (expert, 128 weight rows, <= 128
// tokens) round-robin.  Roles:
//   warps 4..11  loaders: dequantize the packed weight rows (INT2/4/8: z + s*c
//                in fp32, quant.py:110-120, rounded to bf16; bf16 copied) and
//                convert/gather the token rows to bf16, storing both in the
//                canonical K-major no-swizzle UMMA layout (8-row x 16-byte core
//                matrices) of a 4/6-stage shared-memory ring;
//   warp 12      one elected thread issues tcgen05.mma (M = 128 weight rows,
//                N = tokens padded to 16, K = 16) into TMEM and commits each
//                stage back to the loaders and each finished accumulator to
//                the epilogue;
//   warps 0..3   epilogue: tcgen05.ld of their 32 TMEM lanes (= weight rows),
//                SwiGLU (up) or plain store (down).
// Accumulators are double-buffered in TMEM (up: W1 and W3 tiles, 2 x 2 x 128
// columns; down: 2 x 128 columns), so the epilogue of item n overlaps the MMAs
// of item n + 1.  Operands are bf16, accumulation fp32.
#include <cuda_bf16.h>

#include <mutex>

#include "fate_internal.cuh"

namespace fate {
namespace {

constexpr int BM = 128;  // weight rows per item (UMMA M)
constexpr int BK = 64;   // K per stage = one quantization group
constexpr int BN = 128;  // tokens per item (UMMA N <= 128, multiple of 16)
constexpr int kEpiWarps = 4, kLoadWarps = 8;
constexpr int kTcThreads = 32 * (kEpiWarps + kLoadWarps + 1);
constexpr int kMmaWarp = kEpiWarps + kLoadWarps;
constexpr int kUpStages = 4, kDnStages = 6;  // bf16 operand ring (UMMA layout)
constexpr int kTileBytes = BM * BK * 2;  // one 128 x 64 bf16 weight tile (16 KB)
constexpr int kXBytes = BN * BK * 2;     // one token / activation tile (16 KB)
constexpr int kUpStage = 2 * kTileBytes + kXBytes, kDnStage = kTileBytes + kXBytes;
constexpr int kMaxPrefillExperts = FATE_MAX_EXPERTS + 1;  // routed + shared

__device__ __forceinline__ uint32_t su32(const void *p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }

__device__ __forceinline__ void bar_init(uint64_t *b, uint32_t n) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(n));
}
__device__ __forceinline__ void bar_arrive(uint64_t *b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(b)) : "memory");
}
__device__ __forceinline__ void bar_wait(uint64_t *b, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "TCW_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra TCW_%=;\n}" ::"r"(su32(b)),
      "r"(parity)
      : "memory");
}

__device__ __forceinline__ void cp16(void *dst, const void *src, bool valid) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(su32(dst)), "l"(src), "r"(valid ? 16 : 0)
               : "memory");
}
__device__ __forceinline__ void cp8(void *dst, const void *src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(su32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

// Shared-memory matrix descriptor (sm_100 UMMA): start >> 4 in [0,14), leading
// byte offset >> 4 in [16,30) (distance between the two 8-column halves of a
// K = 16 slice), stride byte offset >> 4 in [32,46) (distance between 8-row
// groups), version 1 in [46,48), layout type 0 = no swizzle in [61,64).
__device__ __forceinline__ uint64_t smem_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((saddr >> 4) & 0x3FFFu) | ((uint64_t)((lbo >> 4) & 0x3FFFu) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFFu) << 32) | (1ull << 46);
}

// Instruction descriptor, kind::f16: D fp32, A and B bf16, both K-major.
__device__ __forceinline__ uint32_t idesc_bf16(int M, int N) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

__device__ __forceinline__ void umma(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t idesc, uint32_t accum) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(da), "l"(db), "r"(idesc), "r"(accum));
}

__device__ __forceinline__ void umma_commit(uint64_t *bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(bar))
               : "memory");
}

__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }

// 16 consecutive fp32 columns of this thread's TMEM lane.
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float (&v)[16]) {
  uint32_t r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}

// Byte offset of the 16-byte chunk (row, k8) of an R-row x 64-column bf16
// tile in the canonical K-major no-swizzle layout: K = 16 slices of R*32
// bytes; inside, 8-row groups of 256 bytes; inside, two 128-byte core
// matrices (columns 0-7 | 8-15) of 8 rows x 16 bytes.
__device__ __forceinline__ uint32_t chunk_off(int row, int k8, int R) {
  return (uint32_t)((k8 >> 1) * R * 32 + (row >> 3) * 256 + (k8 & 1) * 128 + (row & 7) * 16);
}

__device__ __forceinline__ uint32_t pack_bf2(float a, float b) {
  const __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<const uint32_t *>(&h);
}

// Dequantize one raw unit (16 bytes of codes of one row + that row's
// (scale, zero) for this 64-column group) into bf16 16-byte chunks of the UMMA
// layout: INT4 -> 4 chunks, INT2 -> 8 chunks, INT8 -> 2 chunks
// (quant.py:110-120: z + s*c, here in fp32, then rounded to bf16).
__device__ __forceinline__ float2 f2fma(float2 a, float2 b, float2 c) {
  unsigned long long d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;"
      : "=l"(d)
      : "l"(*reinterpret_cast<unsigned long long *>(&a)), "l"(*reinterpret_cast<unsigned long long *>(&b)),
        "l"(*reinterpret_cast<unsigned long long *>(&c)));
  return *reinterpret_cast<float2 *>(&d);
}
__device__ __forceinline__ float2 f2sub(float2 a, float2 b) {
  unsigned long long d;
  asm("sub.rn.f32x2 %0, %1, %2;"
      : "=l"(d)
      : "l"(*reinterpret_cast<unsigned long long *>(&a)), "l"(*reinterpret_cast<unsigned long long *>(&b)));
  return *reinterpret_cast<float2 *>(&d);
}
// byte K of v under the exponent of 2^23: the float 2^23 + byte, exactly
template <int K>
__device__ __forceinline__ float m23(uint32_t v) {
  return __uint_as_float(__byte_perm(v, 0x4B000000u, 0x7650 + K));
}
// two codes (as 2^23 + c) -> bf16x2 of z + s*c (quant.py:110-120 in fp32, then RN)
__device__ __forceinline__ uint32_t deq2(float a, float b, float2 s2, float2 z2) {
  const float2 c = f2sub(make_float2(a, b), make_float2(8388608.0f, 8388608.0f));
  const float2 v = f2fma(c, s2, z2);
  return pack_bf2(v.x, v.y);
}

// Dequantize one raw unit (16 bytes of codes of one row + that row's
// (scale, zero) for this 64-column group) into bf16 16-byte chunks of the UMMA
// layout: INT4 -> 4 chunks, INT2 -> 8 chunks, INT8 -> 2 chunks.  Element i of
// a byte sits at bit i*BITS (quant.py:30-39).
template <int BITS>
__device__ __forceinline__ void dequant_unit(const uint8_t *raw, uint8_t *tile, int row, int k8_0) {
  const uint4 q = *reinterpret_cast<const uint4 *>(raw);
  const float2 g = *reinterpret_cast<const float2 *>(raw + 16);
  const float2 s2 = make_float2(g.x, g.x), z2 = make_float2(g.y, g.y);
  const uint32_t w[4] = {q.x, q.y, q.z, q.w};
  if constexpr (BITS == 4) {
    // one word = one 8-element chunk: elements 2k | 2k+1 in byte k of lo | hi
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      const uint32_t lo = w[c] & 0x0F0F0F0Fu, hi = (w[c] >> 4) & 0x0F0F0F0Fu;
      *reinterpret_cast<uint4 *>(tile + chunk_off(row, k8_0 + c, BM)) =
          make_uint4(deq2(m23<0>(lo), m23<0>(hi), s2, z2), deq2(m23<1>(lo), m23<1>(hi), s2, z2),
                     deq2(m23<2>(lo), m23<2>(hi), s2, z2), deq2(m23<3>(lo), m23<3>(hi), s2, z2));
    }
  } else if constexpr (BITS == 2) {
    // one word = two chunks: element 4k + j in byte k of b_j
#pragma unroll
    for (int wi = 0; wi < 4; ++wi) {
      const uint32_t b0 = w[wi] & 0x03030303u, b1 = (w[wi] >> 2) & 0x03030303u;
      const uint32_t b2 = (w[wi] >> 4) & 0x03030303u, b3 = (w[wi] >> 6) & 0x03030303u;
      *reinterpret_cast<uint4 *>(tile + chunk_off(row, k8_0 + 2 * wi, BM)) =
          make_uint4(deq2(m23<0>(b0), m23<0>(b1), s2, z2), deq2(m23<0>(b2), m23<0>(b3), s2, z2),
                     deq2(m23<1>(b0), m23<1>(b1), s2, z2), deq2(m23<1>(b2), m23<1>(b3), s2, z2));
      *reinterpret_cast<uint4 *>(tile + chunk_off(row, k8_0 + 2 * wi + 1, BM)) =
          make_uint4(deq2(m23<2>(b0), m23<2>(b1), s2, z2), deq2(m23<2>(b2), m23<2>(b3), s2, z2),
                     deq2(m23<3>(b0), m23<3>(b1), s2, z2), deq2(m23<3>(b2), m23<3>(b3), s2, z2));
    }
  } else {
    // two words = one chunk of bytes
#pragma unroll
    for (int c = 0; c < 2; ++c) {
      const uint32_t a = w[2 * c], b = w[2 * c + 1];
      *reinterpret_cast<uint4 *>(tile + chunk_off(row, k8_0 + c, BM)) =
          make_uint4(deq2(m23<0>(a), m23<1>(a), s2, z2), deq2(m23<2>(a), m23<3>(a), s2, z2),
                     deq2(m23<0>(b), m23<1>(b), s2, z2), deq2(m23<2>(b), m23<3>(b), s2, z2));
    }
  }
}

struct Item {
  int e, tt, rt;  // expert, token tile, row tile
};

// Profiling builds only (-DFATE_PROF): CTA 0's per-stage timeline of the last
// up-projection launch: [0] loader passed the slot's empty barrier and issued,
// [1] loader's copies landed, [2] loader arrived full (dequant done), [3] MMA
// warp passed full, [4] MMA warp committed (globaltimer ns).
#ifdef FATE_PROF
__device__ unsigned long long g_k4_stage[256][5];
__device__ __forceinline__ unsigned long long k4_time() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#define K4_STAMP(k, i) \
  do { if (UP && blockIdx.x == 0 && (k) < 256) g_k4_stage[k][i] = k4_time(); } while (0)
#else
#define K4_STAMP(k, i) ((void)0)
#endif

// Items are expert-major: for e, for token tile, for row tile.
__device__ __forceinline__ Item item_of(const int *pref, const int *nrt, int n, int idx) {
  // largest e with pref[e] <= idx (binary search; pref is non-decreasing, pref[n] > idx)
  int lo = 0, hi = n - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (pref[mid] <= idx) lo = mid;
    else hi = mid - 1;
  }
  const int e = lo;
  const int local = idx - pref[e];
  return Item{e, local / nrt[e], local % nrt[e]};
}

template <bool UP>
__global__ void __launch_bounds__(kTcThreads, 1)
    k4_tc_kernel(const __nv_bfloat16 *__restrict__ Xb, int H, const PrefillExpert *__restrict__ ex_p, int n,
                 const int32_t *__restrict__ tok_idx, const int32_t *__restrict__ zrow, const int *__restrict__ a_off,
                 __nv_bfloat16 *__restrict__ A, float *__restrict__ Z) {
  constexpr int S = UP ? kUpStages : kDnStages;
  constexpr int kLook = S - 2;  // cp.async stages in flight ahead of the dequant (slot reuse waits on the MMA two stages back)
  constexpr int kStage = UP ? kUpStage : kDnStage;  // [W1 | W3 | X] or [W2 | A]
  constexpr uint32_t kAccCols = UP ? 256 : 128;                 // per accumulator buffer
  extern __shared__ __align__(1024) uint8_t smem[];  // S operand stages
  __shared__ PrefillExpert ex[kMaxPrefillExperts];
  __shared__ int pref[kMaxPrefillExperts + 1], nrt[kMaxPrefillExperts];
  __shared__ __align__(8) uint64_t full[S], empty[S], acc_full[2], acc_empty[2];
  __shared__ uint32_t tmem_base_sh;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  for (int e = tid; e < n; e += kTcThreads) {
    PrefillExpert x = ex_p[e];
    if (x.bits == 0) x.bits = reinterpret_cast<const ExpertHeader *>(x.buf)->bits;  // width that landed
    ex[e] = x;
  }
  __syncthreads();
  if (tid == 0) {
    int acc = 0;
    for (int e = 0; e < n; ++e) {
      pref[e] = acc;
      nrt[e] = (UP ? ex[e].I : H) / BM;
      acc += nrt[e] * ((ex[e].n_tok + BN - 1) / BN);
    }
    pref[n] = acc;
    for (int s = 0; s < S; ++s) {
      bar_init(&full[s], kLoadWarps);
      bar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      bar_init(&acc_full[b], 1);
      bar_init(&acc_empty[b], kEpiWarps);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == kMmaWarp) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(su32(&tmem_base_sh)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_base_sh;
  const int n_items = pref[n];

  if (warp >= kEpiWarps && warp < kMmaWarp) {
    // ================= loaders: cp.async kLook stages ahead, then dequantize
    // the stage that landed.  Thread lt owns weight row (lt % 128) of matrix
    // (lt / 128): the row's packed codes land in its own chunk slots 4.. of
    // the destination tile and its (scale, zero) pair in slot 3; the thread
    // reads them back and overwrites the row with bf16, so only its own
    // cp.async groups need to be complete.  Token / activation chunks go
    // straight to the UMMA layout (rows past the tile's tokens zero-filled).
    const int lt = tid - 32 * kEpiWarps;  // 0..255
    // cursor over this CTA's stage sequence; item fields are resolved once per item
    struct Cur {
      int it, k0, K, e, t0, ntok, npad, r0, bits;
      const __nv_bfloat16 *xrow[BN * 8 / (32 * kLoadWarps)];  // this thread's token / activation rows
    };
    auto load_item = [&](Cur &c) {
      if (c.it >= n_items) return;
      const Item w = item_of(pref, nrt, n, c.it);
      const PrefillExpert &E = ex[w.e];
      c.e = w.e;
      c.K = UP ? H : E.I;
      c.t0 = w.tt * BN;
      c.ntok = min(BN, E.n_tok - c.t0);
      c.npad = (c.ntok + 15) & ~15;
      c.r0 = w.rt * BM;
      c.bits = E.bits;
      const int64_t aoff = UP ? 0 : (int64_t)a_off[w.e];
#pragma unroll
      for (int j = 0; j < BN * 8 / (32 * kLoadWarps); ++j) {
        const int t = (lt + 32 * kLoadWarps * j) >> 3;
        const int tt = t < c.ntok ? t : 0;
        c.xrow[j] = UP ? Xb + (int64_t)tok_idx[E.tok_off + c.t0 + tt] * H
                       : A + aoff + (int64_t)(c.t0 + tt) * E.I;
      }
    };
    auto next = [&](Cur &c) {
      c.k0 += BK;
      if (c.k0 >= c.K) {
        c.k0 = 0;
        c.it += gridDim.x;
        load_item(c);
      }
    };
    auto issue = [&](const Cur &c, int sidx) {
      const PrefillExpert &E = ex[c.e];
      const int bits = c.bits;
      const Layout L = make_layout(H, E.I, bits);
      const uint8_t *p = E.buf + FATE_HEADER_BYTES;
      const int K = c.K;
      const int ntok = c.ntok, r0 = c.r0, npad = c.npad;
      uint8_t *st = smem + (size_t)(sidx % S) * kStage;
      const int mat = lt / BM, row = lt % BM;
      if (mat < (UP ? 2 : 1)) {
        const int64_t grow = r0 + row;
        const uint8_t *codes = p + (UP ? (mat ? L.c3 : L.c1) : L.c2);
        // W1 / W3 rows are row-major; W2 is slab-major (fate_internal.cuh): the K-step's
        // 64 columns of row grow are slab k0/64 (quantized) or slabs k0/8 .. +7 (bf16)
        if (bits == 16) {
#pragma unroll
          for (int k8 = 0; k8 < 8; ++k8) {
            const uint8_t *src = UP ? codes + (grow * K + c.k0 + 8 * k8) * 2
                                    : codes + ((int64_t)(c.k0 / kW2SlabBf16 + k8) * H + grow) * (kW2SlabBf16 * 2);
            cp16(st + mat * kTileBytes + chunk_off(row, k8, BM), src, true);
          }
        } else {
          const uint8_t *sz = p + (UP ? (mat ? L.s3 : L.s1) : L.s2);
          const int units = bits / 2;  // 16-byte code units per 64-column row segment
          const int64_t seg = UP ? (grow * K + c.k0) / kGroup : (int64_t)(c.k0 / kW2SlabQuant) * H + grow;
          const uint8_t *src = codes + seg * (kGroup * bits / 8);
          uint8_t *tl = st + mat * kTileBytes;
          for (int u = 0; u < units; ++u) cp16(tl + chunk_off(row, 4 + u, BM), src + 16 * u, true);
          cp8(tl + chunk_off(row, 3, BM), sz + seg * 8);
        }
      }
      uint8_t *xt = st + (UP ? 2 : 1) * kTileBytes;
#pragma unroll
      for (int j = 0; j < BN * 8 / (32 * kLoadWarps); ++j) {
        const int cc = lt + 32 * kLoadWarps * j, t = cc >> 3, k8 = cc & 7;
        if (t < npad) cp16(xt + chunk_off(t, k8, BN), c.xrow[j] + c.k0 + 8 * k8, t < ntok);
      }
    };
    auto dequant = [&](const Cur &c, int sidx) {
      const int bits = c.bits;
      const int mat = lt / BM, row = lt % BM;
      if (bits == 16 || mat >= (UP ? 2 : 1)) return;
      uint8_t *tl = smem + (size_t)(sidx % S) * kStage + mat * kTileBytes;
      // read the row's raw codes (slots 4..) and (scale, zero) (slot 3) before overwriting
      uint8_t unit[4][32];
      const uint2 g = *reinterpret_cast<const uint2 *>(tl + chunk_off(row, 3, BM));
      const int units = bits / 2;
#pragma unroll
      for (int u = 0; u < 4; ++u)
        if (u < units) {
          *reinterpret_cast<uint4 *>(unit[u]) = *reinterpret_cast<const uint4 *>(tl + chunk_off(row, 4 + u, BM));
          *reinterpret_cast<uint2 *>(unit[u] + 16) = g;
        }
      if (bits == 4) {
        dequant_unit<4>(unit[0], tl, row, 0);
        dequant_unit<4>(unit[1], tl, row, 4);
      } else if (bits == 2) {
        dequant_unit<2>(unit[0], tl, row, 0);
      } else {
#pragma unroll
        for (int u = 0; u < 4; ++u) dequant_unit<8>(unit[u], tl, row, 2 * u);
      }
    };
    Cur ic{(int)blockIdx.x, 0, 0, 0, 0, 0, 0, 0, 0};
    load_item(ic);
    Cur pc = ic;
    int si = 0;  // stages issued
    for (int d = 0; d < kLook; ++d) {
      if (ic.it < n_items) {
        bar_wait(&empty[si % S], ((si / S) & 1) ^ 1);
        issue(ic, si);
        ++si;
        next(ic);
      }
      cp_commit();
    }
    for (int sp = 0; pc.it < n_items; ++sp) {
      if (ic.it < n_items) {
        bar_wait(&empty[si % S], ((si / S) & 1) ^ 1);
        issue(ic, si);
        if (lt == 0) K4_STAMP(si, 0);
        ++si;
        next(ic);
      }
      cp_commit();
      cp_wait<kLook>();  // this thread's copies of stage sp have landed
      if (lt == 0) K4_STAMP(sp, 1);
      dequant(pc, sp);
      // generic-proxy smem writes (cp.async + dequant stores) -> async proxy (tensor core)
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncwarp();
      if (lane == 0) bar_arrive(&full[sp % S]);
      if (lt == 0) K4_STAMP(sp, 2);
      next(pc);
    }
    cp_wait<0>();
  } else if (warp == kMmaWarp) {
    // ================= MMA issuer
    int stage = 0, li = 0, ks = 0;
    uint32_t phase = 0;
    for (int it = blockIdx.x; it < n_items; it += gridDim.x, ++li) {
      const Item w = item_of(pref, nrt, n, it);
      const PrefillExpert &E = ex[w.e];
      const int K = UP ? H : E.I;
      const int ntok = min(BN, E.n_tok - w.tt * BN), npad = (ntok + 15) & ~15;
      const uint32_t idesc = idesc_bf16(BM, npad);
      const int b = li & 1;
      bar_wait(&acc_empty[b], ((li >> 1) & 1) ^ 1);
      tc_fence_after();
      const uint32_t d0 = tmem + b * kAccCols;
      for (int k0 = 0; k0 < K; k0 += BK) {
        bar_wait(&full[stage], phase);
        tc_fence_after();
        if (lane == 0) K4_STAMP(ks, 3);
        if (lane == 0) {
          const uint32_t sb = su32(smem + (size_t)stage * kStage);
          const uint32_t xb = sb + (UP ? 2 : 1) * kTileBytes;
#pragma unroll
          for (int kk = 0; kk < BK / 16; ++kk) {
            const uint64_t db = smem_desc(xb + kk * BN * 32, 128, 256);
            const uint32_t acc = (k0 | kk) != 0;
            umma(d0, smem_desc(sb + kk * BM * 32, 128, 256), db, idesc, acc);
            if (UP) umma(d0 + 128, smem_desc(sb + kTileBytes + kk * BM * 32, 128, 256), db, idesc, acc);
          }
          umma_commit(&empty[stage]);
          K4_STAMP(ks, 4);
        }
        __syncwarp();
        ++ks;
        if (++stage == S) stage = 0, phase ^= 1;
      }
      if (lane == 0) umma_commit(&acc_full[b]);
      __syncwarp();
    }
  } else {
    // ================= epilogue (warps 0..3 own TMEM lanes 32w .. 32w + 31)
    int li = 0;
    for (int it = blockIdx.x; it < n_items; it += gridDim.x, ++li) {
      const Item w = item_of(pref, nrt, n, it);
      const PrefillExpert &E = ex[w.e];
      const int t0 = w.tt * BN, ntok = min(BN, E.n_tok - t0), npad = (ntok + 15) & ~15;
      const int b = li & 1;
      bar_wait(&acc_full[b], (li >> 1) & 1);
      tc_fence_after();
      const int row = w.rt * BM + 32 * warp + lane;  // weight row (up: i, down: h)
      const uint32_t tbase = tmem + ((uint32_t)(32 * warp) << 16) + b * kAccCols;
      for (int c0 = 0; c0 < npad; c0 += 16) {
        float u[16];
        tmem_ld16(tbase + c0, u);
        if (UP) {
          float v[16];
          tmem_ld16(tbase + 128 + c0, v);
          __nv_bfloat16 *dst = A + a_off[w.e] + (int64_t)t0 * E.I + row;
#pragma unroll
          for (int j = 0; j < 16; ++j)
            if (c0 + j < ntok) dst[(int64_t)(c0 + j) * E.I] = __float2bfloat16_rn(u[j] / (1.0f + expf(-u[j])) * v[j]);
        } else {
#pragma unroll
          for (int j = 0; j < 16; ++j)
            if (c0 + j < ntok) Z[(int64_t)zrow[E.tok_off + t0 + c0 + j] * H + row] = u[j];
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) bar_arrive(&acc_empty[b]);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == kMmaWarp) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
  }
}

// per-device one-time setup (kernel attributes live in each device's context)
struct K4Dev {
  int sms = 0;
  bool configured = false;
};
std::mutex g_k4_mu;
K4Dev g_k4[64];

}  // namespace

constexpr size_t kUpSmem = (size_t)kUpStages * kUpStage;
constexpr size_t kDnSmem = (size_t)kDnStages * kDnStage;

static cudaError_t k4_device(int *sms) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  if (dev < 0 || dev >= 64) return cudaErrorInvalidDevice;
  std::lock_guard<std::mutex> lk(g_k4_mu);
  K4Dev &D = g_k4[dev];
  if (!D.configured) {
    e = cudaFuncSetAttribute(k4_tc_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kUpSmem);
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(k4_tc_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kDnSmem);
    if (e == cudaSuccess) e = cudaDeviceGetAttribute(&D.sms, cudaDevAttrMultiProcessorCount, dev);
    if (e != cudaSuccess) return e;
    D.configured = true;
  }
  *sms = D.sms;
  return cudaSuccess;
}

cudaError_t k4_tc_preload() {
  int sms = 0;
  return k4_device(&sms);
}

int k4_tc_items(int n_tok, int I, int H, bool down) { return ((n_tok + BN - 1) / BN) * ((down ? H : I) / BM); }

// A is bf16 activations [sum_e n_e * I_e] at a_off[e]; Z fp32 rows at zrow.
cudaError_t launch_k4_tc(const void *Xb_, int H, const PrefillExpert *ex_dev, int n, const int32_t *tok_idx,
                         const int32_t *zrow, const int *a_off_dev, void *A, float *Z, int items_up, int items_down,
                         cudaStream_t s) {
  int g_sms = 0;
  {
    cudaError_t e = k4_device(&g_sms);
    if (e != cudaSuccess) return e;
  }
  if (n > kMaxPrefillExperts) return cudaErrorInvalidValue;
  __nv_bfloat16 *Ab = reinterpret_cast<__nv_bfloat16 *>(A);
  const __nv_bfloat16 *Xb = reinterpret_cast<const __nv_bfloat16 *>(Xb_);
  if (items_up > 0)
    k4_tc_kernel<true><<<items_up < g_sms ? items_up : g_sms, kTcThreads, kUpSmem, s>>>(Xb, H, ex_dev, n, tok_idx, zrow,
                                                                                      a_off_dev, Ab, Z);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  if (items_down > 0)
    k4_tc_kernel<false><<<items_down < g_sms ? items_down : g_sms, kTcThreads, kDnSmem, s>>>(
        Xb, H, ex_dev, n, tok_idx, zrow, a_off_dev, Ab, Z);
  return cudaGetLastError();
}

}  // namespace fate

extern "C" int fate_k4_profile(uint64_t *out_host) {
#ifdef FATE_PROF
  if (cudaMemcpyFromSymbol(out_host, fate::g_k4_stage, sizeof(unsigned long long) * 256 * 5) != cudaSuccess) {
    fate::set_error("fate_k4_profile: copy failed");
    return FATE_ECUDA;
  }
  return FATE_OK;
#else
  (void)out_host;
  fate::set_error("fate_k4_profile: K4 stage stamps are compiled in only with FATE_PROF=1");
  return FATE_EINVAL;
#endif
}
