// K3: dequant-fused SwiGLU expert FFN for one decode token (bs = 1), sm_100a.
//
// y = sum_j w_j * W2_j (silu(W1_j x) * (W3_j x))  over the routed experts of
// the step (+ the shared expert with weight 1), reading each expert's packed
// buffer straight from HBM (cache slot or freshly landed staging slot).
//
// The op is a chain of GEMVs: pure HBM streaming.  B200 design: one
// persistent CTA per SM (cooperative launch), a TMA-bulk ring per SM and a
// split-K schedule with no mid-kernel dependency:
//  * the work is cut into UNITS = (expert j, slab s of C rows of I): the C
//    rows of W1_j and W3_j plus the matching C columns of W2_j.  The packed
//    format stores W2 slab-major (C = 64 = one quantization group for
//    INT8/4/2, C = 8 for bf16; fate_internal.cuh), so a unit's W2 part is
//    one contiguous H x C block;
//  * a CTA computes its units' activations a = w_j * silu(W1 x) * (W3 x) on
//    chip and immediately multiplies them into its own partial y[H] (shared
//    memory) with the W2 slab: every weight byte crosses HBM exactly once and
//    the W2 stream never waits for other CTAs;
//  * units are assigned statically and deterministically: quantized units
//    round-robin, bf16 units fill every CTA to the same weighted byte count;
//  * weights move global -> shared with cp.async.bulk (SASS UBLKCP) into a
//    ring of 32 KB stages completed on mbarriers; warps 0-3 produce (stage g
//    on warp g mod 4), warps 4-15 consume;
//  * one grid barrier at the very end, then CTA c sums rows of y over the
//    per-CTA partials in fixed CTA order: y is deterministic;
//  * dequant folds the affine map per group: sum_i (z + s c_i) a_i =
//    s * sum_i c_i a_i + z * sum_i a_i, codes become exact floats under the
//    2^23 magic (PRMT / one LOP3 per code) and FFMA2 does two MACs.
#include <cuda_bf16.h>

#include <cstdlib>
#include <mutex>
#include <vector>

#include "fate_internal.cuh"

namespace fate {
namespace {

constexpr int kConsumers = 12;  // consumer warps
constexpr int kProducers = 4;   // producer warps (stage g -> warp g % kProducers);
                                // 16 warps -> 128 registers per thread (allocation in 4-warp units)
constexpr int kThreads = 32 * (kProducers + kConsumers);
constexpr int kStageBytes = 32 * 1024;
constexpr int kMaxStages = 6;
constexpr int kSmemLimit = 227 * 1024;
constexpr int kRowsPerIter = 8 * kConsumers;    // quantized W2 rows per consumer sweep: 4 lanes per row
constexpr int kRowsPerIterBf = 32 * kConsumers; // bf16 W2 rows per consumer sweep: one lane per row

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

// ----------------------------------------------------------------- units
// Unit (j, s): rows [s*C, s*C + C) of W1_j / W3_j and slab s of W2_j.
// A-piece: rows [r0, r0+nr) of the unit; smem [W1 codes nr*rb][W3 codes nr*rb]
//          [W1 sz nr*szb][W3 sz nr*szb] (the layout up_pair reads).
// W-piece: slab rows [h0, h0+nh); smem [codes nh*wrb][sz nh*8].
struct ExpertPlan {
  int C, units;         // slab width, units
  int npa, ra;          // A-pieces per unit, rows per A-piece (last one may be shorter)
  int npw, rw;          // W-pieces per unit, rows per W-piece
  float cost;           // weighted bytes of one unit (balancing only)
};

constexpr int kMaxQList = 32;

struct Plan {
  ExpertPlan ep[kMaxFfnExperts];
  int nq, ns;           // quantized units (round-robin), bf16 units (filled)
  int q_first;          // this CTA's quantized units: q_first, q_first + G, ...
  int nq_mine;
  int s_lo, s_hi;       // this CTA's bf16 units [s_lo, s_hi)
  int nq_open;          // of those quantized units, the ones whose expert is complete at launch
  int qreord;           // qlist holds the order (arrival-gated experts last); 0: identity
  uint8_t qlist[kMaxQList];  // position -> m (this CTA's m-th quantized unit)
};

struct TileMeta {
  int kind;   // 0: A-piece, 1: W-piece, 2: end
  int j, s;   // expert, slab
  int r0, nr; // A: rows within the unit; W: first slab row, rows
  int flag;   // A: last A-piece of its unit (warps then arrive on the unit's activation barrier);
              // W: first W-piece of its unit (warps wait on it)
  int ub;     // activation buffer of the unit (units rotate over kActBufs)
  int par;    // parity of that buffer's barrier for this unit
};

// W-pieces of unit k are streamed after the A-pieces of unit k+1, so a warp
// never waits for the others' activation rows of the unit it is about to
// multiply; four activation buffers keep every unit in flight distinct.
constexpr int kActBufs = 4;

__host__ __device__ __forceinline__ int slab_cols(int bits) { return bits == 16 ? kW2SlabBf16 : kW2SlabQuant; }
__host__ __device__ __forceinline__ int w2_row_bytes(int bits) { return slab_cols(bits) * bits / 8; }
__host__ __device__ __forceinline__ int w2_sz_bytes(int bits) { return bits == 16 ? 0 : 8; }

// relative consumer cost per byte (quantized codes cost ALU work; bf16 streams)
// Relative CTA time per byte.  bf16 units stream at the SM's share of HBM
// (~44 GB/s); quantized units are bound by the consumers' dequant arithmetic
// (measured in the K3 stage timeline: an INT2 unit of 144 KB ~10 us, an INT4
// unit of 240 KB ~11 us), so they count ~3x / ~2.2x per byte.
__device__ __forceinline__ float cost_per_byte(int bits) {
  return bits == 16 ? 1.0f : bits == 8 ? 1.6f : bits == 4 ? 2.2f : 3.0f;
}

__device__ void expert_plan(const FfnExpert &e, int H, ExpertPlan &p) {
  const int bits = e.bits, C = slab_cols(bits);
  const int rb = H * bits / 8, szb = bits == 16 ? 0 : H / 8;
  int rmax = kStageBytes / (2 * (rb + szb));
  rmax = rmax < 1 ? 1 : rmax;
  p.C = C;
  p.units = e.I / C;
  p.npa = (C + rmax - 1) / rmax;
  p.ra = (C + p.npa - 1) / p.npa;
  // W-pieces of whole 96-row blocks (w2_blocks: the whole of H when one stage holds it)
  const int rows = kStageBytes / (w2_row_bytes(bits) + w2_sz_bytes(bits));
  const int per = bits == 16 ? kRowsPerIterBf : kRowsPerIter;
  p.rw = rows >= H ? H : rows / per * per;
  p.npw = (H + p.rw - 1) / p.rw;
  const float bytes = 2.0f * C * (rb + szb) + (float)H * (w2_row_bytes(bits) + w2_sz_bytes(bits));
  p.cost = bytes * cost_per_byte(bits);
}

// (expert, slab) of the i-th unit of a class (quantized or bf16), expert-major
__device__ __forceinline__ void unit_of(const FfnBatch &b, const Plan &p, bool quant, int i, int &j, int &s) {
  for (j = 0; j < b.n; ++j) {
    if ((b.e[j].bits != 16) != quant) continue;
    if (i < p.ep[j].units) break;
    i -= p.ep[j].units;
  }
  s = i;
}

// Start of CTA c's bf16 range in weighted bytes: CTAs c < r carry q+1
// quantized units (round-robin), the others q; each then takes bf16 work up to
// the common target.  One expression with explicit roundings, evaluated the same
// way by every CTA, so neighbouring ranges meet exactly.
__device__ __noinline__ float share_prefix(int c, int r, float sA, float sB) {
  return c < r ? __fmul_rn((float)c, sA) : __fadd_rn(__fmul_rn((float)r, sA), __fmul_rn((float)(c - r), sB));
}

// Warp 0: the assignment in O(1) per CTA (every CTA derives the same one).
// Quantized units go round-robin; bf16 units fill every CTA to the same
// weighted byte count (quantized unit cost = the batch's average).
__device__ __forceinline__ bool gated(const FfnExpert &e, bool gate) { return gate && e.slot >= 0; }

__device__ void make_plan(const FfnBatch &b, Plan &p, int G, int c, int lane) {
  if (lane < b.n) expert_plan(b.e[lane], b.H, p.ep[lane]);
  __syncwarp();
  if (lane == 0) {
    int nq = 0, ns = 0;
    float cq = 0.f, cs = 0.f;
    for (int j = 0; j < b.n; ++j) {
      if (b.e[j].bits != 16) nq += p.ep[j].units, cq += p.ep[j].units * p.ep[j].cost;
      else ns += p.ep[j].units, cs = p.ep[j].cost;
    }
    const float avg = nq ? cq / nq : 0.f;
    const int q = nq / G, r = nq % G;
    const float target = (cq + cs * ns) / G;
    const float sA = fmaxf(0.f, target - (q + 1) * avg), sB = fmaxf(0.f, target - q * avg);
    const float all = share_prefix(G, r, sA, sB);
    const float scale = all > 0.f ? (float)ns / all : 0.f;
    p.nq = nq;
    p.ns = ns;
    p.q_first = c;
    p.nq_mine = q + (c < r ? 1 : 0);
    p.s_lo = c == 0 ? 0 : min(ns, (int)rintf(__fmul_rn(share_prefix(c, r, sA, sB), scale)));
    p.s_hi = c == G - 1 ? ns : min(ns, (int)rintf(__fmul_rn(share_prefix(c + 1, r, sA, sB), scale)));
    if (p.s_hi < p.s_lo) p.s_hi = p.s_lo;
    // experts whose buffer is filled during this step go last in the CTA's
    // sequence, so the units that can run at once are not queued behind a copy
    // (arrival-gated mode).  The order depends on the schedule only, never on
    // which copies happen to be in flight, and is the same in both protocols:
    // y's summation order, hence every bit of y, is timing independent.
    p.nq_open = p.nq_mine;
    p.qreord = 0;
    bool any = false;
    for (int j = 0; j < b.n; ++j) any = any || (b.e[j].late && b.e[j].bits != 16);
    if (any && p.nq_mine <= kMaxQList) {
      int no = 0, n = 0;
      for (int pass = 0; pass < 2; ++pass)
        for (int m = 0; m < p.nq_mine; ++m) {
          int j, s;
          unit_of(b, p, true, c + m * G, j, s);
          if ((b.e[j].late != 0) == (pass == 1)) p.qlist[n++] = (uint8_t)m;
          if (pass == 0) no = n;
        }
      p.nq_open = no;
      p.qreord = no < p.nq_mine;
    }
  }
  __syncwarp();
}

// The k-th unit of this CTA's sequence: quantized and bf16 units interleaved
// evenly (compute-heavy and streaming units overlap in the ring).
// Arrival-gated quantized units follow all the others.
__device__ __forceinline__ void my_unit(const FfnBatch &b, const Plan &p, int G, int k, int &j, int &s) {
  const int nq = p.nq_open, ns = p.s_hi - p.s_lo, m = nq + ns;
  auto quant = [&](int pos) { unit_of(b, p, true, p.q_first + (p.qreord ? p.qlist[pos] : pos) * G, j, s); };
  if (k >= m) {
    quant(k - ns);
    return;
  }
  // quantized unit number floor((k+1)*nq/m) - 1 sits at position k iff the count steps
  const int before = (int)((long long)k * nq / m), after = (int)((long long)(k + 1) * nq / m);
  if (after > before) quant(before);
  else unit_of(b, p, false, p.s_lo + (k - before), j, s);
}

// Arrival gate (producer warps): the copy filling expert j's buffer has landed
// (the copy stream writes landed[slot] = generation behind it).  The host's
// watchdog releases a stuck wait through the abort word.
__device__ __forceinline__ unsigned long long gclock() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// waited: this warp's total wait so far (ns), published as a running maximum
__device__ __forceinline__ void wait_landed(const FfnExpert &e, const uint32_t *landed, const volatile uint32_t *abort,
                                            int lane, unsigned long long &waited, FfnStats *stat) {
  if (lane == 0) {
    uint32_t v;
    unsigned long long t0 = 0;
    for (unsigned n = 1;; ++n) {
      asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(landed + e.slot) : "memory");
      if ((int)(v - e.want) >= 0) break;
      if (n == 1) t0 = gclock();
      if ((n & 1023u) == 0 && abort && *abort == 0x7FFFFFFFu) break;
      // back off: hundreds of pollers on one L2 line slow the copies landing in that slice
      __nanosleep(256);
    }
    if (t0) {
      const unsigned long long t1 = gclock();
      waited += t1 - t0;
      if (stat) {
        atomicMax(&stat->wait_cur, waited);
        atomicMax(&stat->open_max, t1);
      }
    }
    // the bulk copies that follow read the buffer through the async proxy
    asm volatile("fence.proxy.async.global;" ::: "memory");
  }
  __syncwarp();
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

// W-pieces cover whole 96-row blocks (12 consumer warps x 8 row quads),
// B blocks per piece (compile time per format and H); a piece's last block may
// be partial.  Row h0 + 96 b + 8 cw + rq belongs to warp cw, lanes 4 rq .. +3.
template <int BITS, int HT>
__host__ __device__ constexpr int w2_blocks() {
  constexpr int rows = kStageBytes / (BITS == 16 ? kW2SlabBf16 * 2 : kW2SlabQuant * BITS / 8 + 8);
  constexpr int per = BITS == 16 ? kRowsPerIterBf : kRowsPerIter;
  // expert_plan: a piece is the whole of H when one stage holds it (bf16 slabs at
  // H = 2048), else floor(rows / per) whole blocks; HT = 0 (any H): enough for both
  if constexpr (HT == 0) return (rows + per - 1) / per;
  else return rows >= HT ? (HT + per - 1) / per : rows / per;
}

// One W-piece: slab rows [h0, h0+nh) of W2_j against the unit's activations
// aj[C] (w_j folded in).  Each lane first forms its columns' share of its B
// rows in registers (a lane covers 16 columns of a quantized slab, its 16
// activations in registers, or 2 of a bf16 slab), then the four lanes of a row
// are summed in a fixed order and added to the CTA's partial y (one owner per
// row, pieces in stage order: deterministic).  Out-of-range rows of the last
// block read row 0 and are masked by a select, so the loop has no branches.
template <int BITS, int B>
__device__ __forceinline__ void w2_piece(const uint8_t *__restrict__ tile, int h0, int nh,
                                         const float *__restrict__ aj, int cw, int lane, float *__restrict__ ysm) {
  if constexpr (BITS == 16) {
    // bf16 slab rows are 16 bytes: one lane per row (row h0 + 384 b + 32 cw + lane)
    // with the unit's 8 activations in registers; its own accumulator row set
    const float4 av0 = reinterpret_cast<const float4 *>(aj)[0], av1 = reinterpret_cast<const float4 *>(aj)[1];
    float r[B];
#pragma unroll
    for (int b = 0; b < B; ++b) {
      const int hr = kRowsPerIterBf * b + 32 * cw + lane;
      const bool ok = hr < nh;
      const uint4 w = *reinterpret_cast<const uint4 *>(tile + (ok ? hr : 0) * 16);
      float2 p0 = bf_dot(w.x, make_float2(av0.x, av0.y), make_float2(0.f, 0.f));
      float2 p1 = bf_dot(w.y, make_float2(av0.z, av0.w), make_float2(0.f, 0.f));
      p0 = bf_dot(w.z, make_float2(av1.x, av1.y), p0);
      p1 = bf_dot(w.w, make_float2(av1.z, av1.w), p1);
      r[b] = ok ? (p0.x + p0.y) + (p1.x + p1.y) : 0.f;
    }
#pragma unroll
    for (int b = 0; b < B; ++b) {
      const int hr = kRowsPerIterBf * b + 32 * cw + lane;
      if (hr < nh) ysm[h0 + hr] += r[b];
    }
  } else {
  const int rq = lane >> 2, sub = lane & 3;
  const int own = 8 * cw + rq;
  float r[B];
  {
    constexpr int wrb = kW2SlabQuant * BITS / 8;  // 16 / 32 / 64 bytes per slab row
    constexpr int wpl = wrb / 16;                 // 32-bit code words per lane (1, 2, 4)
    // the lane's 16 activations, prescaled for in-place code extraction (exact powers of two)
    float4 xa[4];
    float asum = 0.f;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      float4 v = reinterpret_cast<const float4 *>(aj + 16 * sub)[q];
      asum += (v.x + v.y) + (v.z + v.w);
      if constexpr (BITS == 4) {
        v.y *= 0.0625f, v.z *= 0.00390625f, v.w *= 0.000244140625f;
      } else if constexpr (BITS == 2) {
        const float bb = (q & 1) ? 0.00390625f : 1.0f;
        v.x *= bb, v.y *= bb * 0.25f, v.z *= bb * 0.0625f, v.w *= bb * 0.015625f;
      }
      xa[q] = v;
    }
    asum += __shfl_xor_sync(0xffffffffu, asum, 1);
    asum += __shfl_xor_sync(0xffffffffu, asum, 2);
    const float zsum = sub == 0 ? asum : 0.f;  // the zero-point term once per row
    const float2 *sz = reinterpret_cast<const float2 *>(tile + nh * wrb);
#pragma unroll
    for (int b = 0; b < B; ++b) {
      const int hr = kRowsPerIter * b + own;
      const bool ok = hr < nh;
      const int hs = ok ? hr : 0;
      const uint8_t *src = tile + hs * wrb + sub * (wrb / 4);
      float2 p0 = make_float2(0.f, 0.f), p1 = p0;
      if constexpr (wpl == 1) {
        word_dot<BITS>(*reinterpret_cast<const uint32_t *>(src), xa, p0, p1);
      } else if constexpr (wpl == 2) {
        const uint2 w = *reinterpret_cast<const uint2 *>(src);
        const float4 x0[4] = {xa[0], xa[1], xa[0], xa[1]}, x1[4] = {xa[2], xa[3], xa[2], xa[3]};
        word_dot<BITS>(w.x, x0, p0, p1);
        word_dot<BITS>(w.y, x1, p0, p1);
      } else {
        const uint4 w = *reinterpret_cast<const uint4 *>(src);
        const float4 x0[4] = {xa[0], xa[0], xa[0], xa[0]}, x1[4] = {xa[1], xa[1], xa[1], xa[1]};
        const float4 x2[4] = {xa[2], xa[2], xa[2], xa[2]}, x3[4] = {xa[3], xa[3], xa[3], xa[3]};
        word_dot<BITS>(w.x, x0, p0, p1);
        word_dot<BITS>(w.y, x1, p0, p1);
        word_dot<BITS>(w.z, x2, p0, p1);
        word_dot<BITS>(w.w, x3, p0, p1);
      }
      const float2 z = sz[hs];
      r[b] = ok ? fmaf(z.x, (p0.x + p0.y) + (p1.x + p1.y), z.y * zsum) : 0.f;
    }
  }
#pragma unroll
  for (int b = 0; b < B; ++b) {
    r[b] += __shfl_xor_sync(0xffffffffu, r[b], 1);
    r[b] += __shfl_xor_sync(0xffffffffu, r[b], 2);
  }
  if (sub == 0) {
#pragma unroll
    for (int b = 0; b < B; ++b) {
      const int hr = kRowsPerIter * b + own;
      if (hr < nh) ysm[h0 + hr] += r[b];
    }
  }
  }
}

// Co-residency is guaranteed by the cooperative launch (grid = #SMs, one CTA
// per SM).  The counter belongs to the caller's scratch (one per engine) and is
// never reset: each launch waits for the next multiple of gridDim.x.
__device__ __forceinline__ void grid_barrier(unsigned int *ctr) {
  __threadfence();
  const unsigned int old = atomicAdd(ctr, 1u);
  const unsigned int target = (old / gridDim.x + 1u) * gridDim.x;
  unsigned int v;
  do {
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(ctr) : "memory");
  } while ((int)(v - target) < 0);
}

constexpr int kMaxGrid = 192;

// Profiling builds only (-DFATE_PROF): per-CTA phase stamps (globaltimer ns) of
// the last launch and CTA 0's per-stage consumer timeline (warp 4, lane 0).
#ifdef FATE_PROF
__device__ unsigned long long g_k3_prof[kMaxGrid][8];
__device__ unsigned long long g_k3_stage[256][4];
__device__ __forceinline__ unsigned long long gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#define K3_PROF(i) (g_k3_prof[blockIdx.x][i] = gtime())
#define K3_STAGE(k, i, v) \
  do { if (blockIdx.x == 0 && ctid == 0 && (k) < 256) g_k3_stage[k][i] = (v); } while (0)
#else
#define K3_PROF(i) ((void)0)
#define K3_STAGE(k, i, v) ((void)0)
#endif

template <int HT>
__global__ void __launch_bounds__(kThreads, 1) ffn_kernel(const FfnBatch *__restrict__ batch_p,
                                                          const float4 *__restrict__ xlay, float *__restrict__ part,
                                                          unsigned int *__restrict__ bar, float *__restrict__ y,
                                                          FfnStats *stat, const uint32_t *__restrict__ landed,
                                                          const volatile uint32_t *abort, int stages) {
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ FfnBatch batch;
  __shared__ Plan plan;
  __shared__ Ring ring;
  __shared__ TileMeta meta[kMaxStages];
  __shared__ __align__(8) uint64_t x_bar, act_bar[kActBufs];
  __shared__ __align__(16) float a_sm[kActBufs][kW2SlabQuant];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int G = gridDim.x;
  if (warp == 0) {
    // warp 0: batch copy with 16-byte loads, the plan, the barriers
    const int4 *src = reinterpret_cast<const int4 *>(batch_p);
    int4 *dst = reinterpret_cast<int4 *>(&batch);
    for (int i = lane; i < (int)(sizeof(FfnBatch) / 16); i += 32) dst[i] = __ldg(src + i);
    __syncwarp();
    if (lane < batch.n && batch.e[lane].bits == 0)
      batch.e[lane].bits = reinterpret_cast<const ExpertHeader *>(batch.e[lane].buf)->bits;
    __syncwarp();
    if (lane == 0) {
      for (int s = 0; s < stages; ++s) {
        mbar_init(&ring.full[s], 1);
        mbar_init(&ring.empty[s], kConsumers);
      }
      mbar_init(&x_bar, 1);
      for (int b = 0; b < kActBufs; ++b) mbar_init(&act_bar[b], kConsumers);
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (lane == 0) K3_PROF(0);
#ifdef FATE_PROF
    if (blockIdx.x == 0 && lane == 0 && stat && stat->k1_post_ns) {
      const unsigned long long t = gclock();
      if (t > stat->k1_post_ns) stat->k1k3_ns += t - stat->k1_post_ns, stat->k1k3_n += 1;
      stat->k1_post_ns = 0;
    }
#endif
    make_plan(batch, plan, G, blockIdx.x, lane);
    if (lane == 0) K3_PROF(1);
  }
  __syncthreads();
  const int H = HT ? HT : batch.H;
  const int lay_stride = H / 4 + H / 32;
  uint8_t *ring_buf = smem;
  float4 *xl = reinterpret_cast<float4 *>(smem + (size_t)stages * kStageBytes);  // x layouts of the four widths
  float *ysm = reinterpret_cast<float *>(xl + 4 * lay_stride);                  // partial y[H], quantized W2 rows
  float *ysb = ysm + H;                                                          // partial y[H], bf16 W2 rows
  const int n_units = plan.nq_mine + (plan.s_hi - plan.s_lo);
  if (warp < kProducers) {
    // ================= producers: stage g of the sequence (A- and W-pieces of
    // every unit, then the end marker) belongs to producer g % kProducers, so
    // the issue latency of the bulk copies overlaps across warps.  The ring has
    // more stages than producers, so an empty-barrier parity never aliases.
    const int pw = warp;
    if (pw == 0 && lane == 0) {
      const uint32_t xbytes = (uint32_t)(4 * lay_stride * 16);
      mbar_expect_tx(&x_bar, xbytes);
      bulk_g2s(xl, xlay, xbytes, &x_bar);
      if (blockIdx.x == 0 && stat) {
        unsigned long long bytes = 0;
        for (int j = 0; j < batch.n; ++j) bytes += make_layout(H, batch.e[j].I, batch.e[j].bits).payload;
        atomicAdd(&stat->bytes, bytes);
      }
    }
    const int np = kProducers < stages - 1 ? kProducers : stages - 1;
    if (pw >= np) return;
    int st_ = 0, own_ = 0;  // stage of the next tile, its producer (tile index mod np)
    uint32_t ph_ = 0;
    auto begin = [&](int &stage, uint32_t &phase) -> bool {
      stage = st_;
      phase = ph_;
      const bool mine = own_ == pw;
      if (++st_ == stages) st_ = 0, ph_ ^= 1u;
      if (++own_ == np) own_ = 0;
      if (mine) mbar_wait(&ring.empty[stage], phase ^ 1);
      return mine;
    };
    // stage sequence: A(0) A(1) W(0) A(2) W(1) ... A(m-1) W(m-2) W(m-1)
    auto issue_w = [&](int k, int j, int s) {
      const FfnExpert &ex = batch.e[j];
      const ExpertPlan &ep = plan.ep[j];
      const int bits = ex.bits;
      const Layout Lo = make_layout(H, ex.I, bits);
      const uint8_t *p = ex.buf + FATE_HEADER_BYTES;
      const uint32_t wrb = (uint32_t)w2_row_bytes(bits), wsz = (uint32_t)w2_sz_bytes(bits);
      for (int w = 0; w < ep.npw; ++w) {
        int stage;
        uint32_t phase;
        if (!begin(stage, phase)) continue;
        const int h0 = w * ep.rw, nh = min(ep.rw, H - h0);
        const int64_t row = (int64_t)s * H + h0;
        uint8_t *dst = ring_buf + (size_t)stage * kStageBytes;
        if (lane == 0) {
          meta[stage] = TileMeta{1, j, s, h0, nh, w == 0, k % kActBufs, (k / kActBufs) & 1};
          mbar_expect_tx(&ring.full[stage], (uint32_t)nh * (wrb + wsz));
          bulk_g2s(dst, p + Lo.c2 + row * wrb, nh * wrb, &ring.full[stage]);
        }
        if (lane == 1 && wsz) bulk_g2s(dst + nh * wrb, p + Lo.s2 + row * wsz, nh * wsz, &ring.full[stage]);
      }
    };
    int pj = -1, ps = 0;
    uint32_t open = 0;  // experts known landed (arrival-gated mode)
    unsigned long long waited = 0;
    for (int k = 0; k < n_units; ++k) {
      int j, s;
      my_unit(batch, plan, G, k, j, s);
      const FfnExpert &ex = batch.e[j];
      if (gated(ex, landed != nullptr) && !((open >> j) & 1u)) {
        // finish the previous unit before possibly waiting (its W-pieces would
        // otherwise sit behind this unit's A-pieces), then wait for the copy
        if (pj >= 0) issue_w(k - 1, pj, ps);
        pj = -1;
        wait_landed(ex, landed, abort, lane, waited, stat);
        open |= 1u << j;
      }
      const ExpertPlan &ep = plan.ep[j];
      const int bits = ex.bits;
      const Layout Lo = make_layout(H, ex.I, bits);
      const uint8_t *p = ex.buf + FATE_HEADER_BYTES;
      const uint32_t rb = (uint32_t)H * bits / 8, szb = bits == 16 ? 0u : (uint32_t)H / 8;
      for (int a = 0; a < ep.npa; ++a) {
        int stage;
        uint32_t phase;
        if (!begin(stage, phase)) continue;
        const int r0 = a * ep.ra, nr = min(ep.ra, ep.C - r0);
        const int64_t row = (int64_t)s * ep.C + r0;
        uint8_t *dst = ring_buf + (size_t)stage * kStageBytes;
        if (lane == 0) {
          meta[stage] = TileMeta{0, j, s, r0, nr, a == ep.npa - 1, k % kActBufs, (k / kActBufs) & 1};
          mbar_expect_tx(&ring.full[stage], 2u * nr * (rb + szb));
        }
        __syncwarp();
        if (lane < (szb ? 4 : 2)) {
          // lanes 0..3: W1 codes, W3 codes, W1 (scale, zero), W3 (scale, zero)
          const int64_t src = lane == 0 ? Lo.c1 + row * rb : lane == 1 ? Lo.c3 + row * rb
                            : lane == 2 ? Lo.s1 + row * szb : Lo.s3 + row * szb;
          const uint32_t off = lane == 0 ? 0u : lane == 1 ? nr * rb : lane == 2 ? 2 * nr * rb : 2 * nr * rb + nr * szb;
          bulk_g2s(dst + off, p + src, lane < 2 ? nr * rb : nr * szb, &ring.full[stage]);
        }
      }
      if (pj >= 0) issue_w(k - 1, pj, ps);
      pj = j, ps = s;
    }
    if (pj >= 0) issue_w(n_units - 1, pj, ps);
    {  // end marker
      int stage;
      uint32_t phase;
      if (begin(stage, phase) && lane == 0) {
        meta[stage].kind = 2;
        mbar_arrive(&ring.full[stage]);
      }
    }
    return;
  }
  // ================= consumers
  const int ctid = tid - 32 * kProducers, cw = warp - kProducers;
  // this CTA's partial y, one array per row-ownership pattern (quantized slabs: 4 lanes
  // per row; bf16 slabs: one lane per row), so every row of each has a single writer
  for (int i = ctid; i < 2 * H; i += 32 * kConsumers) ysm[i] = 0.f;
  mbar_wait(&x_bar, 0);  // x layouts landed
  if (ctid == 0) K3_PROF(2);
  int stage = 0, rot = 0;
  uint32_t phase = 0;
#ifdef FATE_PROF
  int kk = 0;
#endif
  for (;;) {
#ifdef FATE_PROF
    K3_STAGE(kk, 0, gtime());
#endif
    mbar_wait(&ring.full[stage], phase);
    const TileMeta tm = meta[stage];
#ifdef FATE_PROF
    K3_STAGE(kk, 1, gtime());
    K3_STAGE(kk, 3, (unsigned long long)(tm.kind * 1000000 + tm.j * 10000 + tm.nr));
#endif
    if (tm.kind == 2) break;
    const uint8_t *tile = ring_buf + (size_t)stage * kStageBytes;
    const FfnExpert &ex = batch.e[tm.j];
    const int bits = ex.bits;
    if (tm.kind == 0) {
      // A-piece: consumer warp w takes the piece's rows whose running index is w mod 12
      const int sl = bits == 16 ? 0 : bits == 8 ? 1 : bits == 4 ? 2 : 3;
      const float4 *xt = xl + sl * lay_stride;
      const float *xs = reinterpret_cast<const float *>(xl + sl * lay_stride + H / 4);
      float *aj = a_sm[tm.ub];
      int row = cw - rot;
      if (row < 0) row += kConsumers;
      for (; row < tm.nr; row += kConsumers) {
        float u, v;
        switch (bits) {
          case 16: up_pair<16, HT>(tile, tm.nr, row, H, xt, xs, lane, u, v); break;
          case 8: up_pair<8, HT>(tile, tm.nr, row, H, xt, xs, lane, u, v); break;
          case 4: up_pair<4, HT>(tile, tm.nr, row, H, xt, xs, lane, u, v); break;
          default: up_pair<2, HT>(tile, tm.nr, row, H, xt, xs, lane, u, v); break;
        }
        u = warp_sum(u);
        v = warp_sum(v);
        if (lane == 0) aj[tm.r0 + row] = ex.weight * (u / (1.0f + expf(-u)) * v);
      }
      rot = (rot + tm.nr) % kConsumers;
      __syncwarp();
      if (tm.flag && lane == 0) mbar_arrive(&act_bar[tm.ub]);  // this warp's rows of the unit are written
    } else {
      // W-piece: the unit's activations are complete once every consumer warp arrived
      if (tm.flag) mbar_wait(&act_bar[tm.ub], (uint32_t)tm.par);
      const float *aj = a_sm[tm.ub];
      switch (bits) {
        case 16: w2_piece<16, w2_blocks<16, HT>()>(tile, tm.r0, tm.nr, aj, cw, lane, ysb); break;
        case 8: w2_piece<8, w2_blocks<8, HT>()>(tile, tm.r0, tm.nr, aj, cw, lane, ysm); break;
        case 4: w2_piece<4, w2_blocks<4, HT>()>(tile, tm.r0, tm.nr, aj, cw, lane, ysm); break;
        default: w2_piece<2, w2_blocks<2, HT>()>(tile, tm.r0, tm.nr, aj, cw, lane, ysm); break;
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&ring.empty[stage]);
#ifdef FATE_PROF
    K3_STAGE(kk, 2, gtime());
    ++kk;
#endif
    if (++stage == stages) stage = 0, phase ^= 1;
  }
  // ---- partial y of this CTA -> global (the four lanes of a row summed in a
  // fixed order); one grid barrier; CTA c sums its rows over the CTAs in order
  if (ctid == 0) K3_PROF(3);
  consumer_sync();
  float *mine = part + (size_t)blockIdx.x * H;
  for (int i = ctid; i < H; i += 32 * kConsumers) mine[i] = ysm[i] + ysb[i];
  consumer_sync();
  if (ctid == 0) {
    K3_PROF(4);
    if (batch.pf_bytes) {
      // this CTA's share of the L2 prefetch (the next step's router rows), issued
      // while the grid gathers at the barrier
      const unsigned long long per = (batch.pf_bytes / G + 15ull) & ~15ull;
      const unsigned long long off = per * blockIdx.x;
      if (off < batch.pf_bytes) {
        const unsigned long long n = batch.pf_bytes - off < per ? batch.pf_bytes - off : per;
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(
                         reinterpret_cast<const uint8_t *>(batch.pf_ptr) + off), "r"((uint32_t)n) : "memory");
      }
    }
    grid_barrier(bar);
    K3_PROF(5);
    // every producer's waits preceded stages its CTA consumed before the barrier
    if (blockIdx.x == 0 && stat && landed) {
      stat->wait_ns += *(volatile unsigned long long *)&stat->wait_cur;
      stat->wait_cur = 0;
    }
  }
  consumer_sync();
  // rows [r0, r0 + nrow) of y: thread (g, r) sums the CTAs c = g, g + ng, ... of row r,
  // then the ng group sums are added in order (one global round trip)
  const int RB = (H + G - 1) / G, r0 = blockIdx.x * RB, nrow = max(0, min(H, r0 + RB) - r0);
  float *red = reinterpret_cast<float *>(ring_buf);  // the ring is idle now
  if (nrow > 0) {
    const int ng = (32 * kConsumers) / nrow;
    const int g = ctid / nrow, r = ctid % nrow;
    if (g < ng) {
      constexpr int kPer = 8;
      float acc = 0.f;
      for (int c0 = g; c0 < G; c0 += kPer * ng) {
        float v[kPer];
#pragma unroll
        for (int m = 0; m < kPer; ++m) {
          const int c = c0 + m * ng;
          v[m] = c < G ? __ldcg(part + (size_t)c * H + r0 + r) : 0.f;
        }
#pragma unroll
        for (int m = 0; m < kPer; ++m) acc += v[m];
      }
      red[g * nrow + r] = acc;
    }
    consumer_sync();
    if (ctid < nrow) {
      float acc = 0.f;
      for (int gg = 0; gg < ng; ++gg) acc += red[gg * nrow + ctid];
      y[r0 + ctid] = acc;
    }
  }
  if (ctid == 0) K3_PROF(6);
#ifdef FATE_PROF
  if (ctid == 0 && stat) atomicMax(&stat->end_max_ns, gclock());
#endif
  if (blockIdx.x == 0 && ctid == 0 && stat) {
    // CTA 0's rows are its last work; the other CTAs finish theirs within ~1 us
    const unsigned long long t = gclock(), o = *(volatile unsigned long long *)&stat->open_max;
    if (landed && o) {
      stat->tail_ns += t - o;
      stat->tail_n += 1;
      stat->open_max = 0;
    }
    stat->end_ns = t;
  }
}

struct DevInfo {
  int sms = 0;
  bool configured = false;
};
std::mutex g_dev_mu;
DevInfo g_dev[64];

cudaError_t configure_device(int dev) {
  cudaError_t e = cudaSuccess;
  const int dyn = (int)(kSmemLimit - 8192);
  for (const void *f : {(const void *)ffn_kernel<0>, (const void *)ffn_kernel<2048>, (const void *)ffn_kernel<4096>}) {
    if (e == cudaSuccess) e = cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, dyn);
    if (e == cudaSuccess) e = cudaFuncSetAttribute(f, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
  }
  cudaFuncAttributes a;
  if (e == cudaSuccess) e = cudaFuncGetAttributes(&a, build_xlay_kernel);
  if (e == cudaSuccess) e = cudaFuncSetAttribute(build_xlay_kernel, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
  if (e == cudaSuccess) e = cudaDeviceGetAttribute(&g_dev[dev].sms, cudaDevAttrMultiProcessorCount, dev);
  return e;
}

// per-device one-time setup (kernel attributes are per device context)
cudaError_t device_info(int *sms) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  if (dev < 0 || dev >= 64) return cudaErrorInvalidDevice;
  std::lock_guard<std::mutex> lk(g_dev_mu);
  if (!g_dev[dev].configured) {
    e = configure_device(dev);
    if (e != cudaSuccess) return e;
    g_dev[dev].configured = true;
  }
  *sms = g_dev[dev].sms;
  return cudaSuccess;
}

// dynamic smem beyond the ring: x layouts of the four widths + the partial y
size_t region_bytes(int H) { return (size_t)4 * (H / 4 + H / 32) * 16 + (size_t)2 * H * 4; }

constexpr size_t kStaticReserve = 8192;  // static shared memory (batch, plan, barriers, loads, activations)

int stages_for(size_t extra) {
  int s = kMaxStages;
  while (s > 2 && (size_t)s * kStageBytes + extra + kStaticReserve > (size_t)kSmemLimit) --s;
  return s;
}

}  // namespace

cudaError_t ffn_preload() {
  int sms = 0;
  return device_info(&sms);
}

size_t ffn_xlay_floats(int H) { return (size_t)4 * (H / 4 + H / 32) * 4; }

size_t ffn_scratch_bytes(int H) {
  int sms = 0;
  if (device_info(&sms) != cudaSuccess || sms < 1) sms = kMaxGrid;
  return ((size_t)sms * H * 4 + 255) / 256 * 256 + 256;  // partials [sms][H] + the barrier word
}

cudaError_t launch_build_xlay(const float *x, int H, float *xlay, cudaStream_t s) {
  build_xlay_kernel<<<1, 512, H * sizeof(float), s>>>(x, H, reinterpret_cast<float4 *>(xlay));
  return cudaGetLastError();
}

cudaError_t launch_ffn_decode(const FfnBatch *batch_dev, const float *xlay, void *scratch, float *y_dev, int H,
                              cudaStream_t s) {
  return launch_ffn_decode_engine(batch_dev, xlay, scratch, y_dev, H, nullptr, nullptr, nullptr, s);
}

cudaError_t launch_ffn_decode_engine(const FfnBatch *batch_dev, const float *xlay, void *scratch, float *y_dev, int H,
                                     FfnStats *stat, const uint32_t *landed,
                                     const volatile uint32_t *abort, cudaStream_t s) {
  int sms = 0;
  cudaError_t e = device_info(&sms);
  if (e != cudaSuccess) return e;
  if (sms > kMaxGrid) sms = kMaxGrid;
  const size_t extra = region_bytes(H);
  const int st = stages_for(extra);
  const size_t smem = (size_t)st * kStageBytes + extra;
  if (smem + kStaticReserve > (size_t)kSmemLimit) return cudaErrorInvalidConfiguration;
  float *part = reinterpret_cast<float *>(scratch);
  unsigned int *bar = reinterpret_cast<unsigned int *>(reinterpret_cast<uint8_t *>(scratch) +
                                                       ((size_t)sms * H * 4 + 255) / 256 * 256);
  const float4 *xl = reinterpret_cast<const float4 *>(xlay);
  // cooperative: every CTA resident (one per SM), which the final grid barrier needs
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(sms);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeCooperative;
  attr[0].val.cooperative = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  if (H == 2048) return cudaLaunchKernelEx(&cfg, ffn_kernel<2048>, batch_dev, xl, part, bar, y_dev, stat, landed, abort, st);
  if (H == 4096) return cudaLaunchKernelEx(&cfg, ffn_kernel<4096>, batch_dev, xl, part, bar, y_dev, stat, landed, abort, st);
  return cudaLaunchKernelEx(&cfg, ffn_kernel<0>, batch_dev, xl, part, bar, y_dev, stat, landed, abort, st);
}

}  // namespace fate

// Profiling builds (FATE_PROF=1): out_host[192*8] per-CTA stamps (ns) of the last
// launch: start, plan, x landed, ring drained, partials written, barrier passed,
// done; then out_host[192*8 + 256*4] CTA 0's per-stage [wait, full, released, tag].
extern "C" int fate_k3_profile(uint64_t *out_host) {
#ifdef FATE_PROF
  if (cudaMemcpyFromSymbol(out_host, fate::g_k3_prof, sizeof(unsigned long long) * fate::kMaxGrid * 8) != cudaSuccess ||
      cudaMemcpyFromSymbol(out_host + fate::kMaxGrid * 8, fate::g_k3_stage, sizeof(unsigned long long) * 256 * 4) !=
          cudaSuccess) {
    fate::set_error("fate_k3_profile: copy failed");
    return FATE_ECUDA;
  }
  return FATE_OK;
#else
  (void)out_host;
  fate::set_error("fate_k3_profile: K3 phase stamps are compiled in only with FATE_PROF=1");
  return FATE_EINVAL;
#endif
}

extern "C" int fate_ffn_decode(const float *x_dev, int H, int n, const uint8_t *const *bufs, const float *weights,
                               float *scratch_dev, float *y_dev, void *stream) {
  using namespace fate;
  if (n < 1 || n > kMaxFfnExperts || H < 128 || H % 128 || H > 4096) {
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
    b.e[j] = FfnExpert{bufs[j], weights[j], h.I, h.bits, 0, -1, 0u};
    off += h.I;
  }
  b.total_I = off;
  FfnBatch *bd = nullptr;
  float *xl = nullptr;
  void *sc = nullptr;
  const size_t scb = ffn_scratch_bytes(H);
  FATE_CUDA(cudaMallocAsync(&bd, sizeof(FfnBatch), s));
  FATE_CUDA(cudaMallocAsync(&xl, ffn_xlay_floats(H) * sizeof(float), s));
  FATE_CUDA(cudaMallocAsync(&sc, scb, s));
  FATE_CUDA(cudaMemsetAsync(sc, 0, scb, s));
  FATE_CUDA(cudaMemcpyAsync(bd, &b, sizeof(b), cudaMemcpyHostToDevice, s));
  FATE_CUDA(launch_build_xlay(x_dev, H, xl, s));
  cudaError_t e = launch_ffn_decode(bd, xl, sc, y_dev, H, s);
  cudaFreeAsync(bd, s);
  cudaFreeAsync(xl, s);
  cudaFreeAsync(sc, s);
  FATE_CUDA(e);
  (void)scratch_dev;
  FATE_CUDA(cudaStreamSynchronize(s));  // b lives on this stack frame
  return FATE_OK;
}

extern "C" int fate_ffn_decode_timed(const float *x_dev, int H, int n, int nsets, const uint8_t *const *bufs,
                                     const float *weights, float *y_dev, int iters, void *stream, float *ms_out) {
  using namespace fate;
  if (n < 1 || n > kMaxFfnExperts || nsets < 1 || nsets > 64 || H < 128 || H % 128 || H > 4096 || iters < 1 ||
      !ms_out) {
    set_error("fate_ffn_decode_timed: bad arguments");
    return FATE_EINVAL;
  }
  cudaStream_t s = (cudaStream_t)stream;
  std::vector<FfnBatch> bs(nsets);
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
      b.e[j] = FfnExpert{buf, weights[j], h.I, h.bits, 0, -1, 0u};
      off += h.I;
    }
    b.total_I = off;
  }
  FfnBatch *bd = nullptr;
  float *xl = nullptr;
  void *sc = nullptr;
  const size_t scb = ffn_scratch_bytes(H);
  FATE_CUDA(cudaMalloc(&bd, sizeof(FfnBatch) * nsets));
  FATE_CUDA(cudaMalloc(&xl, ffn_xlay_floats(H) * sizeof(float)));
  FATE_CUDA(cudaMalloc(&sc, scb));
  FATE_CUDA(cudaMemset(sc, 0, scb));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaError_t e = cudaMemcpyAsync(bd, bs.data(), sizeof(FfnBatch) * nsets, cudaMemcpyHostToDevice, s);
  if (e == cudaSuccess) e = launch_build_xlay(x_dev, H, xl, s);
  for (int i = 0; i < nsets && e == cudaSuccess; ++i) e = launch_ffn_decode(bd + i, xl, sc, y_dev, H, s);
  if (e == cudaSuccess) e = cudaEventRecord(e0, s);
  for (int i = 0; i < iters && e == cudaSuccess; ++i) e = launch_ffn_decode(bd + (i % nsets), xl, sc, y_dev, H, s);
  if (e == cudaSuccess) e = cudaEventRecord(e1, s);
  if (e == cudaSuccess) e = cudaEventSynchronize(e1);
  float ms = 0.f;
  if (e == cudaSuccess) e = cudaEventElapsedTime(&ms, e0, e1);
  *ms_out = ms / iters;
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(bd);
  cudaFree(xl);
  cudaFree(sc);
  FATE_CUDA(e);
  return FATE_OK;
}
