// Internal definitions shared by the sm_100a translation units.
#pragma once

#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <string>

#include "../../include/fate_b200.h"

namespace fate {

// ---------------------------------------------------------------------------
// Error plumbing: every C entry point returns a status and records a message.
void set_error(const std::string &msg);
int cuda_status(cudaError_t e, const char *what);

#define FATE_CUDA(call)                                   \
  do {                                                    \
    cudaError_t _e = (call);                              \
    if (_e != cudaSuccess) return fate::cuda_status(_e, #call); \
  } while (0)

#define FATE_CHECK_LAUNCH(what)                                         \
  do {                                                                  \
    cudaError_t _e = cudaGetLastError();                                \
    if (_e != cudaSuccess) return fate::cuda_status(_e, what);          \
  } while (0)

// ---------------------------------------------------------------------------
// Packed expert buffer: 256-byte header followed by the payload.
//   quantized (bits 8/4/2): codes w1 [I*H*b/8] | codes w3 | codes w2 [H*I*b/8]
//                           | sz w1 [I*H/64 float2] | sz w3 | sz w2
//   bf16 (bits 16):         w1 [I*H] | w3 [I*H] | w2 [H*I]
// W1 / W3 are row-major [I, H] (groups of 64 along H).  W2 [H, I] is stored
// SLAB-MAJOR: slab s holds columns [s*C, s*C + C) of all H rows, row-major
// inside, with C = kW2SlabQuant = 64 (exactly one quantization group of the
// reference's row-major grouping, so codes / scale / zero per group are
// byte-identical, only the group order differs) and C = kW2SlabBf16 = 8 for
// bf16.  K3 thereby reads the W2 columns matching a block of W1/W3 rows as one
// contiguous bulk copy, and K4 reads a 64-column K-step of 128 rows likewise.
// The payload size equals expert_bytes[bits] of quant.py:239-246.  A copy of
// the whole buffer carries its own format, so a cache slot filled by an INT2
// on-demand load is computed as INT2 (the "tag slot bits" decision).
constexpr int kW2SlabQuant = 64;
constexpr int kW2SlabBf16 = 8;
constexpr uint32_t kMagic = 0xFA7EB200u;
constexpr int kGroup = 64;

struct ExpertHeader {
  uint32_t magic;
  int32_t bits;
  int32_t layer;
  int32_t expert;
  int32_t H;
  int32_t I;
  int32_t pad[58];
};
static_assert(sizeof(ExpertHeader) == FATE_HEADER_BYTES, "header size");

struct Layout {
  int64_t c1, c3, c2;  // code (or bf16) offsets within the payload
  int64_t s1, s3, s2;  // float2 (scale, zero) offsets (quantized only)
  int64_t row_bytes_up;   // bytes per row of w1/w3 (H elements)
  int64_t row_bytes_down; // bytes per row of w2 (I elements)
  int64_t payload;
};

__host__ __device__ inline Layout make_layout(int H, int I, int bits) {
  Layout L{};
  const int64_t n = (int64_t)H * I;
  if (bits == 16) {
    L.c1 = 0;
    L.c3 = 2 * n;
    L.c2 = 4 * n;
    L.s1 = L.s3 = L.s2 = 6 * n;
    L.row_bytes_up = 2 * (int64_t)H;
    L.row_bytes_down = 2 * (int64_t)I;
    L.payload = 6 * n;
  } else {
    const int64_t cb = n * bits / 8;
    const int64_t sb = n / kGroup * 8;
    L.c1 = 0;
    L.c3 = cb;
    L.c2 = 2 * cb;
    L.s1 = 3 * cb;
    L.s3 = 3 * cb + sb;
    L.s2 = 3 * cb + 2 * sb;
    L.row_bytes_up = (int64_t)H * bits / 8;
    L.row_bytes_down = (int64_t)I * bits / 8;
    L.payload = 3 * cb + 3 * sb;
  }
  return L;
}

inline int64_t buffer_bytes(int H, int I, int bits) {
  return FATE_HEADER_BYTES + make_layout(H, I, bits).payload;
}

// ---------------------------------------------------------------------------
// K3 launch interface (used both standalone and by the engine).
struct FfnExpert {
  const uint8_t *buf;  // packed buffer (header at buf, payload at buf + 256)
  float weight;
  int I;
  int bits;
  int late;            // 1: the buffer is filled during this step (on-demand / prefetched), so K3
                       // orders its units after the others (decided by the schedule, not by timing)
  int slot;            // >= 0: the buffer is still being filled; K3 reads it once landed[slot] reaches want
  uint32_t want;       // (the copy's generation, written by the copy stream behind the copy)
};
static_assert(sizeof(FfnExpert) == 32, "FfnExpert layout");

constexpr int kMaxFfnExperts = FATE_MAX_TOPK + 2;

struct FfnBatch {
  int n;
  int H;
  int total_I;
  unsigned int work;   // unused (kept zero)
  // optional L2 prefetch issued by the CTAs as they reach the final barrier
  // (the engine: the next decode step's router rows); pf_bytes % 16 == 0
  const void *pf_ptr;
  unsigned long long pf_bytes;
  FfnExpert e[kMaxFfnExperts];
};
static_assert(sizeof(FfnBatch) % 16 == 0, "K3 copies the batch with 16-byte loads");

// K3 launch (one cooperative kernel per step).  xlay: x in every
// chunk-transposed width layout (ffn_xlay_floats(H) floats, see write_xlay);
// scratch: ffn_scratch_bytes(H) bytes owned by ONE caller (per-CTA partial y
// rows + the grid-barrier word; zero-initialised once, launches serialised on
// one stream).  The batch is in DEVICE memory.
cudaError_t launch_ffn_decode(const FfnBatch *batch_dev, const float *xlay, void *scratch, float *y_dev, int H,
                              cudaStream_t s);
// K3 counters in device memory: algorithmic bytes, and (arrival-gated mode)
// the time the most-delayed producer warp of each launch spent waiting for
// copies, summed over launches (wait_cur: the running launch's maximum)
struct FfnStats {
  unsigned long long bytes, wait_ns, wait_cur;
  // diagnostics (globaltimer ns): the running launch's last gate opening, the
  // summed time from it to the launch's end (the K3 work left after the last
  // copy landed) and how many launches waited; the last launch's end
  unsigned long long open_max, tail_ns, tail_n, end_ns;
  // profiling builds: the last CTA's end (max over CTAs), K1's message-posted
  // time, and the summed K1 posted -> K3 CTA start hand-off
  unsigned long long end_max_ns, k1_post_ns, k1k3_ns, k1k3_n;
};

// landed (device memory, per staging buffer) / abort (host-mapped; 0x7FFFFFFF
// releases every wait): the engine's arrival-gated mode, where K3 is launched
// right behind K1 and each expert's pieces start once its copy landed; both
// null = every buffer is complete at launch.
cudaError_t launch_ffn_decode_engine(const FfnBatch *batch_dev, const float *xlay, void *scratch, float *y_dev,
                                     int H, FfnStats *stat, const uint32_t *landed,
                                     const volatile uint32_t *abort, cudaStream_t s);
cudaError_t launch_build_xlay(const float *x, int H, float *xlay, cudaStream_t s);
size_t ffn_xlay_floats(int H);
size_t ffn_scratch_bytes(int H);

// x (in shared memory) -> the four chunk-transposed layouts + chunk sums, by
// a whole thread block: slot s (chunk width 8 << s) at xlay + s*(H/4 + H/32) float4.
__device__ inline void write_xlay(const float *x, int H, float4 *xlay, int tid, int nthr) {
  const int stride = H / 4 + H / 32;
  for (int sl = 0; sl < 4; ++sl) {
    const int cols = 8 << sl, nch = H / cols, nq = cols / 4;
    float4 *xt = xlay + sl * stride;
    float *sums = reinterpret_cast<float *>(xt + H / 4);
    for (int i = tid; i < H / 4; i += nthr) {
      const int c = (4 * i) / cols, m = ((4 * i) % cols) / 4;
      float4 v = reinterpret_cast<const float4 *>(x)[i];
      if (sl == 2) {
        // INT4 width: element 4m+j prescaled by 2^-4j (exact), so K3 reads nibble j of
        // each 16-bit half in place as c * 2^4j (see word_dot<4>); the sums stay unscaled
        v.y *= 0.0625f;
        v.z *= 0.00390625f;
        v.w *= 0.000244140625f;
      } else if (sl == 3) {
        // INT2 width: element e prescaled by 4^-(e mod 8) (word_dot<2>)
        const float b = (m & 1) ? 0.00390625f : 1.0f;  // 4^-4 for odd quads
        v.x *= b;
        v.y *= b * 0.25f;
        v.z *= b * 0.0625f;
        v.w *= b * 0.015625f;
      }
      xt[m * nch + c] = v;
    }
    for (int c = tid; c < nch; c += nthr) {
      float acc = 0.f;
      for (int m = 0; m < nq; ++m) {
        const float4 q = reinterpret_cast<const float4 *>(x)[(c * cols) / 4 + m];
        acc += (q.x + q.y) + (q.z + q.w);
      }
      sums[c] = acc;
    }
  }
}

cudaError_t ffn_preload();

// Dense part of a decode step (dense.cu): attention block + shared-expert gate.
struct DenseDims {
  int H, n_heads, n_kv_heads, head_dim;
  float eps, rope_theta;
  int max_splits;
};
struct DenseLayer {
  const __nv_bfloat16 *wqkv;  // [(nh + 2 nkv) hd, H] row-major
  const float *bqkv;          // [(nh + 2 nkv) hd] or null
  const float *norm;          // RMSNorm weight [H]
  const __nv_bfloat16 *wo;    // [H, nh hd]
  __nv_bfloat16 *kv;          // K/V cache [max_ctx][2][nkv hd]
  const float *shared_gate;   // [H] or null (no gated shared expert)
  float *shared_gate_out;     // sigmoid(w . x) of the step
};
struct DenseScratch {
  float *h, *qkv, *q, *o, *part_o, *a;
  float2 *part_ml;
  unsigned *cnt;  // [n_heads] split-completion counters (zero between steps)
};
constexpr int kDenseMaxSplits = 128;  // context positions <= 32 * kDenseMaxSplits
cudaError_t launch_dense_step(const DenseLayer &Ly, const DenseDims &D, const float *h_prev, const float *y_prev,
                              const double *gate_in, int pos, DenseScratch &S, cudaStream_t s);
cudaError_t launch_embed(const double *gate_in, int H, float *h, cudaStream_t s);
cudaError_t launch_fill_kv(__nv_bfloat16 *kv, int64_t n, uint32_t seed, cudaStream_t s);

// K1 kernels exposed to the engine.
cudaError_t launch_gate_batch(const double *W, double tau, const double *h, int64_t h_stride, int T, int E, int H,
                              double *routing, int32_t *order, int32_t *list_len, int top_k, int policy,
                              double q, cudaStream_t s);

// K4 grouped prefill FFN.
struct PrefillExpert {
  const uint8_t *buf;
  int I;
  int bits;
  int tok_off;   // offset into tok_idx / tok_w
  int n_tok;
};

cudaError_t launch_k4_combine(const float *Z, const float *w, int T, int k, int H, int has_shared, float *Y,
                              cudaStream_t s);
cudaError_t k4_preload();
// K4 on tcgen05 (prefill_tc.cu): Xb bf16 token rows [T, H], A bf16 activations, Z fp32 rows.
cudaError_t launch_k4_tc(const void *Xb, int H, const PrefillExpert *ex_dev, int n, const int32_t *tok_idx,
                         const int32_t *zrow, const int *a_off_dev, void *A, float *Z, int items_up, int items_down,
                         cudaStream_t s);
cudaError_t k4_tc_preload();
int k4_tc_items(int n_tok, int I, int H, bool down);
cudaError_t gate_preload();

}  // namespace fate
