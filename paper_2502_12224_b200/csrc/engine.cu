// The offload engine: device-resident expert cache + prefetch + compute for
// decode (simulate_decoding, pipeline.py:343-517) and prefill
// (simulate_prefill, pipeline.py:536-778) executed on a B200.
//
// Per decode step (token t, layer l) on the compute stream:
//   K1  decode_gate_kernel   fp64 router rows of W_l and W_{l+1} (one CTA per
//       row; each stores its logit into a slot the tail block polls), then the
//       tail block: softmax/top-k of layer l, hit / prefetched / on-demand
//       split (pipeline.py:441-459), cross-layer prediction for l+1 truncated
//       to n and filtered by residency (pipeline.py:390-404), the K3 expert
//       batch and a step message to the host copy manager (warp 0), and this
//       step's ARC update_after_layer (cache.py:212-215, warp 1).
//   WAIT cuStreamWaitValue32 on a host-mapped flag: set by K1 itself when
//       every needed expert is already in HBM, otherwise by the host after
//       the needed copies landed.
//   K3  ffn_up / ffn_down    dequant-fused SwiGLU over the routed + shared
//       experts straight from their HBM buffers.
// The host thread is the transfer channel (pipeline.py:163-264): a FIFO of
// pending copies with on-demand promotion and stale-prefetch dropping, at
// most `max_inflight` copies submitted to the copy stream at a time.
#include <cuda.h>
#include <immintrin.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <unistd.h>
#include <deque>
#include <mutex>
#include <string>
#include <vector>

#include "arc_dev.cuh"
#include "gate_dev.cuh"

namespace fate {

thread_local std::string g_err;

void set_error(const std::string &msg) { g_err = msg; }

int cuda_status(cudaError_t e, const char *what) {
  g_err = std::string(what) + ": " + cudaGetErrorString(e);
  return e == cudaErrorMemoryAllocation ? FATE_ENOMEM : FATE_ECUDA;
}

// Driver entry points resolved through the runtime (no link-time libcuda
// dependency, so the library loads on hosts without a driver).
typedef CUresult (*PFN_wait32)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
typedef CUresult (*PFN_write32)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
static PFN_wait32 p_wait32 = nullptr;
static PFN_write32 p_write32 = nullptr;

static int resolve_driver() {
  if (p_wait32 && p_write32) return FATE_OK;
  cudaDriverEntryPointQueryResult q1, q2;
  void *a = nullptr, *b = nullptr;
  // request the CUDA 12 (v2) ABI of the stream memory operations explicitly
  if (cudaGetDriverEntryPointByVersion("cuStreamWaitValue32", &a, 12000, cudaEnableDefault, &q1) != cudaSuccess ||
      cudaGetDriverEntryPointByVersion("cuStreamWriteValue32", &b, 12000, cudaEnableDefault, &q2) != cudaSuccess ||
      !a || !b || q1 != cudaDriverEntryPointSuccess || q2 != cudaDriverEntryPointSuccess) {
    g_err = "cannot resolve cuStreamWaitValue32/cuStreamWriteValue32 from the CUDA driver";
    return FATE_ECUDA;
  }
  p_wait32 = (PFN_wait32)a;
  p_write32 = (PFN_write32)b;
  return FATE_OK;
}

// Launch-serialised execution (a profiler such as ncu / compute-sanitizer
// injected through CUDA_INJECTION64_PATH, CUDA_LAUNCH_BLOCKING=1, or
// FATE_PROFILE_SERIAL): a kernel launch may block the calling thread until the
// kernel has run, so the engine never enqueues a kernel behind a stream wait
// that this same thread must release.  Each step's expert compute is launched
// only after the host has seen its transfers land.  Same decisions and
// results; only the copy/compute overlap is lost.
static bool serial_launches() {
  static const bool v = [] {
    const char *b = getenv("CUDA_LAUNCH_BLOCKING");
    const char *inj = getenv("CUDA_INJECTION64_PATH");
    const char *pre = getenv("LD_PRELOAD");
    bool prof = (inj && *inj) || (pre && (strstr(pre, "TreeLauncher") || strstr(pre, "nsight") ||
                                          strstr(pre, "Injection") || strstr(pre, "sanitizer")));
    for (char **e = environ; !prof && e && *e; ++e)
      prof = strncmp(*e, "NV_COMPUTE_PROFILER", 19) == 0 || strncmp(*e, "NSIGHT_COMPUTE", 14) == 0 ||
             strncmp(*e, "NV_TPS", 6) == 0;
    const bool on = getenv("FATE_PROFILE_SERIAL") != nullptr || (b && atoi(b) != 0) || prof;
    if (on && getenv("FATE_DEBUG")) fprintf(stderr, "[fate] launch-serialised mode\n");
    return on;
  }();
  return v;
}

static int cu_status(CUresult r, const char *what) {
  g_err = std::string(what) + ": CUDA driver error " + std::to_string((int)r);
  return FATE_ECUDA;
}

#define FATE_CU(call)                                    \
  do {                                                   \
    CUresult _r = (call);                                \
    if (_r != CUDA_SUCCESS) return cu_status(_r, #call); \
  } while (0)

namespace {

constexpr int kGateThreads = 256;

// K1 row -> tail hand-off: every router-row slot holds this bit pattern (a
// signalling NaN with a payload no arithmetic produces) until its row block
// stores the logit; the tail polls the slots themselves (an aligned 8-byte
// store is single-copy atomic), so the value is its own ready flag -- no
// fence, arrive counter or second read -- and re-arms them once consumed.
constexpr unsigned long long kLogitEmpty = 0xFFF4DEADBEEF0001ull;

__device__ __forceinline__ int pop_free(const EngineDev &d) {
  Ctrl &C = *d.ctrl;
  if (C.free_top <= 0) {
    C.err = 1;
    return 0;
  }
  return d.free_stack[--C.free_top];
}

__device__ __forceinline__ void push_free(const EngineDev &d, int b) {
  Ctrl &C = *d.ctrl;
  if (C.free_top >= d.nbuf) {
    C.err = 2;
    return;
  }
  d.free_stack[C.free_top++] = b;
}

// Deferred update_after_layer of the previous step: ARC accesses in ascending
// id order, with buffer hand-over (inserted experts keep the staging buffer
// they were computed from; evicted experts' buffers return to the free
// stack).  Warp 0 only.
__device__ void apply_prev_update(const EngineDev &d, ArcLayer *arc_sm, fate_step_log *log, int32_t *rel) {
  Ctrl &C = *d.ctrl;
  const int lane = threadIdx.x & 31;
  const int pl = C.prev_layer;
  WarpArc arc;
  arc.load(&d.arc[pl], arc_sm);
  int nrel = 0, nvic = 0;
  for (int i = 0; i < C.prev_k; ++i) {
    const int e = C.prev_chosen[i];
    int victim;
    const int hit = arc.access(e, &victim);
    if (lane == 0) {
      if (victim >= 0) {
        int32_t &slot = d.buf_of[pl * d.E + victim];
        if (slot >= 0) rel[nrel++] = slot;
        slot = -1;
        if (log && nvic < KMAX) log[C.prev_step].victims[nvic] = victim;
        ++nvic;
      }
      if (!hit) {
        const int b = C.prev_buf[i];
        if (arc.c >= 1) {
          d.buf_of[pl * d.E + e] = b;
          for (int r = 0; r < nrel; ++r)
            if (rel[r] == b) rel[r] = rel[--nrel], r = nrel;
        } else {
          rel[nrel++] = b;
        }
      }
    }
    __syncwarp();
  }
  arc.store(&d.arc[pl]);
  if (lane == 0) {
    for (int r = 0; r < nrel; ++r) push_free(d, rel[r]);
    if (log) log[C.prev_step].n_victims = nvic;
    C.prev_valid = 0;
  }
  __syncwarp();
}

#ifdef FATE_PROF
__device__ unsigned long long g_k1_upd[4];
__device__ __forceinline__ unsigned long long gtime1();
#endif
// update_after_layer of the step K1 is deciding (cache.py:212-215), by warp 1
// of K1's tail block once warp 0 has made every free-stack edit of the step:
// ARC accesses in ascending id order over the layer's lists (copied into
// shared memory while the router rows ran), buffer hand-over as in
// apply_prev_update, every input from shared memory (chosen ids, their
// buffers, the layer's buffer table, the free-stack top).
__device__ void apply_step_update(const EngineDev &d, ArcLayer *arc_sm, const int32_t *chosen, const int32_t *cbuf,
                                  int32_t *bof, int k, int layer, int top, fate_step_log *lg, int32_t *rel) {
  const int lane = threadIdx.x & 31;
  WarpArc arc;
  arc.attach(arc_sm);
  int nrel = 0, nvic = 0;
#ifdef FATE_PROF
  const unsigned long long u0 = gtime1();
#endif
  for (int i = 0; i < k; ++i) {
    const int e = chosen[i];
    int victim;
    const int hit = arc.access(e, &victim);
    if (lane == 0) {
      if (victim >= 0) {
        const int slot = bof[victim];
        if (slot >= 0) rel[nrel++] = slot;
        bof[victim] = -1;
        d.buf_of[layer * d.E + victim] = -1;
        if (lg && nvic < KMAX) lg->victims[nvic] = victim;
        ++nvic;
      }
      if (!hit) {
        const int b = cbuf[i];
        if (arc.c >= 1) {
          bof[e] = b;
          d.buf_of[layer * d.E + e] = b;
          for (int r = 0; r < nrel; ++r)
            if (rel[r] == b) rel[r] = rel[--nrel], r = nrel;
        } else {
          rel[nrel++] = b;
        }
      }
    }
    __syncwarp();
  }
#ifdef FATE_PROF
  const unsigned long long u1 = gtime1();
#endif
  arc.store(&d.arc[layer]);
#ifdef FATE_PROF
  const unsigned long long u2 = gtime1();
  if (lane == 0) g_k1_upd[0] += u1 - u0, g_k1_upd[1] += u2 - u1, g_k1_upd[2] += 1;
#endif
  if (lane == 0) {
    Ctrl &C = *d.ctrl;
    for (int r = 0; r < nrel; ++r) {
      if (top >= d.nbuf) {
        C.err = 2;
        break;
      }
      d.free_stack[top++] = rel[r];
    }
    C.free_top = top;
    if (lg) lg->n_victims = nvic;
  }
}

// K1 phase timestamps of the last launch (globaltimer ns), diagnostics only:
// [0] block 0 start, [1] tail start, [2] state staged, [3] routed, [4] split,
// [5] predicted, [6] message posted
__device__ unsigned long long g_k1_prof[16];
// FATE_PROF accumulators over a run: [0] sum(K3 end -> K1 block 0 start), [1] n,
// [2] sum(K1 block 0 start -> message posted), [3] n
__device__ unsigned long long g_k1_acc[8];
__device__ unsigned long long g_k1_t0;
#ifdef FATE_PROF
#define K1_STAMP(i) (g_k1_prof[i] = gtime1())
#else
#define K1_STAMP(i) ((void)0)  // phase stamps are compiled in only with -DFATE_PROF
#endif

__device__ __forceinline__ unsigned long long gtime1() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// relaxed system-scope 8-byte store (single-copy atomic) into the mapped ring
__device__ __forceinline__ void st_sys64(uint64_t *p, uint64_t v) {
  asm volatile("st.relaxed.sys.global.b64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

struct TailSmem {
  int32_t bof_l[EMAX], pend_l[EMAX], bof_n[EMAX], bbits_l[EMAX];
  uint32_t pgen_l[EMAX], pdone_l[EMAX];
  int32_t pred_prev[EMAX];
  int32_t c_free_top, c_step, c_pred_valid, c_pred_layer, c_pred_n, shared_present;
  const uint8_t *shared_ptr;
  float shared_w;
  int32_t od_buf[KMAX];
  uint32_t od_gen[KMAX];
  int32_t eap_prev[KMAX], eap_prev_ok;
  double z[2 * EMAX], w[2 * EMAX];
  int32_t ord[2 * EMAX];
  int32_t chosen[KMAX], cbuf[KMAX], csrc[KMAX], chit[KMAX], carr[KMAX];
  int32_t is_chosen[EMAX];
  alignas(16) float xs[4096];  // x = sqrt(H) * gate_in, H <= 4096 (float4-read by write_xlay)
};

__global__ void __launch_bounds__(kGateThreads) decode_gate_kernel(EngineDev d, const double *__restrict__ gate_in,
                                                                   const int32_t *__restrict__ trace_chosen,
                                                                   fate_step_log *__restrict__ log, int layer,
                                                                   volatile uint32_t *ready_host, int token) {
  __shared__ double red[kGateThreads / 32];
  __shared__ TailSmem S;
  __shared__ ArcLayer arc_sm;
  __shared__ int32_t arc_rel[4 * KMAX + 4];
  __shared__ int32_t tchosen[KMAX];
  const int E = d.E, H = d.H, L = d.L;
  const double *h = gate_in + ((int64_t)token * L + layer) * H;
  // block 0: the tail (stages state while the others work); blocks
  // 1..n_rows: router rows; last block: the FFN input x and its K3 layouts.
  // The previous step's update_after_layer ran in the previous K1 (warp 1 of
  // its tail block) and completed before this launch.
  const int n_rows = gridDim.x - 2;
  const int row = blockIdx.x - 1;
  if (blockIdx.x == gridDim.x - 1) {
    // FFN input x = sqrt(H) * gate_in (fp64 product, fp32 storage) -> K3 layouts
    const double sH = sqrt((double)H);
    for (int i = threadIdx.x; i < H; i += kGateThreads) S.xs[i] = (float)(sH * h[i]);
    // launched programmatically behind the previous step's K3: that K3 reads x
    // until it completes (no-op for a normal launch)
    asm volatile("griddepcontrol.wait;" ::: "memory");
    __syncthreads();
    write_xlay(S.xs, H, reinterpret_cast<float4 *>(d.x), threadIdx.x, kGateThreads);
    return;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    K1_STAMP(0);
#ifdef FATE_PROF
    // previous K3's end -> this launch (both globaltimer)
    const unsigned long long e = d.stats->ffn.end_max_ns, now = gtime1();
    if (e && now > e) g_k1_acc[0] += now - e, g_k1_acc[1] += 1;
    g_k1_t0 = now;
#endif
  }
  if (threadIdx.x == 0 && blockIdx.x == 1) K1_STAMP(10);
  if (blockIdx.x > 0) {
    // ---- fp64 router row: each thread sums a fixed strided subset, fixed tree
    const int lrow = row < E ? layer : layer + 1;
    const int e_row = row < E ? row : row - E;
    const double2 *W2 = reinterpret_cast<const double2 *>(d.W + ((int64_t)lrow * E + e_row) * H);
    const double2 *h2 = reinterpret_cast<const double2 *>(h);
    const double tau = d.tau[lrow];
    constexpr int U = 8;  // H <= 2 * U * kGateThreads: every load issued before the first FMA
    double2 a[U], b[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int i = threadIdx.x + u * kGateThreads;
      if (i < H / 2) a[u] = __ldg(W2 + i), b[u] = __ldg(h2 + i);
    }
    double acc = 0.0;
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int i = threadIdx.x + u * kGateThreads;
      if (i < H / 2) {
        acc = fma(a[u].x, b[u].x, acc);
        acc = fma(a[u].y, b[u].y, acc);
      }
    }
    for (int i = threadIdx.x + U * kGateThreads; i < H / 2; i += kGateThreads) {
      const double2 x = __ldg(W2 + i), y = __ldg(h2 + i);
      acc = fma(x.x, y.x, acc);
      acc = fma(x.y, y.y, acc);
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
    __syncthreads();
    if (threadIdx.x == 0) {
      double sum = 0.0;
      for (int w = 0; w < kGateThreads / 32; ++w) sum += red[w];
      const double z = __ddiv_rn(sum, tau);
      asm volatile("st.relaxed.gpu.global.b64 [%0], %1;" ::"l"(d.logits + row), "l"(__double_as_longlong(z))
                   : "memory");
    }
    return;
  }
  // ================= tail block
  Ctrl &C = *d.ctrl;
  // stage every table the tail reads while the router rows are in flight
  const int pl = C.prev_valid ? C.prev_layer : -1;  // layer the ARC block is editing
  for (int i = threadIdx.x; i < E; i += kGateThreads) {
    S.is_chosen[i] = 0;
    const int pb = d.pend_buf[layer * E + i];
    S.pend_l[i] = pb;
    S.pgen_l[i] = d.pend_gen[layer * E + i];
    S.pdone_l[i] = pb >= 0 ? ((volatile uint32_t *)d.buf_done)[pb] : 0u;
    if (pl != layer) {
      const int bb = d.buf_of[layer * E + i];
      S.bof_l[i] = bb;
      S.bbits_l[i] = bb >= 0 ? d.buf_bits[bb] : 0;
    }
    if (pl != layer + 1) S.bof_n[i] = layer + 1 < L ? d.buf_of[(layer + 1) * E + i] : 0;
  }
  if (threadIdx.x < d.k && trace_chosen) tchosen[threadIdx.x] = trace_chosen[((int64_t)token * L + layer) * d.k + threadIdx.x];
  if (threadIdx.x < KMAX) S.eap_prev[threadIdx.x] = threadIdx.x < C.prev_k ? C.prev_chosen[threadIdx.x] : 0;
  // the control block was last written by the previous K1 / ARC update, both
  // complete before this launch (stream order): stage it with the tables
  const int c_pred_n = C.pred_n;
  const int c_top = C.free_top;
  if (threadIdx.x < KMAX) {
    // on-demand pops come off the top of the free stack (at most k): their
    // buffers and generations, so the split does no dependent global loads
    const int i = c_top - 1 - (int)threadIdx.x;
    const int b = i >= 0 && i < d.nbuf ? d.free_stack[i] : 0;
    S.od_buf[threadIdx.x] = b;
    S.od_gen[threadIdx.x] = d.buf_gen[b];
  }
  for (int i = threadIdx.x; i < c_pred_n; i += kGateThreads) S.pred_prev[i] = C.pred_list[i];
  // this layer's ARC lists for warp 1's update (written last by this layer's
  // previous update, in an earlier launch)
  for (int i = threadIdx.x; i < (int)(sizeof(ArcLayer) / 16); i += kGateThreads)
    reinterpret_cast<int4 *>(&arc_sm)[i] = reinterpret_cast<const int4 *>(&d.arc[layer])[i];
  if (threadIdx.x == 0) {
    S.c_step = C.step;
    S.c_pred_valid = C.pred_valid;
    S.c_pred_layer = C.pred_layer;
    S.c_pred_n = c_pred_n;
    S.c_free_top = c_top;
    // EAP observe needs the chosen set of (token, layer - 1): the previous step
    // (prev_valid is cleared once the deferred ARC update ran; the chosen set stays)
    S.eap_prev_ok = layer > 0 && C.step > 0 && C.prev_layer == layer - 1 ? 1 : 0;
    const uint8_t *sh = d.shared ? d.shared[layer] : nullptr;
    S.shared_ptr = sh;
    S.shared_present = sh ? 1 : 0;
    S.shared_w = sh && d.shared_gate ? d.shared_gate[layer] : 1.0f;
  }
  // the router rows: poll each slot until its row block stored the logit,
  // then re-arm it for the next launch
  for (int i = threadIdx.x; i < n_rows; i += kGateThreads) {
    unsigned long long v;
    do {
      asm volatile("ld.relaxed.gpu.global.b64 %0, [%1];" : "=l"(v) : "l"(d.logits + i) : "memory");
    } while (v == kLogitEmpty);
    S.z[i] = __longlong_as_double((long long)v);
    reinterpret_cast<unsigned long long *>(d.logits)[i] = kLogitEmpty;
  }
  if (threadIdx.x == 0) K1_STAMP(1);
  for (int i = threadIdx.x; i < E; i += kGateThreads) {
    if (pl == layer) {
      const int bb = ((volatile int32_t *)d.buf_of)[layer * E + i];
      S.bof_l[i] = bb;
      S.bbits_l[i] = bb >= 0 ? ((volatile int32_t *)d.buf_bits)[bb] : 0;
    }
    if (pl == layer + 1 && layer + 1 < L) S.bof_n[i] = ((volatile int32_t *)d.buf_of)[(layer + 1) * E + i];
  }
  __syncthreads();
  // (2) routing of layer l and the cross-layer prediction for l+1: the two
  // softmaxes on warps 0 and 1 at once, then the ranks by the whole block
  const bool pred_seg = d.use_predictor && d.policy != 2 && layer + 1 < L;
  if ((threadIdx.x >> 5) == 0) warp_softmax(S.z, S.w, E);
  else if ((threadIdx.x >> 5) == 1 && pred_seg) warp_softmax(S.z + E, S.w + E, E);
  __syncthreads();
  if (threadIdx.x < kGateThreads / 2) rank_by_weight(S.w, S.ord, E, threadIdx.x, kGateThreads / 2);
  else if (pred_seg) rank_by_weight(S.w + E, S.ord + E, E, threadIdx.x - kGateThreads / 2, kGateThreads / 2);
  __syncthreads();
  if (threadIdx.x >= 64) return;
  if (threadIdx.x >= 32) {
    // warp 1: update_after_layer of this step (cache.py:212-215) once warp 0
    // has finished every free-stack edit of the step (named barrier 1), in
    // parallel with the K3 batch and the step message
    asm volatile("bar.sync 1, 64;" ::: "memory");
#ifdef FATE_PROF
    const unsigned long long ta = gtime1();
#endif
    apply_step_update(d, &arc_sm, S.chosen, S.cbuf, S.bof_l, d.k, layer, S.c_free_top, log ? log + S.c_step : nullptr,
                      arc_rel);
#ifdef FATE_PROF
    if (threadIdx.x == 32) {
      const unsigned long long tb = gtime1();
      g_k1_acc[4] += ta - g_k1_t0;
      g_k1_acc[5] += tb - g_k1_t0;
      g_k1_acc[6] += 1;
    }
#endif
    return;
  }
  const int lane = threadIdx.x;
  const int k = d.k;
  const int step = S.c_step;
  fate_step_log *lg = log ? log + step : nullptr;
  if (lane == 0) K1_STAMP(2);
  // (2) routing of layer l (gatesim.py:113-123, core.py:159-163): S.w / S.ord above
  const unsigned FULL = 0xffffffffu;
  const unsigned lt = (1u << lane) - 1u;
  // chosen ids in ascending order (pipeline.py:441 iterates sorted(chosen)):
  // lane i < k owns ord[i]; its position = #{j < k : ord[j] < ord[i]}.  When
  // the trace supplies the chosen set (record.chosen, pipeline.py:422) it is
  // what the split and the ARC update use, as in the reference; the recomputed
  // top-k only feeds the mismatch counter (routing weights and predictions
  // always come from the device's fp64 router).
  {
    const int mine = lane < k ? S.ord[lane] : 0x7fffffff;
    int pos = 0;
    for (int j = 0; j < k; ++j) pos += __shfl_sync(FULL, mine, j) < mine;
    if (lane < k) S.csrc[pos] = mine;  // the recomputed set, ascending
  }
  __syncwarp();
  const int own = lane < k ? S.csrc[lane] : 0;
  if (lane < k) {
    const int use = trace_chosen ? tchosen[lane] : own;
    S.chosen[lane] = use;
    S.is_chosen[use] = 1;
  }
  __syncwarp();
  const bool act = lane < k;
  const int ce = act ? S.chosen[lane] : 0;
  {
    int mism = 0;
    if (trace_chosen && act) mism = own != ce;
    mism = __any_sync(FULL, mism);
    // recall of the prediction made one step earlier (pipeline.py:433-436)
    const bool chk = S.c_pred_valid && S.c_pred_layer == layer;
    int inter = 0;
    if (chk)
      for (int i = lane; i < S.c_pred_n; i += 32) inter += S.is_chosen[S.pred_prev[i]];
    for (int o = 16; o; o >>= 1) inter += __shfl_xor_sync(FULL, inter, o);
    if (lane == 0) {
      if (mism) atomicAdd(&d.stats->mismatches, 1ull);
      if (k < E && S.w[S.ord[k - 1]] - S.w[S.ord[k]] < 1e-12) atomicAdd(&d.stats->near_ties, 1ull);
      if (lg) lg->mismatch = mism;
      if (chk) {
        atomicAdd(&d.stats->recall_sum, (double)inter / (double)k);
        atomicAdd(&d.stats->recall_n, 1ull);
        C.pred_valid = 0;
      }
    }
  }
  if (lane == 0) K1_STAMP(3);
  // the previous step's K3 has completed (programmatic launch): it no longer
  // reads the buffers popped below, the batch or x (no-op for a normal launch)
  asm volatile("griddepcontrol.wait;" ::: "memory");
  // (3) hit / prefetched / on-demand split (pipeline.py:441-459), one lane per chosen expert
  DecodeMsg *msg = d.dring + (step % kRing);
  int top = S.c_free_top;
  const int slot_b = act ? S.bof_l[ce] : -1;
  const int pend_b = act && slot_b < 0 ? S.pend_l[ce] : -1;
  const bool hit = act && slot_b >= 0;
  const bool pref = act && !hit && pend_b >= 0;
  const bool odm = act && !hit && !pref;
  const unsigned m_od = __ballot_sync(FULL, odm), m_need = __ballot_sync(FULL, pref);
  const int n_od = __popc(m_od), n_need = __popc(m_need), i_od = __popc(m_od & lt), i_need = __popc(m_need & lt);
  int arr = 0, b = slot_b, src = 16;
  uint32_t want = 0;  // generation K3 waits for in buffer b (copy still in flight)
  if (hit) src = d.cached_bits < 16 ? d.cached_bits : 16;
  if (pref) {
    b = pend_b;
    src = d.prefetch_bits;
    arr = S.pdone_l[ce] == S.pgen_l[ce];
    want = S.pgen_l[ce];
    st_sys64(&msg->need[i_need], msg_entry(step, ce, b, 0u));
  }
  if (odm) {
    // pop n_od buffers off the free stack: the first od takes the top (staged)
    b = S.od_buf[i_od];
    const uint32_t g = S.od_gen[i_od] + 1u;
    d.buf_gen[b] = g;
    want = g;
    src = d.ondemand_bits;
    d.buf_bits[b] = d.ondemand_bits;
    st_sys64(&msg->od[i_od], msg_entry(step, ce, b, g));
    if (lg) lg->ondemand[i_od] = ce;
  }
  top -= n_od;
  if (lane == 0 && n_od) {
    // the on-demand set is final: let the host start those copies now, before
    // the drop list, the prediction and the K3 batch (with nothing to load the
    // full message below carries the step)
    st_sys64(&msg->od_head, ((uint64_t)((uint32_t)step + 1u) << 32) | ((uint64_t)n_od << 23) |
                                ((uint64_t)(d.ondemand_bits & 31) << 18));
  }
  const bool all_landed = __all_sync(FULL, !act || hit || (pref && arr));
  if (act) {
    C.prev_chosen[lane] = ce;
    C.prev_buf[lane] = b;
    S.cbuf[lane] = b;
    if (lg) {
      lg->chosen[lane] = ce;
      lg->src_bits[lane] = src;
      lg->hit[lane] = hit;
      lg->arrived[lane] = arr;
      lg->routing[lane] = (float)S.w[ce];
      lg->fmt_bits[lane] = hit ? S.bbits_l[ce] : src;
    }
  }
  const int n_hit = __popc(__ballot_sync(FULL, hit)), n_arr = __popc(__ballot_sync(FULL, arr != 0));
  const int n_deq = __popc(__ballot_sync(FULL, act && src < 16));
  // (4) prefetched-but-not-chosen experts of this layer: release their buffers
  // and tell the host to drop them if still queued (drop_stale, pipeline.py:438/247-253)
  int n_drop = 0;
  for (int base = 0; base < E; base += 32) {
    const int e = base + lane;
    const int pb = e < E ? S.pend_l[e] : -1;
    if (pb >= 0) d.pend_buf[layer * E + e] = -1;
    const bool drop = pb >= 0 && !S.is_chosen[e];
    const unsigned m = __ballot_sync(FULL, drop);
    if (drop) {
      const int i = n_drop + __popc(m & lt);
      st_sys64(&msg->drop[i], msg_entry(step, e, pb, 0u));
      d.free_stack[top + __popc(m & lt)] = pb;
    }
    top += __popc(m);
    n_drop += __popc(m);
  }
  if (lane == 0) K1_STAMP(4);
  // (5) cross-layer prediction for layer l+1 (predict.py:92-107, pipeline.py:390-404)
  int n_pf = 0, n_pred = -1;
  if (d.use_predictor && d.policy == 2) {
    // EAP observe (pipeline.py:310-315, eap_update predict.py:132-138): every
    // (a, b) in chosen(l-1) x chosen(l) -> counts[l-1][a][b] += 1 (distinct pairs)
    if (S.eap_prev_ok) {
      int32_t *cnt = d.eap_counts + (int64_t)(layer - 1) * E * E;
      for (int i = lane; i < k * k; i += 32) cnt[S.eap_prev[i / k] * E + S.chosen[i % k]] += 1;
      if (lane < k) d.eap_totals[(layer - 1) * E + S.eap_prev[lane]] += k;
    }
    // EAP predict for l+1 (eap_predict predict.py:141-158): Laplace-smoothed
    // row-normalised scores summed over chosen(l) in ascending id order
    // (fp64, IEEE division as numpy), top-k by (-score, id); cold start 0..k-1
    if (layer + 1 < L) {
      const int32_t *cnt = d.eap_counts + (int64_t)layer * E * E;
      const int32_t *tot = d.eap_totals + (int64_t)layer * E;
      int warm = 0;
      for (int j = 0; j < k; ++j) warm |= tot[S.chosen[j]] != 0;
      if (!warm) {
        for (int e = lane; e < E; e += 32) S.ord[E + e] = e;
      } else {
        for (int e = lane; e < E; e += 32) {
          double sc = 0.0;
          for (int j = 0; j < k; ++j) {
            const int a = S.chosen[j];
            sc = __dadd_rn(sc, __ddiv_rn((double)cnt[a * E + e] + 1.0, (double)(tot[a] + E)));
          }
          S.w[E + e] = sc;
        }
        __syncwarp();
        rank_by_weight(S.w + E, S.ord + E, E, lane, 32);
      }
      __syncwarp();
    }
  }
  if (d.use_predictor && layer + 1 < L) {
    const int len = d.policy == 2 ? (k < E ? k : E) : warp_pred_len(S.w + E, S.ord + E, E, k, d.policy, d.q);
    n_pred = len < d.budget_n ? len : d.budget_n;
    for (int base = 0; base < n_pred; base += 32) {
      const int i = base + lane;
      const int e = i < n_pred ? S.ord[E + i] : 0;
      if (i < n_pred) {
        C.pred_list[i] = e;
        if (lg) lg->pred[i] = e;
      }
      const bool issue = i < n_pred && S.bof_n[e] < 0;  // resident: skip (pipeline.py:397)
      const unsigned m = __ballot_sync(FULL, issue);
      if (issue) {
        const int j = n_pf + __popc(m & lt);
        const int nb = d.free_stack[top - 1 - __popc(m & lt)];
        const uint32_t g = d.buf_gen[nb] + 1u;
        d.buf_gen[nb] = g;
        d.buf_bits[nb] = d.prefetch_bits;
        d.pend_buf[(layer + 1) * E + e] = nb;
        d.pend_gen[(layer + 1) * E + e] = g;
        st_sys64(&msg->pf[j], msg_entry(step, e, nb, g));
        if (lg) lg->prefetch[j] = e;
      }
      top -= __popc(m);
      n_pf += __popc(m);
    }
  }
  __syncwarp();
  if (lane == 0) {
    if (top < 0 || top > d.nbuf) C.err = 1;
    C.free_top = top;
    S.c_free_top = top;  // warp 1 pushes the step's released buffers from here
    C.prev_layer = layer;  // (EAP observe of the next step reads the chosen set)
    C.prev_k = k;
    C.prev_step = step;
    if (n_pred >= 0) {
      C.pred_n = n_pred;
      C.pred_layer = layer + 1;
      C.pred_valid = 1;
    }
    if (lg) lg->n_pred = n_pred, lg->n_prefetch = n_pf, lg->n_ondemand = n_od;
    atomicAdd(&d.stats->accesses, (unsigned long long)k);
    atomicAdd(&d.stats->cache_hits, (unsigned long long)n_hit);
    atomicAdd(&d.stats->arrival_hits, (unsigned long long)n_arr);
    atomicAdd(&d.stats->dequant_count, (unsigned long long)n_deq);
    atomicAdd(&d.stats->ondemand_issued, (unsigned long long)n_od);
    atomicAdd(&d.stats->prefetch_issued, (unsigned long long)n_pf);
  }
  __syncwarp();
  asm volatile("bar.arrive 1, 64;" ::: "memory");  // hand the ARC update to warp 1
  if (lane == 0) K1_STAMP(5);
  // (6) the K3 batch: routed experts weighted by their full-softmax routing
  // weight (not renormalised), plus the shared expert with weight 1.
  // storage width of every buffer is known here (hit: the slot's tagged width;
  // fetched: the width requested), so K3 never reads headers on its critical path
  FfnBatch &B = *d.batch;
  if (act)
    B.e[lane] = FfnExpert{d.pool + (int64_t)b * d.buf_stride, (float)S.w[ce], d.I, hit ? S.bbits_l[ce] : src,
                          odm || pref ? 1 : 0, odm || (pref && !arr) ? b : -1, want};
  if (lane == 0) {
    int n = k, off = k * d.I;
    if (S.shared_present) {
      B.e[n] = FfnExpert{S.shared_ptr, S.shared_w, d.I_shared, d.shared_bits, 0, -1, 0u};
      off += d.I_shared;
      ++n;
    }
    B.H = H;
    B.n = n;
    B.total_I = off;
    B.work = 0u;
    {
      // K3 prefetches the router rows the next step's K1 reads (W of its layer
      // and the next one) into L2 while its CTAs gather at the final barrier
      const int nl = layer + 1 < L ? layer + 1 : 0;
      const int nrows = nl + 1 < L ? 2 : 1;
      B.pf_ptr = d.W + (int64_t)nl * E * H;
      B.pf_bytes = (unsigned long long)nrows * E * H * 8ull;
    }
    // (7) self-signal when nothing must be waited for + (8) the step message
    // head (the entries carry their own tags: no fence)
    if (all_landed) ready_host[layer] = (uint32_t)token + 1u;
    st_sys64(&msg->head, ((uint64_t)msg_head_tag(step) << 38) | ((uint64_t)n_od << 33) | ((uint64_t)n_need << 24) |
                             ((uint64_t)n_drop << 15) |
                             ((uint64_t)n_pf << 6) | ((uint64_t)(d.prefetch_bits & 31) << 1) | (all_landed ? 1u : 0u));
    // (9) control block for the next step
    C.cur_token = token;
    C.cur_layer = layer;
    C.step = step + 1;
    if (layer == L - 1) C.next_token = token + 1;
    K1_STAMP(6);
    K1_STAMP(7);
#ifdef FATE_PROF
    const unsigned long long tp = gtime1();
    g_k1_acc[2] += tp - g_k1_t0;
    g_k1_acc[3] += 1;
    d.stats->ffn.k1_post_ns = tp;
#endif
  }
}

// Deferred update_after_layer of the step whose K1 just finished (launched on
// the side stream after every K1, so it overlaps the step's transfers and K3;
// the next K1 waits for it), and the final flush.  No-op if already applied.
__global__ void arc_update_kernel(EngineDev d, fate_step_log *log) {
  __shared__ ArcLayer arc_sm;
  __shared__ int32_t rel[4 * KMAX + 4];
  if (threadIdx.x == 0) K1_STAMP(8);
  if (d.ctrl->prev_valid) apply_prev_update(d, &arc_sm, log, rel);
  if (threadIdx.x == 0) K1_STAMP(9);
}

// Standalone ARC accesses (update_after_layer / arc_access API).  Newly
// resident experts get a buffer popped here; their ids + buffers are returned
// so the host can load the cached_bits copy synchronously.
__global__ void arc_access_kernel(EngineDev d, int layer, const int32_t *experts, int n, int32_t *hits,
                                  int32_t *loads /* [2n]: expert, buffer; -1 terminated */) {
  __shared__ ArcLayer arc_sm;
  const int lane = threadIdx.x;
  WarpArc arc;
  arc.load(&d.arc[layer], &arc_sm);
  int nl = 0;
  for (int i = 0; i < n; ++i) {
    const int e = experts[i];
    int victim;
    const int hit = arc.access(e, &victim);
    if (lane == 0) {
      hits[i] = hit;
      if (victim >= 0) {
        int32_t &slot = d.buf_of[layer * d.E + victim];
        if (slot >= 0) {
          push_free(d, slot);
          for (int j = 0; j < nl; ++j)
            if (loads[2 * j + 1] == slot) loads[2 * j] = -2;  // loaded then evicted: skip copy
        }
        slot = -1;
      }
      if (!hit && arc.c >= 1) {
        const int b = pop_free(d);
        d.buf_bits[b] = d.cached_bits;
        d.buf_of[layer * d.E + e] = b;
        loads[2 * nl] = e;
        loads[2 * nl + 1] = b;
        ++nl;
      }
    }
    __syncwarp();
  }
  arc.store(&d.arc[layer]);
  if (lane == 0) loads[2 * nl] = -1;
}

// seed_resident (cache.py:197-204): append to T1 without ARC bookkeeping.
__global__ void arc_seed_kernel(EngineDev d, int layer, const int32_t *experts, int n, int32_t *loads) {
  if (threadIdx.x) return;
  ArcLayer &a = d.arc[layer];
  int nl = 0;
  for (int i = 0; i < n; ++i) {
    if (a.n1 + a.n2 >= a.c) break;
    const int e = experts[i];
    if (d.buf_of[layer * d.E + e] >= 0) continue;
    a.t1[a.n1++] = e;
    const int b = pop_free(d);
    d.buf_bits[b] = d.cached_bits;
    d.buf_of[layer * d.E + e] = b;
    loads[2 * nl] = e;
    loads[2 * nl + 1] = b;
    ++nl;
  }
  loads[2 * nl] = -1;
}

__global__ void engine_reset_kernel(EngineDev d, const int32_t *caps) {
  const int tid = blockIdx.x * blockDim.x + threadIdx.x;
  const int nth = gridDim.x * blockDim.x;
  for (int i = tid; i < d.L * d.E; i += nth) {
    d.buf_of[i] = -1;
    d.pend_buf[i] = -1;
    d.pend_gen[i] = 0;
  }
  for (int i = tid; i < d.nbuf; i += nth) {
    d.free_stack[i] = d.nbuf - 1 - i;
    d.buf_gen[i] = 0;
    d.buf_done[i] = 0xFFFFFFFFu;
  }
  for (int i = tid; i < 2 * EMAX; i += nth) reinterpret_cast<unsigned long long *>(d.logits)[i] = kLogitEmpty;
  for (int l = tid; l < d.L; l += nth) {
    ArcLayer &a = d.arc[l];
    a.c = caps[l];
    a.n1 = a.n2 = a.nb1 = a.nb2 = 0;
    a.p = 0.0;
  }
  if (tid == 0) {
    Ctrl &C = *d.ctrl;
    C.free_top = d.nbuf;
    C.err = 0;
    C.arrive = 0;
    C.prev_valid = 0;
    C.pred_valid = 0;
    C.next_token = 0;
    C.step = 0;
  }
}

__global__ void run_begin_kernel(EngineDev d) {
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    Ctrl &C = *d.ctrl;
    C.next_token = 0;
    C.step = 0;
    C.arrive = 0;
    C.prev_valid = 0;
    C.pred_valid = 0;
    C.err = 0;
    for (int i = 0; i < 2 * EMAX; ++i) reinterpret_cast<unsigned long long *>(d.logits)[i] = kLogitEmpty;
    // pending prefetches never outlive a run
    for (int i = 0; i < d.L * d.E; ++i) {
      if (d.pend_buf[i] >= 0) push_free(d, d.pend_buf[i]);
      d.pend_buf[i] = -1;
    }
    *d.stats = DevStats{};
  }
}

}  // namespace
}  // namespace fate

using namespace fate;

// ---------------------------------------------------------------------------
// Host side

struct Transfer {
  int kind;  // 0 prefetch, 1 ondemand, 2 signal-only
  int step, layer, expert, bits, buf;
  uint32_t gen;
  int signal_token;   // >= 0: write ready[layer] = signal_token + 1 after this copy
  int signal_layer;
};

struct Inflight {
  uint32_t seq;
  Transfer t;
  int ev;       // index of the start/stop event pair (-1 untimed)
  int stream;   // copy stream (0/1) it was submitted on
  uint32_t sseq;  // per-stream completion sequence number
};

struct fate_engine {
  fate_engine_config cfg{};
  std::vector<int32_t> caps;
  EngineDev d{};
  int64_t buf_stride = 0;
  // device allocations
  void *dev_block = nullptr;
  uint8_t *pool = nullptr;
  int32_t *caps_dev = nullptr;
  int32_t *scratch_i = nullptr;  // small scratch for standalone calls
  void *k3_scratch = nullptr;  // K3 per-CTA partials + grid-barrier word (this engine's launches only)
  // mapped pinned host memory
  StepMsg *ring_host = nullptr;
  DecodeMsg *dring_host = nullptr;
  volatile uint32_t *ready_host = nullptr;     // [L]
  uint32_t *ready_dev = nullptr;
  size_t eap_bytes = 0;  // eap_counts .. end of eap_totals (contiguous in dev_block)
  volatile uint32_t *copy_done_host = nullptr, *copy_done_host2 = nullptr;  // per copy stream
  CUdeviceptr copy_done_dev = 0, copy_done_dev2 = 0;
  // host pools
  const uint8_t *host_pool[17] = {};
  std::vector<const uint8_t *> src_table[17];  // expert-sharded mode: per-(l,e) device/peer sources
  int64_t host_stride[17] = {};
  std::vector<const uint8_t *> shared_dev;
  const uint8_t **shared_table_dev = nullptr;
  int32_t *pf_shared_I = nullptr;
  cudaStream_t cstream = nullptr, xstream = nullptr, xstream2 = nullptr;  // compute, two copy streams
  cudaEvent_t xlast[2] = {nullptr, nullptr};  // last copy submitted on each copy stream
  cudaStream_t astream = nullptr;             // side stream: per-step deferred ARC update
  cudaEvent_t ev_k1 = nullptr, ev_arc = nullptr;
  int max_total_I = 0;
  int prefill_max_tokens = 0;
  int copy_event_stride = 8;  // time every stride-th copy (0: none); fate_engine_set_copy_timing
  bool k3_overlap = true;     // decode: K3 launched behind K1, gated per expert on its copy (fate_engine_set_overlap)
  // prefill scratch
  void *pf_block = nullptr;
  std::mutex mu;
  // last run's timeline (ms from the run's first event)
  // dense part (attention block + shared-expert gate), enabled by fate_engine_set_dense
  bool dense = false;
  DenseDims dd{};
  int max_ctx = 0, ctx0 = 0;
  std::vector<DenseLayer> dl;
  void *dense_block = nullptr;  // K/V cache + scratch + shared-gate outputs
  DenseScratch ds{};
  float *shared_gate_dev = nullptr;
  std::vector<double> step_ms;     // [steps][4]: gate start/end, moe start/end
  std::vector<double> copy_ms;     // [copies][2]
  std::vector<int32_t> copy_meta;  // [copies][5]: kind, step, layer, expert, bits
};

namespace {

int64_t align_up(int64_t x, int64_t a) { return (x + a - 1) / a * a; }

int check_cfg(const fate_engine_config *c) {
  if (!c || c->num_layers < 1 || c->num_experts < 1 || c->num_experts > FATE_MAX_EXPERTS || c->top_k < 1 ||
      c->top_k > c->num_experts || c->top_k > FATE_MAX_TOPK || c->hidden_dim < 128 || c->hidden_dim > 4096 || c->hidden_dim % 128 ||
      c->intermediate_dim < 128 || c->intermediate_dim % 128 || c->shared_intermediate < 0 ||
      c->shared_intermediate % 128 || !c->capacity || c->budget_n < 0 || c->max_tokens < 1) {
    set_error("fate_engine_create: invalid geometry");
    return FATE_EINVAL;
  }
  auto okb = [](int b) { return b == 2 || b == 4 || b == 8 || b == 16; };
  if (!okb(c->prefetch_bits) || !okb(c->ondemand_bits) || !okb(c->cached_bits) ||
      (c->shared_intermediate && !okb(c->shared_bits)) || !okb(c->prefill_ondemand_bits)) {
    set_error("fate_engine_create: bit widths must be 2, 4, 8 or 16");
    return FATE_EINVAL;
  }
  if (c->policy != 0 && c->policy != 1 && c->policy != 2) {
    set_error("fate_engine_create: policy must be 0 (topk), 1 (percentile) or 2 (eap)");
    return FATE_EINVAL;
  }
  for (int l = 0; l < c->num_layers; ++l)
    if (c->capacity[l] < 0 || c->capacity[l] > c->num_experts) {
      set_error("fate_engine_create: capacity must lie in [0, num_experts]");
      return FATE_EINVAL;
    }
  return FATE_OK;
}

int copy_to_buffers(fate_engine *g, const int32_t *loads_dev, int layer, int bits) {
  // loads: pairs (expert, buffer) terminated by -1; -2 marks a skipped entry
  std::vector<int32_t> h(2 * FATE_MAX_EXPERTS + 2);
  FATE_CUDA(cudaMemcpy(h.data(), loads_dev, h.size() * 4, cudaMemcpyDeviceToHost));
  if (!g->host_pool[bits]) {
    set_error("no pinned host pool registered for the cached bit width");
    return FATE_EINVAL;
  }
  const int64_t bytes = buffer_bytes(g->cfg.hidden_dim, g->cfg.intermediate_dim, bits);
  for (int i = 0; h[2 * i] != -1; ++i) {
    if (h[2 * i] < 0) continue;
    const uint8_t *src = g->host_pool[bits] + ((int64_t)layer * g->cfg.num_experts + h[2 * i]) * g->host_stride[bits];
    FATE_CUDA(cudaMemcpyAsync(g->pool + (int64_t)h[2 * i + 1] * g->buf_stride, src, bytes, cudaMemcpyHostToDevice,
                              g->xstream));
  }
  FATE_CUDA(cudaStreamSynchronize(g->xstream));
  return FATE_OK;
}

}  // namespace

static int prefill_preload();

extern "C" int fate_k1_profile(uint64_t *out_host) {
  if (cudaMemcpyFromSymbol(out_host, g_k1_prof, sizeof(unsigned long long) * 16) != cudaSuccess) {
    set_error("fate_k1_profile: copy failed");
    return FATE_ECUDA;
  }
  return FATE_OK;
}

extern "C" int fate_version(void) { return 1; }
extern "C" const char *fate_last_error(void) { return g_err.c_str(); }

extern "C" int fate_device_count(int *count) {
  int n = 0;
  cudaError_t e = cudaGetDeviceCount(&n);
  if (e != cudaSuccess) {
    *count = 0;
    cudaGetLastError();
    return cuda_status(e, "cudaGetDeviceCount");
  }
  *count = n;
  return FATE_OK;
}

extern "C" int fate_engine_create(const fate_engine_config *cfg, fate_engine **out) {
  if (int st = check_cfg(cfg)) return st;
  *out = nullptr;
  if (int st = resolve_driver()) return st;
  fate_engine *g = new fate_engine();
  g->cfg = *cfg;
  g->caps.assign(cfg->capacity, cfg->capacity + cfg->num_layers);
  g->cfg.capacity = g->caps.data();
  if (g->cfg.max_inflight < 1) g->cfg.max_inflight = 2;
  FATE_CUDA(cudaSetDevice(cfg->device));
  const int L = cfg->num_layers, E = cfg->num_experts, k = cfg->top_k, H = cfg->hidden_dim, I = cfg->intermediate_dim;
  int S = 0;
  for (int c : g->caps) S += c;
  // staging: prefetches for l and l+1 in flight plus the step's on-demand loads
  const int n_max = E;  // any later set_strategy may raise n up to E
  const int staging_decode = 2 * n_max + 2 * k + 4;
  const int staging_prefill = 2 * E + 4;
  const int nbuf = S + std::max(staging_decode, staging_prefill);
  if (nbuf > 0xFFFF) {
    set_error("fate_engine_create: more than 65535 expert buffers (the decode message packs buffer ids in 16 bits)");
    delete g;
    return FATE_EINVAL;
  }
  int64_t bb = 0;
  for (int b : {cfg->prefetch_bits, cfg->ondemand_bits, cfg->cached_bits, cfg->prefill_ondemand_bits, 4, 2})
    bb = std::max<int64_t>(bb, buffer_bytes(H, I, b));
  g->buf_stride = align_up(bb, 4096);
  EngineDev &d = g->d;
  d.L = L, d.E = E, d.k = k, d.H = H, d.I = I;
  d.I_shared = cfg->shared_intermediate;
  d.shared_bits = cfg->shared_bits;
  d.cached_bits = cfg->cached_bits;
  d.prefetch_bits = cfg->prefetch_bits;
  d.ondemand_bits = cfg->ondemand_bits;
  d.use_predictor = cfg->use_predictor;
  d.policy = cfg->policy;
  d.budget_n = std::min(cfg->budget_n, E);
  g->cfg.budget_n = d.budget_n;
  d.q = cfg->percentile_q;
  d.nbuf = nbuf;
  d.buf_stride = g->buf_stride;
  g->max_total_I = k * I + cfg->shared_intermediate;
  // one block for the small device state
  size_t off = 0;
  auto carve = [&](size_t bytes) {
    size_t o = off;
    off = (size_t)align_up((int64_t)(off + bytes), 256);
    return o;
  };
  const size_t o_W = carve((size_t)L * E * H * 8), o_tau = carve((size_t)L * 8), o_arc = carve((size_t)L * sizeof(ArcLayer)),
               o_bof = carve((size_t)L * E * 4), o_pb = carve((size_t)L * E * 4), o_pg = carve((size_t)L * E * 4),
               o_fs = carve((size_t)nbuf * 4), o_bg = carve((size_t)nbuf * 4), o_bd = carve((size_t)nbuf * 4),
               o_bb = carve((size_t)nbuf * 4),
               o_ctrl = carve(sizeof(Ctrl)), o_st = carve(sizeof(DevStats)), o_lg = carve(2 * EMAX * 8),
               o_x = carve(ffn_xlay_floats(H) * 4), o_b = carve(sizeof(FfnBatch)), o_caps = carve((size_t)L * 4),
               o_sh = carve((size_t)L * 8), o_si = carve((2 * FATE_MAX_EXPERTS + 2) * 4 * 2),
               o_ec = carve((size_t)std::max(L - 1, 1) * E * E * 4), o_et = carve((size_t)std::max(L - 1, 1) * E * 4);
  FATE_CUDA(cudaMalloc(&g->dev_block, off));
  FATE_CUDA(cudaMemset(g->dev_block, 0, off));
  uint8_t *base = (uint8_t *)g->dev_block;
  d.W = (const double *)(base + o_W);
  d.tau = (const double *)(base + o_tau);
  d.arc = (ArcLayer *)(base + o_arc);
  d.buf_of = (int32_t *)(base + o_bof);
  d.pend_buf = (int32_t *)(base + o_pb);
  d.pend_gen = (uint32_t *)(base + o_pg);
  d.free_stack = (int32_t *)(base + o_fs);
  d.buf_gen = (uint32_t *)(base + o_bg);
  d.buf_done = (uint32_t *)(base + o_bd);
  d.buf_bits = (int32_t *)(base + o_bb);
  d.ctrl = (Ctrl *)(base + o_ctrl);
  d.stats = (DevStats *)(base + o_st);
  d.logits = (double *)(base + o_lg);
  d.x = (float *)(base + o_x);
  d.batch = (FfnBatch *)(base + o_b);
  g->caps_dev = (int32_t *)(base + o_caps);
  g->shared_table_dev = (const uint8_t **)(base + o_sh);
  d.shared = cfg->shared_intermediate ? g->shared_table_dev : nullptr;
  g->scratch_i = (int32_t *)(base + o_si);
  d.eap_counts = (int32_t *)(base + o_ec);
  d.eap_totals = (int32_t *)(base + o_et);
  g->eap_bytes = (size_t)((o_et - o_ec) + (size_t)std::max(L - 1, 1) * E * 4);
  FATE_CUDA(cudaMalloc(&g->pool, (size_t)nbuf * g->buf_stride));
  d.pool = g->pool;
  {
    const size_t kb = ffn_scratch_bytes(H);
    FATE_CUDA(cudaMalloc(&g->k3_scratch, kb));
    FATE_CUDA(cudaMemset(g->k3_scratch, 0, kb));
  }
  FATE_CUDA(cudaMemcpy(g->caps_dev, g->caps.data(), L * 4, cudaMemcpyHostToDevice));
  g->shared_dev.assign(L, nullptr);
  // mapped pinned host memory: mailbox ring, ready flags, copy counter
  void *p = nullptr;
  FATE_CUDA(cudaHostAlloc(&p, sizeof(StepMsg) * kRing, cudaHostAllocMapped));
  memset(p, 0, sizeof(StepMsg) * kRing);
  g->ring_host = (StepMsg *)p;
  void *pd = nullptr;
  FATE_CUDA(cudaHostGetDevicePointer(&pd, p, 0));
  d.ring = (StepMsg *)pd;
  FATE_CUDA(cudaHostAlloc(&p, sizeof(DecodeMsg) * kRing, cudaHostAllocMapped));
  memset(p, 0, sizeof(DecodeMsg) * kRing);
  g->dring_host = (DecodeMsg *)p;
  FATE_CUDA(cudaHostGetDevicePointer(&pd, p, 0));
  d.dring = (DecodeMsg *)pd;
  FATE_CUDA(cudaHostAlloc(&p, 4096, cudaHostAllocMapped));
  memset(p, 0, 4096);
  g->ready_host = (volatile uint32_t *)p;
  g->copy_done_host = (volatile uint32_t *)((uint8_t *)p + 2048);
  g->copy_done_host2 = (volatile uint32_t *)((uint8_t *)p + 2176);
  FATE_CUDA(cudaHostGetDevicePointer(&pd, p, 0));
  g->ready_dev = (uint32_t *)pd;
  g->copy_done_dev = (CUdeviceptr)((uint8_t *)pd + 2048);
  g->copy_done_dev2 = (CUdeviceptr)((uint8_t *)pd + 2176);
  int lo = 0, hi = 0;
  FATE_CUDA(cudaDeviceGetStreamPriorityRange(&lo, &hi));
  FATE_CUDA(cudaStreamCreateWithPriority(&g->cstream, cudaStreamNonBlocking, hi));
  FATE_CUDA(cudaStreamCreateWithPriority(&g->xstream, cudaStreamNonBlocking, lo));
  FATE_CUDA(cudaStreamCreateWithPriority(&g->xstream2, cudaStreamNonBlocking, lo));
  for (auto &e : g->xlast) FATE_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  FATE_CUDA(cudaStreamCreateWithPriority(&g->astream, cudaStreamNonBlocking, hi));
  FATE_CUDA(cudaEventCreateWithFlags(&g->ev_k1, cudaEventDisableTiming));
  FATE_CUDA(cudaEventCreateWithFlags(&g->ev_arc, cudaEventDisableTiming));
  // load every kernel the engine launches now: lazy module loading at first
  // launch can deadlock behind a stream parked on a cuStreamWaitValue32 flag
  {
    cudaFuncAttributes fa;
    FATE_CUDA(cudaFuncGetAttributes(&fa, decode_gate_kernel));
    FATE_CUDA(cudaFuncGetAttributes(&fa, arc_update_kernel));
    // every kernel of the decode step prefers the max shared-memory carveout
    // (K3's 205 KB), so SMs do not reconfigure L1/shared between K1 and K3
    FATE_CUDA(cudaFuncSetAttribute(decode_gate_kernel, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
    FATE_CUDA(cudaFuncSetAttribute(arc_update_kernel, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
    FATE_CUDA(cudaFuncGetAttributes(&fa, arc_access_kernel));
    FATE_CUDA(cudaFuncGetAttributes(&fa, arc_seed_kernel));
    FATE_CUDA(cudaFuncGetAttributes(&fa, run_begin_kernel));
    FATE_CUDA(ffn_preload());
    FATE_CUDA(k4_preload());
    FATE_CUDA(k4_tc_preload());
    FATE_CUDA(gate_preload());
    if (int st = prefill_preload()) return st;
  }
  engine_reset_kernel<<<64, 256, 0, g->cstream>>>(d, g->caps_dev);
  FATE_CHECK_LAUNCH("engine_reset_kernel");
  FATE_CUDA(cudaStreamSynchronize(g->cstream));
  *out = g;
  return FATE_OK;
}

extern "C" int fate_engine_destroy(fate_engine *g) {
  if (!g) return FATE_OK;
  cudaStreamSynchronize(g->cstream);
  cudaStreamSynchronize(g->xstream);
  if (g->xstream2) cudaStreamSynchronize(g->xstream2);
  cudaStreamDestroy(g->cstream);
  cudaStreamDestroy(g->xstream);
  if (g->xstream2) cudaStreamDestroy(g->xstream2);
  for (auto &e : g->xlast)
    if (e) cudaEventDestroy(e);
  if (g->astream) {
    cudaStreamSynchronize(g->astream);
    cudaStreamDestroy(g->astream);
  }
  if (g->ev_k1) cudaEventDestroy(g->ev_k1);
  if (g->ev_arc) cudaEventDestroy(g->ev_arc);
  cudaFree(g->pool);
  cudaFree(g->dev_block);
  if (g->k3_scratch) cudaFree(g->k3_scratch);
  if (g->pf_block) cudaFree(g->pf_block);
  if (g->dense_block) cudaFree(g->dense_block);
  cudaFreeHost(g->ring_host);
  cudaFreeHost(g->dring_host);
  cudaFreeHost((void *)g->ready_host);
  delete g;
  return FATE_OK;
}

// EAP co-activation statistics back to empty (a fresh EapStats, predict.py:110-130).
// The Python layer calls it for every fresh simulate_prefill / simulate_decoding
// with Strategy.eap(); compare_strategies keeps them from prefill into decode.
extern "C" int fate_engine_reset_eap(fate_engine *g) {
  if (!g) {
    fate::set_error("fate_engine_reset_eap: null engine");
    return FATE_EINVAL;
  }
  if (cudaMemsetAsync(g->d.eap_counts, 0, g->eap_bytes, g->cstream) != cudaSuccess) {
    fate::set_error("fate_engine_reset_eap: memset failed");
    return FATE_ECUDA;
  }
  return FATE_OK;
}

extern "C" int fate_engine_set_gate(fate_engine *g, const double *W_host, const double *tau_host) {
  const size_t n = (size_t)g->cfg.num_layers * g->cfg.num_experts * g->cfg.hidden_dim;
  FATE_CUDA(cudaMemcpy((void *)g->d.W, W_host, n * 8, cudaMemcpyHostToDevice));
  FATE_CUDA(cudaMemcpy((void *)g->d.tau, tau_host, g->cfg.num_layers * 8, cudaMemcpyHostToDevice));
  return FATE_OK;
}

extern "C" int fate_engine_set_host_pool(fate_engine *g, int bits, const uint8_t *base, int64_t stride) {
  if (!(bits == 2 || bits == 4 || bits == 8 || bits == 16) ||
      stride < buffer_bytes(g->cfg.hidden_dim, g->cfg.intermediate_dim, bits)) {
    set_error("fate_engine_set_host_pool: bad bits or stride");
    return FATE_EINVAL;
  }
  g->host_pool[bits] = base;
  g->host_stride[bits] = stride;
  return FATE_OK;
}

extern "C" int fate_engine_set_expert_sources(fate_engine *g, int bits, const uint8_t *const *srcs) {
  if (!(bits == 2 || bits == 4 || bits == 8 || bits == 16)) {
    set_error("fate_engine_set_expert_sources: bits must be 2, 4, 8 or 16");
    return FATE_EINVAL;
  }
  auto &t = g->src_table[bits];
  if (!srcs) {
    t.clear();
    return FATE_OK;
  }
  const size_t n = (size_t)g->cfg.num_layers * g->cfg.num_experts;
  t.assign(srcs, srcs + n);
  return FATE_OK;
}

typedef CUresult (*PFN_addr_range)(CUdeviceptr *, size_t *, CUdeviceptr);

// IPC handles name whole allocations: export the allocation that contains
// dev_ptr (a caching allocator may sub-allocate) and return dev_ptr's offset.
extern "C" int fate_ipc_get_handle(const void *dev_ptr, uint8_t *handle64, int64_t *offset) {
  static_assert(sizeof(cudaIpcMemHandle_t) == 64, "IPC handle size");
  static PFN_addr_range p_range = nullptr;
  if (!p_range) {
    void *f = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPointByVersion("cuMemGetAddressRange", &f, 12000, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess || !f) {
      set_error("fate_ipc_get_handle: cuMemGetAddressRange unavailable");
      return FATE_ECUDA;
    }
    p_range = (PFN_addr_range)f;
  }
  CUdeviceptr base = 0;
  size_t size = 0;
  FATE_CU(p_range(&base, &size, (CUdeviceptr)dev_ptr));
  cudaIpcMemHandle_t h;
  FATE_CUDA(cudaIpcGetMemHandle(&h, (void *)base));
  memcpy(handle64, &h, 64);
  *offset = (int64_t)((CUdeviceptr)dev_ptr - base);
  return FATE_OK;
}

extern "C" int fate_ipc_open_handle(const uint8_t *handle64, void **dev_ptr_out) {
  cudaIpcMemHandle_t h;
  memcpy(&h, handle64, 64);
  FATE_CUDA(cudaIpcOpenMemHandle(dev_ptr_out, h, cudaIpcMemLazyEnablePeerAccess));
  return FATE_OK;
}

extern "C" int fate_ipc_close(void *dev_ptr) {
  FATE_CUDA(cudaIpcCloseMemHandle(dev_ptr));
  return FATE_OK;
}

extern "C" int fate_engine_set_overlap(fate_engine *g, int on) {
  g->k3_overlap = on != 0;
  return FATE_OK;
}

extern "C" int fate_engine_set_copy_timing(fate_engine *g, int stride) {
  if (stride < 0) {
    set_error("fate_engine_set_copy_timing: stride must be >= 0");
    return FATE_EINVAL;
  }
  g->copy_event_stride = stride;
  return FATE_OK;
}

extern "C" int fate_host_register(void *host_ptr, int64_t bytes) {
  if (!host_ptr || bytes <= 0) {
    set_error("fate_host_register: bad arguments");
    return FATE_EINVAL;
  }
  FATE_CUDA(cudaHostRegister(host_ptr, (size_t)bytes, cudaHostRegisterPortable));
  return FATE_OK;
}

extern "C" int fate_host_unregister(void *host_ptr) {
  FATE_CUDA(cudaHostUnregister(host_ptr));
  return FATE_OK;
}

extern "C" int fate_engine_set_dense(fate_engine *g, int n_heads, int n_kv_heads, int head_dim, int max_ctx, int ctx0,
                                     float eps, float rope_theta) {
  const int H = g->cfg.hidden_dim, L = g->cfg.num_layers;
  if (H % 256 || head_dim % 32 || head_dim > 128 || n_heads < 1 || n_kv_heads < 1 || n_heads % n_kv_heads ||
      n_heads / n_kv_heads > 32 || max_ctx < 1 || ctx0 < 0 || ctx0 >= max_ctx || max_ctx > 32 * kDenseMaxSplits) {
    set_error("fate_engine_set_dense: unsupported geometry (head_dim <= 128, max_ctx <= 4096)");
    return FATE_EINVAL;
  }
  std::lock_guard<std::mutex> lk(g->mu);
  cudaSetDevice(g->cfg.device);
  if (g->dense_block && g->dd.n_heads == n_heads && g->dd.n_kv_heads == n_kv_heads && g->dd.head_dim == head_dim &&
      g->max_ctx >= max_ctx && g->ctx0 == ctx0) {
    g->dd.eps = eps, g->dd.rope_theta = rope_theta;  // same cache: the prompt positions are kept
    return FATE_OK;
  }
  if (g->dense_block) {
    cudaStreamSynchronize(g->cstream);
    cudaFree(g->dense_block);
    g->dense_block = nullptr;
  }
  const int64_t row = (int64_t)2 * n_kv_heads * head_dim, nq = (int64_t)(n_heads + 2 * n_kv_heads) * head_dim;
  const int64_t kv_elems = (int64_t)L * max_ctx * row;
  size_t off = 0;
  auto carve = [&](size_t bytes) {
    const size_t o = off;
    off += (bytes + 255) / 256 * 256;
    return o;
  };
  const size_t o_kv = carve(kv_elems * 2), o_h = carve(H * 4), o_qkv = carve(nq * 4), o_q = carve(n_heads * head_dim * 4),
               o_o = carve(n_heads * head_dim * 4), o_a = carve(H * 4),
               o_po = carve((size_t)kDenseMaxSplits * n_heads * head_dim * 4),
               o_ml = carve((size_t)kDenseMaxSplits * n_heads * 8), o_sg = carve((size_t)L * 4),
               o_cnt = carve((size_t)n_heads * 4);
  FATE_CUDA(cudaMalloc(&g->dense_block, off));
  uint8_t *b = (uint8_t *)g->dense_block;
  g->ds = DenseScratch{(float *)(b + o_h), (float *)(b + o_qkv), (float *)(b + o_q), (float *)(b + o_o),
                       (float *)(b + o_po), (float *)(b + o_a), (float2 *)(b + o_ml), (unsigned *)(b + o_cnt)};
  FATE_CUDA(cudaMemsetAsync(b + o_cnt, 0, (size_t)n_heads * 4, g->cstream));
  g->shared_gate_dev = (float *)(b + o_sg);
  // the prompt's K/V (positions < ctx0 of every layer): synthetic, deterministic
  FATE_CUDA(launch_fill_kv((__nv_bfloat16 *)(b + o_kv), kv_elems, 0x9e3779b9u, g->cstream));
  FATE_CUDA(cudaStreamSynchronize(g->cstream));
  g->dd = DenseDims{H, n_heads, n_kv_heads, head_dim, eps, rope_theta, kDenseMaxSplits};
  g->max_ctx = max_ctx;
  g->ctx0 = ctx0;
  g->dl.assign(L, DenseLayer{});
  for (int l = 0; l < L; ++l) {
    g->dl[l].kv = (__nv_bfloat16 *)(b + o_kv) + (int64_t)l * max_ctx * row;
    g->dl[l].shared_gate_out = g->shared_gate_dev + l;
  }
  g->dense = false;  // until every layer has its weights
  return FATE_OK;
}

extern "C" int fate_engine_set_dense_layer(fate_engine *g, int layer, const void *wqkv, const float *bqkv,
                                           const float *norm, const void *wo, const float *shared_gate_w) {
  if (!g->dense_block || layer < 0 || layer >= g->cfg.num_layers || !wqkv || !norm || !wo) {
    set_error("fate_engine_set_dense_layer: call fate_engine_set_dense first; wqkv, norm and wo are required");
    return FATE_EINVAL;
  }
  DenseLayer &D = g->dl[layer];
  D.wqkv = (const __nv_bfloat16 *)wqkv;
  D.bqkv = bqkv;
  D.norm = norm;
  D.wo = (const __nv_bfloat16 *)wo;
  D.shared_gate = shared_gate_w;
  bool all = true, gated = false;
  for (const DenseLayer &x : g->dl) all = all && x.wqkv, gated = gated || x.shared_gate;
  g->dense = all;
  // K1 reads the gate only when every layer is gated (else the shared weight stays 1)
  bool every = all;
  for (const DenseLayer &x : g->dl) every = every && x.shared_gate;
  g->d.shared_gate = all && every && gated ? g->shared_gate_dev : nullptr;
  return FATE_OK;
}

extern "C" int fate_engine_set_shared(fate_engine *g, int layer, const uint8_t *buf_dev) {
  if (layer < 0 || layer >= g->cfg.num_layers || !g->cfg.shared_intermediate) {
    set_error("fate_engine_set_shared: bad layer or engine has no shared expert");
    return FATE_EINVAL;
  }
  g->shared_dev[layer] = buf_dev;
  FATE_CUDA(cudaMemcpy(g->shared_table_dev, g->shared_dev.data(), g->cfg.num_layers * sizeof(void *),
                       cudaMemcpyHostToDevice));
  return FATE_OK;
}

extern "C" int fate_engine_reset_cache(fate_engine *g) {
  engine_reset_kernel<<<64, 256, 0, g->cstream>>>(g->d, g->caps_dev);
  FATE_CHECK_LAUNCH("engine_reset_kernel");
  FATE_CUDA(cudaStreamSynchronize(g->cstream));
  return FATE_OK;
}

extern "C" int fate_engine_seed_resident(fate_engine *g, int layer, const int32_t *experts, int n) {
  if (layer < 0 || layer >= g->cfg.num_layers || n < 0 || n > FATE_MAX_EXPERTS) {
    set_error("fate_engine_seed_resident: bad arguments");
    return FATE_EINVAL;
  }
  int32_t *ex = g->scratch_i, *loads = g->scratch_i + FATE_MAX_EXPERTS;
  FATE_CUDA(cudaMemcpy(ex, experts, n * 4, cudaMemcpyHostToDevice));
  arc_seed_kernel<<<1, 32, 0, g->cstream>>>(g->d, layer, ex, n, loads);
  FATE_CHECK_LAUNCH("arc_seed_kernel");
  FATE_CUDA(cudaStreamSynchronize(g->cstream));
  return copy_to_buffers(g, loads, layer, g->cfg.cached_bits);
}

extern "C" int fate_engine_resident(fate_engine *g, int layer, int32_t *out) {
  if (layer < 0 || layer >= g->cfg.num_layers) {
    set_error("fate_engine_resident: bad layer");
    return FATE_EINVAL;
  }
  FATE_CUDA(cudaStreamSynchronize(g->cstream));
  std::vector<int32_t> h(g->cfg.num_experts);
  FATE_CUDA(cudaMemcpy(h.data(), g->d.buf_of + layer * g->cfg.num_experts, h.size() * 4, cudaMemcpyDeviceToHost));
  for (int e = 0; e < g->cfg.num_experts; ++e) out[e] = h[e] >= 0;
  return FATE_OK;
}

extern "C" int fate_engine_access(fate_engine *g, int layer, const int32_t *experts, int n, int32_t *hits) {
  if (layer < 0 || layer >= g->cfg.num_layers || n < 0 || n > FATE_MAX_EXPERTS) {
    set_error("fate_engine_access: bad arguments");
    return FATE_EINVAL;
  }
  for (int i = 0; i < n; ++i)
    if (experts[i] < 0 || experts[i] >= g->cfg.num_experts) {
      set_error("fate_engine_access: expert id out of range");
      return FATE_EINVAL;
    }
  int32_t *ex = g->scratch_i, *loads = g->scratch_i + FATE_MAX_EXPERTS + 1;
  int32_t *hits_dev = g->scratch_i + 3 * FATE_MAX_EXPERTS + 3;
  if (n == 0) return FATE_OK;
  FATE_CUDA(cudaMemcpy(ex, experts, n * 4, cudaMemcpyHostToDevice));
  arc_access_kernel<<<1, 32, 0, g->cstream>>>(g->d, layer, ex, n, hits_dev, loads);
  FATE_CHECK_LAUNCH("arc_access_kernel");
  FATE_CUDA(cudaStreamSynchronize(g->cstream));
  FATE_CUDA(cudaMemcpy(hits, hits_dev, n * 4, cudaMemcpyDeviceToHost));
  return copy_to_buffers(g, loads, layer, g->cfg.cached_bits);
}

extern "C" int fate_engine_arc_state(fate_engine *g, int layer, int32_t *t1, int32_t *t2, int32_t *b1, int32_t *b2,
                                     int32_t *lens, double *p) {
  if (layer < 0 || layer >= g->cfg.num_layers) {
    set_error("fate_engine_arc_state: bad layer");
    return FATE_EINVAL;
  }
  FATE_CUDA(cudaStreamSynchronize(g->cstream));
  ArcLayer a;
  FATE_CUDA(cudaMemcpy(&a, g->d.arc + layer, sizeof(a), cudaMemcpyDeviceToHost));
  const int E = g->cfg.num_experts;
  memcpy(t1, a.t1, std::min(a.n1, E) * 4);
  memcpy(t2, a.t2, std::min(a.n2, E) * 4);
  memcpy(b1, a.b1, std::min(a.nb1, E) * 4);
  memcpy(b2, a.b2, std::min(a.nb2, E) * 4);
  lens[0] = a.n1, lens[1] = a.n2, lens[2] = a.nb1, lens[3] = a.nb2;
  *p = a.p;
  return FATE_OK;
}

// ---------------------------------------------------------------------------
// The transfer channel on the host (pipeline.py:163-264 semantics).

namespace {

struct Channel {
  fate_engine *g;
  std::deque<Transfer> pending;
  std::deque<Inflight> inflight;
  uint32_t submitted = 0;
  int64_t h2d_bytes = 0, d2d_bytes = 0, done = 0, dropped = 0;
  bool timed = false;
  cudaEvent_t t0 = nullptr;      // run start, for absolute copy timestamps
  std::vector<cudaEvent_t> ev;  // pairs, recycled through ev_free once reaped
  std::vector<int> ev_free;
  double copy_ms = 0.0;

  int bytes_of(int bits) const { return (int)buffer_bytes(g->cfg.hidden_dim, g->cfg.intermediate_dim, bits); }

  // launch-serialised mode: completions are seen through events and every flag
  // is set by this thread (no stream memory operations at all)
  bool serial = false;
  bool mark_all = false;  // landed marks behind on-demand copies too (arrival-gated K3)
  std::vector<cudaEvent_t> sev;  // one per in-flight slot
  std::vector<int> sev_free;
  ~Channel() {
    for (auto &e : sev) cudaEventDestroy(e);
  }
  int init_serial() {
    serial = true;
    sev.resize(g->cfg.max_inflight + 2 * FATE_MAX_TOPK + 4);
    for (auto &e : sev) FATE_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    for (int i = (int)sev.size() - 1; i >= 0; --i) sev_free.push_back(i);
    return FATE_OK;
  }

  uint32_t submitted_s[2] = {0u, 0u};
  int next_stream = 0;
  // Copy timing: an event pair around every stride-th copy only.  Each stream op
  // between two copies costs the DMA engine ~7 us of the next copy's start, so
  // timing every copy slowed cold decode by 7 %; the sampled copies' busy time,
  // scaled by bytes, estimates the channel's busy time (copy_busy_ms).
  int stride = 8;
  uint64_t nsub = 0;
  int64_t sampled_bytes = 0;

  // Transfers alternate between two copy streams (two DMA engines), in the
  // channel's FIFO submission order; the completion of each stream is a
  // per-stream counter written behind its copies.  A step's wait flag is
  // written on the stream of the last transfer the step needs, after waiting
  // for the other stream's last copy, so it still follows every one of them.
  //
  // A buffer can be released while a copy into it is still running (a prefetch
  // the gate did not choose is dropped after it started) and be handed to the
  // next transfer at once.  That transfer goes to the same copy stream as the
  // running one, so stream order serialises the two writes and their landed
  // marks (the generation K1 and K3 compare against never goes backwards).
  std::vector<int> buf_si;        // stream of the last copy into each buffer (-1: none)
  std::vector<uint32_t> buf_seq;  // its per-stream sequence number
  int stream_for(int buf) {
    if ((size_t)buf >= buf_si.size()) buf_si.resize(buf + 1, -1), buf_seq.resize(buf + 1, 0u);
    const int last = buf_si[buf];
    if (last >= 0) {
      if (serial) return last;  // completions are not counted per stream there
      const uint32_t c = last ? *g->copy_done_host2 : *g->copy_done_host;
      if ((int32_t)(c - buf_seq[buf]) < 0) return last;  // still in flight
    }
    const int si = next_stream;
    next_stream ^= 1;
    return si;
  }

  int submit_one(const Transfer &t) {
    const int si = t.kind == 2 ? 0 : stream_for(t.buf);
    const cudaStream_t s = si ? g->xstream2 : g->xstream;
    int evi = -1;
    if (t.kind != 2) {
      buf_si[t.buf] = si;
      buf_seq[t.buf] = submitted_s[si] + 1u;  // the sseq this submission gets below
      if (!g->host_pool[t.bits]) {
        set_error("no pinned host pool registered for a requested bit width");
        return FATE_EINVAL;
      }
      const int64_t bytes = bytes_of(t.bits);
      const int64_t le = (int64_t)t.layer * g->cfg.num_experts + t.expert;
      const auto &tab = g->src_table[t.bits];
      const uint8_t *dsrc = tab.empty() ? nullptr : tab[le];  // expert-sharded mode: device / peer copy
      const uint8_t *src = dsrc ? dsrc : g->host_pool[t.bits] + le * g->host_stride[t.bits];
      if (timed && stride > 0 && (nsub++ % (uint64_t)stride) == 0 && !ev_free.empty()) {
        sampled_bytes += bytes;
        evi = ev_free.back();
        ev_free.pop_back();
        FATE_CUDA(cudaEventRecord(ev[evi], s));
      }
      FATE_CUDA(cudaMemcpyAsync(g->pool + (int64_t)t.buf * g->buf_stride, src, bytes,
                                dsrc ? cudaMemcpyDefault : cudaMemcpyHostToDevice, s));
      if (evi >= 0) FATE_CUDA(cudaEventRecord(ev[evi + 1], s));
      // landed marks: K1's arrival check of queued prefetches and, in the
      // arrival-gated decode, K3's per-expert gate (a write-value op behind a
      // copy does not delay the next one; an event record does)
      if ((t.kind == 0 || mark_all) && !serial)
        FATE_CU(p_write32((CUstream)s, (CUdeviceptr)(g->d.buf_done + t.buf), t.gen, 0));
      (dsrc ? d2d_bytes : h2d_bytes) += bytes;
    }
    if (serial) {
      // completion through an event; the host sets the step's flag when it reaps
      const int se = sev_free.back();
      sev_free.pop_back();
      FATE_CUDA(cudaEventRecord(sev[se], s));
      ++submitted;
      inflight.push_back(Inflight{submitted, t, evi, si, (uint32_t)se});
      return FATE_OK;
    }
    // the step's wait flag is released by the copy streams themselves right
    // after the last transfer the step needs (the host also sets it when reaping)
    if (t.signal_token >= 0) {
      // everything submitted so far on the other copy stream precedes the flag
      FATE_CUDA(cudaEventRecord(g->xlast[si ^ 1], si ? g->xstream : g->xstream2));
      FATE_CUDA(cudaStreamWaitEvent(s, g->xlast[si ^ 1], 0));
      FATE_CU(p_write32((CUstream)s, (CUdeviceptr)(g->ready_dev + t.signal_layer), (uint32_t)t.signal_token + 1u, 0));
    }
    ++submitted;
    const uint32_t sseq = ++submitted_s[si];
    // the stream's completion counter is written once behind the last transfer a
    // pump() call puts on it (flush_counters): stream ops between back-to-back
    // copies delay the copy engine; a later counter value also retires the
    // earlier transfers of the stream (stream order)
    counter_due[si] = true;
    inflight.push_back(Inflight{submitted, t, evi, si, sseq});
    return FATE_OK;
  }

  bool counter_due[2] = {false, false};
  int flush_counters() {
    if (serial) return FATE_OK;
    for (int si = 0; si < 2; ++si)
      if (counter_due[si]) {
        counter_due[si] = false;
        FATE_CU(p_write32((CUstream)(si ? g->xstream2 : g->xstream), si ? g->copy_done_dev2 : g->copy_done_dev,
                          submitted_s[si], 0));
      }
    return FATE_OK;
  }

  bool front_done() {
    const Inflight &f = inflight.front();
    if (serial) return cudaEventQuery(sev[f.sseq]) == cudaSuccess;
    const uint32_t c = f.stream ? *g->copy_done_host2 : *g->copy_done_host;
    return (int32_t)(c - f.sseq) >= 0;
  }

  void reap() {
    while (!inflight.empty() && front_done()) {
      Inflight &f = inflight.front();
      if (serial) sev_free.push_back((int)f.sseq);
      if (f.ev >= 0) {
        float ms = 0.f;
        if (cudaEventElapsedTime(&ms, ev[f.ev], ev[f.ev + 1]) == cudaSuccess) copy_ms += ms;
        float a = 0.f, b = 0.f;
        if (t0 && cudaEventElapsedTime(&a, t0, ev[f.ev]) == cudaSuccess &&
            cudaEventElapsedTime(&b, t0, ev[f.ev + 1]) == cudaSuccess) {
          g->copy_ms.push_back(a);
          g->copy_ms.push_back(b);
          const int32_t meta[5] = {f.t.kind, f.t.step, f.t.layer, f.t.expert, f.t.bits};
          g->copy_meta.insert(g->copy_meta.end(), meta, meta + 5);
        }
        ev_free.push_back(f.ev);
      }
      if (f.t.kind != 2) ++done;
      if (f.t.signal_token >= 0) g->ready_host[f.t.signal_layer] = (uint32_t)f.t.signal_token + 1u;
      inflight.pop_front();
    }
  }

  // Prefetches are submitted at most max_inflight at a time (pending ones stay
  // reorderable / droppable, as in the reference's queue); on-demand loads at the
  // front of the queue (promote_ondemand) are urgent and all go to the copy
  // engines at once, back to back, so no host round trip separates them.
  int pump() {
    reap();
    while (!pending.empty() && ((int)inflight.size() < g->cfg.max_inflight || pending.front().kind == 1)) {
      Transfer t = pending.front();
      pending.pop_front();
      if (int st = submit_one(t)) return st;
    }
    return flush_counters();
  }

  // promote_ondemand (pipeline.py:241-245): stable partition, on-demand first
  void promote() {
    std::stable_partition(pending.begin(), pending.end(), [](const Transfer &t) { return t.kind != 0; });
  }
};

}  // namespace

// one tagged word of a decode step message (engine_dev.cuh: DecodeMsg): K1
// stored it before the head the host already saw, so it is at most a few
// PCIe writes away
static int msg_word(const uint64_t *p, int step, uint64_t *out) {
  const uint32_t tag = msg_entry_tag(step);
  for (long spin = 0;; ++spin) {
    const uint64_t w = *(const volatile uint64_t *)p;
    if ((uint32_t)(w >> 56) == tag) {
      *out = w;
      return FATE_OK;
    }
    if (spin > (1l << 28)) {
      set_error("fate_engine_decode: a step-message entry never arrived");
      return FATE_ETIMEOUT;
    }
    _mm_pause();
  }
}
static inline int msg_e(uint64_t w) { return (int)((w >> 48) & 0xFF); }
static inline int msg_b(uint64_t w) { return (int)((w >> 32) & 0xFFFF); }
static inline uint32_t msg_g(uint64_t w) { return (uint32_t)w; }

extern "C" int fate_engine_decode(fate_engine *g, const double *gate_in_dev, const int32_t *chosen_dev, int T,
                                  float *y_dev, fate_step_log *log_dev, fate_run_stats *stats) {
  std::lock_guard<std::mutex> lock(g->mu);
  const int L = g->cfg.num_layers, H = g->cfg.hidden_dim;
  if (T < 0 || T > g->cfg.max_tokens) {
    set_error("fate_engine_decode: T exceeds max_tokens");
    return FATE_EINVAL;
  }
  fate_run_stats st{};
  if (T == 0) {
    if (stats) *stats = st;
    return FATE_OK;
  }
  if (!g->host_pool[g->cfg.ondemand_bits] || (g->cfg.use_predictor && !g->host_pool[g->cfg.prefetch_bits])) {
    set_error("fate_engine_decode: pinned host pool missing for the strategy's bit widths");
    return FATE_EINVAL;
  }
  if (g->cfg.shared_intermediate)
    for (int l = 0; l < L; ++l)
      if (!g->shared_dev[l]) {
        set_error("fate_engine_decode: shared expert buffer missing");
        return FATE_EINVAL;
      }
  cudaSetDevice(g->cfg.device);
  const bool timed = stats != nullptr;
  const int n_steps = T * L;
  Channel ch;
  ch.g = g;
  ch.timed = timed;
  ch.stride = g->copy_event_stride;
  if (serial_launches())
    if (int st = ch.init_serial()) return st;
  std::vector<cudaEvent_t> kev;  // per step: K1 start, K1 end, K3 start (after the wait), K3 end
  std::vector<cudaEvent_t> dev_;  // per step with the dense part: its start, end
  if (g->dense && g->ctx0 + T > g->max_ctx) {
    set_error("fate_engine_decode: prompt context + tokens exceed the dense part's max_ctx");
    return FATE_EINVAL;
  }
  if (timed) {
    ch.ev.resize(2 * (size_t)(g->cfg.max_inflight + 2 * FATE_MAX_TOPK + 4));
    for (auto &e : ch.ev) FATE_CUDA(cudaEventCreate(&e));
    for (int i = (int)ch.ev.size() - 2; i >= 0; i -= 2) ch.ev_free.push_back(i);
    kev.resize(4 * (size_t)n_steps);
    for (auto &e : kev) FATE_CUDA(cudaEventCreate(&e));
    if (g->dense) {
      dev_.resize(2 * (size_t)n_steps);
      for (auto &e : dev_) FATE_CUDA(cudaEventCreate(&e));
    }
    ch.t0 = g->dense ? dev_[0] : kev[0];
  }
  g->step_ms.clear();
  g->copy_ms.clear();
  g->copy_meta.clear();
  for (int l = 0; l < L; ++l) g->ready_host[l] = 0;
  *g->copy_done_host = 0;
  *g->copy_done_host2 = 0;
  memset(g->dring_host, 0, sizeof(DecodeMsg) * kRing);  // tags of an earlier run never match
  const cudaStream_t cs = g->cstream;
  if (getenv("FATE_DEBUG")) fprintf(stderr, "[fate] decode begin T=%d steps=%d\n", T, n_steps);
  run_begin_kernel<<<1, 1, 0, cs>>>(g->d);
  FATE_CHECK_LAUNCH("run_begin_kernel");
  FATE_CUDA(cudaStreamSynchronize(cs));
  if (getenv("FATE_DEBUG")) fprintf(stderr, "[fate] run_begin done\n");
  int launched = 0, processed = 0, k3_next = 0;
  int od_sent = -1;  // last step whose on-demand copies went out at the early post
  const int lookahead = 4;
  const bool k1_pdl = getenv("FATE_K1_NOPDL") == nullptr;  // experiment toggle
  const bool serial = serial_launches();
  // arrival-gated K3: launched right behind K1 (after the step's ARC update),
  // each expert's pieces start once its copy landed, so K3 works through the
  // resident experts while the copies are still on PCIe
  // (not with device-memory sources, expert-sharded mode: a device-to-device
  // cudaMemcpyAsync may run as a copy kernel, which a waiting K3 holding every
  // SM would never let start)
  bool dev_src = false;
  for (const auto &tab : g->src_table) dev_src = dev_src || !tab.empty();
  const bool overlap = g->k3_overlap && !serial && !dev_src;
  ch.mark_all = overlap;
  // per-step kernel events only on every layer of every stride-th token (and the
  // last step): an event record between K1 and K3 sits on the hand-off path, like
  // a copy's events; whole tokens keep every layer equally represented
  const int kstride = std::max(1, g->copy_event_stride);
  auto ksamp = [&](int s) { return timed && ((s / L) % kstride == 0 || s == n_steps - 1); };
  // K3 of step s (routed + shared experts), after the step's wait
  // FATE_HOSTPROF: host time spent in the launch calls (diagnostics)
  const bool hprof = getenv("FATE_HOSTPROF") != nullptr;
  double h_k3 = 0.0, h_k3max = 0.0, h_front = 0.0, h_frontmax = 0.0, h_msg = 0.0;
  auto hnow = [] { return std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now().time_since_epoch()).count(); };
  auto ffn_step = [&](int s) -> int {
    const int t = s / L, l = s % L;
    const double h0 = hprof ? hnow() : 0.0;
    if (ksamp(s)) FATE_CUDA(cudaEventRecord(kev[4 * s + 2], cs));
    FATE_CUDA(launch_ffn_decode_engine(g->d.batch, g->d.x, g->k3_scratch, y_dev + ((int64_t)t * L + l) * H, H,
                                       &g->d.stats->ffn, overlap ? g->d.buf_done : nullptr,
                                       overlap ? (const volatile uint32_t *)g->ready_dev : nullptr, cs));
    if (ksamp(s)) FATE_CUDA(cudaEventRecord(kev[4 * s + 3], cs));
    if (hprof) {
      const double d = hnow() - h0;
      h_k3 += d;
      h_k3max = std::max(h_k3max, d);
    }
    return FATE_OK;
  };
  int status = FATE_OK;
  auto last_progress = std::chrono::steady_clock::now();
  const int rows_pred = g->cfg.use_predictor && g->cfg.policy != 2 ? 2 : 1;  // EAP needs no W_{l+1} rows
  const bool dbg = getenv("FATE_DEBUG") != nullptr;
  auto last_beat = std::chrono::steady_clock::now();
  unsigned idle_spins = 0;
  while (processed < n_steps) {
    if (dbg && std::chrono::steady_clock::now() - last_beat > std::chrono::seconds(2)) {
      last_beat = std::chrono::steady_clock::now();
      fprintf(stderr, "[fate] beat processed=%d launched=%d pending=%zu inflight=%zu submitted=%u copy_done=%u seq=%u\n",
              processed, launched, ch.pending.size(), ch.inflight.size(), ch.submitted, *g->copy_done_host,
              (unsigned)(g->dring_host[processed % kRing].head >> 38));
    }
    // profiling mode (FATE_PROFILE_SERIAL, e.g. under ncu, which serializes
    // launches): K3 of a step is enqueued only after the host has serviced that
    // step's message and submitted its transfers, so the launch never blocks on
    // a stream wait that this thread itself must release.  Same decisions and
    // results; only the overlap is lost.
    while (serial && k3_next < launched && k3_next < processed) {
      const int s = k3_next, t = s / L, l = s % L;
      // every transfer this step needs has landed (the flag the stream waits on)
      while (((volatile uint32_t *)g->ready_host)[l] < (uint32_t)t + 1u) {
        if ((status = ch.pump())) break;
        _mm_pause();
        if (std::chrono::steady_clock::now() - last_progress > std::chrono::seconds(30)) {
          status = FATE_ETIMEOUT;
          set_error("fate_engine_decode: transfers of a step never completed (serial mode)");
          break;
        }
      }
      if (status) break;
      if ((status = ffn_step(s))) break;
      ++k3_next;
    }
    if (status) break;
    // enqueue compute for steps up to `lookahead` beyond the host's progress
    while (launched < n_steps && launched < processed + (serial ? 1 : lookahead) && (!serial || k3_next == launched)) {
      const int s = launched, t = s / L, l = s % L;
      const double hf0 = hprof ? hnow() : 0.0;
      // tail block + router rows of W_l (and W_{l+1} when predicting) + the x block
      const int rows = ((rows_pred == 2 && l + 1 < L) ? 2 * g->cfg.num_experts : g->cfg.num_experts) + 2;
      // any ARC update the side stream still runs (cache protocol calls before the run)
      if (s == 0) FATE_CUDA(cudaStreamWaitEvent(cs, g->ev_arc, 0));
      if (g->dense) {
        // the dense part of (t, l): attention block + shared-expert gate (dense.cu)
        if (ksamp(s)) FATE_CUDA(cudaEventRecord(dev_[2 * s], cs));
        const double *gi = gate_in_dev + ((int64_t)t * L + l) * H;
        if (l == 0) FATE_CUDA(launch_embed(gi, H, g->ds.a, cs));
        FATE_CUDA(launch_dense_step(g->dl[l], g->dd, g->ds.a, l == 0 ? nullptr : y_dev + ((int64_t)t * L + l - 1) * H,
                                    gi, g->ctx0 + t, g->ds, cs));
        if (ksamp(s)) FATE_CUDA(cudaEventRecord(dev_[2 * s + 1], cs));
      }
      if (ksamp(s)) FATE_CUDA(cudaEventRecord(kev[4 * s], cs));
      {
        // programmatic launch behind the previous K3 (its launch processing and
        // the router rows overlap K3's last CTAs; the tail and x blocks wait
        // for K3's completion before touching anything K3 reads).  Not with the
        // dense part, whose kernels produce K1's inputs.
        cudaLaunchConfig_t lc = {};
        lc.gridDim = dim3(rows);
        lc.blockDim = dim3(kGateThreads);
        lc.stream = cs;
        cudaLaunchAttribute la[1];
        la[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        la[0].val.programmaticStreamSerializationAllowed = 1;
        lc.attrs = la;
        lc.numAttrs = (k1_pdl && !g->dense && !serial && s > 0) ? 1 : 0;
        FATE_CUDA(cudaLaunchKernelEx(&lc, decode_gate_kernel, g->d, (const double *)gate_in_dev,
                                     (const int32_t *)chosen_dev, log_dev, l, (volatile uint32_t *)g->ready_dev, t));
      }
      FATE_CHECK_LAUNCH("decode_gate_kernel");
      if (ksamp(s)) FATE_CUDA(cudaEventRecord(kev[4 * s + 1], cs));
      // update_after_layer of this step (pipeline.py:483) runs inside K1 (warp 1
      // of the tail block), so K3 follows K1 directly on this stream
      if (dbg && s < 2) fprintf(stderr, "[fate] launched K1 step %d\n", s);
      // serial mode: no stream wait at all (the host enqueues K3 only once the flag is set);
      // arrival-gated: K3 itself waits per expert
      if (!overlap && !serial)
        FATE_CU(p_wait32((CUstream)cs, (CUdeviceptr)(g->ready_dev + l), (uint32_t)t + 1u, CU_STREAM_WAIT_VALUE_GEQ));
      if (dbg && s < 2) fprintf(stderr, "[fate] enqueued wait step %d\n", s);
      if (!serial && (status = ffn_step(s))) break;
      if (dbg && s < 2) fprintf(stderr, "[fate] launched K3 step %d\n", s);
      ++launched;
      if (hprof) {
        const double d = hnow() - hf0;
        h_front += d;
        h_frontmax = std::max(h_frontmax, d);
      }
    }
    // service the step message of the next unprocessed step
    DecodeMsg &m = g->dring_host[processed % kRing];
    const uint64_t head = *(volatile uint64_t *)&m.head;
    const bool head_ok = (uint32_t)(head >> 38) == msg_head_tag(processed);
    // arrival-gated: the on-demand copies start as soon as K1 posts the set
    // (they go ahead of every queued prefetch, as promote_ondemand orders them)
    if (overlap && od_sent != processed && !head_ok) {
      const uint64_t oh = *(volatile uint64_t *)&m.od_head;
      if ((uint32_t)(oh >> 32) == (uint32_t)processed + 1u) {
        const int t = processed / L, l = processed % L;
        const int n_od = (int)((oh >> 23) & 0x1FF), od_bits = (int)((oh >> 18) & 31);
        for (int i = 0; i < n_od && status == FATE_OK; ++i) {
          uint64_t w;
          if ((status = msg_word(&m.od[i], processed, &w))) break;
          status = ch.submit_one(Transfer{1, t, l, msg_e(w), od_bits, msg_b(w), msg_g(w), -1, -1});
        }
        if (status == FATE_OK) status = ch.flush_counters();
        if (status) break;
        od_sent = processed;
      }
    }
    if (head_ok) {
      const double hm0 = hprof ? hnow() : 0.0;
      const int t = processed / L, l = processed % L;
      const int n_need = (int)((head >> 24) & 0x1FF), n_drop = (int)((head >> 15) & 0x1FF);
      const int n_pf = (int)((head >> 6) & 0x1FF), pf_bits = (int)((head >> 1) & 31);
      const int n_od_h = (int)((head >> 33) & 31);
      const bool self_signaled = head & 1u;
      uint64_t w;
      // drop queued prefetches for this step that the gate did not choose
      for (int i = 0; i < n_drop && status == FATE_OK; ++i) {
        if ((status = msg_word(&m.drop[i], processed, &w))) break;
        const int e = msg_e(w);
        auto it = std::find_if(ch.pending.begin(), ch.pending.end(), [&](const Transfer &x) {
          return x.kind == 0 && x.layer == l && x.expert == e && x.step == t;
        });
        if (it != ch.pending.end()) {
          ch.pending.erase(it);
          ++ch.dropped;
        }
      }
      // prefetches for layer l+1 (issued at gate start, pipeline.py:414-417)
      for (int i = 0; i < n_pf && status == FATE_OK; ++i) {
        if ((status = msg_word(&m.pf[i], processed, &w))) break;
        ch.pending.push_back(Transfer{0, t, l + 1, msg_e(w), pf_bits, msg_b(w), msg_g(w), -1, -1});
      }
      // on-demand loads for this step, promoted ahead of every prefetch (unless
      // already submitted when the set was posted)
      if (od_sent != processed && n_od_h > 0 && status == FATE_OK) {
        // od_head may still be on its way (the head can overtake it)
        uint64_t oh = 0;
        for (long spin = 0;; ++spin) {
          oh = *(volatile uint64_t *)&m.od_head;
          if ((uint32_t)(oh >> 32) == (uint32_t)processed + 1u) break;
          if (spin > (1l << 28)) {
            status = FATE_ETIMEOUT;
            set_error("fate_engine_decode: a step's on-demand set never arrived");
            break;
          }
          _mm_pause();
        }
        const int n_od = status == FATE_OK ? n_od_h : 0, od_bits = (int)((oh >> 18) & 31);
        for (int i = 0; i < n_od && status == FATE_OK; ++i) {
          if ((status = msg_word(&m.od[i], processed, &w))) break;
          ch.pending.push_back(Transfer{1, t, l, msg_e(w), od_bits, msg_b(w), msg_g(w), -1, -1});
        }
      }
      if (status) break;
      ch.promote();
      if (!self_signaled && !overlap) {
        // the compute stream may proceed once every needed transfer landed:
        // attach the signal to the last needed one still queued, else signal
        // behind everything already submitted.
        int need_e[EMAX];
        for (int j = 0; j < n_need && status == FATE_OK; ++j) {
          status = msg_word(&m.need[j], processed, &w);
          need_e[j] = msg_e(w);
        }
        if (status) break;
        int last = -1;
        for (int i = 0; i < (int)ch.pending.size(); ++i) {
          const Transfer &x = ch.pending[i];
          bool need = x.kind == 1 && x.layer == l && x.step == t;
          for (int j = 0; !need && j < n_need; ++j) need = x.kind == 0 && x.layer == l && x.expert == need_e[j];
          if (need) last = i;
        }
        if (last >= 0) {
          ch.pending[last].signal_token = t;
          ch.pending[last].signal_layer = l;
        } else {
          ch.pending.push_front(Transfer{2, t, l, -1, 0, -1, 0, t, l});
        }
      }
      {
        // clear every word of this step's message: a slot's entries are reused 64
        // steps later, and an entry tag only has 7 bits of step, so a stale word
        // must never be left for a later step to mistake for its own
        const int n_od_w = n_od_h;
        volatile uint64_t *vm = reinterpret_cast<volatile uint64_t *>(&m);
        auto clear = [&](const uint64_t *w, int n) {
          for (int i = 0; i < n; ++i) vm[&w[i] - reinterpret_cast<const uint64_t *>(&m)] = 0;
        };
        clear(m.od, n_od_w);
        clear(m.need, n_need);
        clear(m.drop, n_drop);
        clear(m.pf, n_pf);
        vm[0] = 0;  // od_head
        vm[1] = 0;  // head
      }
      if (dbg)
        fprintf(stderr, "[fate] msg step=%d t=%d l=%d self=%d need=%d drop=%d pf=%d pending=%zu inflight=%zu\n",
                processed, t, l, (int)self_signaled, n_need, n_drop, n_pf, ch.pending.size(), ch.inflight.size());
      ++processed;
      last_progress = std::chrono::steady_clock::now();
      if ((status = ch.pump())) break;
      if (hprof) h_msg += hnow() - hm0;
    }
    // (not between the two halves of a step's message: queued prefetches of this
    // step may still be dropped)
    if (od_sent != processed && (status = ch.pump())) break;
    if (!head_ok) {
      _mm_pause();
      // the fault / watchdog checks cost a driver call: every 256th idle spin, so
      // the poll for the next message word stays a few hundred ns
      if ((++idle_spins & 255u) != 0u) continue;
      const cudaError_t qe = cudaStreamQuery(cs);
      if (qe != cudaSuccess && qe != cudaErrorNotReady) {
        status = cuda_status(qe, "decode compute stream (device fault)");
        break;
      }
      if (std::chrono::steady_clock::now() - last_progress > std::chrono::seconds(30)) {
        // watchdog: release the compute stream so the GPU is never left hung
        for (int l = 0; l < L; ++l) g->ready_host[l] = 0x7FFFFFFFu;
        status = FATE_ETIMEOUT;
        set_error("fate_engine_decode: no progress for 30 s (copy or kernel stalled)");
        break;
      }
    }
  }
  if (status != FATE_OK) {
    // never leave the compute stream parked on a flag nobody will write
    for (int l = 0; l < L; ++l) g->ready_host[l] = 0x7FFFFFFFu;
    std::atomic_thread_fence(std::memory_order_seq_cst);
  }
  if (hprof) {
    fprintf(stderr, "[fate] host us/step: launch block %.2f (max %.1f) of which K3 launch %.2f (max %.1f); "
            "message service + submit %.2f\n", h_front / n_steps, h_frontmax, h_k3 / n_steps, h_k3max, h_msg / n_steps);
    cudaStreamSynchronize(cs);
    DevStats dsp{};
    cudaMemcpy(&dsp, g->d.stats, sizeof(dsp), cudaMemcpyDeviceToHost);
    unsigned long long acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
#ifdef FATE_PROF
    cudaMemcpyFromSymbol(acc, g_k1_acc, sizeof(acc));
    const unsigned long long z[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    cudaMemcpyToSymbol(g_k1_acc, z, sizeof(z));
    if (acc[6])
      fprintf(stderr, "[fate] K1 warp-1 ARC update from K1 block start: begins %.2f us, ends %.2f us\n",
              acc[4] * 1e-3 / acc[6], acc[5] * 1e-3 / acc[6]);
    unsigned long long upd[4] = {0, 0, 0, 0};
    cudaMemcpyFromSymbol(upd, g_k1_upd, sizeof(upd));
    cudaMemcpyToSymbol(g_k1_upd, z, sizeof(upd));
    if (upd[2])
      fprintf(stderr, "[fate] K1 warp-1 ARC update: accesses %.2f us, list store %.2f us\n", upd[0] * 1e-3 / upd[2],
              upd[1] * 1e-3 / upd[2]);
#endif
    fprintf(stderr, "[fate] device us/step: K3 tail after its last gate opened %.2f (%llu launches waited); "
            "K3 last CTA end -> K1 block start %.2f; K1 block start -> message posted %.2f; "
            "K1 posted -> K3 CTA 0 start %.2f (profiling builds)\n",
            dsp.ffn.tail_n ? dsp.ffn.tail_ns * 1e-3 / dsp.ffn.tail_n : 0.0, dsp.ffn.tail_n,
            acc[1] ? acc[0] * 1e-3 / acc[1] : 0.0, acc[3] ? acc[2] * 1e-3 / acc[3] : 0.0,
            dsp.ffn.k1k3_n ? dsp.ffn.k1k3_ns * 1e-3 / dsp.ffn.k1k3_n : 0.0);
  }
  if (getenv("FATE_DEBUG"))
    fprintf(stderr, "[fate] decode loop exit status=%d processed=%d/%d pending=%zu inflight=%zu err=%s\n", status,
            processed, n_steps, ch.pending.size(), ch.inflight.size(), g_err.c_str());
  // drain remaining copies (stale prefetches for a layer past the end)
  while (status == FATE_OK && (!ch.pending.empty() || !ch.inflight.empty())) {
    // every message has been processed: whatever is still queued was needed by
    // some step (unneeded prefetches were dropped at their step), so finish it
    if ((status = ch.pump())) break;
    _mm_pause();
    if (std::chrono::steady_clock::now() - last_progress > std::chrono::seconds(30)) {
      status = FATE_ETIMEOUT;
      set_error("fate_engine_decode: copies never completed while draining");
      for (int l = 0; l < L; ++l) g->ready_host[l] = 0x7FFFFFFFu;
      break;
    }
  }
  // profiling mode: the last step's K3 (its transfers were drained above)
  while (status == FATE_OK && serial && k3_next < launched) {
    if ((status = ffn_step(k3_next))) break;
    ++k3_next;
  }
  cudaStreamWaitEvent(cs, g->ev_arc, 0);
  arc_update_kernel<<<1, 32, 0, cs>>>(g->d, log_dev);
  cudaError_t fe = cudaGetLastError();
  cudaError_t se = cudaStreamSynchronize(cs);
  if (se == cudaSuccess) se = cudaStreamSynchronize(g->astream);
  cudaError_t xe = cudaStreamSynchronize(g->xstream);
  if (xe == cudaSuccess) xe = cudaStreamSynchronize(g->xstream2);
  if (status == FATE_OK && fe != cudaSuccess) status = cuda_status(fe, "arc_update_kernel");
  if (status == FATE_OK && se != cudaSuccess) status = cuda_status(se, "decode compute stream");
  if (status == FATE_OK && xe != cudaSuccess) status = cuda_status(xe, "decode copy stream");
  DevStats ds{};
  Ctrl cc{};
  if (status == FATE_OK) {
    FATE_CUDA(cudaMemcpy(&ds, g->d.stats, sizeof(ds), cudaMemcpyDeviceToHost));
    FATE_CUDA(cudaMemcpy(&cc, g->d.ctrl, sizeof(cc), cudaMemcpyDeviceToHost));
    if (cc.err) {
      set_error("fate_engine_decode: staging buffer pool exhausted");
      status = FATE_ENOMEM;
    }
  }
  if (timed && status == FATE_OK) {
    float ms = 0.f;
    const cudaEvent_t t0 = ch.t0;
    cudaEventElapsedTime(&ms, t0, kev[4 * (n_steps - 1) + 3]);
    st.gpu_ms = ms;
    double ffn = 0.0, gate = 0.0, dense = 0.0;
    int n_samp = 0;
    g->step_ms.assign(4 * (size_t)n_steps, std::nan(""));  // unsampled steps stay NaN
    for (int s = 0; s < n_steps; ++s) {
      if (!ksamp(s)) continue;
      ++n_samp;
      float t[4] = {0.f, 0.f, 0.f, 0.f};
      for (int j = 0; j < 4; ++j)
        if (s || j || g->dense) cudaEventElapsedTime(&t[j], t0, kev[4 * s + j]);
      for (int j = 0; j < 4; ++j) g->step_ms[4 * (size_t)s + j] = t[j];
      gate += t[1] - t[0];
      ffn += t[3] - t[2];
      if (g->dense) {
        float d = 0.f;
        cudaEventElapsedTime(&d, dev_[2 * s], dev_[2 * s + 1]);
        dense += d;
      }
    }
    // sampled sums scaled to every step
    const double scale = n_samp ? (double)n_steps / n_samp : 0.0;
    st.ffn_ms = ffn * scale;
    st.gate_ms = gate * scale;
    st.dense_ms = dense * scale;
  }
  if (timed) {
    for (auto &e : ch.ev) cudaEventDestroy(e);
    for (auto &e : kev) cudaEventDestroy(e);
    for (auto &e : dev_) cudaEventDestroy(e);
  }
  st.steps = n_steps;
  st.accesses = (int64_t)ds.accesses;
  st.cache_hits = (int64_t)ds.cache_hits;
  st.arrival_hits = (int64_t)ds.arrival_hits;
  st.dequant_count = (int64_t)ds.dequant_count;
  st.prefetch_issued = (int64_t)ds.prefetch_issued;
  st.ondemand_issued = (int64_t)ds.ondemand_issued;
  st.transfers_done = ch.done;
  st.transfers_dropped = ch.dropped;
  st.h2d_bytes = ch.h2d_bytes;
  st.d2d_bytes = ch.d2d_bytes;
  // busy time of the sampled copies, scaled to every byte the channel moved
  st.copy_busy_ms = ch.sampled_bytes > 0 ? ch.copy_ms * (double)(ch.h2d_bytes + ch.d2d_bytes) / (double)ch.sampled_bytes
                                         : 0.0;
  st.recall_sum = ds.recall_sum;
  st.recall_n = (int64_t)ds.recall_n;
  st.trace_mismatches = (int64_t)ds.mismatches;
  st.near_ties = (int64_t)ds.near_ties;
  st.ffn_bytes = (int64_t)ds.ffn.bytes;
  st.k3_wait_ms = ds.ffn.wait_ns * 1e-6;
  st.error = status;
  if (stats) *stats = st;
  return status;
}

extern "C" int fate_engine_timeline(fate_engine *g, double *step_ms, int max_steps, double *copy_ms, int32_t *copy_meta,
                                    int max_copies, int32_t *counts) {
  const int ns = (int)(g->step_ms.size() / 4), nc = (int)(g->copy_ms.size() / 2);
  counts[0] = ns;
  counts[1] = nc;
  if (step_ms) memcpy(step_ms, g->step_ms.data(), sizeof(double) * 4 * std::min(ns, max_steps));
  if (copy_ms) memcpy(copy_ms, g->copy_ms.data(), sizeof(double) * 2 * std::min(nc, max_copies));
  if (copy_meta) memcpy(copy_meta, g->copy_meta.data(), sizeof(int32_t) * 5 * std::min(nc, max_copies));
  return FATE_OK;
}

extern "C" int fate_engine_set_strategy(fate_engine *g, const fate_engine_config *c) {
  if (int st = check_cfg(c)) return st;
  const int H = g->cfg.hidden_dim, I = g->cfg.intermediate_dim;
  for (int b : {c->prefetch_bits, c->ondemand_bits, c->cached_bits, c->prefill_ondemand_bits})
    if (buffer_bytes(H, I, b) > g->buf_stride) {
      set_error("fate_engine_set_strategy: strategy needs wider expert buffers than the engine was built with");
      return FATE_EINVAL;
    }
  g->cfg.cached_bits = c->cached_bits;
  g->cfg.prefetch_bits = c->prefetch_bits;
  g->cfg.ondemand_bits = c->ondemand_bits;
  g->cfg.use_predictor = c->use_predictor;
  g->cfg.policy = c->policy;
  g->cfg.percentile_q = c->percentile_q;
  g->cfg.budget_n = std::min(c->budget_n, g->cfg.num_experts);
  g->cfg.prefill_use_predictor = c->prefill_use_predictor;
  g->cfg.reorder_prefill = c->reorder_prefill;
  g->cfg.p_int2 = c->p_int2;
  g->cfg.prefill_ondemand_bits = c->prefill_ondemand_bits;
  if (c->max_inflight > 0) g->cfg.max_inflight = c->max_inflight;
  EngineDev &d = g->d;
  d.cached_bits = c->cached_bits;
  d.prefetch_bits = c->prefetch_bits;
  d.ondemand_bits = c->ondemand_bits;
  d.use_predictor = c->use_predictor;
  d.policy = c->policy;
  d.q = c->percentile_q;
  d.budget_n = g->cfg.budget_n;
  return FATE_OK;
}

// ===========================================================================
// Prefill (simulate_prefill, pipeline.py:536-778) on the device.
//
// Per layer l, on the compute stream:
//   prefill_x_kernel       X = sqrt(H) * gate_in[:, l]             (fp32)
//   K1p gate_batch x2      routing/order for layer l and for l+1 (top-k policy, pipeline.py:600)
//   prefill_plan_kernel    chosen sets, actives + counts, popularity profile
//                          of the l+1 predictions (prefill_merge) and its bit
//                          map (assign_bits), prefetch list for l+1 (skip
//                          resident), resident / requested / on-demand split of
//                          layer l, per-expert token lists for K4, host message
//   WAIT                   flag set once every needed copy landed
//   K4 up/down + combine   grouped dequant-fused SwiGLU over the actives (+ shared)
//   prefill_arc_kernel     update_after_layer(l, actives) with buffer hand-over
// The host processes the plan message at "block end": prefetches of layer l
// that have not been submitted yet are re-issued as on-demand loads at the
// on-demand width (drop_stale((0, l)) + pipeline.py:701-719).
// ===========================================================================

namespace fate {
namespace {

struct PfScratch {
  double *routing;   // [T, E] layer l
  int32_t *order;    // [T, E] layer l
  int32_t *order_n;  // [T, E] layer l+1
  float *X;          // [T, H]
  __nv_bfloat16 *Xb; // [T, H] the same rows in bf16 (K4 operand)
  int32_t *chosen;   // [T, k] ascending
  float *cw;         // [T, k]
  int32_t *tok_idx;  // [T*(k+1)]
  int32_t *zrow;     // [T*(k+1)]
  PrefillExpert *ex; // [E+1]
  int32_t *a_off;    // [E+1]
  int32_t *stage;    // [E] buffer used by each active expert in this layer
  int32_t *actives;  // [E]
  int32_t *victims;  // [L, E+1]: count then ids
  float *A;
  float *Z;
};

__global__ void prefill_x_kernel(const double *gate_in, int T, int L, int layer, int H, float *X,
                                 __nv_bfloat16 *Xb) {
  const double sH = sqrt((double)H);
  const int64_t n = (int64_t)T * H;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t t = i / H, h = i % H;
    const float x = (float)(sH * gate_in[(t * L + layer) * H + h]);
    X[i] = x;
    Xb[i] = __float2bfloat16_rn(x);
  }
}

__device__ void sort_by_count_desc(int32_t *ids, const int32_t *cnt, int n) {
  // insertion sort by (-count, id); n <= E <= 256, single thread
  for (int i = 1; i < n; ++i) {
    const int v = ids[i];
    int j = i;
    while (j > 0 && (cnt[ids[j - 1]] < cnt[v] || (cnt[ids[j - 1]] == cnt[v] && ids[j - 1] > v))) {
      ids[j] = ids[j - 1];
      --j;
    }
    ids[j] = v;
  }
}

// EAP prefill (pipeline.py:652-665), one thread per token, between layer l's
// gate and the plan kernel: record the token's transition l-1 -> l into the
// co-activation counts (eap_update; s.chosen still holds layer l-1), then
// write its EAP list for l+1 (eap_predict predict.py:141-158; top-k by
// (-score, id), cold start 0..k-1) into s.order_n for prefill_merge.
__global__ void eap_prefill_kernel(EngineDev d, PfScratch s, int layer, int T, int predict) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= T) return;
  const int E = d.E, k = d.k;
  int32_t cur[KMAX];
  for (int j = 0; j < k; ++j) cur[j] = s.order[(int64_t)t * E + j];
  for (int i = 1; i < k; ++i)
    for (int j = i; j > 0 && cur[j - 1] > cur[j]; --j) {
      const int x = cur[j];
      cur[j] = cur[j - 1];
      cur[j - 1] = x;
    }
  if (layer > 0) {
    int32_t *cnt = d.eap_counts + (int64_t)(layer - 1) * E * E;
    for (int i = 0; i < k; ++i) {
      const int a = s.chosen[t * k + i];
      for (int j = 0; j < k; ++j) atomicAdd(&cnt[a * E + cur[j]], 1);
      atomicAdd(&d.eap_totals[(layer - 1) * E + a], k);
    }
  }
  if (!predict) return;
  const int32_t *cnt = d.eap_counts + (int64_t)layer * E * E;
  const int32_t *tot = d.eap_totals + (int64_t)layer * E;
  int warm = 0;
  for (int j = 0; j < k; ++j) warm |= tot[cur[j]] != 0;
  int32_t *out = s.order_n + (int64_t)t * E;
  if (!warm) {
    for (int j = 0; j < k; ++j) out[j] = j;
    return;
  }
  double best[KMAX];
  int32_t bid[KMAX];
  int nb = 0;
  for (int e = 0; e < E; ++e) {
    double sc = 0.0;
    for (int j = 0; j < k; ++j) {
      const int a = cur[j];
      sc = __dadd_rn(sc, __ddiv_rn((double)cnt[a * E + e] + 1.0, (double)(tot[a] + E)));
    }
    // insert into the running top-k (ids ascend, so an equal score keeps the lower id first)
    int pos = nb;
    while (pos > 0 && sc > best[pos - 1]) --pos;
    if (pos >= k) continue;
    for (int i = (nb < k ? nb : k - 1); i > pos; --i) best[i] = best[i - 1], bid[i] = bid[i - 1];
    best[pos] = sc;
    bid[pos] = e;
    if (nb < k) ++nb;
  }
  for (int j = 0; j < k; ++j) out[j] = bid[j];
}

__global__ void __launch_bounds__(1024) prefill_plan_kernel(EngineDev d, PfScratch s, int layer, int T, int predict,
                                                            int reorder, double p_int2, int od_bits,
                                                            const int32_t *__restrict__ trace_chosen,
                                                            int32_t *shared_I_out) {
  __shared__ int32_t cnt[EMAX], pcnt[EMAX], fill[EMAX], order[EMAX], bits_of[EMAX], mark[EMAX];
  __shared__ int32_t first_seen[EMAX], fs_n;
  __shared__ int mism;
  const int E = d.E, k = d.k, L = d.L;
  for (int e = threadIdx.x; e < E; e += blockDim.x) cnt[e] = 0, pcnt[e] = 0, fill[e] = 0, mark[e] = 0;
  if (threadIdx.x == 0) mism = 0;
  __syncthreads();
  // (1) chosen sets of layer l (ascending) with their routing weights; counts
  for (int t = threadIdx.x; t < T; t += blockDim.x) {
    int32_t c[KMAX];
    for (int j = 0; j < k; ++j) c[j] = s.order[(int64_t)t * E + j];
    for (int i = 1; i < k; ++i)
      for (int j = i; j > 0 && c[j - 1] > c[j]; --j) {
        const int x = c[j];
        c[j] = c[j - 1];
        c[j - 1] = x;
      }
    // the trace's chosen set (record.chosen, ascending) drives actives and the
    // ARC update when supplied, as in the reference (pipeline.py:620-631); the
    // recomputed top-k only feeds the mismatch counter
    if (trace_chosen)
      for (int j = 0; j < k; ++j) {
        const int tc = trace_chosen[((int64_t)t * L + layer) * k + j];
        if (tc != c[j]) atomicExch(&mism, 1);
        c[j] = tc;
      }
    for (int j = 0; j < k; ++j) {
      s.chosen[t * k + j] = c[j];
      s.cw[t * k + j] = (float)s.routing[(int64_t)t * E + c[j]];
      atomicAdd(&cnt[c[j]], 1);
    }
    if (predict)
      for (int j = 0; j < k; ++j) atomicAdd(&pcnt[s.order_n[(int64_t)t * E + j]], 1);
  }
  __syncthreads();
  if (threadIdx.x != 0) return;
  StepMsg *msg = d.ring + (layer % kRing);
  if (mism) atomicAdd(&d.stats->mismatches, 1ull);
  msg->mismatch = mism;
  // (2) popularity profile of the predictions for l+1 (prefill_merge, assign_bits)
  int n_pf = 0, n_pred = 0;
  if (predict) {
    for (int e = 0; e < E; ++e)
      if (pcnt[e] > 0) order[n_pred++] = e;
    sort_by_count_desc(order, pcnt, n_pred);
    const int m = (int)floor(p_int2 * (double)n_pred);
    for (int i = 0; i < n_pred; ++i) {
      bits_of[order[i]] = d.prefetch_bits >= 16 ? 16 : (i >= n_pred - m ? 2 : 4);
      msg->pred_order[i] = order[i];
      msg->pred_cnt[i] = pcnt[order[i]];
    }
    int32_t *issue = order;
    int n_issue = n_pred;
    if (!reorder) {  // token-request order: token ascending, ids ascending within (pipeline.py:524-533)
      fs_n = 0;
      for (int t = 0; t < T; ++t) {
        int32_t c[KMAX];
        for (int j = 0; j < k; ++j) c[j] = s.order_n[(int64_t)t * E + j];
        for (int i = 1; i < k; ++i)
          for (int j = i; j > 0 && c[j - 1] > c[j]; --j) {
            const int x = c[j];
            c[j] = c[j - 1];
            c[j - 1] = x;
          }
        for (int j = 0; j < k; ++j)
          if (!mark[c[j]]) mark[c[j]] = 1, first_seen[fs_n++] = c[j];
      }
      for (int e = 0; e < E; ++e) mark[e] = 0;
      issue = first_seen;
      n_issue = fs_n;
    }
    for (int i = 0; i < n_issue; ++i) {
      const int e = issue[i];
      if (d.buf_of[(layer + 1) * E + e] >= 0 || d.pend_buf[(layer + 1) * E + e] >= 0) continue;
      const int b = pop_free(d);
      const uint32_t g = ++d.buf_gen[b];
      d.buf_bits[b] = bits_of[e];
      d.pend_buf[(layer + 1) * E + e] = b;
      d.pend_gen[(layer + 1) * E + e] = g;
      msg->pf_e[n_pf] = e;
      msg->pf_b[n_pf] = b;
      msg->pf_g[n_pf] = g;
      msg->pf_bits_each[n_pf] = bits_of[e];
      ++n_pf;
    }
    atomicAdd(&d.stats->prefetch_issued, (unsigned long long)n_pf);
  }
  msg->n_pred = n_pred;
  msg->n_pf = n_pf;
  // (3) actives of layer l and the resident / requested / on-demand split
  int n_act = 0, n_res = 0, n_need = 0, n_od = 0, n_arr = 0, n_deq = 0;
  bool all_landed = true;
  for (int e = 0; e < E; ++e)
    if (cnt[e] > 0) {
      s.actives[n_act] = e;
      msg->active_e[n_act] = e;
      msg->active_cnt[n_act] = cnt[e];
      ++n_act;
    }
  // recall of the layer-l prediction made one layer earlier (pipeline.py:676-680)
  Ctrl &C = *d.ctrl;
  if (C.pred_valid && C.pred_layer == layer && n_act > 0) {
    int inter = 0;
    for (int i = 0; i < C.pred_n; ++i) inter += cnt[C.pred_list[i]] > 0;
    d.stats->recall_sum += (double)inter / (double)n_act;
    d.stats->recall_n += 1;
  }
  // this layer's profile becomes the prediction checked at layer l+1
  C.pred_valid = predict;
  if (predict) {
    C.pred_n = n_pred;
    C.pred_layer = layer + 1;
    for (int i = 0; i < n_pred; ++i) C.pred_list[i] = msg->pred_order[i];
  }
  int32_t *od_order = first_seen;  // reuse as scratch for the on-demand order
  int n_unpl = 0;
  for (int i = 0; i < n_act; ++i) {
    const int e = s.actives[i];
    const int b = d.buf_of[layer * E + e];
    if (b >= 0) {
      s.stage[e] = b;
      msg->res_e[n_res++] = e;
      n_deq += (d.cached_bits < 16);
    } else if (d.pend_buf[layer * E + e] >= 0) {
      const int pb = d.pend_buf[layer * E + e];
      s.stage[e] = pb;
      const bool arr = ((volatile uint32_t *)d.buf_done)[pb] == d.pend_gen[layer * E + e];
      n_arr += arr;
      all_landed = all_landed && arr;
      msg->need_e[n_need] = e;
      msg->need_b[n_need] = pb;
      ++n_need;
    } else {
      od_order[n_unpl++] = e;
    }
  }
  if (reorder) sort_by_count_desc(od_order, cnt, n_unpl);
  else {  // first-seen order of this layer's chosen sets
    int nfs = 0;
    for (int t = 0; t < T && nfs < n_unpl; ++t)
      for (int j = 0; j < k; ++j) {
        const int e = s.chosen[t * k + j];
        bool unpl = false;
        for (int i = 0; i < n_unpl; ++i) unpl |= od_order[i] == e;
        if (unpl && !mark[e]) mark[e] = 1, fill[nfs++] = e;
      }
    for (int i = 0; i < n_unpl; ++i) od_order[i] = fill[i];
    for (int e = 0; e < E; ++e) mark[e] = 0, fill[e] = 0;
    // first-seen rank of every active expert: the host orders the on-demand
    // loads, prefetches converted at block end included, by it
    int r = 0;
    for (int t = 0; t < T && r < n_act; ++t)
      for (int j = 0; j < k; ++j) {
        const int e = s.chosen[t * k + j];
        if (!mark[e]) mark[e] = 1, fill[e] = r++;
      }
    for (int i = 0; i < n_act; ++i) msg->active_fs[i] = fill[s.actives[i]];
    for (int e = 0; e < E; ++e) mark[e] = 0, fill[e] = 0;
  }
  for (int i = 0; i < n_unpl; ++i) {
    const int e = od_order[i];
    const int b = pop_free(d);
    const uint32_t g = ++d.buf_gen[b];
    d.buf_bits[b] = od_bits;
    s.stage[e] = b;
    msg->od_e[n_od] = e;
    msg->od_b[n_od] = b;
    msg->od_g[n_od] = g;
    ++n_od;
    all_landed = false;
  }
  // prefetched for l but inactive: release + drop (pipeline.py:682)
  int n_drop = 0;
  for (int e = 0; e < E; ++e) {
    const int b = d.pend_buf[layer * E + e];
    if (b < 0) continue;
    d.pend_buf[layer * E + e] = -1;
    if (cnt[e] > 0) continue;
    msg->drop_e[n_drop] = e;
    msg->drop_b[n_drop] = b;
    ++n_drop;
    push_free(d, b);
  }
  // (4) token lists per active expert, in ascending expert order, tokens ascending
  int off = 0;
  int64_t aoff = 0;
  for (int i = 0; i < n_act; ++i) {
    const int e = s.actives[i];
    fill[e] = off;
    s.ex[i] = PrefillExpert{d.pool + (int64_t)s.stage[e] * d.buf_stride, d.I, 0, off, cnt[e]};
    s.a_off[i] = (int32_t)aoff;
    off += cnt[e];
    aoff += (int64_t)cnt[e] * d.I;
  }
  for (int t = 0; t < T; ++t)
    for (int j = 0; j < k; ++j) {
      const int e = s.chosen[t * k + j];
      const int pos = fill[e]++;
      s.tok_idx[pos] = t;
      s.zrow[pos] = t * (k + 1) + j;
    }
  int n_ex = n_act;
  if (d.shared && d.shared[layer]) {
    const int Is = d.I_shared;
    s.ex[n_ex] = PrefillExpert{d.shared[layer], Is, 0, off, T};
    s.a_off[n_ex] = (int32_t)aoff;
    for (int t = 0; t < T; ++t) {
      s.tok_idx[off + t] = t;
      s.zrow[off + t] = t * (k + 1) + k;
    }
    ++n_ex;
    *shared_I_out = Is;
  } else {
    *shared_I_out = 0;
  }
  // src bits: resident -> cached, requested -> its prefetch width, on-demand -> od width
  for (int i = 0; i < n_need; ++i) n_deq += (d.buf_bits[msg->need_b[i]] < 16);
  n_deq += n_od * (od_bits < 16);
  msg->n_active = n_act;
  msg->n_res = n_res;
  msg->n_need = n_need;
  msg->n_od = n_od;
  msg->n_drop = n_drop;
  msg->od_bits = od_bits;
  msg->pf_bits = d.prefetch_bits;
  msg->step = layer;
  msg->token = 0;
  msg->layer = layer;
  atomicAdd(&d.stats->accesses, (unsigned long long)n_act);
  atomicAdd(&d.stats->cache_hits, (unsigned long long)n_res);
  atomicAdd(&d.stats->arrival_hits, (unsigned long long)n_arr);
  atomicAdd(&d.stats->ondemand_issued, (unsigned long long)n_od);
  atomicAdd(&d.stats->dequant_count, (unsigned long long)n_deq);
  const int self = all_landed ? 1 : 0;
  msg->self_signaled = self;
  if (self) ((volatile uint32_t *)d.ready)[layer] = 1u;
  __threadfence_system();
  msg->seq = (uint32_t)layer + 1u;
  __threadfence_system();
}

// update_after_layer(l, actives) with buffer hand-over (cf. apply_prev_update).
__global__ void prefill_arc_kernel(EngineDev d, PfScratch s, int layer, int n_act) {
  __shared__ ArcLayer arc_sm;
  __shared__ int32_t rel[EMAX + 4];
  const int lane = threadIdx.x;
  WarpArc arc;
  arc.load(&d.arc[layer], &arc_sm);
  int nrel = 0, nvic = 0;
  int32_t *vic = s.victims + (int64_t)layer * (d.E + 1);
  for (int i = 0; i < n_act; ++i) {
    const int e = s.actives[i];
    int victim;
    const int hit = arc.access(e, &victim);
    if (lane == 0) {
      if (victim >= 0) {
        int32_t &slot = d.buf_of[layer * d.E + victim];
        if (slot >= 0) rel[nrel++] = slot;
        slot = -1;
        vic[1 + nvic++] = victim;
      }
      if (!hit) {
        const int b = s.stage[e];
        if (arc.c >= 1) {
          // the slot keeps the width that actually landed (a prefetch the host
          // re-issued as an on-demand load carries the narrower header)
          d.buf_bits[b] = reinterpret_cast<const ExpertHeader *>(d.pool + (int64_t)b * d.buf_stride)->bits;
          d.buf_of[layer * d.E + e] = b;
          for (int r = 0; r < nrel; ++r)
            if (rel[r] == b) rel[r] = rel[--nrel], r = nrel;
        } else {
          rel[nrel++] = b;
        }
      }
    }
    __syncwarp();
  }
  arc.store(&d.arc[layer]);
  if (lane == 0) {
    for (int r = 0; r < nrel; ++r) push_free(d, rel[r]);
    vic[0] = nvic;
  }
}

__global__ void prefill_begin_kernel(EngineDev d) {
  Ctrl &C = *d.ctrl;
  C.pred_valid = 0;
  C.err = 0;
  for (int i = 0; i < d.L * d.E; ++i) {
    if (d.pend_buf[i] >= 0) push_free(d, d.pend_buf[i]);
    d.pend_buf[i] = -1;
  }
  *d.stats = DevStats{};
}

}  // namespace
}  // namespace fate

static int ensure_prefill_scratch(fate_engine *g, PfScratch &s, int T) {
  const int E = g->cfg.num_experts, k = g->cfg.top_k, H = g->cfg.hidden_dim, L = g->cfg.num_layers;
  const int Tm = g->cfg.max_tokens;
  const int64_t a_floats = (int64_t)Tm * k * g->cfg.intermediate_dim + (int64_t)Tm * g->cfg.shared_intermediate;
  size_t off = 0;
  auto carve = [&](size_t bytes) {
    size_t o = off;
    off = (size_t)align_up((int64_t)(off + bytes), 256);
    return o;
  };
  const size_t o_r = carve((size_t)Tm * E * 8), o_o = carve((size_t)Tm * E * 4), o_on = carve((size_t)Tm * E * 4),
               o_x = carve((size_t)Tm * H * 4), o_xb = carve((size_t)Tm * H * 2), o_c = carve((size_t)Tm * k * 4), o_cw = carve((size_t)Tm * k * 4),
               o_ti = carve((size_t)Tm * (k + 1) * 4), o_zr = carve((size_t)Tm * (k + 1) * 4),
               o_ex = carve(sizeof(PrefillExpert) * (E + 1)), o_ao = carve(4 * (E + 1)), o_st = carve(4 * E),
               o_ac = carve(4 * E), o_v = carve(4 * (size_t)L * (E + 1)), o_si = carve(16),
               o_A = carve(4 * (size_t)a_floats), o_Z = carve(4 * (size_t)Tm * (k + 1) * H);
  if (!g->pf_block) FATE_CUDA(cudaMalloc(&g->pf_block, off));
  uint8_t *b = (uint8_t *)g->pf_block;
  s.routing = (double *)(b + o_r);
  s.order = (int32_t *)(b + o_o);
  s.order_n = (int32_t *)(b + o_on);
  s.X = (float *)(b + o_x);
  s.Xb = (__nv_bfloat16 *)(b + o_xb);
  s.chosen = (int32_t *)(b + o_c);
  s.cw = (float *)(b + o_cw);
  s.tok_idx = (int32_t *)(b + o_ti);
  s.zrow = (int32_t *)(b + o_zr);
  s.ex = (PrefillExpert *)(b + o_ex);
  s.a_off = (int32_t *)(b + o_ao);
  s.stage = (int32_t *)(b + o_st);
  s.actives = (int32_t *)(b + o_ac);
  s.victims = (int32_t *)(b + o_v);
  g->pf_shared_I = (int32_t *)(b + o_si);
  s.A = (float *)(b + o_A);
  s.Z = (float *)(b + o_Z);
  (void)T;
  return FATE_OK;
}

extern "C" int fate_engine_prefill(fate_engine *g, const double *gate_in_dev, const int32_t *chosen_dev, int T,
                                   float *Y_dev, fate_prefill_log *log_host, fate_run_stats *stats) {
  std::lock_guard<std::mutex> lock(g->mu);
  const int L = g->cfg.num_layers, E = g->cfg.num_experts, k = g->cfg.top_k, H = g->cfg.hidden_dim;
  const int I = g->cfg.intermediate_dim;
  if (T < 1 || T > g->cfg.max_tokens) {
    set_error("fate_engine_prefill: T must lie in [1, max_tokens]");
    return FATE_EINVAL;
  }
  const int predict = g->cfg.prefill_use_predictor && g->cfg.use_predictor;
  const int od_bits = g->cfg.prefill_ondemand_bits;
  if (!g->host_pool[od_bits] || (predict && g->cfg.prefetch_bits < 16 && (!g->host_pool[4] || !g->host_pool[2])) ||
      (predict && g->cfg.prefetch_bits >= 16 && !g->host_pool[16])) {
    set_error("fate_engine_prefill: pinned host pool missing for the strategy's bit widths");
    return FATE_EINVAL;
  }
  cudaSetDevice(g->cfg.device);
  PfScratch s;
  if (int st = ensure_prefill_scratch(g, s, T)) return st;
  const cudaStream_t cs = g->cstream;
  const bool timed = stats != nullptr;
  const bool dbg = getenv("FATE_DEBUG") != nullptr;
  Channel ch;
  ch.g = g;
  ch.timed = timed;
  ch.stride = g->copy_event_stride;
  if (serial_launches())
    if (int st = ch.init_serial()) return st;
  std::vector<cudaEvent_t> kev;
  if (timed) {
    ch.ev.resize(2 * (size_t)(g->cfg.max_inflight + 4));
    for (auto &e : ch.ev) FATE_CUDA(cudaEventCreate(&e));
    for (int i = (int)ch.ev.size() - 2; i >= 0; i -= 2) ch.ev_free.push_back(i);
    kev.resize(4 * (size_t)L);
    for (auto &e : kev) FATE_CUDA(cudaEventCreate(&e));
    ch.t0 = kev[0];
  }
  g->step_ms.clear();
  g->copy_ms.clear();
  g->copy_meta.clear();
  for (int l = 0; l < L; ++l) g->ready_host[l] = 0;
  *g->copy_done_host = 0;
  *g->copy_done_host2 = 0;
  for (int i = 0; i < kRing; ++i) g->ring_host[i].seq = 0, g->ring_host[i].seq_od = 0;
  EngineDev d = g->d;
  d.ready = g->ready_dev;
  prefill_begin_kernel<<<1, 1, 0, cs>>>(d);
  FATE_CHECK_LAUNCH("prefill_begin_kernel");
  FATE_CUDA(cudaStreamSynchronize(cs));
  double flops = 0.0;
  int status = FATE_OK;
  std::vector<double> tau(L);
  FATE_CUDA(cudaMemcpy(tau.data(), g->d.tau, L * 8, cudaMemcpyDeviceToHost));
  auto launch_front = [&](int l) -> int {
    if (timed) FATE_CUDA(cudaEventRecord(kev[4 * l], cs));
    prefill_x_kernel<<<148 * 4, 256, 0, cs>>>(gate_in_dev, T, L, l, H, s.X, s.Xb);
    FATE_CHECK_LAUNCH("prefill_x_kernel");
    FATE_CUDA(launch_gate_batch(g->d.W + (int64_t)l * E * H, tau[l], gate_in_dev + (int64_t)l * H, (int64_t)L * H, T,
                                E, H, s.routing, s.order, nullptr, k, 0, 0.5, cs));
    const int pred_here = predict && l + 1 < L;
    const bool eap = g->cfg.use_predictor && g->cfg.policy == 2;
    if (eap && (l > 0 || pred_here)) {
      eap_prefill_kernel<<<(T + 127) / 128, 128, 0, cs>>>(d, s, l, T, pred_here);
      FATE_CHECK_LAUNCH("eap_prefill_kernel");
    }
    if (pred_here && !eap)
      FATE_CUDA(launch_gate_batch(g->d.W + (int64_t)(l + 1) * E * H, tau[l + 1], gate_in_dev + (int64_t)l * H,
                                  (int64_t)L * H, T, E, H, nullptr, s.order_n, nullptr, k, 0, 0.5, cs));
    prefill_plan_kernel<<<1, 1024, 0, cs>>>(d, s, l, T, pred_here, g->cfg.reorder_prefill, g->cfg.p_int2, od_bits,
                                            chosen_dev, g->pf_shared_I);
    FATE_CHECK_LAUNCH("prefill_plan_kernel");
    if (timed) FATE_CUDA(cudaEventRecord(kev[4 * l + 1], cs));
    return FATE_OK;
  };
  if ((status = launch_front(0))) return status;
  std::vector<int> pf_bits_cur(E, 0);  // widths of the prefetches issued for the current layer
  auto last_progress = std::chrono::steady_clock::now();
  for (int l = 0; l < L && status == FATE_OK; ++l) {
    StepMsg &m = g->ring_host[l % kRing];
    while (m.seq != (uint32_t)l + 1u) {
      if ((status = ch.pump())) break;
      _mm_pause();
      if (std::chrono::steady_clock::now() - last_progress > std::chrono::seconds(60)) {
        status = FATE_ETIMEOUT;
        set_error("fate_engine_prefill: no plan message for 60 s");
        break;
      }
    }
    if (status) break;
    std::atomic_thread_fence(std::memory_order_acquire);
    last_progress = std::chrono::steady_clock::now();
    fate_prefill_log *lg = log_host ? log_host + l : nullptr;
    if (lg) memset(lg, 0, sizeof(*lg));
    // drop prefetches of layer l the gate did not activate
    for (int i = 0; i < m.n_drop; ++i) {
      auto it = std::find_if(ch.pending.begin(), ch.pending.end(),
                             [&](const Transfer &x) { return x.kind == 0 && x.layer == l && x.expert == m.drop_e[i]; });
      if (it != ch.pending.end()) ch.pending.erase(it), ++ch.dropped;
    }
    // block end: requested prefetches that have not started become on-demand loads
    std::vector<int> started, converted;
    for (int i = 0; i < m.n_need; ++i) {
      const int e = m.need_e[i];
      auto it = std::find_if(ch.pending.begin(), ch.pending.end(),
                             [&](const Transfer &x) { return x.kind == 0 && x.layer == l && x.expert == e; });
      if (it != ch.pending.end()) {
        Transfer t = *it;
        ch.pending.erase(it);
        ++ch.dropped;
        converted.push_back(e);
        (void)t;
      } else {
        started.push_back(e);
      }
    }
    std::vector<int> cnt(E, 0);
    for (int i = 0; i < m.n_active; ++i) cnt[m.active_e[i]] = m.active_cnt[i];
    // the on-demand set in (-count, id) order (pipeline.py:703-704); non-reordered strategies keep device order
    std::vector<std::pair<int, int>> od;  // expert, buffer
    std::vector<uint32_t> od_gen;
    for (int i = 0; i < m.n_od; ++i) od.push_back({m.od_e[i], m.od_b[i]});
    for (int i = 0; i < m.n_od; ++i) od_gen.push_back(m.od_g[i]);
    for (int e : converted) {
      int b = -1;
      for (int i = 0; i < m.n_need; ++i)
        if (m.need_e[i] == e) b = m.need_b[i];
      od.push_back({e, b});
      od_gen.push_back(0);
    }
    std::vector<int> idx(od.size());
    for (size_t i = 0; i < idx.size(); ++i) idx[i] = (int)i;
    if (g->cfg.reorder_prefill) {
      std::stable_sort(idx.begin(), idx.end(), [&](int a, int b) {
        const int ea = od[a].first, eb = od[b].first;
        return cnt[ea] != cnt[eb] ? cnt[ea] > cnt[eb] : ea < eb;
      });
    } else {
      // token-request (first-seen) order over every unplanned expert, converted
      // prefetches included (pipeline.py:701-719 with _first_seen_order :524-533)
      std::vector<int> rank(E, 1 << 30);
      for (int i = 0; i < m.n_active; ++i) rank[m.active_e[i]] = m.active_fs[i];
      std::stable_sort(idx.begin(), idx.end(), [&](int a, int b) { return rank[od[a].first] < rank[od[b].first]; });
    }
    // prefetches for l+1 (issued at predict_at, before this layer's on-demand loads)
    for (int i = 0; i < m.n_pf; ++i)
      ch.pending.push_back(Transfer{0, 0, l + 1, m.pf_e[i], m.pf_bits_each[i], m.pf_b[i], m.pf_g[i], -1, -1});
    for (int i : idx) {
      // converted prefetches reuse their buffer; bump the generation by the device's next value
      uint32_t gen = od_gen[i];
      ch.pending.push_back(Transfer{1, 0, l, od[i].first, od_bits, od[i].second, gen, -1, -1});
    }
    ch.promote();
    if (!m.self_signaled) {
      int last = -1;
      for (int i = 0; i < (int)ch.pending.size(); ++i)
        if (ch.pending[i].kind == 1 && ch.pending[i].layer == l) last = i;
      if (last >= 0) {
        ch.pending[last].signal_token = 0;
        ch.pending[last].signal_layer = l;
      } else {
        ch.pending.push_front(Transfer{2, 0, l, -1, 0, -1, 0, 0, l});
      }
    }
    if ((status = ch.pump())) break;
    // host log (timing-independent fields + this run's started set)
    if (lg) {
      lg->n_pred = m.n_pred;
      for (int i = 0; i < m.n_pred; ++i) lg->pred_order[i] = m.pred_order[i], lg->pred_counts[i] = m.pred_cnt[i];
      lg->n_prefetch = m.n_pf;
      for (int i = 0; i < m.n_pf; ++i) lg->prefetch[i] = m.pf_e[i], lg->prefetch_bits[i] = m.pf_bits_each[i];
      lg->n_active = m.n_active;
      for (int i = 0; i < m.n_active; ++i) lg->actives[i] = m.active_e[i], lg->counts[i] = m.active_cnt[i];
      lg->n_resident = m.n_res;
      for (int i = 0; i < m.n_res; ++i) lg->resident[i] = m.res_e[i];
      lg->n_started = (int)started.size();
      lg->n_planned = (int)started.size();
      for (size_t i = 0; i < started.size(); ++i) lg->started[i] = started[i], lg->planned[i] = started[i];
      lg->n_ondemand = (int)idx.size();
      for (size_t i = 0; i < idx.size(); ++i) lg->ondemand[i] = od[idx[i]].first;
      lg->mismatch = m.mismatch;
      for (int i = 0; i < m.n_active; ++i) {
        const int e = m.active_e[i];
        int b = g->cfg.cached_bits < 16 ? g->cfg.cached_bits : 16;  // resident (pipeline.py:689)
        if (std::find(started.begin(), started.end(), e) != started.end()) b = pf_bits_cur[e];
        for (size_t j = 0; j < od.size(); ++j)
          if (od[j].first == e) b = od_bits;
        lg->src_bits[i] = b;
      }
    }
    for (int e = 0; e < E; ++e) pf_bits_cur[e] = 0;
    for (int i = 0; i < m.n_pf; ++i) pf_bits_cur[m.pf_e[i]] = m.pf_bits_each[i];
    // expert compute for layer l once every needed copy landed
    if (serial_launches()) {
      // launch-serialised mode: the host waits for the flag, then enqueues K4
      while (((volatile uint32_t *)g->ready_host)[l] < 1u) {
        if ((status = ch.pump())) break;
        _mm_pause();
        if (std::chrono::steady_clock::now() - last_progress > std::chrono::seconds(60)) {
          status = FATE_ETIMEOUT;
          set_error("fate_engine_prefill: transfers of a layer never completed (serial mode)");
          break;
        }
      }
      if (status) break;
    } else {
      FATE_CU(p_wait32((CUstream)cs, (CUdeviceptr)(g->ready_dev + l), 1u, CU_STREAM_WAIT_VALUE_GEQ));
    }
    if (timed) FATE_CUDA(cudaEventRecord(kev[4 * l + 2], cs));
    int tiles_up = 0, tiles_down = 0;
    for (int i = 0; i < m.n_active; ++i) {
      tiles_up += k4_tc_items(m.active_cnt[i], I, H, false);
      tiles_down += k4_tc_items(m.active_cnt[i], I, H, true);
      flops += 6.0 * H * I * m.active_cnt[i];
    }
    int n_ex = m.n_active;
    const int has_shared = g->cfg.shared_intermediate && g->shared_dev[l] ? 1 : 0;
    if (has_shared) {
      tiles_up += k4_tc_items(T, g->cfg.shared_intermediate, H, false);
      tiles_down += k4_tc_items(T, g->cfg.shared_intermediate, H, true);
      flops += 6.0 * H * g->cfg.shared_intermediate * T;
      ++n_ex;
    }
    FATE_CUDA(launch_k4_tc(s.Xb, H, s.ex, n_ex, s.tok_idx, s.zrow, s.a_off, s.A, s.Z, tiles_up, tiles_down, cs));
    FATE_CUDA(launch_k4_combine(s.Z, s.cw, T, k, H, has_shared, Y_dev + (int64_t)l * T * H, cs));
    prefill_arc_kernel<<<1, 32, 0, cs>>>(d, s, l, m.n_active);
    FATE_CHECK_LAUNCH("prefill_arc_kernel");
    if (timed) FATE_CUDA(cudaEventRecord(kev[4 * l + 3], cs));
    if (l + 1 < L && (status = launch_front(l + 1))) break;
    if (dbg) fprintf(stderr, "[fate] prefill layer %d act=%d res=%d need=%d started=%zu od=%zu pf=%d\n", l, m.n_active,
                     m.n_res, m.n_need, started.size(), idx.size(), m.n_pf);
  }
  if (status != FATE_OK)
    for (int l = 0; l < L; ++l) g->ready_host[l] = 0x7FFFFFFFu;
  auto drain_start = std::chrono::steady_clock::now();
  while (status == FATE_OK && (!ch.pending.empty() || !ch.inflight.empty())) {
    ch.pending.erase(std::remove_if(ch.pending.begin(), ch.pending.end(),
                                    [&](const Transfer &x) { return x.kind == 0 && x.layer >= L; }),
                     ch.pending.end());
    if ((status = ch.pump())) break;
    _mm_pause();
    if (std::chrono::steady_clock::now() - drain_start > std::chrono::seconds(60)) {
      status = FATE_ETIMEOUT;
      set_error("fate_engine_prefill: copies never completed while draining");
      for (int l = 0; l < L; ++l) g->ready_host[l] = 0x7FFFFFFFu;
    }
  }
  cudaError_t se = cudaStreamSynchronize(cs), xe = cudaStreamSynchronize(g->xstream);
  if (xe == cudaSuccess) xe = cudaStreamSynchronize(g->xstream2);
  if (status == FATE_OK && se != cudaSuccess) status = cuda_status(se, "prefill compute stream");
  if (status == FATE_OK && xe != cudaSuccess) status = cuda_status(xe, "prefill copy stream");
  DevStats ds{};
  fate_run_stats st{};
  if (status == FATE_OK) {
    FATE_CUDA(cudaMemcpy(&ds, g->d.stats, sizeof(ds), cudaMemcpyDeviceToHost));
    Ctrl cc;
    FATE_CUDA(cudaMemcpy(&cc, g->d.ctrl, sizeof(cc), cudaMemcpyDeviceToHost));
    if (cc.err) {
      set_error("fate_engine_prefill: staging buffer pool exhausted");
      status = FATE_ENOMEM;
    }
    if (log_host) {
      std::vector<int32_t> vic((size_t)L * (E + 1));
      FATE_CUDA(cudaMemcpy(vic.data(), s.victims, vic.size() * 4, cudaMemcpyDeviceToHost));
      for (int l = 0; l < L; ++l) {
        fate_prefill_log &lg = log_host[l];
        lg.n_victims = vic[(size_t)l * (E + 1)];
        for (int i = 0; i < lg.n_victims; ++i) lg.victims[i] = vic[(size_t)l * (E + 1) + 1 + i];
      }
    }
  }
  if (timed && status == FATE_OK) {
    g->step_ms.assign(4 * (size_t)L, 0.0);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, kev[0], kev[4 * (L - 1) + 3]);
    st.gpu_ms = ms;
    double ffn = 0.0, gate = 0.0;
    for (int l = 0; l < L; ++l) {
      float t[4] = {0.f, 0.f, 0.f, 0.f};
      for (int j = 0; j < 4; ++j)
        if (l || j) cudaEventElapsedTime(&t[j], kev[0], kev[4 * l + j]);
      for (int j = 0; j < 4; ++j) g->step_ms[4 * (size_t)l + j] = t[j];
      gate += t[1] - t[0];
      ffn += t[3] - t[2];
    }
    st.ffn_ms = ffn;
    st.gate_ms = gate;
  }
  if (timed) {
    for (auto &e : ch.ev) cudaEventDestroy(e);
    for (auto &e : kev) cudaEventDestroy(e);
  }
  st.steps = L;
  st.accesses = (int64_t)ds.accesses;
  st.cache_hits = (int64_t)ds.cache_hits;
  st.arrival_hits = (int64_t)ds.arrival_hits;
  st.dequant_count = (int64_t)ds.dequant_count;
  st.prefetch_issued = (int64_t)ds.prefetch_issued;
  st.ondemand_issued = (int64_t)ds.ondemand_issued;
  st.transfers_done = ch.done;
  st.transfers_dropped = ch.dropped;
  st.h2d_bytes = ch.h2d_bytes;
  st.d2d_bytes = ch.d2d_bytes;
  // busy time of the sampled copies, scaled to every byte the channel moved
  st.copy_busy_ms = ch.sampled_bytes > 0 ? ch.copy_ms * (double)(ch.h2d_bytes + ch.d2d_bytes) / (double)ch.sampled_bytes
                                         : 0.0;
  st.recall_sum = ds.recall_sum;
  st.recall_n = (int64_t)ds.recall_n;
  st.trace_mismatches = (int64_t)ds.mismatches;
  st.ffn_flops = flops;
  st.error = status;
  if (stats) *stats = st;
  return status;
}

static int prefill_preload() {
  cudaFuncAttributes fa;
  FATE_CUDA(cudaFuncGetAttributes(&fa, prefill_x_kernel));
  FATE_CUDA(cudaFuncGetAttributes(&fa, prefill_plan_kernel));
  FATE_CUDA(cudaFuncGetAttributes(&fa, prefill_arc_kernel));
  FATE_CUDA(cudaFuncGetAttributes(&fa, prefill_begin_kernel));
  return FATE_OK;
}
