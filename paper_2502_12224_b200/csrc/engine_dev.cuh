// Device-side state of the offload engine: ARC tables, expert->buffer maps,
// the staging free stack, the step control block and the host mailbox.
#pragma once

#include "fate_internal.cuh"

namespace fate {

constexpr int EMAX = FATE_MAX_EXPERTS;
constexpr int KMAX = FATE_MAX_TOPK;

// One layer's ARC lists (cache.py:104-179), LRU first.
struct alignas(16) ArcLayer {
  int32_t c, n1, n2, nb1, nb2, pad0;
  double p;
  int32_t t1[EMAX], t2[EMAX], b1[EMAX], b2[EMAX];
};

// Step message, device -> host (mapped pinned memory).  `seq` is written last;
// `seq_od` earlier, as soon as the on-demand set (n_od, od_*) is final.
struct StepMsg {
  volatile uint32_t seq;
  volatile uint32_t seq_od;
  int32_t step, token, layer;
  int32_t self_signaled;
  int32_t n_od, n_need, n_drop, n_pf;
  int32_t od_bits, pf_bits;
  int32_t od_e[EMAX], od_b[EMAX];
  uint32_t od_g[EMAX];
  int32_t need_e[EMAX], need_b[EMAX];
  int32_t drop_e[EMAX], drop_b[EMAX];
  int32_t pf_e[EMAX], pf_b[EMAX], pf_bits_each[EMAX];
  uint32_t pf_g[EMAX];
  // prefill extras (host-side log + ordering)
  int32_t n_active, n_res;
  int32_t active_e[EMAX], active_cnt[EMAX], res_e[EMAX];
  int32_t active_fs[EMAX];  // prefill, reorder off: first-seen rank of active_e[i] (pipeline.py:524-533)
  int32_t pred_order[EMAX], pred_cnt[EMAX], n_pred;
  int32_t mismatch;
};

constexpr int kRing = 64;

// Decode step message, device -> host (mapped pinned memory), as
// self-validating 64-bit words: every word carries a tag of its step, so the
// host accepts each word once its tag matches and K1 needs no system-scope
// fence (an aligned 8-byte store arrives whole).  A run starts from a zeroed
// ring; tags are never zero.
//   od_head: [63:32] step+1  [31:23] n_od  [22:18] od_bits
//   head:    [63:38] (step+1) mod 2^26  [37:33] n_od  [32:24] n_need  [23:15] n_drop
//            [14:6] n_pf  [5:1] pf_bits  [0] self_signaled
// (the two heads may reach the host in either order: the head repeats n_od so
// the host knows whether to wait for od_head).  The host clears every word it
// consumed, so a slot never holds a stale word a later step could take for its
// own (entry tags only carry 7 bits of the step).
//   entries: [63:56] entry tag  [55:48] expert  [47:32] buffer  [31:0] generation
struct DecodeMsg {
  uint64_t od_head;
  uint64_t head;
  uint64_t od[KMAX];
  uint64_t need[KMAX];
  uint64_t drop[EMAX];
  uint64_t pf[EMAX];
};
__host__ __device__ inline uint32_t msg_entry_tag(int step) { return ((uint32_t)(step + 1) & 0x7Fu) | 0x80u; }
__host__ __device__ inline uint64_t msg_entry(int step, int e, int b, uint32_t g) {
  return ((uint64_t)msg_entry_tag(step) << 56) | ((uint64_t)(e & 0xFF) << 48) | ((uint64_t)(b & 0xFFFF) << 32) | g;
}
__host__ __device__ inline uint32_t msg_head_tag(int step) { return (uint32_t)(step + 1) & 0x3FFFFFFu; }

// Control block for the step sequence.
struct Ctrl {
  int32_t next_token;
  int32_t cur_token, cur_layer;
  int32_t prev_valid, prev_layer, prev_k, prev_step;
  int32_t prev_chosen[EMAX], prev_buf[EMAX];
  int32_t free_top;
  int32_t err;
  uint32_t arrive;        // K1 last-block detector
  int32_t pred_valid, pred_layer, pred_n;
  int32_t pred_list[EMAX];
  int32_t step;           // global step counter (token*L + layer)
};

struct DevStats {
  unsigned long long accesses, cache_hits, arrival_hits, dequant_count, prefetch_issued, ondemand_issued;
  unsigned long long mismatches, near_ties, recall_n;
  FfnStats ffn;
  double recall_sum;
};

// All device pointers of an engine, passed to kernels by value.
struct EngineDev {
  int L, E, k, H, I, I_shared, shared_bits;
  int cached_bits, prefetch_bits, ondemand_bits;
  int use_predictor, policy, budget_n;  // policy: 0 top-k, 1 percentile (cross-layer), 2 EAP
  int32_t *eap_counts;        // [L-1, E, E] co-activation counts (EapStats, predict.py:110-130)
  int32_t *eap_totals;        // [L-1, E] their row sums
  double q;
  int nbuf;
  int64_t buf_stride;
  uint8_t *pool;              // nbuf * buf_stride
  const uint8_t **shared;     // [L] shared-expert buffers (or null)
  const float *shared_gate;   // [L] sigmoid gate of the shared expert (dense part), or null: weight 1
  const double *W;            // [L, E, H]
  const double *tau;          // [L]
  ArcLayer *arc;              // [L]
  int32_t *buf_of;            // [L, E]
  int32_t *pend_buf;          // [L, E]
  uint32_t *pend_gen;         // [L, E]
  int32_t *free_stack;        // [nbuf]
  uint32_t *buf_gen;          // [nbuf]
  uint32_t *buf_done;         // [nbuf]  written by the copy stream
  int32_t *buf_bits;          // [nbuf]  storage width requested into each buffer
  uint32_t *ready;            // [L]     wait flags of the compute stream
  Ctrl *ctrl;
  DevStats *stats;
  double *logits;             // [2E]
  float *x;                   // x in the four chunk-transposed K3 layouts (write_xlay)
  FfnBatch *batch;
  StepMsg *ring;              // mapped pinned [kRing] (prefill)
  DecodeMsg *dring;           // mapped pinned [kRing] (decode)
};

}  // namespace fate
