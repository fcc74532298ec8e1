/*
 * fate_b200.h — C ABI of the B200-native Fate offloaded-MoE hot path.
 *
 * The reference (moesim, /root/reference/pkg/src/moesim) is a pure-Python
 * package with no FFI; its "plugin boundary" is the Python API plus the two
 * injection seams of the engine entry points (pipeline.py:343-353 and
 * pipeline.py:536-545).  Every entry point below replaces one reference
 * function (cited per declaration); the Python package
 * paper_2502_12224_b200 binds them with ctypes.
 *
 * Conventions
 *   - every function returns an int status: FATE_OK or one of FATE_E*; the
 *     Python wrapper maps these onto the reference's SimError classes;
 *   - buffers are caller-owned; "_dev" pointers are CUDA device pointers,
 *     "_host" pointers are host memory (pinned where stated);
 *   - `stream` is a cudaStream_t passed as void* (0 = legacy default stream);
 *   - no C++ exception crosses this boundary; no allocation in hot calls
 *     except inside fate_engine_create.
 */
#ifndef FATE_B200_H
#define FATE_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define FATE_OK 0
#define FATE_EINVAL 1     /* InvalidConfig            (errors.py:21)  */
#define FATE_EMISMATCH 2  /* TraceMismatch            (errors.py:39)  */
#define FATE_EBUDGET 3    /* BudgetTooSmall           (errors.py:63)  */
#define FATE_ECODES 4     /* CorruptCodes             (errors.py:75)  */
#define FATE_ECUDA 5      /* CUDA runtime/driver failure               */
#define FATE_ENOMEM 6     /* device or pinned allocation failed        */
#define FATE_ETIMEOUT 7   /* engine watchdog fired (copy never landed) */

#define FATE_MAX_EXPERTS 256
#define FATE_MAX_TOPK 16
#define FATE_HEADER_BYTES 256

/* ---- library ------------------------------------------------------------ */
int fate_version(void);
/* Last error message of the calling thread (never NULL). */
const char *fate_last_error(void);
/* Number of visible CUDA devices, 0 if none; nonzero status if the driver is unusable. */
int fate_device_count(int *count);

/* ---- K5 quantization: quant.py:67-107 (quantize) and :30-39 (_pack) ------
 * Group-wise min/max affine quantization of w[n] (fp32 on device) with
 * fp64 arithmetic and round-half-even, groups of `group` consecutive
 * elements, packed little-endian within each byte.  Writes
 *   codes_dev   : ceil(n*bits/8) bytes,
 *   sz_dev      : optional fp32 (scale, zero) pairs per group (device format),
 *   scale64_dev / zero64_dev : optional fp64 per-group values (reference format).
 * bits in {8,4,2}.  bits == 16 converts to bf16 into codes_dev (2n bytes). */
int fate_quant_pack(const float *w_dev, int64_t n, int bits, int group, uint8_t *codes_dev,
                    float *sz_dev, double *scale64_dev, double *zero64_dev, void *stream);

/* Same as fate_quant_pack for fp64 input (the reference quantizes fp64 arrays). */
int fate_quant_pack64(const double *w_dev, int64_t n, int bits, int group, uint8_t *codes_dev, float *sz_dev,
                      double *scale64_dev, double *zero64_dev, void *stream);

/* dequantize (quant.py:110-120): out[n] fp32 = zero + code*scale from the
 * device format (fp32 scale/zero); bits 16 reads bf16. */
int fate_dequant(const uint8_t *codes_dev, const float *sz_dev, int64_t n, int bits, int group,
                 float *out_dev, void *stream);

/* fp64 dequantization from the reference representation (fp64 scales/zeros),
 * zero + code*scale with the reference's two roundings (quant.py:110-120). */
int fate_dequant64(const uint8_t *codes_dev, const double *scale64_dev, const double *zero64_dev, int64_t n,
                   int bits, int group, double *out_dev, void *stream);

/* Pack one expert (w1 [I,H], w3 [I,H], w2 [H,I], fp32 on device) into the
 * engine's self-describing buffer layout: 256-byte header + payload of
 * exactly expert_bytes[bits] bytes (quant.py:239-246 formula).  Returns
 * the payload layout via fate_expert_layout. */
int fate_pack_expert(const float *w1_dev, const float *w3_dev, const float *w2_dev, int H, int I, int bits,
                     int layer, int expert, uint8_t *dst_dev, void *stream);
/* Byte size of one packed expert buffer (header + payload) for (H, I, bits). */
int64_t fate_expert_buffer_bytes(int H, int I, int bits);

/* ---- K1 gate + cross-layer predictor --------------------------------------
 * gatesim.py:113-123 (gate_forward), core.py:159-163 (top_k_set),
 * predict.py:84-107 (nearest_rank_percentile, cross_layer_predict).
 * For T hidden vectors h[T,H] (fp64): routing[T,E] = softmax(W h / tau) in
 * fp64; order[T,E] = experts sorted by (-routing, id); list_len[T] = length
 * of the policy's prediction prefix of `order` (policy 0 = top-k: k;
 * policy 1 = percentile q: max(k, #{w > nearest-rank(q)})). */
int fate_gate_forward(const double *W_dev, double tau, const double *h_dev, int T, int E, int H,
                      double *routing_dev, int32_t *order_dev, int32_t *list_len_dev, int top_k,
                      int policy, double q, void *stream);

/* ---- K3 decode expert FFN (replaces the t_moe charge, pipeline.py:477-479)
 * y[H] = sum_j weight[j] * W2_j (silu(W1_j x) * (W3_j x)) over n experts
 * whose packed buffers (fate_pack_expert layout) are at bufs[j] (device
 * pointers, host array).  fp32 accumulation.  scratch_dev >= sum_j I_j floats. */
int fate_ffn_decode(const float *x_dev, int H, int n, const uint8_t *const *bufs, const float *weights,
                    float *scratch_dev, float *y_dev, void *stream);

/* Measurement: K3 launched `iters` times back to back on `stream`, cycling
 * over `nsets` expert sets (bufs[nsets*n], set q = bufs[q*n .. q*n+n)) so the
 * working set can exceed L2; batches and layouts are built once; *ms_out =
 * mean kernel time in ms from CUDA events around the launches. */
int fate_ffn_decode_timed(const float *x_dev, int H, int n, int nsets, const uint8_t *const *bufs,
                          const float *weights, float *y_dev, int iters, void *stream, float *ms_out);

/* Diagnostics: per-CTA phase timestamps (globaltimer ns) of the last K3
 * launch, out_host[160*8]: start, consumers start, x layouts done, phase A
 * done, grid barrier passed, activation layouts done, phase B done, producer
 * done; then out_host[160*8 + 17*48*3]: CTA 0 per-warp tile trace in SM
 * cycles, [warp][tile][3] (producer: empty-wait start, empty passed, issued;
 * consumers: full-wait start, full passed, released); then [8][4] cycles of
 * consumer warp 1's first phase-A rows (dots done, sums done, store done). */
int fate_k3_profile(uint64_t *out_host);
/* Profiling builds only (FATE_PROF=1): CTA 0's per-stage K4 timeline of the last
 * up-projection launch, out_host[256*5] (ns): issued, landed, dequantized, MMA saw
 * full, MMA committed. */
int fate_k4_profile(uint64_t *out_host);
/* Diagnostics: phase timestamps of the last K1 launch, out_host[8] ns. */
int fate_k1_profile(uint64_t *out_host);

/* ---- K4 prefill grouped expert FFN (replaces pipeline.py:733-750) ----------
 * For T tokens X[T,H] (fp32 on device), n experts: token lists tok_idx
 * (concatenated, device int32) with per-expert offsets off[n+1] (host) and
 * routing weights tok_w (device fp32, aligned with tok_idx):
 *   Y[t] += tok_w * W2_e(silu(W1_e x_t) * W3_e x_t)  (Y zeroed by the caller).
 * bf16 operands (dequantized in shared memory), fp32 accumulation. */
int fate_ffn_prefill(const float *X_dev, int T, int H, int n, const uint8_t *const *bufs,
                     const int32_t *tok_idx_dev, const float *tok_w_dev, const int32_t *off_host,
                     float *Y_dev, void *stream);

/* ---- Engine: device-resident expert cache + prefetch + compute ------------
 * The engine owns: the fp64 router weights, a pool of expert buffers on the
 * GPU (plan slots + staging), the per-layer ARC tables and expert->buffer
 * maps (cache.py:104-215), pinned host pools (INT2/INT4/INT8/bf16 copies of
 * every expert), a copy stream and a host copy manager thread
 * (the transfer channel, pipeline.py:163-264). */
typedef struct fate_engine fate_engine;

typedef struct fate_engine_config {
  int num_layers, num_experts, top_k, hidden_dim, intermediate_dim;
  int shared_intermediate;       /* 0 = no shared expert                    */
  int shared_bits;               /* 16, 8, 4 or 2                           */
  const int32_t *capacity;       /* [num_layers] CachePlan.per_layer_capacity */
  int cached_bits;               /* CachePlan.cached_bits (reported src bits) */
  int prefetch_bits;             /* Strategy.prefetch_bits()   (pipeline.py:96-97)  */
  int ondemand_bits;             /* Strategy.ondemand_bits()   (pipeline.py:99-101) */
  int use_predictor;             /* fate: 1, lod: 0                         */
  int policy;                    /* 0 topk, 1 percentile (predict.py:21-47), 2 EAP co-activation (predict.py:110-158, decode) */
  double percentile_q;
  int budget_n;                  /* transfer_budget (pipeline.py:151-156)   */
  int prefill_use_predictor;     /* fate prefill prediction (pipeline.py:568) */
  int reorder_prefill;           /* Strategy.reorder_prefill                */
  double p_int2;                 /* QuantPolicy.p_int2 (prefill INT2 share) */
  int prefill_ondemand_bits;     /* 2 for fate (pipeline.py:701), 16 otherwise */
  int max_tokens;                /* decode/prefill capacity for scratch     */
  int max_inflight;              /* copy-engine issue depth (preemption granularity) */
  int device;
} fate_engine_config;

int fate_engine_create(const fate_engine_config *cfg, fate_engine **out);
int fate_engine_destroy(fate_engine *eng);
/* Change the Strategy knobs (pipeline.py:44-104) of an existing engine,
 * keeping its cache state (compare_strategies chaining, pipeline.py:835-850). */
int fate_engine_set_strategy(fate_engine *eng, const fate_engine_config *cfg);
/* Timeline of the last timed run (pipeline.py:107-132): step_ms[4*s..] =
 * gate start, gate end, moe start, moe end (ms from the run start);
 * copy_ms[2*c..] = start, end; copy_meta[5*c..] = kind (0 prefetch,
 * 1 on-demand), step, layer, expert, bits.  counts = {steps, copies}. */
int fate_engine_timeline(fate_engine *eng, double *step_ms, int max_steps, double *copy_ms, int32_t *copy_meta,
                         int max_copies, int32_t *counts);
/* Copy timing of timed runs: an event pair around every stride-th transfer only
 * (default 8; 1 = every transfer, as the timeline of collect_cache_events wants;
 * 0 = none).  Events between copies delay the copy engine; copy_busy_ms is the
 * sampled copies' busy time scaled by bytes.  Decode's per-step kernel events
 * follow the same stride (max(1, stride); the last step always): gate_ms /
 * ffn_ms / dense_ms are the sampled steps scaled to all, the timeline's
 * unsampled steps are NaN. */
int fate_engine_set_copy_timing(fate_engine *eng, int stride);
/* Decode step protocol.  on = 1 (default): K3 is launched right behind K1 and
 * waits per expert for that expert's copy (a generation mark the copy stream
 * writes behind it), so the resident experts and the shared expert are computed
 * while the copies are on PCIe.  on = 0: the compute stream waits for every
 * copy of the step before K3 starts (K3's event time is then its compute time
 * alone, which the bench's roofline uses).  Same decisions and results. */
int fate_engine_set_overlap(fate_engine *eng, int on);

/* Router weights W[L,E,H] fp64 and temperatures tau[L] (host arrays; copied). */
int fate_engine_set_gate(fate_engine *eng, const double *W_host, const double *tau_host);
/* EAP baseline (policy 2): co-activation statistics back to empty, i.e. a fresh
 * EapStats (predict.py:110-130).  Replaces constructing EapDecodePredictor /
 * EapStats (pipeline.py:301-336, 572-574); prefill and decode otherwise share them. */
int fate_engine_reset_eap(fate_engine *eng);
/* Register the pinned host pool for one bit width: experts (l,e) at
 * base + (l*E + e) * stride, each a packed buffer (header + payload). */
int fate_engine_set_host_pool(fate_engine *eng, int bits, const uint8_t *base_host, int64_t stride);
/* Expert-sharded peer-fetch mode: per-expert source buffers for
 * one bit width, srcs[l*E + e] = a packed buffer (header + payload) in device
 * memory of this GPU or of a peer GPU mapped into this process (CUDA IPC,
 * fate_ipc_open_handle), or NULL to keep the pinned host copy.  A miss of
 * (l, e) at that width is then a device/peer copy (cudaMemcpyDefault: NVLink
 * for peers) instead of a host fetch; decisions are unchanged.  srcs == NULL
 * clears the table.  The array is copied. */
int fate_engine_set_expert_sources(fate_engine *eng, int bits, const uint8_t *const *srcs);
/* CUDA IPC for the home shards of the expert-sharded mode: export the device
 * allocation containing dev_ptr (64-byte handle + dev_ptr's byte offset in it),
 * map a peer's allocation (add the offset to the returned base), unmap it. */
int fate_ipc_get_handle(const void *dev_ptr, uint8_t *handle64, int64_t *offset);
int fate_ipc_open_handle(const uint8_t *handle64, void **dev_ptr_out);
int fate_ipc_close(void *dev_ptr);
/* Node-wide shared expert pools: page-lock an existing host
 * mapping (a /dev/shm segment every rank maps) in this process, portable
 * across devices, so transfers from it are pinned-memory DMA; and undo it.
 * Replaces the per-process pinned pools the reference's single-process
 * simulator never needed (it keeps no weights). */
int fate_host_register(void *host_ptr, int64_t bytes);
/* Transfer channel C1 as a standalone object (SURVEY §8b prefetch_{enqueue,
 * promote,drop_stale,wait}): the reference's _Channel (pipeline.py:163-264) over
 * real copies.  Pending transfers are a host FIFO; pump / wait start them in
 * queue order as cudaMemcpyAsync on the channel's copy stream (<= max_inflight
 * in flight for pump), each followed by an event.  device < 0: queue
 * bookkeeping only, no CUDA calls.  The decode / prefill engine runs the same
 * discipline internally. */
typedef struct fate_channel fate_channel;
int fate_channel_create(int device, int max_inflight, fate_channel **out);
int fate_channel_destroy(fate_channel *ch);
/* _Channel.enqueue (pipeline.py:196): kind 0 prefetch / 1 on-demand for step
 * (token, layer), a copy of `bytes` from src (pinned host or device) to dst. */
int fate_channel_enqueue(fate_channel *ch, int kind, int token, int layer, int expert, int bits, const void *src,
                         void *dst, int64_t bytes, int64_t *id_out);
/* _Channel.promote_ondemand (pipeline.py:241): on-demand ahead of prefetch, stably. */
int fate_channel_promote(fate_channel *ch);
/* _Channel.drop_stale (pipeline.py:247): discard pending prefetches with step <= (token, layer). */
int fate_channel_drop_stale(fate_channel *ch, int token, int layer, int *n_dropped);
/* _Channel.settle (pipeline.py:214): retire finished copies, start pending ones while < max_inflight. */
int fate_channel_pump(fate_channel *ch);
/* _Channel.completion (pipeline.py:222) for a consumer stream: start everything up to
 * transfer `id` in queue order, then cudaStreamWaitEvent(stream, its event). */
int fate_channel_wait(fate_channel *ch, int64_t id, void *stream);
/* _Channel.find (pipeline.py:232): state -1 none, 0 pending, 1 in flight, 2 complete. */
int fate_channel_find(fate_channel *ch, int token, int layer, int expert, int *state, int64_t *id_out);
/* The pending queue in order (ids) and the number of copies in flight. */
int fate_channel_pending(fate_channel *ch, int64_t *ids, int max, int *n, int *n_inflight);

/* Dense part of one decode step (replaces the t_attn / t_gate
 * constants, reference core.py:79-83, pipeline.py:418, 484): h = h_prev + y_prev,
 * qkv = Wqkv RMSNorm(h) + b, RoPE at pos, K/V appended to the bf16 cache
 * kv[pos] ([ctx][2][nkv*hd]), o = decode attention over positions 0..pos (GQA),
 * a = h + Wo o, and the shared-expert gate sigmoid(gate_w . sqrt(H) gate_in) into
 * *gate_out when gate_w is given.  Device pointers; bf16 weights; synchronous.
 * The engine runs the same kernels inside its step loop (fate_engine_set_dense). */
int fate_dense_step(int H, int n_heads, int n_kv_heads, int head_dim, float eps, float rope_theta, const void *wqkv,
                    const float *bqkv, const float *norm, const void *wo, void *kv, const float *gate_w,
                    float *gate_out, const float *h_prev, const float *y_prev, const double *gate_in, int pos, float *h,
                    float *qkv, float *q, float *o, float *a, float *part_o, float *part_ml, void *stream);
int fate_host_unregister(void *host_ptr);
/* The dense part of every decode step (replacing the t_attn /
 * t_gate constants of core.py:79-83): attention geometry, K/V cache capacity
 * max_ctx positions per layer with the prompt's ctx0 positions pre-filled
 * (synthetic), RMSNorm eps and RoPE theta; then per layer the device weights
 * (bf16 Wqkv [(nh+2nkv)hd, H], optional fp32 bias, fp32 RMSNorm weight, bf16 Wo
 * [H, nh hd], optional fp32 shared-expert gate [H]; caller-owned).  Decode token
 * t then runs at position ctx0 + t; with every layer gated, the shared expert's
 * routing weight is sigmoid(gate . x) instead of 1. */
int fate_engine_set_dense(fate_engine *eng, int n_heads, int n_kv_heads, int head_dim, int max_ctx, int ctx0,
                          float eps, float rope_theta);
int fate_engine_set_dense_layer(fate_engine *eng, int layer, const void *wqkv, const float *bqkv, const float *norm,
                                const void *wo, const float *shared_gate_w);
/* Shared expert for layer l: a packed device buffer (resident, dense bytes). */
int fate_engine_set_shared(fate_engine *eng, int layer, const uint8_t *buf_dev);

/* Cache control: LayeredExpertCache(plan) fresh state (cache.py:185-187),
 * seed_resident (cache.py:197-204; loads the experts' cached_bits copies). */
int fate_engine_reset_cache(fate_engine *eng);
int fate_engine_seed_resident(fate_engine *eng, int layer, const int32_t *experts, int n);
/* contains() (cache.py:192-195) for every expert of a layer: out[E] in {0,1}. */
int fate_engine_resident(fate_engine *eng, int layer, int32_t *out_host);
/* Standalone ARC accesses in order (update_after_layer, cache.py:212-215):
 * hits_host[n] receives 1 on a resident hit.  Buffers of newly inserted
 * experts are loaded from the cached_bits host pool synchronously. */
int fate_engine_access(fate_engine *eng, int layer, const int32_t *experts, int n, int32_t *hits_host);
/* ARC state export: lists LRU-first; lens[4] = |T1|,|T2|,|B1|,|B2|; each list
 * array must hold num_experts entries. */
int fate_engine_arc_state(fate_engine *eng, int layer, int32_t *t1, int32_t *t2, int32_t *b1,
                          int32_t *b2, int32_t *lens, double *p);

/* Per-step parity log (timing-independent fields of pipeline.py:406-490). */
typedef struct fate_step_log {
  int32_t chosen[FATE_MAX_TOPK];           /* ascending                          */
  int32_t src_bits[FATE_MAX_TOPK];         /* source bits per chosen expert      */
  int32_t hit[FATE_MAX_TOPK];              /* 1 if cache-resident at gate time   */
  int32_t ondemand[FATE_MAX_TOPK];
  int32_t victims[FATE_MAX_TOPK];
  int32_t n_ondemand, n_victims, n_pred, n_prefetch;
  int32_t arrived[FATE_MAX_TOPK];          /* prefetched AND landed at gate time (timing-dependent) */
  int32_t pred[FATE_MAX_EXPERTS];          /* entries[:n] for layer+1, rank order */
  int32_t prefetch[FATE_MAX_EXPERTS];      /* issued (pred minus resident)        */
  float routing[FATE_MAX_TOPK];            /* fp32 copy of the chosen weights     */
  int32_t fmt_bits[FATE_MAX_TOPK];         /* storage width of the buffer computed from */
  int32_t mismatch;                        /* 1 if device top-k != trace chosen   */
  int32_t pad;
} fate_step_log;

typedef struct fate_run_stats {
  double gpu_ms;              /* CUDA-event time of the whole run          */
  double ffn_ms;              /* summed K3/K4 kernel time (event pairs)    */
  double gate_ms;             /* summed K1 time                            */
  int64_t steps, accesses, cache_hits, arrival_hits, dequant_count;
  int64_t prefetch_issued, ondemand_issued, transfers_done, transfers_dropped;
  int64_t h2d_bytes;
  double copy_busy_ms;        /* copy-stream busy time (event pairs)       */
  double recall_sum; int64_t recall_n;
  int64_t trace_mismatches;   /* device top-k differing from trace chosen  */
  int64_t ffn_bytes;          /* algorithmic bytes of executed experts     */
  double ffn_flops;           /* prefill: 2*3*H*I*tokens summed            */
  int64_t near_ties;          /* k-th/(k+1)-th weight gap < 1e-12           */
  int64_t d2d_bytes;          /* misses served from device memory (local or
                                 peer HBM over NVLink, expert-sharded mode)    */
  int32_t error; int32_t pad;
  double dense_ms;            /* summed dense-part time (attention block +
                                 shared-expert gate, fate_engine_set_dense)    */
  double k3_wait_ms;          /* arrival-gated decode: per K3 launch, the
                                 longest time one of its producer warps waited
                                 for copies, summed (ffn_ms - k3_wait_ms ~ the
                                 K3 compute time; 0 with overlap off)          */
} fate_run_stats;

/* Decode T tokens (simulate_decoding, pipeline.py:343-517).
 * gate_in_dev [T,L,H] fp64 gate inputs, chosen_dev [T,L,k] (trace ids for the
 * mismatch check, may be NULL); y_dev [T,L,H] fp32 expert outputs;
 * log_dev [T*L] fate_step_log or NULL.  Blocks until done. */
int fate_engine_decode(fate_engine *eng, const double *gate_in_dev, const int32_t *chosen_dev, int T,
                       float *y_dev, fate_step_log *log_dev, fate_run_stats *stats);

/* Per-layer prefill log (timing-independent fields of pipeline.py:608-753). */
typedef struct fate_prefill_log {
  int32_t n_pred, n_prefetch, n_active, n_resident, n_planned, n_ondemand, n_victims, n_started;
  int32_t pred_order[FATE_MAX_EXPERTS], pred_counts[FATE_MAX_EXPERTS];
  int32_t prefetch[FATE_MAX_EXPERTS], prefetch_bits[FATE_MAX_EXPERTS];
  int32_t actives[FATE_MAX_EXPERTS], counts[FATE_MAX_EXPERTS];
  int32_t resident[FATE_MAX_EXPERTS], planned[FATE_MAX_EXPERTS], ondemand[FATE_MAX_EXPERTS];
  int32_t src_bits[FATE_MAX_EXPERTS];      /* aligned with actives           */
  int32_t victims[FATE_MAX_EXPERTS];
  int32_t started[FATE_MAX_EXPERTS];       /* this layer's prefetches that began before block end */
  int32_t mismatch;
  int32_t pad;
} fate_prefill_log;

/* Prefill T tokens (simulate_prefill, pipeline.py:536-778).  Y_dev [L,T,H] fp32. */
int fate_engine_prefill(fate_engine *eng, const double *gate_in_dev, const int32_t *chosen_dev, int T,
                        float *Y_dev, fate_prefill_log *log_host, fate_run_stats *stats);

#ifdef __cplusplus
}
#endif
#endif /* FATE_B200_H */
