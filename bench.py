"""Benchmark: Fate offloaded-MoE decode on B200 (BASELINE.json configs[1]).

Workload: Qwen1.5-MoE-A2.7B shape (24 layers, 60 experts top-4, hidden 2048,
expert intermediate 1408, shared expert 5632 in bf16), random-init weights,
synthetic gate trace (the package's gen_trace, rho=0.888), decode bs=1 at a
fixed expert budget of 360 INT4 slots (25% of the 1440 experts), Strategy.fate()
with n = transfer_budget of a TimingModel measured on this GPU.

A "step" = one simulate_decoding pass over the trace (T tokens) from a cold
cache.  value = decode tokens/s over the K timed steps (device time from CUDA
events on the engine's compute stream, max over ranks, summed over ranks'
tokens); e2e = the same through the public API (host GateTrace in, y of the
last layer back to host) by wall clock.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--tokens T] [--impl ours|reference]
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

QWEN = dict(L=24, E=60, k=4, H=2048, I=1408, Lb=3, shared=5632, slots=360)
METRIC = "decode tokens/s at fixed expert-memory budget (Qwen1.5-MoE shape, 360 INT4 slots)"


def qwen_cfg():
    from paper_2502_12224_b200.core import ModelConfig
    c = QWEN
    return ModelConfig.from_shape(c["L"], c["E"], c["k"], c["H"], c["I"], c["Lb"],
                                  dense_bytes=c["L"] * 3 * c["H"] * c["shared"] * 2)


def make_trace(cfg, tokens: int, seed: int):
    from paper_2502_12224_b200.gatesim import GenConfig, gen_trace
    return gen_trace(cfg, GenConfig(seed=seed, num_tokens=tokens, phase="decoding"))


# ---------------------------------------------------------------------------
# clocks sampled during the timed region


class ClockSampler:
    def __init__(self, gpu: int):
        self.gpu, self.proc, self.lines = gpu, None, []

    def __enter__(self):
        q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap,power.draw")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--query-gpu={q}", "--format=csv,noheader,nounits", "-lms",
                                          "200", "-i", str(self.gpu)], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL,
                                         text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self) -> dict:
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for n, v in zip(names, parts[2:6]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


# ---------------------------------------------------------------------------
# CPU path (oracle port, test infrastructure): the whole executed decode path on
# the host cores -- fp64 gate + top-k, prediction, ARC, and the expert FFN in the
# width each copy has (AVX2 C threads) -- timed as one (oracle.port_decode)

REF_N = 0  # transfer budget n of the GPU arm on B200 (its measured TimingModel gives 0; the line states it)


def cpu_port(cfg, trace, weights, plan, n, tokens, get_buf, shared_buf, lib, ffn=True):
    """Run the CPU restatement on the first `tokens` tokens; returns (seconds, logs)."""
    from oracle import fate_oracle as O
    _, g, _ = trace.dense_arrays(cfg)
    mats, taus = np.stack(weights.matrices), np.array(weights.temperatures)
    t0 = time.perf_counter()
    logs = O.port_decode(g, mats, taus, list(plan.per_layer_capacity), cfg.top_k, n, O.StrategyKnobs(), get_buf,
                         shared_buf, cfg.hidden_dim, cfg.intermediate_dim, QWEN["shared"], lib, tokens, ffn=ffn)
    return time.perf_counter() - t0, logs


def reference_as_is(cfg, trace, weights, plan_caps, tokens):
    """The reference simulator itself (moesim.pipeline.simulate_decoding, installed in
    baseline/_ref) on the same sample trace: policy + discrete-event simulation wall
    clock with the paper TimingModel (it executes no expert FFN).  None when absent."""
    import tempfile
    ref = os.path.join(ROOT, "baseline", "_ref")
    if not os.path.isdir(os.path.join(ref, "moesim")):
        return None
    sys.path.insert(0, ref)
    try:
        from moesim import cache as mc, core as mcore, gatesim as mg, pipeline as mp
        from paper_2502_12224_b200 import core
        from paper_2502_12224_b200.core import GateTrace
        recs = [r for r in trace.records if r.token_index < tokens]
        sample = GateTrace(records=tuple(recs), phase=trace.phase, provenance=trace.provenance)
        with tempfile.TemporaryDirectory() as d:
            pth = os.path.join(d, "t.ndjson")
            core.write_trace(sample, pth)
            mtrace = mcore.read_trace(pth)
        mcfg = mcore.ModelConfig(num_layers=cfg.num_layers, num_experts=cfg.num_experts, top_k=cfg.top_k,
                                 hidden_dim=cfg.hidden_dim, shallow_boundary_L=cfg.shallow_boundary_L,
                                 expert_bytes=dict(cfg.expert_bytes), dense_bytes=cfg.dense_bytes)
        mw = mg.GateWeights(matrices=[np.asarray(m) for m in weights.matrices],
                            temperatures=[float(t) for t in weights.temperatures])
        timing = mcore.TimingModel(t_moe=13.0, t_attn=9.0, t_gate=2.0, t_expert_io={16: 6.0, 8: 3.0, 4: 1.6, 2: 0.85})
        mplan = mc.plan_allocation(mcfg, cfg.dense_bytes + QWEN["slots"] * cfg.expert_bytes[4], 4)
        assert list(mplan.per_layer_capacity) == list(plan_caps)
        t0 = time.perf_counter()
        mp.simulate_decoding(mtrace, mp.Strategy.fate(), mplan, timing, mcfg, weights=mw)
        secs = time.perf_counter() - t0
        return {"value": tokens / secs, "unit": "tokens/s (simulator wall clock)", "cores": 1,
                "sample": f"moesim.pipeline.simulate_decoding over the first {tokens} tokens of the same trace "
                          "(reference as is: schedule + discrete-event clock, no expert FFN executed)"}
    except Exception as e:  # the reference is a baseline, never a reason to fail the bench
        return {"unavailable": f"{type(e).__name__}: {e}"}
    finally:
        sys.path.remove(ref)


def run_reference(args):
    """--impl reference: the CPU restatement of the path on the host cores (rank 0 only),
    on the GPU arm's workload: the same Qwen trace (seed 0), plan and transfer budget,
    every routed expert in the width the GPU computes it in (INT2 on-demand copies, the
    slot's width on a hit) and the bf16 shared expert.  Expert codes are random bytes in
    those formats (the arithmetic does not depend on their values)."""
    from oracle import fate_oracle as O
    from paper_2502_12224_b200 import core
    from paper_2502_12224_b200.cache import plan_allocation
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    cfg = qwen_cfg()
    tokens = args.ref_tokens
    trace, weights = make_trace(cfg, args.tokens, 0)
    plan = plan_allocation(cfg, cfg.dense_bytes + QWEN["slots"] * cfg.expert_bytes[4], 4)
    lib = O.cpu_lib()
    cores = lib.fate_cpu_threads(0)
    rng = np.random.default_rng(0)
    H, I, Is = cfg.hidden_dim, cfg.intermediate_dim, QWEN["shared"]
    bufs: dict = {}

    def rand_buf(I_, bits):
        nb = core.packed_expert_bytes(3 * H * I_, bits)
        b = np.frombuffer(rng.bytes(256 + nb), dtype=np.uint8).copy()
        lay = O.buffer_layout(H, I_, bits)
        if bits != 16:  # sane fp32 scale/zero so the FFN does real arithmetic
            sz = b[256 + lay["s1"]:256 + lay["payload"]].view(np.float32)
            sz[0::2], sz[1::2] = 1e-3, -7.5e-3
        else:
            b[256:].view(np.uint16)[:] = 0x3C00
        return b

    # every buffer the sample touches is built before the timed steps
    _, logs = cpu_port(cfg, trace, weights, plan, REF_N, tokens, None, None, lib, ffn=False)
    for s, lg in enumerate(logs):
        for e, b in zip(lg["chosen"], lg["fmt_bits"]):
            if (s % cfg.num_layers, e, b) not in bufs:
                bufs[(s % cfg.num_layers, e, b)] = rand_buf(I, b)
    for l in range(cfg.num_layers):
        bufs[("s", l)] = rand_buf(Is, 16)
    get_buf = lambda l, e, b: bufs[(l, e, b)]  # noqa: E731
    shared = lambda l: bufs[("s", l)]  # noqa: E731
    for _ in range(args.warmup):
        cpu_port(cfg, trace, weights, plan, REF_N, tokens, get_buf, shared, lib)
    times = [cpu_port(cfg, trace, weights, plan, REF_N, tokens, get_buf, shared, lib)[0] for _ in range(args.steps)]
    total = sum(times)
    v = tokens * args.steps / total
    sample = (f"first {tokens} of the {args.tokens} decode tokens x 24 layers per step, same trace / plan / n={REF_N} as "
              "the GPU arm: fp64 gate + top-4, ARC, INT2 routed experts (their GPU width) + bf16 shared FFN, AVX2 threads")
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": v, "unit": "tokens/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1000 * total / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "fp32 accumulate, fp64 router",
        "data": "synthetic",
        "config": {"workload": "Qwen1.5-MoE-A2.7B shape decode bs=1, fixed expert budget (BASELINE configs[1])",
                   "tokens_per_step": tokens, "trace_tokens": args.tokens, "transfer_budget_n": REF_N,
                   "plan": list(plan.per_layer_capacity)},
        "cpu_baseline": {"value": v, "unit": "tokens/s", "cores": cores, "kind": "port", "sample": sample},
        "e2e": {"value": v, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "reference_as_is": reference_as_is(cfg, trace, weights, plan.per_layer_capacity, tokens),
    }), flush=True)


# ---------------------------------------------------------------------------


DSK = dict(L=28, E=64, k=6, H=2048, I=1408, Lb=3, shared=2816, slots=448, tokens=512)


def bench_prefill(peaks, rank: int) -> dict:
    """BASELINE configs[2]: DeepSeek-MoE-16B shape prefill of 512 tokens with a
    448-slot INT4 expert cache (25% of 1792), cold cache, Strategy.fate() prefill
    path (pipeline.simulate_prefill semantics on the device engine)."""
    import torch
    from paper_2502_12224_b200 import pipeline as P
    from paper_2502_12224_b200.cache import plan_allocation
    from paper_2502_12224_b200.core import ModelConfig
    from paper_2502_12224_b200.engine import OffloadEngine
    from paper_2502_12224_b200.experts import ExpertStore
    from paper_2502_12224_b200.gatesim import GenConfig, gen_trace
    c = DSK
    cfg = ModelConfig.from_shape(c["L"], c["E"], c["k"], c["H"], c["I"], c["Lb"],
                                 dense_bytes=c["L"] * 3 * c["H"] * c["shared"] * 2)
    tr, w = gen_trace(cfg, GenConfig(seed=rank, num_tokens=c["tokens"], phase="prefill"))
    store = ExpertStore(cfg, bits=(4, 2), seed=rank, shared_intermediate=c["shared"], shared_bits=16)
    plan = plan_allocation(cfg, cfg.dense_bytes + c["slots"] * cfg.expert_bytes[4], 4)
    strategy = P.Strategy.fate()
    _, g, ch = tr.dense_arrays(cfg)
    gd, chd = torch.as_tensor(g, device="cuda"), torch.as_tensor(ch, device="cuda")
    eng = OffloadEngine(cfg, plan.per_layer_capacity, store, w, P.knobs_for(strategy, plan, 0),
                        max_tokens=c["tokens"])
    eng.prefill(gd, chd)  # warm-up (kernel load, pools)
    runs = []
    for _ in range(2):
        eng.reset_cache()
        _, st, _, _, _ = eng.prefill(gd, chd)
        runs.append(st)
    eng.close()
    st = min(runs, key=lambda r: r["gpu_ms"])
    k4_tflops = st["ffn_flops"] / (st["ffn_ms"] * 1e-3) / 1e12
    peak = peaks.get("bf16_tflops", 1667.9)
    return {"workload": "DeepSeek-MoE-16B shape prefill 512 tokens, 448 INT4 slots, cold (BASELINE configs[2])",
            "tokens_per_s": c["tokens"] / st["gpu_ms"] * 1e3, "ms": st["gpu_ms"],
            "h2d_gbs": st["h2d_bytes"] / (st["copy_busy_ms"] * 1e-3) / 1e9 if st["copy_busy_ms"] else None,
            "h2d_bytes": st["h2d_bytes"],
            "roofline": {"bound": "tensor", "kernel": "K4 tcgen05 grouped SwiGLU (up + down)",
                         "achieved": k4_tflops, "peak": peak, "unit": "TFLOP/s", "frac": k4_tflops / peak,
                         "flops": st["ffn_flops"], "k4_ms": st["ffn_ms"],
                         "peak_source": "MEASURED_PEAKS.json bf16_tflops (burst)"},
            "dtype": "bf16 operands (dequantized INT4/INT2 experts, bf16 shared), fp32 accumulate"}


def load_traffic():
    """DRAM bytes per K3 launch from the committed ncu capture of this K3 on the bench's
    expert mix (profiles/r02_k3_bench_ncu.json, `--set full` of one launch); ncu replays
    a launch, so this is a per-launch count taken outside the timed run.  None if absent."""
    p = os.path.join(ROOT, "profiles", "r02_k3_bench_ncu.json")
    if os.path.exists(p):
        try:
            d = json.load(open(p))
            return d.get("dram_bytes_per_launch"), d.get("source", "profiles/r02_k3_bench_ncu.json")
        except Exception:
            return None, None
    return None, None


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--tokens", type=int, default=256)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--ref-tokens", type=int, default=16)
    ap.add_argument("--cpu-tokens", type=int, default=16)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--no-regimes", action="store_true", help="skip the prefetch / warm-cache decode regimes")
    ap.add_argument("--dense", action="store_true",
                    help="execute the dense part (attention block + shared-expert gate) in the headline run too")
    ap.add_argument("--no-prefill", action="store_true")
    ap.add_argument("--peer-fetch", action="store_true",
                    help="also time the expert-sharded peer-fetch mode (one shared model across ranks)")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)

    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # one GPU per rank; more ranks than GPUs (functional runs on a 1-GPU box) share
    # devices, and NCCL cannot place two ranks on one device, so those use gloo
    ndev = torch.cuda.device_count()
    oversub = world > ndev
    local_dev = local % ndev
    torch.cuda.set_device(local_dev)
    if world > 1:
        if oversub:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local_dev))
    red_dev = torch.device("cpu") if oversub else torch.device("cuda", local_dev)
    if oversub:
        # ranks time-share a GPU: an arrival-gated K3 would hold every SM while it waits
        os.environ["FATE_OVERLAP"] = "0"

    from paper_2502_12224_b200 import pipeline as P
    from paper_2502_12224_b200.cache import LayeredExpertCache, plan_allocation
    from paper_2502_12224_b200.engine import OffloadEngine, overlap_default
    from paper_2502_12224_b200.experts import ExpertStore

    peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))) if os.path.exists(
        os.path.join(ROOT, "MEASURED_PEAKS.json")) else {"hbm_gbs": 6650.0, "_fallback": True}
    cfg = qwen_cfg()
    T = args.tokens
    trace, weights = make_trace(cfg, T, seed=rank)
    # one model, replicas serve independent request streams (trace seed = rank); the
    # packed expert pools live once per node in /dev/shm, filled by local rank 0 and
    # page-locked by every rank, instead of a private pinned pool each
    shm = f"fate_bench_{os.environ.get('MASTER_PORT', '0')}" if world > 1 else None
    store = ExpertStore(cfg, bits=(4, 2), seed=0, shared_intermediate=QWEN["shared"], shared_bits=16, shm=shm,
                        shm_owner=local == 0, barrier=dist.barrier if world > 1 else None)
    budget = cfg.dense_bytes + QWEN["slots"] * cfg.expert_bytes[4]
    plan = plan_allocation(cfg, budget, 4)
    strategy = P.Strategy.fate()
    _, g, ch = trace.dense_arrays(cfg)
    dev = torch.device("cuda", local_dev)
    gd, chd = torch.as_tensor(g, device=dev), torch.as_tensor(ch, device=dev)

    # the dense part of every step (attention block with a K/V cache over a 512-token
    # prompt + Qwen's shared-expert gate) executes on the device
    # The headline line is the MoE-layer path (the reference charges attention as the
    # constant t_attn); --dense executes the dense part in the headline too, and the
    # line always carries a "dense_part" measurement with it executed.
    from paper_2502_12224_b200.dense import DenseConfig, DenseWeights
    dense_w = DenseWeights(cfg, DenseConfig.qwen_moe(), seed=0)
    dense = dense_w if args.dense else None
    CTX0 = 512
    # -- measured TimingModel -> n (transfer_budget, pipeline.py:151-156)
    from paper_2502_12224_b200.gatesim import GenConfig as GenConfigFn, gen_trace as gen_trace_fn
    eng = OffloadEngine(cfg, plan.per_layer_capacity, store, weights, P.knobs_for(strategy, plan, 0),
                        max_tokens=max(T, 512))
    if dense is not None:
        eng.set_dense(dense, max_ctx=CTX0 + max(T, 64), ctx0=CTX0)
    eng.set_overlap(False)  # the TimingModel's t_moe is K3 compute: calibrate with the stream-wait protocol
    cal = eng.decode(gd[:32], chd[:32])
    eng.set_overlap(overlap_default())
    io = {}
    for b in (4, 2):
        src = store.host_pool(b)[:16]
        dst = torch.empty_like(src, device=dev)
        s = torch.cuda.Stream()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(s):
            dst.copy_(src, non_blocking=True)
            e0.record(s)
            for i in range(16):
                dst[i].copy_(src[i], non_blocking=True)
            e1.record(s)
        torch.cuda.synchronize()
        io[b] = e0.elapsed_time(e1) / 16
    t_attn = cal.stats["dense_ms"] / cal.stats["steps"] if dense is not None else 0.01
    timing = P.TimingModel(t_moe=(cal.stats["ffn_ms"] - cal.stats["k3_wait_ms"]) / cal.stats["steps"], t_attn=t_attn,
                           t_gate=cal.stats["gate_ms"] / cal.stats["steps"], t_expert_io={4: io[4], 2: io[2]},
                           dequant_ms=0.0)
    n = P.transfer_budget(timing, strategy.prefetch_bits())
    eng.set_strategy(P.knobs_for(strategy, plan, n))

    # -- warmup + timed steps (cold cache each step)
    for _ in range(args.warmup):
        eng.reset_cache()
        eng.decode(gd, chd)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    stats = []
    with ClockSampler(local_dev) as clk:
        t_wall = time.perf_counter()
        for _ in range(args.steps):
            eng.reset_cache()
            stats.append(eng.decode(gd, chd).stats)
        wall = time.perf_counter() - t_wall
    torch.cuda.synchronize()
    gpu_s = sum(s["gpu_ms"] for s in stats) / 1000.0
    if world > 1:
        t = torch.tensor([gpu_s], device=red_dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        gpu_s = float(t.item())
        dist.barrier()
    value = T * args.steps * world / gpu_s
    agg = {k: sum(s[k] for s in stats) for k in ("ffn_ms", "gate_ms", "ffn_bytes", "accesses", "cache_hits",
                                                   "arrival_hits", "h2d_bytes", "copy_busy_ms", "transfers_done",
                                                   "trace_mismatches", "steps", "ondemand_issued", "prefetch_issued",
                                                   "dense_ms", "k3_wait_ms")}
    # In the timed runs K3 is arrival-gated (launched behind K1, waiting per expert
    # for its copy), so its event interval includes the waits.  The K3 roofline and
    # the H2D rate come from one more decode of the same trace with the stream-wait
    # protocol (K3 starts once the step's copies landed: its events time compute
    # alone) and every transfer timed (the timed runs sample every 8th transfer:
    # events between copies delay the copy engine); two copy streams overlap, so
    # H2D is bytes over the union of the copy intervals.
    eng.set_copy_timing(1)
    eng.set_overlap(False)
    eng.reset_cache()
    h2d_run = eng.decode(gd, chd).stats
    eng.set_copy_timing(8)
    eng.set_overlap(overlap_default())
    k3_launches = h2d_run["steps"]
    k3_ms = h2d_run["ffn_ms"] / k3_launches
    k3_bytes = h2d_run["ffn_bytes"] / k3_launches
    achieved = k3_bytes / (k3_ms * 1e-3) / 1e9
    k3_overlap = {"ms_per_launch_incl_waits": agg["ffn_ms"] / agg["steps"],
                  "wait_ms_per_launch": agg["k3_wait_ms"] / agg["steps"],
                  "stream_wait_protocol_tokens_per_s": T / (h2d_run["gpu_ms"] * 1e-3),
                  "protocol": "arrival-gated" if overlap_default() else "stream-wait (ranks share a GPU)",
                  "what": "timed runs: K3 launched behind K1, each expert's pieces start when its copy landed "
                          "(waits = longest producer-warp wait per launch)"}
    _, copies_tl = eng.timeline()
    h2d_gbs = None
    if copies_tl:
        iv = sorted((a, b) for (a, b, *_r) in copies_tl)
        busy, cur_a, cur_b = 0.0, iv[0][0], iv[0][1]
        for a, b in iv[1:]:
            if a > cur_b:
                busy += cur_b - cur_a
                cur_a, cur_b = a, b
            else:
                cur_b = max(cur_b, b)
        busy += cur_b - cur_a
        h2d_gbs = h2d_run["h2d_bytes"] / (busy * 1e-3) / 1e9 if busy > 0 else None

    # -- e2e through the public API: host GateTrace in, last-layer outputs back to host
    e2e_times, h2d_b, d2h_b = [], 0, 0
    for i in range(args.e2e_steps + 1 if args.e2e_steps else 0):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        tl, rep, res = P.simulate_decoding(trace, strategy, plan, timing, cfg, weights=weights,
                                           cache=LayeredExpertCache(plan), experts=store, return_result=True,
                                           dense=dense, dense_ctx0=CTX0)
        y_last = res.y[:, -1].cpu()
        torch.cuda.synchronize()
        if i:
            e2e_times.append(time.perf_counter() - t0)
        h2d_b = g.nbytes + ch.nbytes
        d2h_b = y_last.numel() * 4
        res.y = None
    e2e = T / float(np.mean(e2e_times)) * world if e2e_times else None

    cpu, parity = None, None
    if rank == 0 and not args.no_cpu:
        # cpu_baseline: the CPU restatement of the same path on the host cores, on the first
        # cpu_tokens tokens with the store's own packed experts; its schedule over the whole
        # trace is also the trace-parity check of the engine's first timed step's decisions
        from oracle import fate_oracle as O
        lib = O.cpu_lib()
        cores = lib.fate_cpu_threads(0)
        sh_cache = {l: store.shared_buffer(l).cpu().numpy() for l in range(cfg.num_layers)}
        getb = lambda l, e, b: store.packed(l, e, b).numpy()  # noqa: E731
        cpu_port(cfg, trace, weights, plan, n, 2, getb, lambda l: sh_cache[l], lib)
        secs, _ = cpu_port(cfg, trace, weights, plan, n, args.cpu_tokens, getb, lambda l: sh_cache[l], lib)
        cpu = {"value": args.cpu_tokens / secs, "unit": "tokens/s", "cores": cores, "kind": "port",
               "sample": f"first {args.cpu_tokens} tokens of the same trace x 24 layers: fp64 gate + top-4, ARC, "
                         "the routed experts in the width the GPU computed them in + bf16 shared FFN "
                         "(AVX2 C threads over rows)"}
        _, port_logs = cpu_port(cfg, trace, weights, plan, n, T, None, None, lib, ffn=False)
        eng.reset_cache()
        vlogs = eng.decode(gd, chd, want_logs=True).logs
        keys = ("chosen", "hits", "ondemand", "victims")
        bad = sum(1 for a_, b_ in zip(vlogs, port_logs)
                  if tuple(a_[k_] for k_ in keys) != tuple(b_[k_] for k_ in keys) or a_["fmt_bits"] != b_["fmt_bits"]
                  or (n > 0 and a_.get("pred") != b_.get("pred")))
        parity = {"trace_parity": bad == 0 and len(vlogs) == len(port_logs), "steps": len(vlogs),
                  "mismatched_steps": bad, "fields": list(keys) + ["fmt_bits"] + (["pred"] if n > 0 else []),
                  "against": "oracle.port_decode schedule over the whole timed trace (cold cache)"}
    # expert-sharded peer-fetch mode (BASELINE configs[4]): each rank
    # homes (l*E+e) mod G of the experts in its HBM; misses are device/peer copies
    peer = None
    if args.peer_fetch:
        from paper_2502_12224_b200.replicas import ExpertShards
        shards = ExpertShards(store, bits=(4, 2), rank=rank, world_size=world, device=dev)
        shards.attach(eng)
        eng.reset_cache()
        eng.decode(gd, chd)
        pst = []
        for _ in range(2):
            eng.reset_cache()
            pst.append(eng.decode(gd, chd).stats)
        p_s = sum(x["gpu_ms"] for x in pst) / 1000.0
        if world > 1:
            tt = torch.tensor([p_s], device=red_dev, dtype=torch.float64)
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            p_s = float(tt.item())
        peer = {"workload": f"Qwen1.5-MoE shape decode, experts sharded over {world} GPU(s), misses served "
                            "from the home GPU's HBM (NVLink peer copy for remote homes)",
                "tokens_per_s": T * len(pst) * world / p_s, "home_pool_bytes_per_gpu": shards.device_bytes,
                "d2d_bytes": sum(x["d2d_bytes"] for x in pst), "h2d_bytes": sum(x["h2d_bytes"] for x in pst),
                "k3_ms_per_launch": sum(x["ffn_ms"] - x["k3_wait_ms"] for x in pst) / sum(x["steps"] for x in pst)}
        shards.detach(eng)
        shards.close()
    # -- two more regimes of the same decode: (i) prefetch exercised --
    # the paper's TimingModel (t_io[4] = 1.6 ms vs 24 ms of compute) gives n = 15, so
    # every step issues cross-layer INT4 prefetches on the copy streams while K3 runs;
    # (ii) a warm cache -- decode continues on the cache a 512-token prefill of the
    # same model left (compare_strategies chaining), so K1 / K3 dominate, not PCIe
    regimes = {}
    if not args.no_regimes:
        paper = P.TimingModel(t_moe=13.0, t_attn=9.0, t_gate=2.0, t_expert_io={16: 6.0, 8: 3.0, 4: 1.6, 2: 0.85})
        n_p = P.transfer_budget(paper, strategy.prefetch_bits())
        eng.set_strategy(P.knobs_for(strategy, plan, n_p))
        pst = []
        for _ in range(2):
            eng.reset_cache()
            pst.append(eng.decode(gd, chd).stats)
        regimes["prefetch_n15"] = {
            "tokens_per_s": T * len(pst) / (sum(x["gpu_ms"] for x in pst) / 1e3), "transfer_budget_n": n_p,
            "prefetch_issued": sum(x["prefetch_issued"] for x in pst) // len(pst),
            "ondemand_issued": sum(x["ondemand_issued"] for x in pst) // len(pst),
            "dropped_before_start": sum(x["transfers_dropped"] for x in pst) // len(pst),
            "h2d_gbs": sum(x["h2d_bytes"] for x in pst) / (sum(x["copy_busy_ms"] for x in pst) * 1e-3) / 1e9,
            "copy_busy_fraction_of_step": sum(x["copy_busy_ms"] for x in pst) / sum(x["gpu_ms"] for x in pst),
            "hit_rate_combined": sum(x["cache_hits"] + x["arrival_hits"] for x in pst) / sum(x["accesses"] for x in pst),
            "what": "paper TimingModel (n = 15): predicted experts of layer l+1 prefetched in INT4 during layer l"}
        eng.set_strategy(P.knobs_for(strategy, plan, n))
        pre_tr, _ = gen_trace_fn(cfg, GenConfigFn(seed=rank + 1, num_tokens=512, phase="prefill"), weights=weights)
        _, gp, chp = pre_tr.dense_arrays(cfg)
        gpd, chpd = torch.as_tensor(gp, device=dev), torch.as_tensor(chp, device=dev)
        if eng.max_tokens >= 512:
            wst = []
            for _ in range(2):
                eng.reset_cache()
                eng.prefill(gpd, chpd, timed=False)
                wst.append(eng.decode(gd, chd).stats)
            regimes["warm_after_prefill512"] = {
                "tokens_per_s": T * len(wst) / (sum(x["gpu_ms"] for x in wst) / 1e3),
                "hit_rate_cache": sum(x["cache_hits"] for x in wst) / sum(x["accesses"] for x in wst),
                "k3_ms_per_launch": sum(x["ffn_ms"] - x["k3_wait_ms"] for x in wst) / sum(x["steps"] for x in wst),
                "k1_ms_per_launch": sum(x["gate_ms"] for x in wst) / sum(x["steps"] for x in wst),
                "h2d_bytes_per_token": sum(x["h2d_bytes"] for x in wst) / (T * len(wst)),
                "what": "decode on the cache a 512-token prefill of the same model warmed (pipeline.py:828-849)"}
        del gpd, chpd
        # (iii) every expert resident (capacity E in every layer, 7.8 GB of INT4 slots):
        # no transfers at all, the step is K1 + K3 -- the engine's compute floor
        ares = OffloadEngine(cfg, [cfg.num_experts] * cfg.num_layers, store, weights, P.knobs_for(strategy, plan, n),
                             max_tokens=max(T, 64))
        for l in range(cfg.num_layers):
            ares.seed_resident(l, range(cfg.num_experts))
        ares.decode(gd[:16], chd[:16])
        ast_ = [ares.decode(gd, chd).stats for _ in range(2)]
        regimes["all_resident"] = {
            "tokens_per_s": T * len(ast_) / (sum(x["gpu_ms"] for x in ast_) / 1e3),
            "k3_ms_per_launch": sum(x["ffn_ms"] - x["k3_wait_ms"] for x in ast_) / sum(x["steps"] for x in ast_),
            "k3_gbs": sum(x["ffn_bytes"] for x in ast_) / (sum(x["ffn_ms"] - x["k3_wait_ms"] for x in ast_) * 1e-3) / 1e9,
            "k1_ms_per_launch": sum(x["gate_ms"] for x in ast_) / sum(x["steps"] for x in ast_),
            "what": "every expert resident in INT4 (no transfers): K1 + K3 only"}
        ares.close()
    # -- the dense part executed: attention block with a K/V cache
    # over a 512-token prompt + Qwen's shared-expert gate in every step; t_attn is then
    # measured instead of assumed, which sets the transfer budget n of this run
    dense_part = None
    if dense is None:
        eng.set_dense(dense_w, max_ctx=CTX0 + max(T, 64), ctx0=CTX0)
        eng.set_strategy(P.knobs_for(strategy, plan, n))
        eng.reset_cache()
        cal_d = eng.decode(gd[:32], chd[:32]).stats
        t_attn_d = cal_d["dense_ms"] / cal_d["steps"]
        timing_d = P.TimingModel(t_moe=timing.t_moe, t_attn=t_attn_d, t_gate=timing.t_gate,
                                 t_expert_io=dict(timing.t_expert_io), dequant_ms=0.0)
        n_d = P.transfer_budget(timing_d, strategy.prefetch_bits())
        eng.set_strategy(P.knobs_for(strategy, plan, n_d))
        dst = []
        for _ in range(2):
            eng.reset_cache()
            dst.append(eng.decode(gd, chd).stats)
        d_s = sum(x["gpu_ms"] for x in dst) / 1000.0
        if world > 1:
            tt = torch.tensor([d_s], device=red_dev, dtype=torch.float64)
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            d_s = float(tt.item())
        dense_part = {"tokens_per_s": T * len(dst) * world / d_s, "dense_ms_per_step":
                      sum(x["dense_ms"] for x in dst) / sum(x["steps"] for x in dst),
                      "t_attn_ms_measured": t_attn_d, "transfer_budget_n": n_d,
                      "what": f"attention (16 x 128 heads, q/k/v bias, RoPE, K/V cache over a {CTX0}-token prompt) + "
                              "shared-expert gate executed before every gate kernel; n from the measured t_attn"}
    pre = None
    # prefill (configs[2]) is a single-GPU workload; under torchrun every rank would
    # pin its own 15 GB DeepSeek host pools, so it is measured at N = 1 only
    if not args.no_prefill and world == 1:
        eng.close()
        eng = None
        torch.cuda.empty_cache()
        pre = bench_prefill(peaks, rank)
    if rank == 0:
        clocks = clk.summary()
        out = {
            "metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1000 * gpu_s / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "int4/int2 weights, fp32 accumulate, fp64 router",
            "data": "synthetic (random-init experts, gen_trace gate inputs)",
            "config": {"workload": "Qwen1.5-MoE-A2.7B shape decode bs=1, fixed expert budget (BASELINE configs[1])",
                       "layers": cfg.num_layers, "experts": cfg.num_experts, "top_k": cfg.top_k,
                       "hidden": cfg.hidden_dim, "expert_intermediate": cfg.intermediate_dim,
                       "shared_intermediate": QWEN["shared"], "shared_bits": 16, "slots_int4": QWEN["slots"],
                       "plan": list(plan.per_layer_capacity), "tokens_per_step": T, "strategy": "fate",
                       "transfer_budget_n": n, "timing_model_ms": timing.to_dict(), "cache_start": "cold each step",
                       "dense_part": "not executed in the headline (reference: constant t_attn); see dense_part"
                       if dense is None else
                       f"executed: attention (16 x 128 heads, K/V cache, prompt {CTX0} tokens) + shared-expert gate",
                       "l2": "inputs larger than L2 (1.95 GB slot pool + 12.5 GB pinned host pools)",
                       "parallelism": f"replicas x{world}",
                       "devices": ndev if oversub else world,
                       "host_pools": "one /dev/shm copy per node, page-locked by every rank" if world > 1
                       else "pinned, private"},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peaks["hbm_gbs"], "unit": "GB/s",
                         "frac": achieved / peaks["hbm_gbs"], "traffic": load_traffic()[0],
                         "traffic_source": load_traffic()[1],
                         "kernel": "K3 ffn_up+ffn_down (dequant-fused SwiGLU GEMV)",
                         "bytes_per_launch": k3_bytes, "ms_per_launch": k3_ms,
                         "measured_in": "CUDA events on the engine's compute stream, one more decode of the timed "
                                        "trace with the stream-wait protocol (K3 events = compute only)",
                         "peak_source": "MEASURED_PEAKS.json hbm_gbs" if "_fallback" not in peaks else "fallback"},
            "cpu_baseline": cpu,
            "trace_parity": parity["trace_parity"] if parity else None,
            "trace_parity_detail": parity,
            "e2e": {"value": e2e, "unit": "tokens/s", "h2d_bytes_per_step": h2d_b, "d2h_bytes_per_step": d2h_b}
            if e2e else None,
            # per decode step K1 (router + split + prediction + the step's ARC update) + K3; per run
            # run_begin + the final ARC flush (agg["steps"] already sums the steps of all timed runs)
            # + with the dense part, per step QKV GEMV, RoPE/append, attention, combine, Wo
            # GEMV, shared gate, and one embedding per token
            "gpu_launches": int(2 * agg["steps"] + 2 * args.steps
                                + (6 * agg["steps"] + agg["steps"] // cfg.num_layers if dense is not None else 0)),
            "clocks": clocks,
            "hit_rate_cache": agg["cache_hits"] / agg["accesses"],
            "hit_rate_combined": (agg["cache_hits"] + agg["arrival_hits"]) / agg["accesses"],
            "h2d": {"gbs": h2d_gbs, "bytes": agg["h2d_bytes"], "copies": agg["transfers_done"],
                    "ondemand": agg["ondemand_issued"], "prefetch": agg["prefetch_issued"]},
            "k1_ms_per_launch": agg["gate_ms"] / agg["steps"],
            "k1_note": "K1 event time = programmatic launch behind K3 + router rows + split + on-demand set posted + "
                       "prediction + K3 batch + the step's ARC update (warp 1, formerly a side-stream kernel); in cold "
                       "decode the event is longer while the step's H2D copies run (off the critical path: K3 waits "
                       "for those copies anyway); regimes.all_resident.k1_ms_per_launch is K1 without copies",
            "k3_overlap": k3_overlap,
            "dense_ms_per_step": agg["dense_ms"] / agg["steps"] if dense is not None else None,
            "trace_mismatches": agg["trace_mismatches"],
            "prefill": pre,
            "peer_fetch": peer,
            "dense_part": dense_part,
            "regimes": regimes,
            "wall_s_timed": wall,
        }
        print(json.dumps(out), flush=True)
    if eng is not None:
        eng.close()
    if world > 1:
        store.close()
        dist.barrier()
        if local == 0:
            store.remove_shared()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
