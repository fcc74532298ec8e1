"""Kernel-level measurement harness (not a bench line).

  k3      : K3 (ffn_up + ffn_down) standalone at the Qwen decode shape: 4 routed
            INT4 experts + the bf16 shared expert (5632), rotating over 24
            expert sets so the working set (~2 GB) exceeds L2; CUDA-event timed.
  allhit  : the decode engine on the Qwen shape with every expert resident
            (capacity = E in every layer), so no step waits on the host; used
            for ncu captures of K1/K3 inside the real step sequence.
Usage: python tools/profile_kernels.py k3|allhit [iters]
"""
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2502_12224_b200 import ops  # noqa: E402


def k3(iters: int):
    H, I, Is = 2048, 1408, 5632
    g = torch.Generator(device="cuda").manual_seed(0)
    sets = []
    for s in range(24):
        bufs = []
        for j in range(4):
            w = [torch.randn(sh, generator=g, device="cuda") * 0.02 for sh in ((I, H), (I, H), (H, I))]
            bufs.append(ops.pack_expert(*w, 4 if j != 3 else 2))
        w = [torch.randn(sh, generator=g, device="cuda") * 0.02 for sh in ((Is, H), (Is, H), (H, Is))]
        bufs.append(ops.pack_expert(*w, 16))
        sets.append(bufs)
    x = torch.randn(H, device="cuda")
    nbytes = [sum(b.numel() - 256 for b in s) for s in sets]
    for s in sets[:4]:
        ops.ffn_decode(x, s, [0.3, 0.2, 0.1, 0.05, 1.0])
    torch.cuda.synchronize()
    # the standalone entry point synchronizes per call; time the device span with events
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(iters)]
    for i in range(iters):
        s = sets[i % len(sets)]
        ev[i][0].record()
        ops.ffn_decode(x, s, [0.3, 0.2, 0.1, 0.05, 1.0])
        ev[i][1].record()
    torch.cuda.synchronize()
    ms = np.array([a.elapsed_time(b) for a, b in ev])
    by = np.array([nbytes[i % len(sets)] for i in range(iters)])
    out = {"k3_ms_median": float(np.median(ms)), "bytes": int(by[0]), "gbs_median": float(np.median(by / (ms * 1e-3)) / 1e9)}
    print(json.dumps(out))


def k3sweep(iters: int):
    """K3 alone (fate_ffn_decode_timed) on expert sets of one format each and on
    the Qwen mixes, cycling over enough copies of each set that the working set
    exceeds 2x L2 (so every launch streams from HBM)."""
    H, I, Is = 2048, 1408, 5632
    g = torch.Generator(device="cuda").manual_seed(0)

    def mk(I_, bits):
        w = [torch.randn(sh, generator=g, device="cuda") * 0.02 for sh in ((I_, H), (I_, H), (H, I_))]
        return ops.pack_expert(*w, bits)
    x = torch.randn(H, device="cuda")
    specs = {"bf16_shared": [(Is, 16)], "int4x4": [(I, 4)] * 4, "int2x4": [(I, 2)] * 4, "int8x4": [(I, 8)] * 4,
             "qwen_mix_int4": [(I, 4)] * 4 + [(Is, 16)], "qwen_mix_int2": [(I, 2)] * 3 + [(I, 4), (Is, 16)],
             "int4x12": [(I, 4)] * 12, "qwen_bench_mix": [(I, 2)] * 4 + [(Is, 16)]}
    out = {}
    only = os.environ.get("K3_ONLY")
    for name, spec in specs.items():
        if only and name != only:
            continue
        one = sum(make_layout_bytes(H, i, b) for i, b in spec)
        nsets = max(2, min(64, int(np.ceil(300e6 / one))))
        sets = [[mk(i, b) for i, b in spec] for _ in range(nsets)]
        _, ms = ops.ffn_decode_timed(x, sets, [0.1] * len(spec), iters)
        out[name] = {"ms": ms, "MB": one / 1e6, "gbs": one / (ms * 1e-3) / 1e9, "sets": nsets}
        del sets
        torch.cuda.empty_cache()
        print(name, json.dumps(out[name]))
    print(json.dumps(out))


def k3prof(iters: int):
    """Profiling build only (FATE_PROF=1): K3 phase stamps per CTA and CTA 0's
    per-stage consumer timeline, for each K3_SPECS mix (default: the bench mix)."""
    from paper_2502_12224_b200 import _lib
    H, I, Is = 2048, 1408, 5632
    g = torch.Generator(device="cuda").manual_seed(0)

    def mk(I_, bits, H_=H):
        w = [torch.randn(sh, generator=g, device="cuda") * 0.02 for sh in ((I_, H_), (I_, H_), (H_, I_))]
        return ops.pack_expert(*w, bits)
    specs = {"bf16_shared": [(Is, 16)], "int2x4": [(I, 2)] * 4, "qwen_bench_mix": [(I, 2)] * 4 + [(Is, 16)],
             "int4x4": [(I, 4)] * 4}
    want = os.environ.get("K3_SPECS", "qwen_bench_mix,bf16_shared,int2x4").split(",")
    x = torch.randn(H, device="cuda")
    for name in want:
        spec = specs[name]
        sets = [[mk(i, b) for i, b in spec] for _ in range(4)]
        _, ms = ops.ffn_decode_timed(x, sets, [0.1] * len(spec), iters)
        buf = np.zeros(192 * 8 + 256 * 4, dtype=np.uint64)
        _lib.load().fate_k3_profile(buf.ctypes.data)
        P = buf[:192 * 8].reshape(192, 8).astype(np.int64)
        P = P[:148]
        t0 = P[:, 0].min()
        names = ["start", "plan", "x", "drained", "partials", "barrier", "done"]
        print(f"== {name}: {ms * 1e3:.2f} us per launch")
        for i, nm in enumerate(names):
            v = (P[:, i] - t0) / 1e3
            print(f"  {nm:9s} median {np.median(v):7.2f}  min {v.min():7.2f}  max {v.max():7.2f}  argmax {int(v.argmax())}")
        nq = sum(i // 64 for i, b in spec if b != 16)
        dr = (P[:, 3] - t0) / 1e3
        if 0 < nq < 148:
            print(f"  drained: CTAs with a quantized unit (< {nq}) median {np.median(dr[:nq]):.2f} max {dr[:nq].max():.2f}"
                  f" | bf16 only median {np.median(dr[nq:]):.2f} max {dr[nq:].max():.2f}")
        S = buf[192 * 8:].reshape(256, 4).astype(np.int64)
        n = int((S[:, 1] > 0).sum())
        print("  CTA0 stages: [wait-start, full, released] us, tag (kind*1e6 + j*1e4 + rows)")
        for k in range(min(n, 40)):
            print(f"   {k:3d} {(S[k, 0] - t0) / 1e3:7.2f} {(S[k, 1] - t0) / 1e3:7.2f} {(S[k, 2] - t0) / 1e3:7.2f}  {S[k, 3]}")
        del sets
        torch.cuda.empty_cache()


def k4prof(tokens: int):
    """Profiling build only (FATE_PROF=1): CTA 0's per-stage K4 timeline of the
    last up-projection launch of an all-resident DeepSeek-shape prefill."""
    from paper_2502_12224_b200 import _lib
    prefill(tokens, modes=("allhit",))
    buf = np.zeros(256 * 5, dtype=np.uint64)
    _lib.load().fate_k4_profile(buf.ctypes.data)
    S = buf.reshape(256, 5).astype(np.int64)
    n = int((S[:, 0] > 0).sum())
    t0 = S[:n][S[:n] > 0].min()
    print("stage: issued landed dequantized mma_full mma_committed (us from the first stamp)")
    for k in range(min(n, 80)):
        print(f"  {k:3d} " + " ".join(f"{(S[k, i] - t0) / 1e3:8.2f}" if S[k, i] else "       -" for i in range(5)))
    d = np.diff(S[:n, 4]) / 1e3
    print(f"per-stage period (commit to commit) median {np.median(d):.3f} us; landed-issued median "
          f"{np.median((S[:n, 1] - S[:n, 0]) / 1e3):.3f}; dequant {np.median((S[:n, 2] - S[:n, 1]) / 1e3):.3f}; "
          f"full->commit {np.median((S[:n, 4] - S[:n, 3]) / 1e3):.3f}; arrive->mma saw full "
          f"{np.median((S[:n, 3] - S[:n, 2]) / 1e3):.3f}")


def make_layout_bytes(H, I, bits):
    n = 3 * H * I
    return n * 2 if bits == 16 else n * bits // 8 + n // 64 * 8


def print_k3_trace(_lib, mhz=1965.0):
    buf = np.zeros(160 * 8 + 17 * 48 * 3 + 32, dtype=np.uint64)
    _lib.load().fate_k3_profile(buf.ctypes.data)
    prof = buf[:1280].reshape(160, 8)
    P = prof[:148].astype(np.float64)
    rel = (P - P[:, 0].min()) / 1000.0
    names = ["start", "cons", "xlay", "phaseA", "gbar", "alay", "phaseB", "prod_done"]
    print("K3 phase timestamps (us from first CTA start): median / max over CTAs")
    for i, nm in enumerate(names):
        print(f"  {nm:10s} {np.median(rel[:, i]):8.2f} {rel[:, i].max():8.2f}")
    tr = buf[1280:1280 + 17 * 48 * 3].view(np.int64).reshape(17, 48, 3).astype(np.float64)
    sub = buf[1280 + 17 * 48 * 3:].view(np.int64).reshape(8, 4).astype(np.float64)
    nz = tr[tr > 0]
    t0 = nz.min() if nz.size else 0.0
    us = np.where(tr > 0, (tr - t0) / mhz, np.nan)
    for t in range(8):
        if sub[t, 0] > 0:
            print(f"  sub tile {t}: dots done {(sub[t,0]-t0)/mhz:7.2f} sums {(sub[t,1]-t0)/mhz:7.2f} "
                  f"store {(sub[t,2]-t0)/mhz:7.2f}")
    print("CTA0 trace (us): producer [wait-start pre-copy issued] | consumer w1 [wait full released] | "
          "max over consumers of release")
    for t in range(48):
        if np.all(np.isnan(us[:, t, :])):
            break
        rel_max = np.nanmax(us[1:, t, 2]) if not np.all(np.isnan(us[1:, t, 2])) else np.nan
        full_min = np.nanmin(us[1:, t, 1]) if not np.all(np.isnan(us[1:, t, 1])) else np.nan
        print(f"  {t:2d} P[{us[0,t,0]:6.2f} {us[0,t,1]:6.2f} {us[0,t,2]:6.2f}] "
              f"C1[{us[1,t,0]:6.2f} {us[1,t,1]:6.2f} {us[1,t,2]:6.2f}] first_full {full_min:6.2f} last_rel {rel_max:6.2f}")


def prefill(tokens: int, modes=("allhit", "cold448")):
    """DeepSeek-MoE-16B shape prefill (BASELINE configs[2]): 28 layers, 64 experts
    top-6 + shared 2 x 1408 (as one 2816 expert, bf16), T tokens; (a) every expert
    resident (pure K4 tensor-core time), (b) 448 INT4 slots cold (the bench case)."""
    from paper_2502_12224_b200.core import ModelConfig
    from paper_2502_12224_b200.engine import OffloadEngine, StrategyKnobs
    from paper_2502_12224_b200.experts import ExpertStore
    from paper_2502_12224_b200.gatesim import GenConfig, gen_trace
    from paper_2502_12224_b200.cache import plan_allocation
    cfg = ModelConfig.from_shape(28, 64, 6, 2048, 1408, 3, dense_bytes=28 * 3 * 2048 * 2816 * 2)
    tr, w = gen_trace(cfg, GenConfig(seed=0, num_tokens=tokens, phase="prefill"))
    store = ExpertStore(cfg, bits=(4, 2), shared_intermediate=2816, shared_bits=16)
    _, g, ch = tr.dense_arrays(cfg)
    gd, chd = torch.as_tensor(g, device="cuda"), torch.as_tensor(ch, device="cuda")
    out = {}
    for mode in modes:
        if mode == "allhit":
            caps = [64] * 28
        else:
            caps = list(plan_allocation(cfg, cfg.dense_bytes + 448 * cfg.expert_bytes[4], 4).per_layer_capacity)
        eng = OffloadEngine(cfg, caps, store, w, StrategyKnobs(budget_n=0), max_tokens=max(tokens, 64))
        if mode == "allhit":
            for l in range(28):
                eng.seed_resident(l, range(64))
        eng.prefill(gd, chd)
        if mode == "allhit":
            for l in range(28):
                eng.seed_resident(l, range(64))
        else:
            eng.reset_cache()
        t0 = time.perf_counter()
        Y, st, logs, step_ms, copies = eng.prefill(gd, chd)
        wall = time.perf_counter() - t0
        out[mode] = {"gpu_ms": st["gpu_ms"], "tok_s": tokens / st["gpu_ms"] * 1e3, "k4_ms": st["ffn_ms"],
                     "k4_tflops": st["ffn_flops"] / (st["ffn_ms"] * 1e-3) / 1e12, "wall_s": wall,
                     "h2d_gb": st["h2d_bytes"] / 1e9}
        eng.close()
        print(mode, json.dumps(out[mode]), flush=True)
    print(json.dumps(out))


def timeline(tokens: int):
    """Per-step critical path of the bench decode (Qwen shape, 360 INT4 slots, cold):
    K1, K1 end -> first copy start, copy span, last copy end -> K3 start, K3, K3 end ->
    next K1 (all from the engine's CUDA events, ms relative to the run start)."""
    sys.path.insert(0, ROOT)
    import bench as B
    from paper_2502_12224_b200 import pipeline as P
    from paper_2502_12224_b200.cache import plan_allocation
    from paper_2502_12224_b200.engine import OffloadEngine
    from paper_2502_12224_b200.experts import ExpertStore
    cfg = B.qwen_cfg()
    trace, weights = B.make_trace(cfg, tokens, 0)
    store = ExpertStore(cfg, bits=(4, 2), seed=0, shared_intermediate=B.QWEN["shared"], shared_bits=16)
    plan = plan_allocation(cfg, cfg.dense_bytes + B.QWEN["slots"] * cfg.expert_bytes[4], 4)
    _, g, ch = trace.dense_arrays(cfg)
    gd, chd = torch.as_tensor(g, device="cuda"), torch.as_tensor(ch, device="cuda")
    eng = OffloadEngine(cfg, plan.per_layer_capacity, store, weights, P.knobs_for(P.Strategy.fate(), plan, 0),
                        max_tokens=max(tokens, 64))
    eng.set_copy_timing(1)  # every transfer in the timeline
    eng.decode(gd, chd)
    eng.reset_cache()
    res = eng.decode(gd, chd)
    sm, copies = eng.timeline()
    n = sm.shape[0]
    by_step = {}
    for (a, b, kind, step, layer, e, bits) in copies:
        by_step.setdefault(step * cfg.num_layers + layer if False else None, None)
    # copies carry (token, layer): map to the flat step index
    cs = {}
    for (a, b, kind, tok, layer, e, bits) in copies:
        cs.setdefault(tok * cfg.num_layers + layer, []).append((a, b, kind))
    rows = []
    for s in range(n):
        k1a, k1b, k3a, k3b = sm[s]
        c = cs.get(s, [])
        od = [x for x in c if x[2] == 1]
        first = min((x[0] for x in od), default=np.nan)
        last = max((x[1] for x in od), default=np.nan)
        nxt = sm[s + 1][0] if s + 1 < n else np.nan
        rows.append([k1b - k1a, first - k1b, last - first, k3a - last if od else k3a - k1b, k3b - k3a, nxt - k3b,
                     len(od)])
    for s_ in (300, 301, 302):
        print("step", s_, "K1 %.1f-%.1f K3 %.1f-%.1f" % tuple(1e3 * x for x in sm[s_]),
              "copies", [("%.1f-%.1f k%d e%d b%d" % (1e3 * a, 1e3 * b, kd, e, bt))
                         for (a, b, kd, tok, layer, e, bt) in copies if tok * cfg.num_layers + layer == s_])
    R = np.array(rows) * np.array([1e3] * 6 + [1])
    names = ["K1", "K1end->copy0", "copy span", "copyN->K3", "K3", "K3end->nextK1", "n_od"]
    med = np.nanmedian(R, axis=0)
    mean = np.nanmean(R, axis=0)
    print(json.dumps({"steps": n, "tok_s": tokens / res.stats["gpu_ms"] * 1e3,
                      "median_us": dict(zip(names, [round(float(v), 2) for v in med])),
                      "mean_us": dict(zip(names, [round(float(v), 2) for v in mean])),
                      "step_us_mean": float((sm[-1][3] - sm[0][0]) / n * 1e3)}))


def mixtral(tokens: int):
    """BASELINE configs[3]: Mixtral-8x7B shape (32 layers, 8 experts top-2, H 4096,
    I 14336), decode with quantized prefetch (Strategy.fate()), budget sweep
    S in {0, 32, 64, 128, 192, 256} INT4 slots (0-100% of 256), cold cache."""
    from paper_2502_12224_b200 import pipeline as P
    from paper_2502_12224_b200.cache import plan_allocation
    from paper_2502_12224_b200.core import ModelConfig
    from paper_2502_12224_b200.engine import OffloadEngine
    from paper_2502_12224_b200.experts import ExpertStore
    from paper_2502_12224_b200.gatesim import GenConfig, gen_trace
    cfg = ModelConfig.from_shape(32, 8, 2, 4096, 14336, 1, dense_bytes=0)
    tr, w = gen_trace(cfg, GenConfig(seed=0, num_tokens=tokens, phase="decoding"))
    store = ExpertStore(cfg, bits=(4, 2), seed=0)
    _, g, ch = tr.dense_arrays(cfg)
    gd, chd = torch.as_tensor(g, device="cuda"), torch.as_tensor(ch, device="cuda")
    strategy = P.Strategy.fate()
    rows = []
    for S in (0, 32, 64, 128, 192, 256):
        plan = plan_allocation(cfg, cfg.dense_bytes + S * cfg.expert_bytes[4], 4)
        # n = 2: the whole percentile-0.75 prediction at E = 8 (= top-2) is prefetched
        eng = OffloadEngine(cfg, plan.per_layer_capacity, store, w, P.knobs_for(strategy, plan, 2),
                            max_tokens=max(tokens, 64))
        eng.decode(gd[:4], chd[:4])
        eng.reset_cache()
        res = eng.decode(gd, chd)
        st = res.stats
        rows.append({"slots": S, "plan": list(plan.per_layer_capacity)[:4], "tok_s": tokens / st["gpu_ms"] * 1e3,
                     "hit_rate_cache": st["cache_hits"] / st["accesses"],
                     "hit_rate_combined": (st["cache_hits"] + st["arrival_hits"]) / st["accesses"],
                     "h2d_gb": st["h2d_bytes"] / 1e9, "k3_ms": st["ffn_ms"] / st["steps"],
                     "k3_gbs": st["ffn_bytes"] / st["steps"] / (st["ffn_ms"] / st["steps"] * 1e-3) / 1e9})
        eng.close()
        print(json.dumps(rows[-1]), flush=True)
    print(json.dumps({"workload": "Mixtral-8x7B shape decode, budget sweep (BASELINE configs[3])", "tokens": tokens,
                      "rows": rows}))


def allhit(iters: int):
    from paper_2502_12224_b200.core import ModelConfig
    from paper_2502_12224_b200.engine import OffloadEngine, StrategyKnobs
    from paper_2502_12224_b200.experts import ExpertStore
    from paper_2502_12224_b200.gatesim import GenConfig, gen_trace
    cfg = ModelConfig.from_shape(24, 60, 4, 2048, 1408, 3)
    tr, w = gen_trace(cfg, GenConfig(seed=0, num_tokens=iters))
    store = ExpertStore(cfg, bits=(4, 2), shared_intermediate=5632, shared_bits=16)
    eng = OffloadEngine(cfg, [60] * 24, store, w, StrategyKnobs(budget_n=0), max_tokens=max(iters, 64))
    for l in range(24):
        eng.seed_resident(l, range(60))
    _, g, ch = tr.dense_arrays(cfg)
    gd, chd = torch.as_tensor(g, device="cuda"), torch.as_tensor(ch, device="cuda")
    eng.decode(gd[:4], chd[:4])
    t0 = time.perf_counter()
    res = eng.decode(gd, chd)
    wall = time.perf_counter() - t0
    st = res.stats
    from paper_2502_12224_b200 import _lib
    print_k3_trace(_lib)
    k1 = np.zeros(16, dtype=np.uint64)
    _lib.load().fate_k1_profile(k1.ctypes.data)
    k1 = (k1.astype(np.float64) - float(k1[0])) / 1000.0
    print("K1 (us from tail-block start): row1_start %.2f last_row_arrival %.2f arc_start %.2f arc_end %.2f "
          "tail_sees_all %.2f staged %.2f routed %.2f split %.2f predicted %.2f posted %.2f tail_end %.2f" %
          (k1[10], k1[11], k1[8], k1[9], k1[1], k1[2], k1[3], k1[4], k1[5], k1[6], k1[7]))
    print(json.dumps({"tokens": iters, "gpu_ms": st["gpu_ms"], "tok_s": iters / st["gpu_ms"] * 1e3, "wall_s": wall,
                      "k3_ms": st["ffn_ms"] / st["steps"], "k1_ms": st["gate_ms"] / st["steps"],
                      "k3_gbs": st["ffn_bytes"] / st["steps"] / (st["ffn_ms"] / st["steps"] * 1e-3) / 1e9,
                      "hits": st["cache_hits"], "accesses": st["accesses"]}))


if __name__ == "__main__":
    mode = sys.argv[1]
    it = int(sys.argv[2]) if len(sys.argv) > 2 else 64
    {"k3": k3, "allhit": allhit, "k3sweep": k3sweep, "prefill": prefill, "timeline": timeline, "k4prof": k4prof,
     "mixtral": mixtral, "k3prof": k3prof}[mode](it)
