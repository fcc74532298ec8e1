"""Generate golden vectors by running the REFERENCE (`moesim`) in this container.

Run from the repo root:  python tests/golden/make_golden.py
It needs /root/reference (read-only, present only in the build container);
its outputs are committed under tests/golden/ so the tests never read the
reference at run time.  The script only *observes* the reference: it wraps
the cache, predictor and transfer channel of ``pipeline.simulate_decoding`` /
``simulate_prefill`` with logging subclasses and records what they did.
"""

from __future__ import annotations

import hashlib
import json
import os
import sys
import tempfile

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
sys.dont_write_bytecode = True

from moesim import cache as mcache  # noqa: E402
from moesim import core as mcore  # noqa: E402
from moesim import gatesim as mgate  # noqa: E402
from moesim import pipeline as mpipe  # noqa: E402
from moesim import predict as mpred  # noqa: E402
from moesim import quant as mquant  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))
PAPER_TIMING = dict(t_moe=13.0, t_attn=9.0, t_gate=2.0, t_expert_io={16: 6.0, 8: 3.0, 4: 1.6, 2: 0.85})


def ebytes(n_params: int) -> dict:
    out = {16: 2 * n_params}
    for b in (8, 4, 2):
        out[b] = -(-n_params * b // 8) + 8 * (-(-n_params // 64))
    return out


CONFIGS = {
    "tiny": dict(L=4, E=8, k=2, H=256, I=512, Lb=1, S=12, dec_tokens=64, pre_tokens=32),
    "qwen": dict(L=24, E=60, k=4, H=2048, I=1408, Lb=3, S=360, dec_tokens=8, pre_tokens=16),
    "dsk": dict(L=28, E=64, k=6, H=2048, I=1408, Lb=3, S=448, dec_tokens=4, pre_tokens=64),
    "mixtral": dict(L=32, E=8, k=2, H=4096, I=14336, Lb=1, S=64, dec_tokens=8, pre_tokens=8),
}


def model_cfg(c):
    return mcore.ModelConfig(num_layers=c["L"], num_experts=c["E"], top_k=c["k"], hidden_dim=c["H"],
                             shallow_boundary_L=c["Lb"], expert_bytes=ebytes(3 * c["H"] * c["I"]),
                             dense_bytes=0)


def trace_sha(trace) -> str:
    with tempfile.TemporaryDirectory() as d:
        p = os.path.join(d, "t.ndjson")
        mcore.write_trace(trace, p)
        return hashlib.sha256(open(p, "rb").read()).hexdigest()


def traces_for(cfg, c, seed=0):
    """Decode + prefill traces sharing gate weights (experiments.py:158-183 pattern)."""
    dec, w = mgate.gen_trace(cfg, mgate.GenConfig(seed=seed, num_tokens=c["dec_tokens"], phase="decoding"))
    pre, _ = mgate.gen_trace(cfg, mgate.GenConfig(seed=seed + 1, num_tokens=c["pre_tokens"], phase="prefill"), weights=w)
    return dec, pre, w


# ---------------------------------------------------------------------------
# Instrumentation (observation only)

LOG: dict = {}


class LogChannel(mpipe._Channel):
    def enqueue(self, kind, token, layer, expert, bits, duration, now):
        LOG.setdefault("enqueue", []).append((kind, token, layer, expert, bits))
        return super().enqueue(kind, token, layer, expert, bits, duration, now)

    def drop_stale(self, current_step):
        before = [(t.kind, t.token, t.layer, t.expert, t.bits) for t in self.pending]
        super().drop_stale(current_step)
        after = {(t.kind, t.token, t.layer, t.expert, t.bits) for t in self.pending}
        for x in before:
            if x not in after:
                LOG.setdefault("dropped", []).append(x)


class LogArc(mcache.ArcState):
    layer_id = -1

    def access(self, expert):
        before = self.resident()
        hit = super().access(expert)
        after = self.resident()
        for v in sorted(before - after):
            LOG["updates"][-1].append(v)
        return hit


_orig_update = mpipe.update_after_layer


def _logged_update(cache, layer, chosen):
    LOG.setdefault("updates", []).append([])
    return _orig_update(cache, layer, chosen)


mpipe.update_after_layer = _logged_update


class LogCache(mcache.LayeredExpertCache):
    def __init__(self, plan):
        super().__init__(plan)
        self.layers = []
        for i, c in enumerate(plan.per_layer_capacity):
            a = LogArc(capacity=c)
            a.layer_id = i
            self.layers.append(a)


class LogPredictor(mpipe.CrossLayerDecodePredictor):
    def predict(self, token, source_layer, record, chosen):
        pl = super().predict(token, source_layer, record, chosen)
        LOG.setdefault("pred", []).append((token, source_layer + 1, list(pl.experts())))
        return pl


class LogEapPredictor(mpipe.EapDecodePredictor):
    def predict(self, token, source_layer, record, chosen):
        pl = super().predict(token, source_layer, record, chosen)
        LOG.setdefault("pred", []).append((token, source_layer + 1, list(pl.experts())))
        return pl


def arc_states(cache):
    return [{"t1": list(a.t1), "t2": list(a.t2), "b1": list(a.b1), "b2": list(a.b2), "p": float(a.p_arc)}
            for a in cache.layers]


def report_dict(rep):
    return {k: getattr(rep, k) for k in ("num_tokens", "total_ms", "ttft_ms", "tpot_ms", "tokens_per_s",
                                         "recall", "hit_rate", "stall_ms", "dequant_count")}


def run_decode_logged(trace, strategy, plan, timing, cfg, weights, cache, eap_stats=None):
    LOG.clear()
    mpipe._Channel = LogChannel
    if strategy.kind == "fate":
        pred = LogPredictor(weights, strategy.prefetch_policy, cfg.top_k)
    elif strategy.kind == "eap":
        pred = LogEapPredictor(cfg.num_layers, cfg.num_experts, cfg.top_k, stats=eap_stats)
    else:
        pred = None
    tl, rep = mpipe.simulate_decoding(trace, strategy, plan, timing, cfg, weights=weights, cache=cache,
                                      predictor=pred, collect_cache_events=True)
    n = mpipe.transfer_budget(timing, strategy.prefetch_bits())
    steps = []
    by_tok = trace.by_token()
    enq = LOG.get("enqueue", [])
    preds = {(t, l): lst for t, l, lst in LOG.get("pred", [])}
    for t in sorted(by_tok):
        for l in range(cfg.num_layers):
            ch = sorted(by_tok[t][l].chosen)
            rec = {"token": t, "layer": l, "chosen": ch}
            if (t, l + 1) in preds:
                rec["pred"] = preds[(t, l + 1)][:n]
                rec["prefetch"] = [e for (k, tt, ll, e, b) in enq if k == "prefetch" and tt == t and ll == l + 1]
            rec["ondemand"] = [e for (k, tt, ll, e, b) in enq if k == "ondemand" and tt == t and ll == l]
            steps.append(rec)
    # cache hits: cache-resident at decision time = chosen - prefetched-for-step - ondemand
    pref = {}
    for (k, tt, ll, e, b) in enq:
        if k == "prefetch":
            pref.setdefault((tt, ll), set()).add(e)
    for rec in steps:
        t, l = rec["token"], rec["layer"]
        rec["hits"] = [e for e in rec["chosen"] if e not in pref.get((t, l), set()) and e not in rec["ondemand"]]
    ups = LOG.get("updates", [])
    assert len(ups) == len(steps)
    for rec, v in zip(steps, ups):
        rec["victims"] = v
    return {"n": n, "steps": steps, "report": report_dict(rep), "arcs": arc_states(cache),
            "transfers": {"prefetch": sum(1 for x in enq if x[0] == "prefetch"),
                          "ondemand": sum(1 for x in enq if x[0] == "ondemand")}}


def run_prefill_logged(trace, strategy, plan, timing, cfg, weights, cache, eap_stats=None):
    LOG.clear()
    mpipe._Channel = LogChannel
    tl, rep = mpipe.simulate_prefill(trace, strategy, plan, timing, cfg, weights=weights, cache=cache,
                                     eap_stats=eap_stats)
    enq = LOG.get("enqueue", [])
    dropped = LOG.get("dropped", [])
    layers = []
    ups = LOG.get("updates", [])
    assert len(ups) == cfg.num_layers
    for l in range(cfg.num_layers):
        iss = [(e, b) for (k, t, ll, e, b) in enq if k == "prefetch" and ll == l]
        drp = {e for (k, t, ll, e, b) in dropped if k == "prefetch" and ll == l}
        layers.append({
            "layer": l,
            "prefetch_for_next": [[e, b] for (k, t, ll, e, b) in enq if k == "prefetch" and ll == l + 1],
            "started": [e for e, b in iss if e not in drp],
            "ondemand": [[e, b] for (k, t, ll, e, b) in enq if k == "ondemand" and ll == l],
            "victims": ups[l],
        })
    return {"layers": layers, "report": report_dict(rep), "arcs": arc_states(cache)}


def dump_trace_arrays(trace, cfg):
    by = trace.by_token()
    T = len(by)
    g = np.zeros((T, cfg.num_layers, cfg.hidden_dim))
    ch = np.zeros((T, cfg.num_layers, cfg.top_k), dtype=np.int64)
    for t in sorted(by):
        for l in range(cfg.num_layers):
            r = by[t][l]
            g[t, l] = r.probe_hidden["gate_in_cur"]
            ch[t, l] = sorted(r.chosen)
    return g, ch


def eap_entries(sched):
    """EAP baseline decode (pipeline.py:301-321, predict.py:110-158) from a cold cache."""
    for name in ("tiny", "qwen"):
        c = CONFIGS[name]
        cfg = model_cfg(c)
        dec, pre, w = traces_for(cfg, c)
        timing = mcore.TimingModel(**PAPER_TIMING)
        budget = cfg.dense_bytes + c["S"] * cfg.expert_bytes[4]
        plan = mcache.plan_allocation(cfg, budget, 4)
        cache = LogCache(plan)
        sched[name]["decode_eap"] = run_decode_logged(dec, mpipe.Strategy.eap(), plan, timing, cfg, w, cache)
        # compare_strategies chaining (pipeline.py:828-849): prefill then decode share one EapStats
        cache = LogCache(plan)
        stats = mpred.EapStats(num_layers=cfg.num_layers, num_experts=cfg.num_experts)
        sched[name]["prefill_eap"] = run_prefill_logged(pre, mpipe.Strategy.eap(), plan, timing, cfg, w, cache,
                                                        eap_stats=stats)
        sched[name]["decode_eap_warm"] = run_decode_logged(dec, mpipe.Strategy.eap(), plan, timing, cfg, w, cache,
                                                           eap_stats=stats)


def main():
    golden: dict = {}
    # -------------------------------------------------------------- SPEC KATs
    kat = {}
    kat["softmax"] = mgate.softmax(np.array([2.0, 1.0, 0.0, -1.0])).tolist()
    kat["cosine"] = mgate.cosine_similarity(np.array([1.0, 0.0]), np.array([1.0, 1.0]))
    w60 = np.random.default_rng(7).random(60)
    w60 = w60 / w60.sum()
    kat["percentile_60"] = {"w": w60.tolist(), "q": 0.75,
                            "thr": mpred.nearest_rank_percentile(w60, 0.75)}
    tiny_w = mgate.GateWeights(matrices=(np.eye(60),) * 2, temperatures=(1.0, 1.0))
    pl = mpred.cross_layer_predict(w60, tiny_w, 1, mpred.PrefetchPolicy("percentile", 0.75), 4)
    kat["percentile_60"]["list"] = list(pl.experts())
    kat["recall_fig5"] = mpred.prefetch_recall([5, 11, 21, 36], [5, 21, 31, 36])
    plan_cfg = mcore.ModelConfig(num_layers=24, num_experts=60, top_k=4, hidden_dim=8, shallow_boundary_L=3,
                                 expert_bytes={16: 100, 4: 10}, dense_bytes=0)
    kat["plan_300"] = list(mcache.plan_allocation(plan_cfg, 300 * 10, 4).per_layer_capacity)
    kat["plan_100"] = list(mcache.plan_allocation(plan_cfg, 100 * 10, 4).per_layer_capacity)
    kat["plan_1500"] = list(mcache.plan_allocation(plan_cfg, 1500 * 10, 4).per_layer_capacity)
    a = mcache.ArcState(capacity=2)
    kat["arc_c2"] = [a.access(x) for x in [0, 1, 0, 2, 0]]
    a = mcache.ArcState(capacity=1)
    kat["arc_c1"] = [a.access(x) for x in [0, 0]]
    q = mquant.quantize(np.array([0.0, 1.0, 2.0, 3.0]), 2, group_size=4)
    kat["quant_2bit"] = {"codes": q.codes.tolist(), "scales": q.scales.tolist(), "zeros": q.zeros.tolist()}
    q = mquant.quantize(np.full(10, 0.37), 4, group_size=4)
    kat["quant_const"] = {"codes": q.codes.tolist(), "scales": q.scales.tolist(), "zeros": q.zeros.tolist(),
                          "deq": mquant.dequantize(q).tolist()}
    kat["pack4_0_15"] = mquant._pack(np.arange(16, dtype=np.uint8), 4).tolist()
    tm = mcore.TimingModel(t_moe=13, t_attn=9, t_gate=2, t_expert_io={4: 6, 16: 12})
    kat["transfer_budget"] = mpipe.transfer_budget(tm, 4)
    tm2 = mcore.TimingModel(**PAPER_TIMING)
    kat["transfer_budget_paper"] = mpipe.transfer_budget(tm2, 4)
    prof = mquant.PopularityProfile.from_counts(0, {i: 10 - i for i in range(8)})
    kat["assign_bits_8"] = {str(k): v for k, v in mquant.assign_bits(prof, mquant.QuantPolicy(p_int2=0.25), "prefill").items()}
    lists = [mpred.PrefetchList(1, (mpred.PrefetchEntry(1, 0.5, None), mpred.PrefetchEntry(2, 0.4, None)))] * 3
    prof = mpred.prefill_merge(lists)
    kat["prefill_merge"] = {"counts": {str(k): v for k, v in prof.counts.items()}, "ordering": list(prof.ordering)}
    kat["topk_ties"] = sorted(mcore.top_k_set(np.full(5, 0.2), 2))
    golden["kat"] = kat

    # ------------------------------------------------------------- quantize
    rng = np.random.default_rng(123)
    qcases = []
    for shape in [(7, 9), (3, 64), (16, 128), (8, 200)]:
        x = rng.standard_normal(shape) * 0.02
        x.reshape(-1)[5:70] = 0.125  # a constant run spanning a whole group
        for bits in (8, 4, 2):
            q = mquant.quantize(x, bits, group_size=64)
            qcases.append({"shape": list(shape), "bits": bits, "x": x.reshape(-1).tolist(),
                           "codes": q.codes.tolist(), "scales": q.scales.tolist(), "zeros": q.zeros.tolist()})
    golden["quant"] = qcases

    # ------------------------------------------------------------------ ARC
    rng = np.random.default_rng(99)
    arc_cases = []
    for i in range(400):
        c = int(rng.integers(0, 9))
        u = int(rng.integers(2, 17))
        seq = rng.integers(0, u, size=int(rng.integers(1, 80))).tolist()
        st = mcache.ArcState(capacity=c)
        hits = [bool(st.access(int(x))) for x in seq]
        arc_cases.append({"c": c, "seq": seq, "hits": hits,
                          "final": {"t1": st.t1, "t2": st.t2, "b1": st.b1, "b2": st.b2, "p": st.p_arc}})
    golden["arc"] = arc_cases

    # ---------------------------------------------------------- schedules
    sched = {}
    for name, c in CONFIGS.items():
        cfg = model_cfg(c)
        dec, pre, w = traces_for(cfg, c)
        timing = mcore.TimingModel(**PAPER_TIMING)
        strat = mpipe.Strategy.fate()
        budget = cfg.dense_bytes + c["S"] * cfg.expert_bytes[4]
        plan = mcache.plan_allocation(cfg, budget, 4)
        entry = {"cfg": {**c, "expert_bytes": {str(k): v for k, v in cfg.expert_bytes.items()}},
                 "plan": list(plan.per_layer_capacity),
                 "dec_sha": trace_sha(dec), "pre_sha": trace_sha(pre),
                 "taus": list(w.temperatures)}
        # decode from a cold cache
        cache = LogCache(plan)
        entry["decode_cold"] = run_decode_logged(dec, strat, plan, timing, cfg, w, cache)
        # prefill from a cold cache, then decode on the warmed cache (compare_strategies chaining)
        cache = LogCache(plan)
        entry["prefill_cold"] = run_prefill_logged(pre, strat, plan, timing, cfg, w, cache)
        entry["decode_warm"] = run_decode_logged(dec, strat, plan, timing, cfg, w, cache)
        sched[name] = entry
        if name == "tiny":
            g, ch = dump_trace_arrays(dec, cfg)
            gp, chp = dump_trace_arrays(pre, cfg)
            np.savez_compressed(os.path.join(OUT, "tiny_traces.npz"), dec_gate_in=g, dec_chosen=ch,
                                pre_gate_in=gp, pre_chosen=chp,
                                gate_w=np.stack(w.matrices), taus=np.array(w.temperatures))
            # zero-n variant (B200-like timings: no prefetch)
            t0 = mcore.TimingModel(t_moe=0.02, t_attn=0.01, t_gate=0.005,
                                   t_expert_io={16: 0.3, 8: 0.16, 4: 0.1, 2: 0.06}, dequant_ms=0.0)
            cache = LogCache(plan)
            entry["decode_cold_n0"] = run_decode_logged(dec, strat, plan, t0, cfg, w, cache)
            # top-k policy, LoD
            cache = LogCache(plan)
            entry["decode_cold_topk"] = run_decode_logged(
                dec, mpipe.Strategy.fate(prefetch_policy=mpred.PrefetchPolicy("topk")), plan, timing, cfg, w, cache)
            lod_plan = mcache.zero_plan(cfg, budget)
            cache = LogCache(lod_plan)
            entry["decode_lod"] = run_decode_logged(dec, mpipe.Strategy.lod(), lod_plan, timing, cfg, w, cache)
        print(name, "decode hit", entry["decode_cold"]["report"]["hit_rate"],
              "prefill", entry["prefill_cold"]["report"]["tokens_per_s"], flush=True)
    eap_entries(sched)
    golden["schedules"] = sched
    with open(os.path.join(OUT, "golden.json"), "w") as fh:
        json.dump(golden, fh, separators=(",", ":"))
    print("wrote", os.path.join(OUT, "golden.json"))


if __name__ == "__main__":
    main()
