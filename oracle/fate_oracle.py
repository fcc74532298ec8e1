"""CPU oracle for Fate's offloaded-MoE hot path (arXiv 2502.12224).

TEST INFRASTRUCTURE ONLY.  Nothing in ``paper_2502_12224_b200`` imports this
module; only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may use it, and only as the
checker or as the timed CPU baseline.

This is a numpy restatement of the reference's arithmetic for the path the
B200 framework executes.  Each function cites the reference ``moesim`` source
it follows (paths relative to ``/root/reference/pkg/src/moesim``).  Parity is
PINNED: ``tests/test_oracle_golden.py`` checks every function here against
golden vectors produced by running the reference itself
(``tests/golden/make_golden.py``), including the full per-step decode and
prefill schedules of ``pipeline.simulate_decoding`` / ``simulate_prefill``.

The reference has no expert FFN (it is a time constant, pipeline.py:477-479);
``ffn_swiglu`` is the repo's own fp64 definition of the expert compute the GPU
path executes and is pinned only by construction.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

# ---------------------------------------------------------------------------
# Gate, top-k, cross-layer prediction


def softmax64(z: np.ndarray) -> np.ndarray:
    """Max-subtracted fp64 softmax (gatesim.py:106-110)."""
    z = np.asarray(z, dtype=np.float64)
    ez = np.exp(z - z.max())
    return ez / ez.sum()


def gate_routing(mat: np.ndarray, tau: float, h: np.ndarray) -> np.ndarray:
    """softmax(W_l h / tau_l) in fp64 (gatesim.py:113-123)."""
    return softmax64((np.asarray(mat, np.float64) @ np.asarray(h, np.float64)) / tau)


def rank_order(w: np.ndarray) -> list[int]:
    """Experts sorted by (-w, id): the tie rule of core.py:159-163 and predict.py:80."""
    w = np.asarray(w)
    return [int(i) for i in np.lexsort((np.arange(w.shape[0]), -w))]


def top_k(w: np.ndarray, k: int) -> list[int]:
    """Top-k ids in rank order (core.py:159-163 returns the same set)."""
    return rank_order(w)[:k]


def nearest_rank_threshold(w: np.ndarray, q: float) -> float:
    """Value at rank ceil(q*n) of the ascending sample (predict.py:84-89)."""
    s = np.sort(np.asarray(w))
    r = min(max(int(math.ceil(q * s.shape[0])), 1), s.shape[0])
    return float(s[r - 1])


def predicted_list(w: np.ndarray, kind: str, q: float, k: int) -> list[int]:
    """Ordered prediction list of cross_layer_predict (predict.py:92-107).

    topk: the k best.  percentile: {w > thr} | top-k, sorted by (-w, id).
    """
    order = rank_order(w)
    if kind == "topk":
        return order[:k]
    thr = nearest_rank_threshold(w, q)
    keep = set(order[:k]) | {int(e) for e in np.nonzero(np.asarray(w) > thr)[0]}
    return [e for e in order if e in keep]


def transfer_budget(t_moe: float, t_attn: float, t_gate: float, t_io: float) -> int:
    """n = floor((t_moe + t_attn + t_gate) / t_io) (pipeline.py:151-156)."""
    return math.floor((t_moe + t_attn + t_gate) / t_io)


# ---------------------------------------------------------------------------
# Capacity plan and ARC


def plan_capacities(num_layers: int, num_experts: int, boundary: int, cache_total: int) -> list[int]:
    """Shallow-favoring split of ``cache_total`` slots (cache.py:42-74)."""
    cap = [0] * num_layers
    left = cache_total
    for layer in range(min(boundary, num_layers)):
        if left == 0:
            break
        cap[layer] = min(num_experts, left)
        left -= cap[layer]
    n_deep = num_layers - boundary
    if left > 0 and n_deep > 0:
        per = min(num_experts, left // n_deep)
        spare = left - per * n_deep if per < num_experts else 0
        for layer in range(boundary, num_layers):
            cap[layer] = per + (1 if layer - boundary < spare else 0)
    return cap


def slots_for_budget(budget: int, dense_bytes: int, slot_bytes: int) -> int:
    """(budget - dense) // expert_bytes[cached_bits] (cache.py:32-39)."""
    if budget < dense_bytes:
        raise ValueError("budget below dense footprint")
    return (budget - dense_bytes) // slot_bytes


@dataclass
class Arc:
    """One layer's ARC lists, LRU first (cache.py:104-179).

    Restated from Megiddo & Modha's ARC as the reference realises it: the
    replace() rule of cache.py:128-135 and the four access cases of
    cache.py:137-179 (T hit, B1 ghost, B2 ghost, full miss IV-A / IV-B).
    """

    c: int
    t1: list = field(default_factory=list)
    t2: list = field(default_factory=list)
    b1: list = field(default_factory=list)
    b2: list = field(default_factory=list)
    p: float = 0.0

    def resident(self) -> set:
        return set(self.t1) | set(self.t2)

    def _evict_one(self, x: int) -> int | None:
        """REPLACE: demote the LRU of T1 or T2 to its ghost list; returns the victim."""
        n1 = len(self.t1)
        if n1 and (n1 > self.p or (x in self.b2 and n1 == self.p)):
            v = self.t1.pop(0)
            self.b1.append(v)
            return v
        if self.t2:
            v = self.t2.pop(0)
            self.b2.append(v)
            return v
        if self.t1:
            v = self.t1.pop(0)
            self.b1.append(v)
            return v
        return None

    def access(self, x: int) -> tuple[bool, int | None]:
        """Returns (hit, victim removed from residency or None)."""
        c = self.c
        if c < 1:
            return False, None
        if x in self.t1 or x in self.t2:
            (self.t1 if x in self.t1 else self.t2).remove(x)
            self.t2.append(x)
            return True, None
        if x in self.b1:
            self.p = min(float(c), self.p + max(1.0, len(self.b2) / len(self.b1)))
            v = self._evict_one(x)
            self.b1.remove(x)
            self.t2.append(x)
            return False, v
        if x in self.b2:
            self.p = max(0.0, self.p - max(1.0, len(self.b1) / len(self.b2)))
            v = self._evict_one(x)
            self.b2.remove(x)
            self.t2.append(x)
            return False, v
        v = None
        if len(self.t1) + len(self.b1) == c:
            if len(self.t1) < c:
                self.b1.pop(0)
                v = self._evict_one(x)
            else:
                v = self.t1.pop(0)
        else:
            tot = len(self.t1) + len(self.b1) + len(self.t2) + len(self.b2)
            if tot >= c:
                if tot == 2 * c:
                    self.b2.pop(0)
                v = self._evict_one(x)
        self.t1.append(x)
        return False, v

    def state(self) -> dict:
        return {"t1": list(self.t1), "t2": list(self.t2), "b1": list(self.b1),
                "b2": list(self.b2), "p": float(self.p)}


def seed_arc(arc: Arc, experts) -> None:
    """LayeredExpertCache.seed_resident (cache.py:197-204)."""
    for e in experts:
        if len(arc.t1) + len(arc.t2) >= arc.c:
            break
        if int(e) not in arc.resident():
            arc.t1.append(int(e))


# ---------------------------------------------------------------------------
# Group-wise affine quantization (quant.py:30-120), vectorised


def pack_codes(codes: np.ndarray, bits: int) -> np.ndarray:
    """Little-endian-in-byte packing: element i of a byte at bit i*bits (quant.py:30-39)."""
    per = 8 // bits
    c = np.asarray(codes, dtype=np.uint8).reshape(-1)
    pad = (-c.shape[0]) % per
    if pad:
        c = np.concatenate([c, np.zeros(pad, np.uint8)])
    c = c.reshape(-1, per).astype(np.uint16)
    shifts = (np.arange(per, dtype=np.uint16) * bits)
    return (c << shifts).sum(axis=1).astype(np.uint8)


def unpack_codes(packed: np.ndarray, bits: int, n: int) -> np.ndarray:
    """Inverse of pack_codes (quant.py:42-48)."""
    per = 8 // bits
    p = np.asarray(packed, dtype=np.uint8).reshape(-1, 1)
    shifts = (np.arange(per, dtype=np.uint8) * bits).reshape(1, -1)
    return ((p >> shifts) & ((1 << bits) - 1)).reshape(-1)[:n].astype(np.uint8)


def quantize(w: np.ndarray, bits: int, group: int = 64):
    """Min/max affine group quantization, round-half-even (quant.py:67-107).

    Returns (packed codes uint8, scales f64, zeros f64).  Vectorised over
    groups; a short tail group is handled separately so the arithmetic per
    element is exactly the reference's fp64 sequence.
    """
    flat = np.asarray(w, dtype=np.float64).reshape(-1)
    n = flat.shape[0]
    levels = (1 << bits) - 1
    n_groups = max(1, math.ceil(n / group))
    scales = np.zeros(n_groups)
    zeros = np.zeros(n_groups)
    codes = np.zeros(n, dtype=np.uint8)
    full = n // group

    def _do(x: np.ndarray):
        mn = x.min(axis=1)
        mx = x.max(axis=1)
        rng = mx - mn
        sc = np.where(rng == 0.0, 0.0, rng / levels)
        safe = np.where(sc == 0.0, 1.0, sc)
        q = np.rint((x - mn[:, None]) / safe[:, None])
        q = np.where((sc == 0.0)[:, None], 0.0, np.clip(q, 0, levels))
        return mn, sc, q.astype(np.uint8)

    if full:
        mn, sc, q = _do(flat[: full * group].reshape(full, group))
        zeros[:full], scales[:full] = mn, sc
        codes[: full * group] = q.reshape(-1)
    if n > full * group:
        mn, sc, q = _do(flat[full * group:].reshape(1, -1))
        zeros[full], scales[full] = mn[0], sc[0]
        codes[full * group:] = q.reshape(-1)
    return pack_codes(codes, bits), scales, zeros


def dequantize(packed, scales, zeros, bits: int, shape, group: int = 64) -> np.ndarray:
    """zero + code*scale in fp64 (quant.py:110-120)."""
    n = int(np.prod(shape))
    c = unpack_codes(packed, bits, n).astype(np.float64)
    gi = np.arange(n) // group
    return (np.asarray(zeros, np.float64)[gi] + c * np.asarray(scales, np.float64)[gi]).reshape(shape)


def expert_bytes(n_params: int, bits: int, group: int = 64) -> int:
    """Packed size ceil(n*b/8) + 8*ceil(n/group) (quant.py:239-246); bf16 = 2n."""
    if bits == 16:
        return 2 * n_params
    return math.ceil(n_params * bits / 8) + 8 * math.ceil(n_params / group)


# ---------------------------------------------------------------------------
# Popularity and bit assignment (quant.py:123-185, predict.py:179-195)


def popularity(lists) -> tuple[dict, list]:
    """counts[e] = #lists containing e; ordering by (-count, id)."""
    counts: dict[int, int] = {}
    for lst in lists:
        for e in set(int(x) for x in lst):
            counts[e] = counts.get(e, 0) + 1
    order = sorted(counts, key=lambda e: (-counts[e], e))
    return counts, order


def assign_bits_prefill(order: list, p_int2: float) -> dict:
    """floor(p*|active|) least popular -> 2 bits, rest 4 (quant.py:168-185)."""
    m = math.floor(p_int2 * len(order))
    low = set(order[len(order) - m:]) if m > 0 else set()
    return {e: (2 if e in low else 4) for e in order}


# ---------------------------------------------------------------------------
# Expert FFN (repo-defined; the reference has none)


def silu(x):
    return x / (1.0 + np.exp(-x))


def ffn_swiglu(x: np.ndarray, w1: np.ndarray, w3: np.ndarray, w2: np.ndarray) -> np.ndarray:
    """W2 (silu(W1 x) * (W3 x)) in fp64.  x [..., H]; w1,w3 [I, H]; w2 [H, I]."""
    x = np.asarray(x, np.float64)
    a = silu(x @ np.asarray(w1, np.float64).T) * (x @ np.asarray(w3, np.float64).T)
    return a @ np.asarray(w2, np.float64).T


# ---------------------------------------------------------------------------
# Timing-independent decode / prefill schedules


@dataclass
class StrategyKnobs:
    """The Strategy fields the schedule reads (pipeline.py:44-104)."""

    kind: str = "fate"            # fate | eap | lod
    policy_kind: str = "percentile"
    q: float = 0.75
    quant: bool = True            # quant_policy is not None
    p_int2: float = 0.25
    decode_bits: int = 4
    cache_bits: int = 4
    reorder_prefill: bool = True

    @property
    def prefetch_bits(self) -> int:
        return self.decode_bits if self.quant else 16

    @property
    def ondemand_bits(self) -> int:
        return 2 if self.quant else 16


def eap_list(counts_l: np.ndarray, chosen, k: int) -> list[int]:
    """eap_predict (predict.py:138-158): Laplace-smoothed, row-normalised
    co-activation scores summed over the chosen set in ascending id order,
    top-k by (-score, id); cold start (every relevant row empty) -> 0..k-1."""
    E = counts_l.shape[1]
    ch = sorted(int(a) for a in chosen)
    totals = {a: int(counts_l[a].sum()) for a in ch}
    if all(v == 0 for v in totals.values()):
        return list(range(k))
    score = np.zeros(E)
    for a in ch:
        score += (counts_l[a] + 1.0) / (totals[a] + E)
    return sorted(range(E), key=lambda e: (-score[e], e))[:k]


def decode_schedule(gate_in, chosen, mats, taus, caps, k: int, budget_n: int,
                    knobs: StrategyKnobs, cached_bits: int, arcs: list | None = None,
                    eap_counts: np.ndarray | None = None) -> dict:
    """Timing-independent fields of simulate_decoding (pipeline.py:343-517).

    gate_in [T, L, H] fp64, chosen [T][L] ids.  Per (token, layer) step:
    predicted list for layer+1 truncated to n (pipeline.py:390-393), the
    prefetch-issued set (skip resident, :397), cache-hit flags (:442),
    on-demand set (:450-459), source bits (:444, :453, :459), the ARC victims
    of update_after_layer (:483) and the recall contribution (:433-436).
    """
    T, L = len(chosen), len(chosen[0])
    arcs = arcs if arcs is not None else [Arc(c) for c in caps]
    issued: dict = {}
    pred_sets: dict = {}
    steps = []
    recall_sum, recall_n, dequant = 0.0, 0, 0
    cache_hits = 0
    use_pred = knobs.kind == "fate"
    use_eap = knobs.kind == "eap"
    E = int(np.asarray(mats).shape[1])
    # EapStats (predict.py:110-130); shared with a preceding prefill when chained
    counts = eap_counts if eap_counts is not None else np.zeros((max(L - 1, 1), E, E), dtype=np.int64)
    for t in range(T):
        for l in range(L):
            rec = {"token": t, "layer": l}
            if use_pred and l + 1 < L:
                w = gate_routing(mats[l + 1], taus[l + 1], gate_in[t][l])
                lst = predicted_list(w, knobs.policy_kind, knobs.q, k)[:budget_n]
                pred_sets[(t, l + 1)] = set(lst)
                iss = [e for e in lst if e not in arcs[l + 1].resident()]
                issued[(t, l + 1)] = iss
                rec["pred"] = lst
                rec["prefetch"] = iss
            ch = sorted(int(e) for e in chosen[t][l])
            rec["chosen"] = ch
            if use_eap:
                # observe (pipeline.py:310-315, eap_update predict.py:132-138), then
                # predict l+1 from l's chosen set at gate end (pipeline.py:421-428)
                if l > 0:
                    prev = sorted(int(e) for e in chosen[t][l - 1])
                    for a in prev:
                        counts[l - 1, a, ch] += 1
                if l + 1 < L:
                    lst = eap_list(counts[l], ch, k)[:budget_n]
                    pred_sets[(t, l + 1)] = set(lst)
                    iss = [e for e in lst if e not in arcs[l + 1].resident()]
                    issued[(t, l + 1)] = iss
                    rec["pred"] = lst
                    rec["prefetch"] = iss
            if (t, l) in pred_sets:
                recall_sum += len(pred_sets.pop((t, l)) & set(ch)) / len(ch)
                recall_n += 1
            res = arcs[l].resident()
            iss_here = set(issued.pop((t, l), []))
            hits, od, src = [], [], []
            for e in ch:
                if e in res:
                    hits.append(e)
                    src.append(cached_bits if cached_bits < 16 else 16)
                elif e in iss_here:
                    src.append(knobs.prefetch_bits)
                else:
                    od.append(e)
                    src.append(knobs.ondemand_bits)
            cache_hits += len(hits)
            dequant += sum(1 for b in src if b < 16)
            victims = []
            for e in ch:
                _, v = arcs[l].access(e)
                if v is not None:
                    victims.append(v)
            rec.update({"hits": hits, "ondemand": od, "src_bits": src, "victims": victims})
            steps.append(rec)
    return {"steps": steps, "recall": (recall_sum / recall_n) if recall_n else 0.0,
            "dequant_count": dequant, "cache_hits": cache_hits,
            "accesses": T * L * k, "arcs": [a.state() for a in arcs]}


def prefill_schedule(gate_in, chosen, mats, taus, caps, k: int, knobs: StrategyKnobs,
                     cached_bits: int, started: dict | None = None, arcs: list | None = None,
                     eap_counts: np.ndarray | None = None) -> dict:
    """Timing-independent fields of simulate_prefill (pipeline.py:536-778).

    ``started[layer]`` is the set of that layer's prefetches that had begun
    by the layer's block end (timing-dependent: pipeline.py:682 drops the
    rest, which are then fetched on demand at ondemand_bits, :701-719).  When
    ``None`` every issued prefetch counts as started.
    """
    T, L = len(chosen), len(chosen[0])
    arcs = arcs if arcs is not None else [Arc(c) for c in caps]
    issued: dict = {}
    profiles: dict = {}
    layers = []
    recall_sum, recall_n, dequant = 0.0, 0, 0
    if knobs.kind == "eap" and eap_counts is None:
        E = int(np.asarray(mats).shape[1])
        eap_counts = np.zeros((max(L - 1, 1), E, E), dtype=np.int64)
    for l in range(L):
        rec = {"layer": l}
        lists = None
        if knobs.kind == "eap":
            # EAP prefill (pipeline.py:652-665): every token's transition l-1 -> l
            # first (eap_update), then per-token EAP lists for l+1 (merged_topk_lists)
            if l > 0:
                for t in range(T):
                    nxt = sorted(int(x) for x in chosen[t][l])
                    for a in sorted(int(x) for x in chosen[t][l - 1]):
                        eap_counts[l - 1, a, nxt] += 1
            if l + 1 < L:
                lists = [eap_list(eap_counts[l], chosen[t][l], k) for t in range(T)]
        elif knobs.kind == "fate" and l + 1 < L:
            lists = []
            for t in range(T):
                w = gate_routing(mats[l + 1], taus[l + 1], gate_in[t][l])
                lists.append(top_k(w, k))
        if lists is not None:
            counts, order = popularity(lists)
            bits = assign_bits_prefill(order, knobs.p_int2) if knobs.quant else {e: 16 for e in order}
            if not knobs.reorder_prefill:
                seen, order_iss = set(), []
                for lst in lists:
                    for e in sorted(lst):
                        if e not in seen:
                            seen.add(e)
                            order_iss.append(e)
            else:
                order_iss = order
            res_next = arcs[l + 1].resident()
            iss = [(e, bits[e]) for e in order_iss if e not in res_next]
            issued[l + 1] = iss
            profiles[l + 1] = (counts, order)
            rec.update({"pred_order": order, "pred_counts": [counts[e] for e in order],
                        "prefetch": iss})
        counts = {}
        for t in range(T):
            for e in chosen[t][l]:
                counts[int(e)] = counts.get(int(e), 0) + 1
        actives = sorted(counts)
        rec["actives"] = actives
        rec["counts"] = [counts[e] for e in actives]
        if l in profiles:
            pc, po = profiles.pop(l)
            recall_sum += len(set(po) & set(actives)) / len(actives)
            recall_n += 1
        res = arcs[l].resident()
        iss_here = dict(issued.pop(l, []))
        st = iss_here.keys() if started is None else set(started.get(l, ()))
        resident, planned, unplanned = [], [], []
        src = {}
        for e in actives:
            if e in res:
                resident.append(e)
                src[e] = cached_bits if cached_bits < 16 else 16
            elif e in iss_here and e in st:
                planned.append(e)
                src[e] = iss_here[e]
            else:
                unplanned.append(e)
        od_bits = knobs.ondemand_bits if knobs.kind == "fate" else 16
        by_pop = lambda e: (-counts[e], e)
        first_seen, seen = [], set()
        for t in range(T):
            for e in sorted(int(x) for x in chosen[t][l]):
                if e not in seen:
                    seen.add(e)
                    first_seen.append(e)
        unp = set(unplanned)
        od_order = (sorted(unplanned, key=by_pop) if knobs.reorder_prefill
                    else [e for e in first_seen if e in unp])
        for e in od_order:
            src[e] = od_bits
        dequant += sum(1 for e in actives if src[e] < 16)
        rec.update({"resident": resident, "planned": planned, "ondemand": od_order,
                    "src_bits": [src[e] for e in actives],
                    "compute_order": (sorted(resident, key=by_pop) + sorted(planned, key=by_pop) + od_order)
                    if knobs.reorder_prefill else first_seen})
        victims = []
        for e in actives:
            _, v = arcs[l].access(e)
            if v is not None:
                victims.append(v)
        rec["victims"] = victims
        layers.append(rec)
    return {"layers": layers, "recall": (recall_sum / recall_n) if recall_n else 0.0,
            "dequant_count": dequant, "arcs": [a.state() for a in arcs]}


# ---------------------------------------------------------------------------
# Packed expert buffers (the repo's device layout; see csrc/fate_internal.cuh)


def buffer_layout(H: int, I: int, bits: int) -> dict:
    n = H * I
    if bits == 16:
        return {"c1": 0, "c3": 2 * n, "c2": 4 * n, "payload": 6 * n}
    cb, sb = n * bits // 8, n // 64 * 8
    return {"c1": 0, "c3": cb, "c2": 2 * cb, "s1": 3 * cb, "s3": 3 * cb + sb, "s2": 3 * cb + 2 * sb,
            "payload": 3 * cb + 3 * sb}


def unpack_buffer(buf: np.ndarray, H: int, I: int, bits: int) -> dict:
    """Split a packed expert buffer into (codes, fp32 sz) per projection and
    its fp64 dequantized matrices (zero + code*scale with the stored fp32 scale/zero)."""
    buf = np.asarray(buf, dtype=np.uint8)
    hdr = buf[:256].view(np.int32)
    p = buf[256:]
    lay = buffer_layout(H, I, bits)
    n = H * I
    out = {"header": {"bits": int(hdr[1]), "layer": int(hdr[2]), "expert": int(hdr[3]), "H": int(hdr[4]),
                      "I": int(hdr[5])}}
    shapes = {"1": (I, H), "3": (I, H), "2": (H, I)}
    for j in ("1", "3", "2"):
        c0 = lay["c" + j]
        if bits == 16:
            raw = p[c0:c0 + 2 * n].view(np.uint16).astype(np.uint32) << 16
            w = raw.view(np.float32).astype(np.float64)
            out["w" + j] = w.reshape(shapes[j]) if j != "2" else w2_from_slabs(w, H, I, W2_SLAB_BF16)
            continue
        codes = p[c0:c0 + n * bits // 8]
        sz = p[lay["s" + j]:lay["s" + j] + n // 64 * 8].view(np.float32).reshape(-1, 2)
        if j == "2":
            # slab-major W2: group order (slab, row) -> the reference's row-major (row, slab)
            g = (n * bits // 8) // (n // 64)
            codes = codes.reshape(I // 64, H, g).transpose(1, 0, 2).reshape(-1)
            sz = sz.reshape(I // 64, H, 2).transpose(1, 0, 2).reshape(-1, 2)
        out["codes" + j] = np.ascontiguousarray(codes)
        out["sz" + j] = np.ascontiguousarray(sz)
        out["w" + j] = dequantize(out["codes" + j], out["sz" + j][:, 0].astype(np.float64),
                                  out["sz" + j][:, 1].astype(np.float64), bits, shapes[j])
    return out


W2_SLAB_BF16 = 8  # bf16 W2 slab width of the packed format (quantized: 64 = one group)


def pack_buffer(w1: np.ndarray, w3: np.ndarray, w2: np.ndarray, bits: int, layer: int = 0,
                expert: int = 0) -> np.ndarray:
    """The packed expert buffer in numpy (test / CPU-baseline use): 256-byte header,
    W1 / W3 row-major, W2 slab-major, quantized with the reference's quantize."""
    I, H = w1.shape
    lay = buffer_layout(H, I, bits)
    buf = np.zeros(256 + lay["payload"], np.uint8)
    buf[:24].view(np.int32)[:] = [np.int32(np.uint32(0xFA7EB200).view(np.int32)), bits, layer, expert, H, I]
    p = buf[256:]
    C = W2_SLAB_BF16 if bits == 16 else 64
    w2s = np.asarray(w2, np.float32).reshape(H, I // C, C).transpose(1, 0, 2).reshape(-1)
    for j, w in (("1", w1), ("3", w3), ("2", w2s)):
        w = np.asarray(w, np.float32).reshape(-1)
        c0 = lay["c" + j]
        if bits == 16:
            u = w.view(np.uint32)
            # round-to-nearest-even fp32 -> bf16 (as __float2bfloat16_rn)
            r = ((u + 0x7FFF + ((u >> 16) & 1)) >> 16).astype(np.uint16)
            p[c0:c0 + 2 * w.size] = r.view(np.uint8)
            continue
        codes, sc, zr = quantize(w.astype(np.float64), bits)
        p[c0:c0 + codes.size] = codes
        sz = np.stack([sc.astype(np.float32), zr.astype(np.float32)], axis=1).reshape(-1)
        p[lay["s" + j]:lay["s" + j] + 4 * sz.size] = sz.view(np.uint8)
    return buf


def w2_from_slabs(flat: np.ndarray, H: int, I: int, C: int) -> np.ndarray:
    """Slab-major W2 (slab s = columns [s*C, s*C+C) of all H rows) back to [H, I]."""
    return np.ascontiguousarray(flat.reshape(I // C, H, C).transpose(1, 0, 2).reshape(H, I))


# ---------------------------------------------------------------------------
# C restatement of the expert FFN (oracle/ffn_cpu.c), for CPU timing only


def cpu_lib():
    import ctypes
    import os
    import subprocess

    here = os.path.dirname(os.path.abspath(__file__))
    so = os.path.join(here, "libfate_oracle.so")
    if not os.path.exists(so):
        subprocess.run(["make", "-s", "-C", here], check=True)
    lib = ctypes.CDLL(so)
    P = ctypes.POINTER
    lib.fate_cpu_ffn.argtypes = [P(ctypes.c_float), ctypes.c_int, ctypes.c_int, P(ctypes.c_void_p), P(ctypes.c_int),
                                 P(ctypes.c_int), P(ctypes.c_float), P(ctypes.c_float), P(ctypes.c_float)]
    lib.fate_cpu_ffn.restype = None
    lib.fate_cpu_threads.argtypes = [ctypes.c_int]
    lib.fate_cpu_threads.restype = ctypes.c_int
    return lib


def cpu_scratch_floats(H: int, I: list) -> int:
    """Scratch of fate_cpu_ffn: activations + their group sums + x's group sums."""
    tot = int(sum(I))
    return tot + tot // 64 + H // 64


def cpu_ffn(lib, x: np.ndarray, bufs: list, I: list, bits: list, w: list, scratch: np.ndarray) -> np.ndarray:
    import ctypes

    n = len(bufs)
    H = x.shape[0]
    need = cpu_scratch_floats(H, I)
    if scratch.dtype != np.float32 or scratch.size < need:
        raise ValueError(f"cpu_ffn scratch needs {need} float32, got {scratch.size} {scratch.dtype}")
    y = np.empty(H, np.float32)
    arr = (ctypes.c_void_p * n)(*[b.ctypes.data for b in bufs])
    f = lambda a: a.ctypes.data_as(ctypes.POINTER(ctypes.c_float))  # noqa: E731
    xc = np.ascontiguousarray(x, np.float32)
    lib.fate_cpu_ffn(f(xc), H, n, arr, (ctypes.c_int * n)(*I), (ctypes.c_int * n)(*bits), (ctypes.c_float * n)(*w),
                     f(y), f(scratch))
    return y


# ---------------------------------------------------------------------------
# CPU restatement of the whole executed decode path (bench cpu_baseline /
# --impl reference legs): schedule + FFN, timed together


def port_decode(gate_in, mats, taus, caps, k: int, n: int, knobs: StrategyKnobs, get_buf, shared_buf, H: int,
                I: int, Is: int, lib, tokens: int, ffn: bool = True) -> list:
    """Per (token, layer) step: the fp64 gate and top-k (gatesim.py:113-123,
    core.py:159-163), the cross-layer prediction entries[:n] issued for layer+1
    minus residents (pipeline.py:390-404, predict.py:92-107), the hit /
    prefetched / on-demand split (pipeline.py:441-459), the expert FFN of the
    chosen experts in the width their copy has (a cache slot keeps the width
    that landed; prefetch = decode_bits, miss = ondemand_bits) plus the shared
    expert with weight 1 (C threads, oracle/ffn_cpu.c), then update_after_layer
    (cache.py:212-215).  Returns the per-step decision log.

    get_buf(layer, expert, bits) -> packed buffer; shared_buf(layer) -> packed
    bf16 shared expert (or None when Is == 0)."""
    L = len(caps)
    arcs = [Arc(c) for c in caps]
    fmt = [dict() for _ in range(L)]
    issued: dict = {}
    logs = []
    sizes = [I] * k + ([Is] if Is else [])
    scratch = np.empty(cpu_scratch_floats(H, sizes), np.float32)
    sH = np.sqrt(H)
    for t in range(tokens):
        for l in range(L):
            h = gate_in[t, l]
            w = gate_routing(mats[l], taus[l], h)
            ch = sorted(top_k(w, k))
            rec = {"chosen": ch}
            if n > 0 and knobs.kind == "fate" and l + 1 < L:
                wn = gate_routing(mats[l + 1], taus[l + 1], h)
                lst = predicted_list(wn, knobs.policy_kind, knobs.q, k)[:n]
                res_n = arcs[l + 1].resident()
                issued[(t, l + 1)] = {e for e in lst if e not in res_n}
                rec["pred"] = lst
            res = arcs[l].resident()
            iss = issued.pop((t, l), set())
            bits, hits, od = [], [], []
            for e in ch:
                if e in res:
                    bits.append(fmt[l][e])
                    hits.append(e)
                elif e in iss:
                    bits.append(knobs.prefetch_bits)
                else:
                    bits.append(knobs.ondemand_bits)
                    od.append(e)
            if ffn:
                x = (sH * h).astype(np.float32)
                bufs = [get_buf(l, e, b) for e, b in zip(ch, bits)]
                wts = [float(w[e]) for e in ch]
                if Is:
                    bufs.append(shared_buf(l))
                    wts.append(1.0)
                cpu_ffn(lib, x, bufs, sizes, bits + ([16] if Is else []), wts, scratch)
            victims = []
            for e, b in zip(ch, bits):
                hit, v = arcs[l].access(e)
                if v is not None:
                    victims.append(v)
                    fmt[l].pop(v, None)
                if not hit and arcs[l].c >= 1:
                    fmt[l][e] = b
            rec.update({"hits": hits, "ondemand": od, "victims": victims, "fmt_bits": bits})
            logs.append(rec)
    return logs
