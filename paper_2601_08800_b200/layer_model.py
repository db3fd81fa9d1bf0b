"""Layout selection from the fused layer's own measured costs (config E).

The reference selector (:mod:`.analyzer`, cm:111-153) prices MoE tensor
parallelism as an all-reduce of ``b*s*h`` and expert parallelism as an
all-to-all of the mean per-rank volume.  The fused B200 layer does neither:
on one NVSwitch box it moves deduplicated (token, host) rows one hop, pre-
reduces them per pair, and its TP sharding shrinks the grouped GEMMs' K and
N -- which costs tensor-core efficiency the reference model cannot see.
Measured at config B, 4 GPUs: EP4 0.319 ms vs TP2xEP2 0.341 ms on a uniform
router, the reverse under Zipf skew (profiles/r01_configE_n4.jsonl), while
the reference model ranks TP2xEP2 first at every skew.

This module predicts the layer time of every ``(n, m)`` layout from the
routing itself, with the same algorithmic bytes/flops ``bench.py`` reports
per phase and per-phase efficiencies calibrated on measured bench lines:

* segments separated by the layer's device barriers -- (route, layout,
  dispatch), (expand, GEMM1, GEMM2, pair pre-reduction), (combine) -- each
  costs its slowest rank (the barrier waits for it);
* a phase costs ``bytes / (eff * peak)`` (HBM or NVLink) or
  ``flops / (eff * bf16 peak)``; GEMM efficiency depends on the TP shard
  ``I/m`` (it sets GEMM1's N and GEMM2's K);
* route + layout and each barrier are fixed latencies.

:func:`select_layout` ranks the candidate layouts; tests pin it to the
measured config-E ordering.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

__all__ = ["LayerCalibration", "routing_stats", "predict_layer", "select_layout"]


@dataclass(frozen=True)
class LayerCalibration:
    """Peaks and per-phase efficiencies (achieved / peak).  Only their
    product -- the phase's measured throughput -- enters a prediction.  The
    defaults are the round-1 B200 measurements (profiles/r01_n{1,2,4}_bench.json
    ``rooflines``) expressed against the round-2 denominators bench.py
    divides by: MEASURED_PEAKS.json's HBM copy (6446.3 GB/s) and burst bf16
    matmul (1668.3 TF/s), and the same-run NVLink probe at 4 GPUs (651 GB/s,
    profiles/r02_n4_tp2_bench.json); ``from_bench`` re-derives them from
    newer lines."""

    hbm_gbs: float = 6446.3
    nvlink_gbs: float = 651.0
    bf16_tflops: float = 1668.3
    # GEMM efficiency vs the TP shard I/m: {I/m: (gemm1, gemm2)}
    gemm_eff: dict = field(default_factory=lambda: {384: (0.5612, 0.5025),
                                                    768: (0.6952, 0.6114)})
    eff: dict = field(default_factory=lambda: {
        "dispatch_nvlink": 0.6978, "dispatch_hbm": 0.8724, "expand": 0.7101,
        "pair_reduce": 0.6087, "pair_push_nvlink": 0.5796, "combine_nvlink": 0.4731,
        "combine_hbm": 0.6391})
    route_layout_us: float = 32.0
    barrier_us: float = 6.0   # graph replay: ~5 us intrinsic (barrier_bench) + skew

    # bench.py phase (and the bound it was judged against) -> efficiency key
    _PHASE_EFF = {("dispatch", "nvlink"): "dispatch_nvlink", ("dispatch", "hbm"): "dispatch_hbm",
                  ("expand", "hbm"): "expand", ("pair_reduce", "hbm"): "pair_reduce",
                  ("pair_reduce", "nvlink"): "pair_push_nvlink",
                  ("combine", "nvlink"): "combine_nvlink", ("combine", "hbm"): "combine_hbm"}

    @classmethod
    def from_bench(cls, lines, base: "LayerCalibration | None" = None) -> "LayerCalibration":
        """Recalibrate from measured ``bench.py`` JSON lines (a dict or a
        list; later lines win): every phase's achieved / peak becomes its
        efficiency, the GEMM fractions are filed under the line's TP shard
        ``I/m``, route + layout is the measured latency, and the peaks are
        the ones the line was judged against.  The device barriers keep
        ``base``'s figure (phase-mode barriers carry event-node overhead)."""
        c = base or cls()
        if isinstance(lines, dict):
            lines = [lines]
        eff, gemm_eff = dict(c.eff), dict(c.gemm_eff)
        hbm, nvl, tf, rl = c.hbm_gbs, c.nvlink_gbs, c.bf16_tflops, c.route_layout_us
        for line in lines:
            roof = line.get("rooflines", {})
            cfg = line.get("config", {})
            for ph, r in roof.items():
                key = cls._PHASE_EFF.get((ph, r["bound"]))
                if key:
                    eff[key] = float(r["frac"])
                if r["bound"] == "hbm":
                    hbm = float(r["peak"])
                elif r["bound"] == "nvlink":
                    nvl = float(r["peak"])
                elif r["bound"] == "tensor":
                    tf = float(r["peak"])
            if "gemm1_swiglu" in roof and "gemm2" in roof and cfg.get("moe_intermediate"):
                shard = int(cfg["moe_intermediate"]) // int(cfg.get("tp_m", 1))
                gemm_eff[shard] = (float(roof["gemm1_swiglu"]["frac"]), float(roof["gemm2"]["frac"]))
            ph_us = line.get("phases_us", {})
            if "route" in ph_us and "layout" in ph_us:
                rl = float(ph_us["route"]) + float(ph_us["layout"])
        return cls(hbm_gbs=hbm, nvlink_gbs=nvl, bf16_tflops=tf, gemm_eff=gemm_eff, eff=eff,
                   route_layout_us=rl, barrier_us=c.barrier_us)

    def gemm(self, shard: int):
        ks = sorted(self.gemm_eff)
        if shard <= ks[0]:
            return self.gemm_eff[ks[0]]
        if shard >= ks[-1]:
            return self.gemm_eff[ks[-1]]
        for lo, hi in zip(ks, ks[1:]):
            if lo <= shard <= hi:
                f = (shard - lo) / (hi - lo)
                a, b = self.gemm_eff[lo], self.gemm_eff[hi]
                return tuple(x + f * (y - x) for x, y in zip(a, b))
        return self.gemm_eff[ks[-1]]


def routing_stats(ids, n: int, num_experts: int):
    """Per-group slot and (token, host) pair counts of a routing.

    ``ids``: [T_global, k] expert ids, tokens split into ``n`` contiguous
    groups (sim:575-580), experts placed ``e*n//E`` (sim:210-212).
    Returns ``S[j][d]`` (slots of group j hosted on d) and ``U[j][d]``
    (tokens of group j with at least one expert on d)."""
    ids = np.asarray(ids, dtype=np.int64)
    Tg = ids.shape[0]
    if Tg % n:
        raise ValueError("tokens do not split evenly over the groups")
    T = Tg // n
    host = (ids * n) // num_experts
    grp = np.repeat(np.arange(n), T)
    S = np.zeros((n, n), dtype=np.int64)
    U = np.zeros((n, n), dtype=np.int64)
    for d in range(n):
        on_d = host == d
        S[:, d] = np.bincount(grp, weights=on_d.sum(axis=1), minlength=n).astype(np.int64)
        U[:, d] = np.bincount(grp, weights=on_d.any(axis=1), minlength=n).astype(np.int64)
    return S, U


def predict_layer(ids, n: int, m: int, num_experts: int, hidden: int, inter: int,
                  calib: LayerCalibration | None = None, elt: int = 2) -> dict:
    """Predicted seconds per layer forward of layout ``(n, m)`` (token wire
    for n*m > 1, slot wire on one GPU), with the per-segment breakdown."""
    c = calib or LayerCalibration()
    S, U = routing_stats(ids, n, num_experts)
    Tg = np.asarray(ids).shape[0]
    T = Tg // n
    hb = hidden * elt
    W = n * m
    shard = inter // m
    e1, e2 = c.gemm(shard)
    hbm, nvl, tf = c.hbm_gbs * 1e9, c.nvlink_gbs * 1e9, c.bf16_tflops * 1e12
    seg = {"pre": 0.0, "expert": 0.0, "combine": 0.0}
    for d in range(n):
        S_d = int(S[:, d].sum())
        local = int(S[d, d])
        remote_in = S_d - local
        pairs = int(U[:, d].sum())
        remote_pairs = pairs - int(U[d, d])
        g1 = 2.0 * S_d * hidden * 2 * shard / (e1 * tf)
        g2 = 2.0 * S_d * shard * hidden / (e2 * tf)
        if W == 1:
            disp = (T + S_d) * hb / (c.eff["dispatch_hbm"] * hbm)
            comb = (S_d + T) * hb / (c.eff["combine_hbm"] * hbm)
            pre, expert = disp, g1 + g2
        else:
            disp = max(remote_pairs * hb / (c.eff["dispatch_nvlink"] * nvl),
                       (T + local) * hb / (c.eff["dispatch_hbm"] * hbm))
            exp_ = (remote_pairs + remote_in) * hb / (c.eff["expand"] * hbm)
            # pre-reduction: reads the host's slot partials, pushes each pair
            # row's shards into the owners (NVLink except the own shard)
            own = int(U[d, d])
            push = (pairs - own) * hb + own * hb * (m - 1) // m
            pr = max(S_d * hb / (c.eff["pair_reduce"] * hbm),
                     push / (c.eff["pair_push_nvlink"] * nvl))
            # owner: local ZIN planes, y shard pushed to the TP peers
            zin = int(U[d].sum()) * hb
            ypush = T * hidden * (m - 1) // m * elt
            comb = max(zin / (c.eff["combine_hbm"] * hbm),
                       ypush / (c.eff["combine_nvlink"] * nvl))
            pre, expert = disp, exp_ + g1 + g2 + pr
        seg["pre"] = max(seg["pre"], pre)
        seg["expert"] = max(seg["expert"], expert)
        seg["combine"] = max(seg["combine"], comb)
    fixed = c.route_layout_us * 1e-6 + (4 * c.barrier_us * 1e-6 if W > 1 else 0.0)
    total = fixed + seg["pre"] + seg["expert"] + seg["combine"]
    return {"layout": f"TP{m}xEP{n}", "n": n, "m": m, "seconds": total, "fixed_s": fixed,
            "segments_s": seg, "host_slots_max": int(S.sum(axis=0).max())}


def select_layout(ids, world: int, num_experts: int, hidden: int, inter: int,
                  calib: LayerCalibration | None = None, tp_choices=(1, 2, 4, 8)):
    """Rank the ``(n, m)`` layouts of ``world`` GPUs the expert shapes allow
    (``(I/m) % 128 == 0``, ``n`` divides the tokens) by predicted time."""
    Tg = np.asarray(ids).shape[0]
    out = []
    for m in tp_choices:
        if world % m or (inter // m) % 128 or inter % m:
            continue
        n = world // m
        if Tg % n or num_experts < n:
            continue
        out.append(predict_layer(ids, n, m, num_experts, hidden, inter, calib))
    out.sort(key=lambda r: r["seconds"])
    return out
