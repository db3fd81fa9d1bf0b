"""Freeze the reference selector's outputs (run in the build container).

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_selector_golden.py

Imports the unmodified reference ``moeplan`` and records, for a grid of
model / cluster / workload / calibration cases: enumeration order, memory
checks, indicator vectors, rankings for every objective, compare reports,
the Eq. 12/13 comparison and calibration fits.  Also copies the
reference's own frozen ``pkg/tests/golden/report_2x2.json`` (written by the
reference under Python 3.10) as ``ref_report_2x2.json``.
"""
from __future__ import annotations

import gzip
import json
import shutil
from dataclasses import asdict
from pathlib import Path

from moeplan.analyzer import (ProfilingObservation, calibrate, compare_report,
                              select_strategy)
from moeplan.config import (CalibrationCoefficients, ClusterConfig,
                            ModelHyperparams, WorkloadSpec)
from moeplan.costmodel import (indicators, lambda_ep_baseline, lambda_mix)
from moeplan.strategy import (check_memory, classify_dp_ep, enumerate_strategies,
                              format_strategy, parse_strategy)

HERE = Path(__file__).resolve().parent

MODELS = {
    "small": dict(hidden_dim=64, num_layers=4, top_k=2, num_routed_experts=8,
                  num_shared_experts=1, psi_attn=1e6, psi_moe=8e6, psi_active=2e6),
    "mid": dict(hidden_dim=1024, num_layers=8, top_k=2, num_routed_experts=32,
                num_shared_experts=1, psi_attn=1e8, psi_moe=8e8, psi_active=2e8),
    "qwen3": dict(hidden_dim=2048, num_layers=48, top_k=8, num_routed_experts=128,
                  num_shared_experts=0, psi_attn=1.5e9, psi_moe=2.9e10, psi_active=3.3e9),
    "dsr1": dict(hidden_dim=7168, num_layers=61, top_k=8, num_routed_experts=256,
                 num_shared_experts=1, psi_attn=1.1e10, psi_moe=6.6e11, psi_active=3.7e10,
                 bytes_per_element=1),
}
CLUSTERS = {
    "c2x2": (2, 2, 1e-6, 100e9, 2e-6, 10e9, 64e9, 1e12),
    "c4x8": (4, 8, 1e-6, 100e9, 5e-6, 10e9, 64e9, 1e13),
    "b200x8": (2, 4, 3e-6, 770e9, 3e-6, 770e9, 180e9, 2.25e15),
    "h20": (2, 8, 2e-6, 450e9, 8e-6, 50e9, 96e9, 1.5e14),
}
WORKLOADS = {
    "w_small": (8, 128, 128, 64, 10.0),
    "w_serve": (16, 256, 256, 64, 5.0),
    "w_prefill": (16, 4096, 4096, 256, 2.0),
}
CALIBS = {"default": {}, "c13": {"compute_coeff": 1e-13},
          "nonlit": {"compute_coeff": 1e-14, "ar_literal": False},
          "taulit": {"compute_coeff": 1e-16, "tau_literal": True}}


def est_dict(e):
    d = asdict(e)
    d["ttft"], d["w_q"] = repr(e.ttft), repr(e.w_q)  # inf-safe
    return d


def main():
    cases = []
    for mk, mv in MODELS.items():
        for ck, cv in CLUSTERS.items():
            for wk, wv in WORKLOADS.items():
                for calk, calv in CALIBS.items():
                    if (mk, ck) in (("small", "c4x8"), ("dsr1", "c2x2")) and calk != "c13":
                        continue
                    model = ModelHyperparams(**mv)
                    cluster = ClusterConfig(*cv)
                    wl = WorkloadSpec(*wv)
                    calib = CalibrationCoefficients(**calv)
                    strats = enumerate_strategies(cluster, model)
                    per = []
                    for s in strats:
                        mem = check_memory(s, model, cluster, wl)
                        try:
                            case = asdict(classify_dp_ep(s))
                        except Exception as exc:  # noqa: BLE001
                            case = {"error": type(exc).__name__}
                        row = {"strategy": format_strategy(s), "mem": [mem.feasible, mem.required_bytes],
                               "dp_ep": case}
                        try:
                            e = indicators(s, model, wl, cluster, calib)
                            row["est"] = {k: (repr(v) if isinstance(v, float) else v)
                                          for k, v in asdict(e).items() if k != "breakdown"}
                        except Exception as exc:  # noqa: BLE001
                            row["est_error"] = type(exc).__name__
                        per.append(row)
                    rankings = {}
                    for obj in ("ttft", "itl", "throughput", "pareto"):
                        try:
                            r = select_strategy(model, cluster, wl, calib, objective=obj)
                            rankings[obj] = [[format_strategy(e.strategy), e.on_front] for e in r.entries]
                            if obj == "ttft":
                                rep = compare_report(r, 5)
                                rankings["report"] = json.loads(json.dumps(rep, sort_keys=True))
                        except Exception as exc:  # noqa: BLE001
                            rankings[obj] = {"error": type(exc).__name__, "msg": str(exc)}
                    cases.append({"model": mv, "cluster": list(cv), "workload": list(wv),
                                  "calib": calv, "strategies": per, "rankings": rankings,
                                  "lambda": [repr(lambda_ep_baseline(model, wl, cluster, calib)),
                                             repr(lambda_mix(model, wl, cluster, calib))]})
    # calibration fits
    fits = []
    for seed, (ia, ib, ea, eb, c) in enumerate([(1e-6, 200e9, 8e-6, 20e9, 3e-13),
                                                (3e-6, 770e9, 3.5e-6, 700e9, 1e-15),
                                                (0.0, 50e9, 1e-5, 5e9, 2e-14)]):
        obs = []
        for scope, (a, b) in (("intra", (ia, ib)), ("inter", (ea, eb))):
            for size in (1e4, 1e5, 1e6, 1e7, 3e7):
                for d in (2, 4, 8):
                    j = 1.0 + 0.01 * ((size / 1e4 + d + seed) % 3 - 1)
                    obs.append(["RS", size, d, scope, j * (a + (size / d) / b)])
                    obs.append(["A2A", size, d, scope, j * (d - 1) * (a + (size / d) / b)])
                    obs.append(["AR", size, d, scope, j * 2 * (a + (size / d / d) / b)])
                obs.append(["P2P", size, 1, scope, a + size / b])
        obs += [["MoE_compute", ops, 1, "intra", c * ops * (1.0 + 0.001 * i)]
                for i, ops in enumerate((1e7, 1e8, 1e9, 5e9))]
        cal = calibrate([ProfilingObservation(*o) for o in obs])
        fits.append({"obs": obs, "calib": {k: (repr(v) if isinstance(v, float) else v)
                                           for k, v in asdict(cal).items()}})
    grammar = {}
    for text in ["TP=4 + DP=8, TP=4 + EP=8", "TP=8 [PP=4]", "DP=2 + TP=2, EP=2 + TP=2",
                 "TP=1", "TP=2 + DP=2, TP=2 + EP=2 [PP=2]", " TP = 8 ,  EP = 8 ",
                 "EP=4, TP=4", "TP=3", "TP=2 + DP=2", "TP=2, DP=2", "", "TP=2 + TP=2, EP=4",
                 "TP=2 + DP=2 + EP=2, TP=8", "TP=4, TP=2"]:
        try:
            s = parse_strategy(text)
            grammar[text] = {"ok": format_strategy(s),
                             "deg": [s.attn_tp, s.attn_dp, s.moe_tp, s.moe_ep, s.d_pp]}
        except Exception as exc:  # noqa: BLE001
            grammar[text] = {"error": type(exc).__name__, "msg": str(exc)}
    seen = set()  # keep one full compare report per (model, cluster, workload)
    for c in cases:
        key = (json.dumps(c["model"], sort_keys=True), tuple(c["cluster"]), tuple(c["workload"]))
        if key in seen:
            c["rankings"].pop("report", None)
        seen.add(key)
    with gzip.open(HERE / "ref_selector.json.gz", "wt") as f:
        json.dump({"cases": cases, "fits": fits, "grammar": grammar}, f, sort_keys=True)
    shutil.copy("/root/reference/pkg/tests/golden/report_2x2.json", HERE / "ref_report_2x2.json")
    print(f"{len(cases)} selector cases written")


if __name__ == "__main__":
    main()
