"""Strategy selector pinned to the reference (CPU only).

Fixtures: ``tests/golden/ref_selector.json.gz`` (reference outputs over a
model x cluster x workload x calibration grid, make_selector_golden.py) and
the reference's own frozen ``report_2x2.json``.  The acceptance criteria
C4-C8 of the reference suite (pkg/tests/test_acceptance.py:128-296) are
restated against this implementation.
"""
import gzip
import json
import math
import random

import pytest

from conftest import GOLDEN
from paper_2601_08800_b200 import analyzer as an
from paper_2601_08800_b200.analyzer import (ProfilingObservation, calibrate,
                                            compare_report, save_report, select_strategy)
from paper_2601_08800_b200.config import (CalibrationCoefficients, ClusterConfig,
                                          ModelHyperparams, WorkloadSpec)
from paper_2601_08800_b200.costmodel import (LinkClass, a2a_cost, ar_cost, indicators,
                                             lambda_ep_baseline, lambda_ep_terms, lambda_mix,
                                             lambda_mix_terms, queuing_delay, rs_cost)
from paper_2601_08800_b200.errors import GrammarError, SaturationError, StrategyError
from paper_2601_08800_b200.strategy import (check_memory, classify_dp_ep,
                                            enumerate_strategies, format_strategy,
                                            parse_strategy)

with gzip.open(GOLDEN / "ref_selector.json.gz", "rt") as _f:
    REF = json.load(_f)


def _close(a, b):
    a, b = float(a), float(b)
    if math.isinf(a) or math.isinf(b):
        return a == b
    # the reference here runs Python 3.12 (compensated builtin sum); ours sums
    # left to right like the 3.10 run that wrote its goldens -> ULP-level drift
    return a == b or abs(a - b) <= 1e-12 * max(abs(a), abs(b))


def _objs(case):
    return (ModelHyperparams(**case["model"]), ClusterConfig(*case["cluster"]),
            WorkloadSpec(*case["workload"]), CalibrationCoefficients(**case["calib"]))


@pytest.mark.parametrize("idx", range(len(REF["cases"])))
def test_strategies_indicators_and_rankings_match_reference(idx):
    case = REF["cases"][idx]
    model, cluster, wl, calib = _objs(case)
    strats = enumerate_strategies(cluster, model)
    assert [format_strategy(s) for s in strats] == [r["strategy"] for r in case["strategies"]]
    for s, row in zip(strats, case["strategies"]):
        mem = check_memory(s, model, cluster, wl)
        assert [mem.feasible, mem.required_bytes] == row["mem"]
        try:
            dp = classify_dp_ep(s)
            assert {"case": dp.case, "num_parallel_groups": dp.num_parallel_groups,
                    "group_size": dp.group_size,
                    "redundancy_factor": dp.redundancy_factor} == row["dp_ep"]
        except StrategyError:
            assert row["dp_ep"] == {"error": "StrategyError"}
        if "est" in row:
            est = indicators(s, model, wl, cluster, calib)
            for k, v in row["est"].items():
                mine = getattr(est, k)
                if isinstance(v, str):
                    assert _close(mine, float(v)), (k, mine, v)
                else:
                    assert mine == v, (k, mine, v)
        else:
            with pytest.raises(Exception):
                indicators(s, model, wl, cluster, calib)
    for obj in ("ttft", "itl", "throughput", "pareto"):
        want = case["rankings"][obj]
        if isinstance(want, dict):
            with pytest.raises(Exception) as ei:
                select_strategy(model, cluster, wl, calib, objective=obj)
            assert type(ei.value).__name__ == want["error"]
            continue
        got = select_strategy(model, cluster, wl, calib, objective=obj)
        assert [[format_strategy(e.strategy), e.on_front] for e in got.entries] == want
    ep, mix = case["lambda"]
    assert _close(lambda_ep_baseline(model, wl, cluster, calib), float(ep))
    assert _close(lambda_mix(model, wl, cluster, calib), float(mix))
    if "report" in case["rankings"]:
        rep = json.loads(json.dumps(compare_report(
            select_strategy(model, cluster, wl, calib), 5), sort_keys=True))
        want = case["rankings"]["report"]
        assert _json_close(rep, want)


def _json_close(a, b):
    if isinstance(a, dict):
        return a.keys() == b.keys() and all(_json_close(a[k], b[k]) for k in a)
    if isinstance(a, list):
        return len(a) == len(b) and all(_json_close(x, y) for x, y in zip(a, b))
    if isinstance(a, float) or isinstance(b, float):
        return _close(a, b)
    return a == b


def test_report_2x2_byte_exact(tmp_path):
    """The reference's frozen report (pkg/tests/golden/report_2x2.json, written
    under Python 3.10) is reproduced byte for byte: term sums accumulate left
    to right like 3.10's sum()."""
    model = ModelHyperparams(hidden_dim=64, num_layers=4, top_k=2, num_routed_experts=8,
                             num_shared_experts=1, psi_attn=1e6, psi_moe=8e6, psi_active=2e6)
    wl = WorkloadSpec(batch_size=8, seq_len=128, input_len=128, output_len=64, arrival_rate=10.0)
    cluster = ClusterConfig(2, 2, 1e-6, 100e9, 2e-6, 10e9, 64e9, 1e12)
    ranked = select_strategy(model, cluster, wl, CalibrationCoefficients(compute_coeff=1e-13))
    path = tmp_path / "report.json"
    save_report(compare_report(ranked, 5), path)
    assert path.read_bytes() == (GOLDEN / "ref_report_2x2.json").read_bytes()


@pytest.mark.parametrize("i", range(3))
def test_calibration_fit_matches_reference(i):
    fit = REF["fits"][i]
    cal = calibrate([ProfilingObservation(*o) for o in fit["obs"]])
    for k, v in fit["calib"].items():
        mine = getattr(cal, k)
        if isinstance(v, str):
            assert abs(mine - float(v)) <= 1e-9 * abs(float(v)) + 1e-30, (k, mine, v)
        else:
            assert mine == v


@pytest.mark.parametrize("text", sorted(REF["grammar"]))
def test_grammar_matches_reference(text):
    want = REF["grammar"][text]
    if "error" in want:
        with pytest.raises((GrammarError, StrategyError)) as ei:
            parse_strategy(text)
        assert type(ei.value).__name__ == want["error"]
        assert str(ei.value) == want["msg"]
    else:
        s = parse_strategy(text)
        assert format_strategy(s) == want["ok"]
        assert [s.attn_tp, s.attn_dp, s.moe_tp, s.moe_ep, s.d_pp] == want["deg"]
        assert format_strategy(parse_strategy(format_strategy(s))) == want["ok"]


# ---- acceptance criteria C4-C8 of the reference, restated
def test_c4_tp_sharding_cuts_inter_volume():
    for ratio in (0.5, 0.25, 0.125):
        for n_proc in (2, 4, 8):
            for k in (2, 4, 8):
                cl = ClusterConfig(4, n_proc, 1e-6, 100e9, 5e-6, 100e9 * ratio, 64e9, 1e12)
                m = ModelHyperparams(hidden_dim=1024, num_layers=4, top_k=k, num_routed_experts=16,
                                     num_shared_experts=0, psi_attn=1e6, psi_moe=8e6,
                                     psi_active=2e6)
                wl = WorkloadSpec(8, 256, 256, 64, 0.0)
                ep = [t for t in lambda_ep_terms(m, wl, cl) if t["op"] == "a2a"]
                mix = [t for t in lambda_mix_terms(m, wl, cl) if t["op"] == "a2a"]
                assert all(b["size_bytes"] * n_proc == a["size_bytes"] for a, b in zip(ep, mix))
                full = 8 * 256 * 1024 * k * 2
                shard = full / n_proc
                saving = 2 * 3 * (full - shard) / 4 / (100e9 * ratio)
                added = 1e-6 + (shard / n_proc) / 100e9
                assert (lambda_mix(m, wl, cl) < lambda_ep_baseline(m, wl, cl)) == (saving > added)


def test_c5_argmin_and_invariances(monkeypatch):
    m = ModelHyperparams(hidden_dim=1024, num_layers=8, top_k=2, num_routed_experts=32,
                         num_shared_experts=1, psi_attn=1e8, psi_moe=8e8, psi_active=2e8)
    cl = ClusterConfig(4, 8, 1e-6, 100e9, 5e-6, 10e9, 64e9, 1e13)
    wl = WorkloadSpec(16, 256, 256, 64, 5.0)
    cal = CalibrationCoefficients(compute_coeff=1e-13)
    for obj, val in (("ttft", lambda e: e.ttft), ("itl", lambda e: e.itl),
                     ("throughput", lambda e: -e.theta)):
        best = min((not indicators(s, m, wl, cl, cal).stable, val(indicators(s, m, wl, cl, cal)),
                    format_strategy(s)) for s in enumerate_strategies(cl, m)
                   if check_memory(s, m, cl, wl).feasible)
        assert format_strategy(select_strategy(m, cl, wl, cal, obj).best.strategy) == best[2]
    order = [format_strategy(e.strategy) for e in select_strategy(m, cl, wl, cal).entries]
    orig = an.enumerate_strategies
    monkeypatch.setattr(an, "enumerate_strategies",
                        lambda *a: random.Random(42).sample(orig(*a), len(orig(*a))))
    assert [format_strategy(e.strategy) for e in select_strategy(m, cl, wl, cal).entries] == order
    monkeypatch.undo()
    quiet = WorkloadSpec(16, 256, 256, 64, 0.0)
    scaled = CalibrationCoefficients(compute_coeff=7e-13, intra_alpha=7e-6, intra_beta=100e9 / 7,
                                     inter_alpha=35e-6, inter_beta=10e9 / 7)
    a = select_strategy(m, cl, quiet, cal)
    b = select_strategy(m, cl, quiet, scaled)
    assert [format_strategy(e.strategy) for e in a.entries] == \
        [format_strategy(e.strategy) for e in b.entries]
    assert b.best.estimate.ttft == pytest.approx(7 * a.best.estimate.ttft)


def test_c6_calibration_round_trip():
    truth = {"intra": (1e-6, 200e9), "inter": (8e-6, 20e9)}
    obs = []
    for scope, (a, b) in truth.items():
        for size in (1e4, 1e5, 1e6, 1e7):
            for d in (2, 4, 8):
                obs.append(ProfilingObservation("RS", size, d, scope, a + (size / d) / b))
                obs.append(ProfilingObservation("A2A", size, d, scope,
                                                (d - 1) * (a + (size / d) / b)))
    obs += [ProfilingObservation("MoE_compute", x, 1, "intra", 3e-13 * x) for x in (1e7, 1e8, 1e9)]
    c = calibrate(obs)
    assert c.intra_alpha == pytest.approx(1e-6, rel=0.01)
    assert c.intra_beta == pytest.approx(200e9, rel=0.01)
    assert c.inter_alpha == pytest.approx(8e-6, rel=0.01)
    assert c.inter_beta == pytest.approx(20e9, rel=0.01)
    assert c.compute_coeff == pytest.approx(3e-13, rel=0.01)


def test_c7_queue_closed_form():
    for rate in (0.0, 0.1, 1.0, 10.0, 100.0):
        for svc in (1e-4, 1e-3, 1e-2, 9e-3):
            if rate * svc >= 1:
                with pytest.raises(SaturationError):
                    queuing_delay(rate, svc)
            else:
                mu = 1 / svc
                assert queuing_delay(rate, svc) == pytest.approx(rate / (mu * (mu - rate)),
                                                                 rel=1e-15, abs=0)


def test_c8_bandwidth_regime_changes_winner():
    def order(cluster, k):
        m = ModelHyperparams(hidden_dim=1024, num_layers=8, top_k=k, num_routed_experts=32,
                             num_shared_experts=1, psi_attn=4e9, psi_moe=32e9, psi_active=2e9)
        wl = WorkloadSpec(64, 512, 512, 128, 1.0)
        cal = CalibrationCoefficients(compute_coeff=1e-14, ar_literal=False)
        scored = []
        for label, text in (("equal", "TP=8 + DP=4, TP=8 + EP=4"),
                            ("dp_greater", "TP=4 + DP=8, TP=8 + EP=4"),
                            ("dp_less", "TP=8 + DP=4, TP=4 + EP=8")):
            s = parse_strategy(text)
            if check_memory(s, m, cluster, wl).feasible:
                scored.append((indicators(s, m, wl, cluster, cal).ttft, label))
        return [lab for _, lab in sorted(scored)]
    assert order(ClusterConfig(4, 8, 5e-6, 6e9, 8e-6, 25e9, 4.5e9, 1e14), 1)[0] == "equal"
    assert order(ClusterConfig(4, 8, 2e-6, 400e9, 5e-6, 25e9, 4.5e9, 1e14), 8)[0] == "dp_less"


def test_collective_hand_arithmetic():
    link = LinkClass(0.0, 1e9)
    assert rs_cost(8192, 4, link) == pytest.approx(2.048e-6)
    assert ar_cost(8192, 2, link, literal=True) == pytest.approx(4.096e-6)
    assert a2a_cost(1024, 4, link) == pytest.approx(768e-9)
    assert rs_cost(5, 1, link) == 0.0


def test_b200_cluster_from_calibration_selects_a_layout():
    """Measured-style NVLink rows (same fabric for both scopes) -> fit ->
    ClusterConfig of one 8-GPU box -> a ranked MoE layout."""
    from paper_2601_08800_b200.calibration import b200_cluster
    obs = []
    for size in (1 << 16, 1 << 20, 1 << 24, 1 << 26):
        for scope in ("intra", "inter"):
            obs.append(ProfilingObservation("RS", size, 8, scope, 8e-6 + size / 8 / 700e9))
            obs.append(ProfilingObservation("A2A", size, 8, scope, 7 * (9e-6 + size / 8 / 650e9)))
    obs += [ProfilingObservation("MoE_compute", x, 1, "intra", x / 6e14) for x in (1e9, 1e10, 1e11)]
    cal = calibrate(obs, ar_literal=False)
    assert cal.intra_beta == pytest.approx(cal.inter_beta)
    cl = b200_cluster(cal, 2, 4)
    m = ModelHyperparams(hidden_dim=2048, num_layers=48, top_k=8, num_routed_experts=128,
                         num_shared_experts=0, psi_attn=1.5e9, psi_moe=2.9e10, psi_active=3.3e9)
    ranked = select_strategy(m, cl, WorkloadSpec(16, 4096, 4096, 256, 0.5), cal)
    best = ranked.best.strategy
    assert best.moe_tp * best.moe_ep * best.d_pp == 8
