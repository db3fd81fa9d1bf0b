"""Config E: Zipf-skewed routers and the skew-aware strategy ranking.

The skew term must (1) vanish exactly on balanced routers, so every
reference ranking fixture still holds, and (2) price each strategy's A2A on
its hottest expert host under skew."""
import gzip
import json

import numpy as np
import pytest

from conftest import GOLDEN
from paper_2601_08800_b200.analyzer import select_strategy
from paper_2601_08800_b200.config import (CalibrationCoefficients, ClusterConfig,
                                          ModelHyperparams, WorkloadSpec)
from paper_2601_08800_b200.costmodel import comm_terms, indicators
from paper_2601_08800_b200.errors import AnalyzerError
from paper_2601_08800_b200.skew import (expert_counts, host_loads, host_skew, zipf_logits,
                                        zipf_popularity)
from paper_2601_08800_b200.strategy import enumerate_strategies, format_strategy

with gzip.open(GOLDEN / "ref_selector.json.gz", "rt") as _f:
    REF = json.load(_f)


def _objs(case):
    return (ModelHyperparams(**case["model"]), ClusterConfig(*case["cluster"]),
            WorkloadSpec(*case["workload"]), CalibrationCoefficients(**case["calib"]))


def test_zipf_popularity_shape():
    p = zipf_popularity(128, 1.2, seed=3)
    assert p.shape == (128,) and abs(p.sum() - 1) < 1e-12
    assert np.all(p > 0)
    ranks = np.sort(p)[::-1]
    assert ranks[0] / ranks[1] == pytest.approx(2 ** 1.2)
    assert np.array_equal(p, zipf_popularity(128, 1.2, seed=3))       # deterministic
    assert not np.array_equal(p, zipf_popularity(128, 1.2, seed=4))   # order permuted
    assert np.all(zipf_popularity(16, 0.0) == 1 / 16)                 # s = 0: uniform
    with pytest.raises(ValueError):
        zipf_popularity(8, -1)


def test_host_loads_and_skew_by_hand():
    load = np.array([4, 0, 1, 1, 1, 1, 0, 0], float)     # hosts of ep=4: 4,2,2,0
    assert host_loads(load, 4).tolist() == [4, 2, 2, 0]
    assert host_skew(load, 4) == 4 / 2
    assert host_skew(load, 2) == 6 / 4
    assert host_skew(load, 1) == 1.0
    assert host_skew(None, 8) == 1.0
    assert host_skew(np.ones(128), 8) == 1.0               # balanced: exactly 1
    assert host_skew(np.ones(4), 8) == 1.0                 # ep > E: empty hosts ignored
    with pytest.raises(ValueError):
        host_loads(load, 0)


@pytest.mark.parametrize("s", [0.8, 1.0, 1.2])
def test_skew_grows_with_exponent_and_degree(s):
    p = zipf_popularity(128, s, seed=0)
    q = zipf_popularity(128, s + 0.2, seed=0)
    ks = [host_skew(p, d) for d in (1, 2, 4, 8, 16)]
    assert ks[0] == 1.0 and all(a <= b for a, b in zip(ks, ks[1:]))
    assert all(host_skew(q, d) >= host_skew(p, d) for d in (2, 4, 8))


def test_expert_counts_from_logits():
    import torch
    g = torch.Generator().manual_seed(0)
    lg = zipf_logits(4096, 64, 1.2, seed=1, generator=g)
    ids = torch.topk(lg, 8, dim=1).indices.numpy()
    c = expert_counts(ids, 64)
    assert c.sum() == 4096 * 8
    # the popular experts of the law are the popular experts of the router
    p = zipf_popularity(64, 1.2, seed=1)
    assert np.argmax(c) == np.argmax(p)
    assert host_skew(c, 8) > 1.3


@pytest.mark.parametrize("idx", range(0, len(REF["cases"]), 3))
def test_balanced_load_reproduces_reference_ranking(idx):
    """kappa == 1.0 exactly on a balanced router: same estimates, same order."""
    case = REF["cases"][idx]
    model, cluster, workload, calib = _objs(case)
    uniform = np.full(model.num_routed_experts, 7.0)
    for obj in ("ttft", "throughput"):
        try:
            a = select_strategy(model, cluster, workload, calib, objective=obj)
        except AnalyzerError:
            with pytest.raises(AnalyzerError):
                select_strategy(model, cluster, workload, calib, objective=obj,
                                expert_load=uniform)
            continue
        b = select_strategy(model, cluster, workload, calib, objective=obj, expert_load=uniform)
        assert [format_strategy(e.strategy) for e in a.entries] == \
               [format_strategy(e.strategy) for e in b.entries]
        for x, y in zip(a.entries, b.entries):
            assert (x.estimate.ttft, x.estimate.itl, x.estimate.theta) == \
                   (y.estimate.ttft, y.estimate.itl, y.estimate.theta)


def test_skew_prices_a2a_on_the_hottest_host():
    case = REF["cases"][0]
    model, cluster, workload, calib = _objs(case)
    p = zipf_popularity(model.num_routed_experts, 1.2, seed=0)
    for strat in enumerate_strategies(cluster, model):
        base = comm_terms(strat, model, workload, cluster, calib)
        sk = comm_terms(strat, model, workload, cluster, calib, expert_load=p)
        kappa = host_skew(p, strat.moe_ep)
        for t0, t1 in zip(base, sk):
            if t0["op"] == "a2a":
                assert t1["size_bytes"] == t0["size_bytes"] * kappa
                assert t1["host_skew"] == kappa
                assert t1["seconds"] >= t0["seconds"]
            else:
                assert t1 == t0
        e0 = indicators(strat, model, workload, cluster, calib)
        e1 = indicators(strat, model, workload, cluster, calib, p)
        if strat.moe_ep == 1:
            assert e1.ttft == e0.ttft
        else:
            assert e1.ttft >= e0.ttft


def test_skew_moves_selection_toward_tensor_parallel_experts():
    """On a B200-calibrated 2x4 box the hottest-host penalty grows with the EP
    degree, so the TTFT gap between EP-heavy and TP-heavy MoE layouts widens
    monotonically with the Zipf exponent."""
    from paper_2601_08800_b200.calibration import b200_cluster
    from paper_2601_08800_b200.analyzer import ProfilingObservation, calibrate
    obs = []
    for size in (1 << 16, 1 << 20, 1 << 24, 1 << 26):
        for scope in ("intra", "inter"):
            obs.append(ProfilingObservation("RS", size, 8, scope, 8e-6 + size / 8 / 700e9))
            obs.append(ProfilingObservation("A2A", size, 8, scope, 7 * (9e-6 + size / 8 / 650e9)))
    obs += [ProfilingObservation("MoE_compute", x, 1, "intra", x / 6e14) for x in (1e9, 1e10, 1e11)]
    cal = calibrate(obs, ar_literal=False)
    cl = b200_cluster(cal, 2, 4)
    m = ModelHyperparams(hidden_dim=2048, num_layers=48, top_k=8, num_routed_experts=128,
                         num_shared_experts=0, psi_attn=1.5e9, psi_moe=2.9e10, psi_active=3.3e9)
    wl = WorkloadSpec(16, 4096, 4096, 256, 0.5)
    gaps = []
    for s in (0.0, 0.8, 1.0, 1.2):
        r = select_strategy(m, cl, wl, cal, expert_load=zipf_popularity(128, s, seed=0))
        by = {format_strategy(e.strategy): e.estimate.ttft for e in r.entries}
        gaps.append(by["DP=8, EP=8"] - by["DP=8, TP=4 + EP=2"])
        assert r.best.strategy.moe_ep <= 2
    assert all(a < b for a, b in zip(gaps, gaps[1:]))
