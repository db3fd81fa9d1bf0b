"""Layout selection from the fused layer's measured costs (config E).

Pins :mod:`paper_2601_08800_b200.layer_model` to the round-1 B200
measurements: the ranking of TP1xEP4 vs TP2xEP2 on 4 GPUs flips with the
router's skew exactly as measured (profiles/r01_configE_n4.jsonl), and the
absolute predictions stay near the measured bench lines."""
import numpy as np
import pytest
import torch

from paper_2601_08800_b200.layer_model import (LayerCalibration, predict_layer,
                                               routing_stats, select_layout)
from paper_2601_08800_b200.skew import zipf_logits

H, I, E, K, TG = 2048, 768, 128, 8, 8192


def _ids(s, seed=0):
    g = torch.Generator().manual_seed(seed)
    return torch.topk(zipf_logits(TG, E, s, seed=1, generator=g), K, dim=1).indices.numpy()


def test_routing_stats_by_hand():
    # 4 tokens, 2 groups of 2, 4 experts (host = e*2//4), top-2
    ids = np.array([[0, 1], [0, 2], [3, 2], [1, 3]])
    S, U = routing_stats(ids, 2, 4)
    # group 0 tokens: {0,1}->host0 x2 ; {0,2}->host0,host1
    # group 1 tokens: {3,2}->host1 x2 ; {1,3}->host0,host1
    assert S.tolist() == [[3, 1], [1, 3]]
    assert U.tolist() == [[2, 1], [1, 2]]
    with pytest.raises(ValueError):
        routing_stats(ids[:3], 2, 4)


def test_layouts_respect_the_tp_shard_rule():
    ids = _ids(0.0)
    names = [r["layout"] for r in select_layout(ids, 8, E, H, I)]
    assert set(names) == {"TP1xEP8", "TP2xEP4"}       # I/4 = 192 is not a multiple of 128


@pytest.mark.parametrize("s,best", [(0.0, "TP1xEP4"), (0.8, "TP2xEP2"), (1.0, "TP2xEP2"),
                                    (1.2, "TP2xEP2")])
def test_ranking_matches_measured_config_e(s, best):
    """Measured at 4 x B200 (round 1, profiles/r01_configE_n4.jsonl): EP4
    0.319 ms vs TP2xEP2 0.341 ms at s=0; TP2xEP2 0.348-0.351 ms vs EP4
    0.375-0.395 ms for s >= 0.8."""
    assert select_layout(_ids(s), 4, E, H, I)[0]["layout"] == best


@pytest.mark.parametrize("n,m,measured_ms", [(1, 1, 0.688), (2, 1, 0.446), (2, 2, 0.344),
                                             (4, 1, 0.317)])
def test_predictions_near_measured(n, m, measured_ms):
    # measured: bench.py lines of profiles/r01_n{1,2,4}_bench.json
    # (value and layout_ep_only), uniform router
    pred = predict_layer(_ids(0.0), n, m, E, H, I)["seconds"] * 1e3
    assert abs(pred - measured_ms) / measured_ms < 0.15, pred


def test_skew_only_hurts_expert_parallel_layouts():
    u, z = _ids(0.0), _ids(1.2)
    one = predict_layer(u, 1, 1, E, H, I)["seconds"]
    assert predict_layer(z, 1, 1, E, H, I)["seconds"] == pytest.approx(one, rel=1e-9)
    assert predict_layer(z, 4, 1, E, H, I)["seconds"] > predict_layer(u, 4, 1, E, H, I)["seconds"]


def test_calibration_interpolates_gemm_efficiency():
    c = LayerCalibration()
    assert c.gemm(768) == (0.6952, 0.6114) and c.gemm(384) == (0.5612, 0.5025)
    g1, g2 = c.gemm(576)
    assert 0.5612 < g1 < 0.6952 and 0.5025 < g2 < 0.6114
    assert c.gemm(192) == c.gemm(384) and c.gemm(2048) == c.gemm(768)
    # the round-1 throughputs behind the defaults: 0.83 of 1397.3 TF/s (GEMM1, I/m = 768)
    assert c.gemm(768)[0] * c.bf16_tflops == pytest.approx(0.83 * 1397.3, rel=1e-3)


@pytest.mark.parametrize("s,layout", [(0.0, (4, 1)), (1.2, (2, 2))])
def test_layout_for_auto_follows_the_model(s, layout):
    from paper_2601_08800_b200.layer import layout_for
    assert layout_for(4, "auto", routing=_ids(s), num_experts=E, hidden=H, inter=I) == layout
    assert layout_for(4) == (2, 2)                       # default: config B's TP2
    with pytest.raises(ValueError):
        layout_for(4, "auto")
    with pytest.raises(ValueError):                      # no TP shard of I=200 is 128-aligned
        layout_for(4, "auto", routing=_ids(s), num_experts=E, hidden=H, inter=200)


def test_calibration_from_measured_bench_lines():
    """Recalibrating from the round's bench lines reproduces the defaults
    (which were read off them) and tracks the newer 4-GPU kernels."""
    import json
    from pathlib import Path
    prof = Path(__file__).resolve().parents[1] / "profiles"
    lines = [json.loads((prof / f).read_text()) for f in
             ("r01_n1_bench.json", "r01_n2_bench.json", "r01_n4_bench.json")]
    d = LayerCalibration()

    def close(a, b):  # throughputs (efficiency x the peak it was taken against)
        return abs(a - b) / b < 0.025

    one = LayerCalibration.from_bench(lines[0])           # slot wire, 1 GPU
    assert close(one.eff["dispatch_hbm"] * one.hbm_gbs, d.eff["dispatch_hbm"] * d.hbm_gbs)
    assert close(one.eff["combine_hbm"] * one.hbm_gbs, d.eff["combine_hbm"] * d.hbm_gbs)
    c = LayerCalibration.from_bench(lines)
    assert c.nvlink_gbs == 770.0 and c.hbm_gbs == 6539.5  # the round-1 lines' denominators
    assert close(c.eff["pair_reduce"] * c.hbm_gbs, d.eff["pair_reduce"] * d.hbm_gbs)
    assert close(c.eff["combine_nvlink"] * c.nvlink_gbs, d.eff["combine_nvlink"] * d.nvlink_gbs)
    assert close(c.eff["pair_push_nvlink"] * c.nvlink_gbs, d.eff["pair_push_nvlink"] * d.nvlink_gbs)
    assert close(c.gemm(768)[0] * c.bf16_tflops, d.gemm(768)[0] * d.bf16_tflops)
    assert close(c.gemm(384)[0] * c.bf16_tflops, d.gemm(384)[0] * d.bf16_tflops)
    newer = LayerCalibration.from_bench(json.loads((prof / "r01b_n4_bench.json").read_text()), c)
    assert newer.eff["pair_push_nvlink"] > c.eff["pair_push_nvlink"]   # bulk-copy pre-reduction
    assert newer.eff["expand"] > 0.6
    pred = predict_layer(_ids(0.0), 2, 2, E, H, I, newer)["seconds"] * 1e3
    assert abs(pred - 0.332) / 0.332 < 0.15, pred


def test_model_tracks_round_two_lines():
    """Recalibrated from the round-2 4-GPU lines (denominators: HBM copy,
    burst bf16, same-run NVLink probe), the model still predicts the
    measured TP2 x EP2 and EP4 layer times within 15% and ranks EP4 first
    on the uniform router, as measured (0.309 vs 0.337 ms)."""
    import json
    from pathlib import Path
    prof = Path(__file__).resolve().parents[1] / "profiles"
    lines = [json.loads((prof / f).read_text()) for f in
             ("r02_n4_tp2_bench.json", "r02_n4_ep4_bench.json")]
    c = LayerCalibration.from_bench(lines)
    assert c.nvlink_gbs == pytest.approx(651.0, rel=0.01) and c.bf16_tflops == 1668.3
    u = _ids(0.0)
    tp2 = predict_layer(u, 2, 2, E, H, I, c)["seconds"] * 1e3
    ep4 = predict_layer(u, 4, 1, E, H, I, c)["seconds"] * 1e3
    assert abs(tp2 - 0.337) / 0.337 < 0.15, tp2
    assert abs(ep4 - 0.309) / 0.309 < 0.15, ep4
    assert select_layout(u, 4, E, H, I, c)[0]["layout"] == "TP1xEP4"
