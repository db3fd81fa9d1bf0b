"""Freeze DeepSeek-V3 router outputs from transformers (build container).

    python tests/golden/make_router_golden.py

Calls the UNMODIFIED ``DeepseekV3MoE.route_tokens_to_experts``
(transformers ``models/deepseek_v3/modeling_deepseek_v3.py``, the router
named by BASELINE configs[2] / SURVEY.md §8(f)4) on seeded fp32 logits and a
seeded score-correction bias, with the DeepSeek-R1 settings (256 experts,
8 groups, top-4 groups, top-8, normalised, routed scaling 2.5) and a small
second shape.  ``sorted=False`` leaves the id order unspecified, so each
row's ids are stored sorted with their weights.  The fixture is committed;
tests never import transformers for this.
"""
from pathlib import Path
from types import SimpleNamespace

import numpy as np
import torch
from transformers.models.deepseek_v3.modeling_deepseek_v3 import DeepseekV3MoE

HERE = Path(__file__).resolve().parent
CASES = [  # name, T, E, k, n_group, topk_group, norm, scaling, bias scale, bias offset
    ("r1", 512, 256, 8, 8, 4, True, 2.5, 0.05, 0.0),
    ("small", 300, 64, 6, 4, 2, False, 1.0, 0.3, 0.0),
    # choice keys mostly negative: masked experts (0.0) outrank selected ones
    ("negbias", 200, 64, 8, 8, 2, True, 2.5, 0.3, -0.8),
]


def main():
    out = {}
    for seed, (name, T, E, k, ng, tg, norm, scale, bs, bo) in enumerate(CASES):
        rng = np.random.default_rng(1000 + seed)
        logits = rng.standard_normal((T, E)).astype(np.float32)
        bias = (bo + bs * rng.standard_normal(E)).astype(np.float32)
        fake = SimpleNamespace(gate=SimpleNamespace(e_score_correction_bias=torch.from_numpy(bias)),
                               n_group=ng, topk_group=tg, n_routed_experts=E, top_k=k,
                               norm_topk_prob=norm, routed_scaling_factor=scale)
        idx, w = DeepseekV3MoE.route_tokens_to_experts(fake, torch.from_numpy(logits))
        idx, w = idx.numpy(), w.numpy()
        o = np.argsort(idx, axis=1)
        out[f"{name}_logits"] = logits
        out[f"{name}_bias"] = bias
        out[f"{name}_ids"] = np.take_along_axis(idx, o, axis=1).astype(np.int32)
        out[f"{name}_w"] = np.take_along_axis(w, o, axis=1).astype(np.float32)
        out[f"{name}_cfg"] = np.array([T, E, k, ng, tg, int(norm)], dtype=np.int64)
        out[f"{name}_scaling"] = np.array([scale], dtype=np.float32)
    np.savez_compressed(HERE / "deepseek_router.npz", **out)
    print("wrote", HERE / "deepseek_router.npz")


if __name__ == "__main__":
    main()
