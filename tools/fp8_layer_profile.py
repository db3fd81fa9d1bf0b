"""Config C's layer at N=1 (256 routed fp8 experts + shared expert, h=7168,
DeepSeek-V3 gate, 8192 tokens), three eager forwards: the target for an
ncu capture of the kind::f8f6f4 grouped GEMM (tools/runs/ncu_fp8.sh)."""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2601_08800_b200 import FP8SwiGLUExperts  # noqa: E402
from paper_2601_08800_b200.layer import MoELayer  # noqa: E402
from paper_2601_08800_b200.plan import GateSpec  # noqa: E402


def main():
    T, h, E, k, I, Is = 8192, 7168, 256, 8, 2048, 2048
    ex = FP8SwiGLUExperts.random(E, h, I, shared_inter=Is, seed=0)
    ex.rank_shard(1, 1, 0)
    ex.src = ex.shared = None
    torch.cuda.empty_cache()
    bias = (0.05 * torch.randn(E, generator=torch.Generator().manual_seed(3))).float()
    layer = MoELayer(1, 1, T, h, E, k, I, experts=ex, rank=0,
                     gate=GateSpec.deepseek_v3(bias, groups=8, topk_groups=4, scaling=2.5))
    g = torch.Generator(device="cuda").manual_seed(1000)
    x = torch.randn(T, h, device="cuda", generator=g).to(torch.bfloat16)
    logits = torch.randn(T, E, device="cuda", generator=g)
    for _ in range(3):
        layer.forward(x, logits)
    torch.cuda.synchronize()
    print("ok")


if __name__ == "__main__":
    main()
