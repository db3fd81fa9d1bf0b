"""A small emulated-cluster layer forward for compute-sanitizer (one
process, every rank's heap on one GPU, so the dispatch / expand / pair
pre-reduction / combine kernels run their peer-heap code paths with local
addresses): token wire with enough pairs per SM for the bulk-copy
pre-reduction ring, and the slot wire.

    compute-sanitizer --tool racecheck python tools/sanitize_layer.py
"""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2601_08800_b200 import _native as N  # noqa: E402
from paper_2601_08800_b200 import SwiGLUExperts  # noqa: E402
from paper_2601_08800_b200.plan import LayerPlan  # noqa: E402


def main():
    n, m, T, h, E, k, I = 2, 2, 2400, 256, 16, 4, 256
    ex = SwiGLUExperts.random(E, h, I, seed=1)
    w13, w2 = ex.stacked_shards(n, m)
    g = torch.Generator(device="cuda").manual_seed(2)
    x = torch.randn(n * T, h, device="cuda", generator=g).to(torch.bfloat16)
    logits = torch.randn(n * T, E, device="cuda", generator=g)
    for wire in ("token", "slot"):
        plan = LayerPlan(n, m, T, h, E, k, dtype=torch.bfloat16, expert_kind="swiglu",
                         inter=I, wire=wire)
        y = torch.empty(n * T, h, dtype=torch.bfloat16, device="cuda")
        plan.forward(x, N.ExpertParams(None, None, w13.data_ptr(), w2.data_ptr()),
                     logits=logits, y_out=y)
        torch.cuda.synchronize()
        plan.check()
        plan.close()
        print(wire, "ok", float(y.float().abs().mean()), flush=True)


if __name__ == "__main__":
    main()
