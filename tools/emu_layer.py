"""Config-B layer on the emulated cluster (every rank's kernels on one GPU,
peer stores landing in local HBM): a single-process target for ncu captures
of the token wire's kernels (k_pair_reduce, k_dispatch_token, ...), whose
multi-rank runs may not be profiled.

    ncu --set full -k regex:k_pair_reduce -s 4 -c 1 python tools/emu_layer.py
"""
from __future__ import annotations

import argparse
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main() -> int:
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=2)
    ap.add_argument("--m", type=int, default=2)
    ap.add_argument("--tokens", type=int, default=8192, help="global tokens")
    ap.add_argument("--iters", type=int, default=3)
    a = ap.parse_args()
    from paper_2601_08800_b200 import SwiGLUExperts, _native as N
    from paper_2601_08800_b200.plan import LayerPlan
    n, m = a.n, a.m
    T, h, E, k, I = a.tokens // n, 2048, 128, 8, 768
    ex = SwiGLUExperts.random(E, h, I, seed=0)
    w13, w2 = ex.stacked_shards(n, m)
    gen = torch.Generator(device="cuda").manual_seed(1)
    x = torch.randn(n * T, h, device="cuda", generator=gen).to(torch.bfloat16)
    logits = torch.randn(n * T, E, device="cuda", generator=gen)
    plan = LayerPlan(n, m, T, h, E, k, dtype=torch.bfloat16, expert_kind="swiglu", inter=I,
                     wire="token")
    y = torch.empty(n * T, h, dtype=torch.bfloat16, device="cuda")
    params = N.ExpertParams(None, None, w13.data_ptr(), w2.data_ptr())
    for _ in range(a.iters):
        plan.forward(x, params, logits=logits, y_out=y)
    torch.cuda.synchronize()
    print("ok", float(y.float().abs().mean()))
    plan.close()
    return 0


if __name__ == "__main__":
    sys.exit(main())
