"""Timeline of the overlapped forward (mx_forward's two-stream schedule):
device-clock stamps after each step on its own stream (MX_OVERLAP_STAMPS=1,
stamp slots 30..44), median over iterations, rank 0 prints one JSON line.

    torchrun --nproc-per-node N tools/overlap_timeline.py [--tp M] [--tokens 8192]
"""
import argparse
import json
import os
import sys
from pathlib import Path

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2601_08800_b200 import SwiGLUExperts  # noqa: E402
from paper_2601_08800_b200.layer import MoELayer, layout_for  # noqa: E402

STEPS = ["start", "layout", "dispatch_own", "dispatch_other (side)", "rows_landed (side)",
         "expand (side)", "gemm1_own", "gemm1_other", "gemm2_other", "push_other (side)",
         "gemm2_own", "reduce_own", "zin_complete", "combine", "y_complete"]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--tp", type=int, default=1)
    ap.add_argument("--tokens", type=int, default=8192)
    ap.add_argument("--iters", type=int, default=10)
    a = ap.parse_args()
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    rank, world = dist.get_rank(), dist.get_world_size()
    n, m = layout_for(world, a.tp)
    H, I, E, K = 2048, 768, 128, 8
    T = a.tokens // n
    ex = SwiGLUExperts.random(E, H, I, seed=0)
    w13, w2 = ex.rank_shard(n, m, rank)
    del ex
    layer = MoELayer(n, m, T, H, E, K, I, w13=w13, w2=w2, rank=rank, wire="token")
    g = torch.Generator(device="cuda").manual_seed(1000 + rank // m)
    x = torch.randn(T, H, device="cuda", generator=g).to(torch.bfloat16)
    logits = torch.randn(T, E, device="cuda", generator=g)
    os.environ["MX_OVERLAP_STAMPS"] = "1"
    runs = []
    view = layer.plan.stamps_view(rank)
    for i in range(a.iters + 3):
        layer.plan.barrier()
        layer.forward(x, logits, check=False)
        torch.cuda.synchronize()
        if i >= 3:
            runs.append(view[30:30 + len(STEPS)].cpu().numpy().astype(np.int64))
    del os.environ["MX_OVERLAP_STAMPS"]
    st = np.median(np.stack([r - r[0] for r in runs]), axis=0) / 1e3
    allst = [None] * world
    dist.all_gather_object(allst, [round(float(v), 1) for v in st])
    if rank == 0:
        print(json.dumps({"layout": f"TP{m}xEP{n}", "tokens": a.tokens, "steps_us": STEPS,
                          "ranks": allst}))
    layer.close()
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
