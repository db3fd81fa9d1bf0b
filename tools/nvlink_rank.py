"""One rank of a 2-GPU config-B layer (TP1 x EP2, token wire) for profiling
the NVLink kernels of ONE rank under ncu (tools/runs/nvlink_ncu.sh starts
the other rank as a plain process): a few eager forwards, then exit.

    RANK=r LOCAL_RANK=r WORLD_SIZE=2 MASTER_ADDR=127.0.0.1 MASTER_PORT=p python tools/nvlink_rank.py
"""
import os
import sys
from pathlib import Path

import torch
import torch.distributed as dist

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2601_08800_b200 import SwiGLUExperts  # noqa: E402
from paper_2601_08800_b200.layer import MoELayer  # noqa: E402


def main():
    local = int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dist.init_process_group("gloo")
    rank, world = dist.get_rank(), dist.get_world_size()
    n, m, H, I, E, K = world, 1, 2048, 768, 128, 8
    T = 8192 // n
    ex = SwiGLUExperts.random(E, H, I, seed=0)
    w13, w2 = ex.rank_shard(n, m, rank)
    del ex
    layer = MoELayer(n, m, T, H, E, K, I, w13=w13, w2=w2, rank=rank, wire="token")
    g = torch.Generator(device="cuda").manual_seed(1000 + rank)
    x = torch.randn(T, H, device="cuda", generator=g).to(torch.bfloat16)
    logits = torch.randn(T, E, device="cuda", generator=g)
    for _ in range(int(os.environ.get("FORWARDS", "5"))):
        layer.forward(x, logits, check=False)
    torch.cuda.synchronize()
    dist.barrier()
    layer.close()
    print(f"rank {rank} ok", flush=True)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
