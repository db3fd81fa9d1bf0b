"""Device-barrier latency over NVLink: K barrier kernels replayed in one CUDA
graph, CUDA events around the replay, max over ranks.

    torchrun --nproc-per-node N tools/barrier_bench.py
"""
import os
import sys
from pathlib import Path

import torch
import torch.distributed as dist

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2601_08800_b200.layer import MoELayer, layout_for  # noqa: E402


def main():
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    rank, world = dist.get_rank(), dist.get_world_size()
    n, m = layout_for(world)
    layer = MoELayer(n, m, 128, 256, 16, 2, 0, rank=rank, dtype=torch.float32,
                     expert_kind="affine", scales=[1.0] * 16, biases=[0.0] * 16)
    K = 200
    for _ in range(10):
        layer.plan.barrier()
    torch.cuda.synchronize()
    dist.barrier()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(K):
            layer.plan.barrier()
    g.replay()
    torch.cuda.synchronize()
    dist.barrier()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    g.replay()
    b.record()
    torch.cuda.synchronize()
    t = torch.tensor([a.elapsed_time(b) / K * 1e3], device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    if rank == 0:
        print(f"device barrier over {world} GPUs: {t.item():.2f} us per barrier (graph of {K})")
    layer.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
