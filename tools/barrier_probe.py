"""Cost of the layer's device barrier and of one kernel boundary, replayed
as CUDA graphs (the decode regime's fixed costs).

    torchrun --nproc-per-node N tools/barrier_probe.py

Per rank: a graph of R barriers (mx_comm_barrier: fence, flag store into
every peer, spin on own flags) and a graph of R stamp kernels (one thread
writing %globaltimer: launch + PDL boundary only); µs per node, max over
ranks, one JSON line.
"""
import json
import os
import sys
from pathlib import Path

import torch
import torch.distributed as dist

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2601_08800_b200 import SwiGLUExperts  # noqa: E402
from paper_2601_08800_b200.layer import MoELayer, layout_for  # noqa: E402


def per_node(fn, reps, stream):
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=stream):
        for _ in range(reps):
            fn()
    for _ in range(3):
        g.replay()
    torch.cuda.synchronize()
    dist.barrier()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(stream)
    for _ in range(10):
        g.replay()
    b.record(stream)
    torch.cuda.synchronize()
    t = torch.tensor([a.elapsed_time(b) / 10 / reps * 1e3], device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return round(float(t.item()), 2)


def main():
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    rank, world = dist.get_rank(), dist.get_world_size()
    n, m = layout_for(world, 1)
    ex = SwiGLUExperts.random(128, 2048, 768, seed=0)
    w13, w2 = ex.rank_shard(n, m, rank)
    del ex
    layer = MoELayer(n, m, 16, 2048, 128, 8, 768, w13=w13, w2=w2, rank=rank, wire="token")
    s = torch.cuda.Stream()
    out = {"n_gpus": world}
    with torch.cuda.stream(s):
        out["stamp_kernel_us"] = per_node(lambda: layer.plan.stamp(0, stream=s), 64, s)
        out["barrier_plus_stamp_us"] = per_node(
            lambda: (layer.plan.barrier(stream=s), layer.plan.stamp(0, stream=s)), 32, s)
    if rank == 0:
        print(json.dumps(out))
    layer.close()
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
