"""Probe: two micro-batches on two streams so one's NVLink phases overlap the
other's grouped GEMMs (the paper's comm/compute overlap, at layer level).

    MX_GEMM_CTAS=128 torchrun --nproc-per-node 4 tools/overlap_probe.py

Micro-batch A runs route/layout/dispatch, then its experts, then combine on
stream 0; micro-batch B (its own plan and symmetric heap, T/2 tokens) starts
on stream 1 once A's dispatch is queued, so B's dispatch overlaps A's GEMMs
and A's combine overlaps B's GEMMs.  Captured as one CUDA graph; CUDA
events, max over ranks, L2 flushed per step.  Prints one JSON line.
"""
import argparse
import ctypes as C
import json
import os
import sys
from pathlib import Path

import torch
import torch.distributed as dist

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2601_08800_b200 import SwiGLUExperts, _native as N  # noqa: E402
from paper_2601_08800_b200.layer import MoELayer, layout_for  # noqa: E402
from paper_2601_08800_b200.plan import stream_ptr  # noqa: E402

H, I, E, K = 2048, 768, 128, 8


def pre(layer, x, lg, s):
    p, r = layer.plan, layer.rank
    p.route(logits=lg, rank=r, stream=s)
    p.barrier(stream=s)
    p.layout(rank=r, stream=s)
    p.dispatch(x, rank=r, stream=s)
    p.barrier(stream=s)


def expert(layer, s):
    N.check(N.load().mx_expert(layer.plan._plan, layer.rank, C.byref(layer.params),
                               stream_ptr(s)), "expert")


def post(layer, s):
    p = layer.plan
    p.barrier(stream=s)
    p.combine(rank=layer.rank, stream=s)
    p.barrier(stream=s)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--tokens", type=int, default=8192)
    ap.add_argument("--iters", type=int, default=30)
    ap.add_argument("--mb", type=int, default=2)
    ap.add_argument("--stagger", default="dispatch", choices=["none", "dispatch"])
    args = ap.parse_args()
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    rank, world = dist.get_rank(), dist.get_world_size()
    n, m = layout_for(world)
    g = rank // m
    ex = SwiGLUExperts.random(E, H, I, seed=0)
    w13, w2 = ex.rank_shard(n, m, rank)
    T = args.tokens // n
    gen = torch.Generator(device="cuda").manual_seed(100 + g)
    x = torch.randn(T, H, device="cuda", generator=gen).to(torch.bfloat16)
    lg = torch.randn(T, E, device="cuda", generator=gen)
    mb = args.mb
    Tm = T // mb
    layers = [MoELayer(n, m, Tm, H, E, K, I, w13=w13, w2=w2, rank=rank, wire="token")
              for _ in range(mb)]
    xs = [x[i * Tm:(i + 1) * Tm] for i in range(mb)]
    ls = [lg[i * Tm:(i + 1) * Tm] for i in range(mb)]
    y = torch.empty(T, H, dtype=torch.bfloat16, device="cuda")
    side = [torch.cuda.Stream() for _ in range(mb - 1)]

    def step():
        main_s = torch.cuda.current_stream()   # the capture stream inside the graph
        streams = [main_s] + side
        start = torch.cuda.Event()
        start.record(main_s)
        gate = start
        for i, L in enumerate(layers):
            s = streams[i]
            if i > 0:
                s.wait_event(gate)
            with torch.cuda.stream(s):
                pre(L, xs[i], ls[i], s)
                if args.stagger == "dispatch":   # next micro-batch starts now
                    gate = torch.cuda.Event()
                    gate.record(s)
                expert(L, s)
                post(L, s)
                y[i * Tm:(i + 1) * Tm].copy_(L.y, non_blocking=True)
        for s in side:
            main_s.wait_stream(s)

    for _ in range(2):
        step()
    torch.cuda.synchronize()
    dist.barrier()
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph):
        step()
    torch.cuda.synchronize()
    dist.barrier()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    for _ in range(5):
        graph.replay()
    main_s = torch.cuda.current_stream()
    ev = []
    for _ in range(args.iters):
        flush.fill_(1)
        layers[0].plan.barrier()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(main_s)
        graph.replay()
        b.record(main_s)
        ev.append((a, b))
    torch.cuda.synchronize()
    t = torch.tensor([sum(a.elapsed_time(b) for a, b in ev) / args.iters], device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    if rank == 0:
        print(json.dumps({"n_gpus": world, "layout": f"TP{m}xEP{n}", "micro_batches": mb,
                          "stagger": args.stagger,
                          "gemm_ctas": os.environ.get("MX_GEMM_CTAS", "all"),
                          "ms_per_step": float(t.item()),
                          "tokens_per_s": args.tokens / (float(t.item()) / 1e3)}), flush=True)
    del graph
    for L in layers:
        L.close()
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
