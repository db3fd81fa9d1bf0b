"""Measured Gantt + stamped reference trace of the fused layer (§8(f)1).

    torchrun --nproc-per-node N tools/measured_trace.py --out gpurun_out/mt_nN

Config B shape (Qwen3-30B-A3B MoE layer, 8192 tokens, bf16 SwiGLU experts),
TP2 x EP(N/2), token wire.  Writes ``<out>_gantt.csv`` (reference Gantt
format, timeline.py:216-233), ``<out>_trace.csv`` (reference trace rows,
simcluster.py:99-100, + measured start_s/end_s/phase) and ``<out>.json``
(per-rank phase spans).  Stamps are device clocks (%globaltimer) after each
phase; medians over --iters runs.
"""
import argparse
import json
import os
import sys
from pathlib import Path

import numpy as np
import torch
import torch.distributed as dist

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import bench  # noqa: E402  (phase_model: algorithmic bytes per phase)
from paper_2601_08800_b200 import SwiGLUExperts  # noqa: E402
from paper_2601_08800_b200.layer import MoELayer, layout_for  # noqa: E402
from paper_2601_08800_b200.measured import (gantt_csv, gantt_rows, gather_phases,  # noqa: E402
                                            layer_trace, measure_phases, stamp_trace)

H, I, E, K = 2048, 768, 128, 8


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--tokens", type=int, default=8192)
    ap.add_argument("--iters", type=int, default=10)
    ap.add_argument("--wire", default="token")
    ap.add_argument("--out", required=True)
    args = ap.parse_args()
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    rank, world = dist.get_rank(), dist.get_world_size()
    n, m = layout_for(world)
    group, tp = divmod(rank, m)
    T = args.tokens // n
    ex = SwiGLUExperts.random(E, H, I, seed=0)
    w13, w2 = ex.rank_shard(n, m, rank)
    gen = torch.Generator(device="cuda").manual_seed(100 + group)
    x = torch.randn(T, H, device="cuda", generator=gen).to(torch.bfloat16)
    logits = torch.randn(T, E, device="cuda", generator=gen)
    layer = MoELayer(n, m, T, H, E, K, I, w13=w13, w2=w2, rank=rank, wire=args.wire)
    for _ in range(3):
        layer.forward(x, logits)
    torch.cuda.synchronize()
    phases = measure_phases(layer, x, logits, iters=args.iters)
    per_rank = gather_phases(phases)
    cnt, send = layer.routing_counts()
    U = layer.pair_counts() if args.wire == "token" else None
    model = bench.phase_model(send.astype(np.int64), cnt, n, m, group, tp, T, U, args.wire)
    pb = {k: v.get("bytes", 0) for k, v in model.items()}
    all_pb = [None] * world
    dist.all_gather_object(all_pb, pb)
    events, stages = layer_trace(layer)
    if rank == 0:
        out = Path(args.out)
        rows = gantt_rows(per_rank, all_pb)
        Path(f"{out}_gantt.csv").write_text(gantt_csv(rows))
        Path(f"{out}_trace.csv").write_text(stamp_trace(events, stages, per_rank, args.wire))
        makespan = max(b for ph in per_rank for _, b in ph.values())
        Path(f"{out}.json").write_text(json.dumps({
            "n_gpus": world, "layout": f"TP{m}xEP{n}", "wire": args.wire,
            "global_tokens": args.tokens, "makespan_s": makespan,
            "phases": per_rank, "trace_events": len(events)}, indent=1) + "\n")
        print(json.dumps({"makespan_us": makespan * 1e6, "events": len(events),
                          "rank0": {k: round((b - a) * 1e6, 1) for k, (a, b) in per_rank[0].items()}}))
    layer.close()
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
