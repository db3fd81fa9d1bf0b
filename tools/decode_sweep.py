"""BASELINE configs[3]: decode-regime sweep, fused layer vs NCCL AR+A2A.

    torchrun --nproc-per-node N tools/decode_sweep.py [--out profiles/decode_nN.jsonl]

Qwen3-30B-A3B-shaped layer (h=2048, I=768, 128 experts, top-8, bf16), total
tokens per step T_g in {N, 4N, 16, 64, 128, 256, 512} (multiples of the
group count, sim:575-577), TP2 x EP(N/2) (or --tp).  Per T_g: the fused
forward replayed as one CUDA graph (token and slot wires, with the token
wire's per-phase times from a second graph with event nodes) and the NCCL
baseline (all_to_all_single x2 + TP all_reduce around the same kernels)
graph-captured the same way with this routing's split sizes (and eagerly,
with its host sync, as before), CUDA events, max over ranks.  One JSON line
per T_g.
"""
import argparse
import json
import os
import sys
from pathlib import Path

import torch
import torch.distributed as dist

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2601_08800_b200 import SwiGLUExperts  # noqa: E402
from paper_2601_08800_b200.layer import MoELayer, layout_for  # noqa: E402

H, I, E, K = 2048, 768, 128, 8


def timed(fn, iters, stream, barrier=None):
    ev = []
    for _ in range(iters):
        if barrier:
            barrier()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        fn()
        b.record(stream)
        ev.append((a, b))
    torch.cuda.synchronize()
    t = torch.tensor([sum(a.elapsed_time(b) for a, b in ev) / iters * 1e3], device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=None)
    ap.add_argument("--iters", type=int, default=50)
    ap.add_argument("--tp", type=int, default=None)
    args = ap.parse_args()
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    rank, world = dist.get_rank(), dist.get_world_size()
    n, m = layout_for(world, args.tp)
    g = rank // m
    ex = SwiGLUExperts.random(E, H, I, seed=0)
    w13, w2 = ex.rank_shard(n, m, rank)
    del ex
    stream = torch.cuda.current_stream()
    lines = []
    for tg in sorted({world, 4 * world, 16, 64, 128, 256, 512}):
        if tg % n:
            continue
        T = tg // n
        gen = torch.Generator(device="cuda").manual_seed(100 + g)
        x = torch.randn(T, H, device="cuda", generator=gen).to(torch.bfloat16)
        logits = torch.randn(T, E, device="cuda", generator=gen)
        res = {"T_global": tg, "n_gpus": world, "layout": f"TP{m}xEP{n}"}
        for wire in ("token", "slot"):
            layer = MoELayer(n, m, T, H, E, K, I, w13=w13, w2=w2, rank=rank, wire=wire)
            run = layer.capture(x, logits)
            for _ in range(5):
                run()
            res[f"fused_{wire}_us"] = timed(run, args.iters, stream, layer.plan.barrier)
            if wire == "token":
                ph = layer.capture(x, logits, with_events=True)
                acc = {}
                for _ in range(10):
                    layer.plan.barrier()
                    ph()
                    torch.cuda.synchronize()
                    for k, v in ph.phase_ms():
                        acc.setdefault(k, []).append(v * 1e3)
                res["token_phases_us"] = {k: round(sum(v) / len(v), 1) for k, v in acc.items()}
                del ph
            if wire == "slot":
                bl = layer.capture_baseline(x, logits)
                for _ in range(3):
                    bl()
                res["nccl_us"] = timed(bl, args.iters, stream, layer.plan.barrier)
                res["nccl_captured"] = bl.graph is not None
                del bl
                for _ in range(3):
                    layer.forward_baseline(x, logits)
                res["nccl_eager_us"] = timed(lambda: layer.forward_baseline(x, logits),
                                             max(10, args.iters // 3), stream)
            del run
            layer.close()
        res["speedup_token_vs_nccl"] = res["nccl_us"] / res["fused_token_us"]
        res["speedup_slot_vs_nccl"] = res["nccl_us"] / res["fused_slot_us"]
        lines.append(res)
        if rank == 0:
            print(json.dumps(res), flush=True)
    if rank == 0 and args.out:
        Path(args.out).write_text("".join(json.dumps(r) + "\n" for r in lines))
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
