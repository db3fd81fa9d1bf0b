"""BASELINE configs[2] (DeepSeek-R1-shaped fp8 layer) and configs[4] (Zipf
skew with strategy auto-selection) on the fused layer.

    torchrun --nproc-per-node N tools/config_sweep.py --config C [--out f.jsonl]
    torchrun --nproc-per-node N tools/config_sweep.py --config E [--out f.jsonl]

C: h=7168, moe_intermediate=2048, 256 routed experts top-8 + a 2048-wide
   shared expert, fp8 e4m3 experts (per-channel weight scales, per-row
   activation scales), the DeepSeek-V3 group-limited gate, 8192 tokens,
   every (TP, EP) layout of N GPUs with TP >= 2.  Reports the fused forward (one CUDA graph) in tokens/s and
   the expert FLOP rate.
E: the Qwen3-30B-A3B-shaped bf16 layer (config B) with gate logits
   N(0,1) + log p_e, p_e ∝ rank^-s (s in 0, 0.8, 1.0, 1.2), at every
   (TP, EP) layout of N GPUs.  Per s: measured latency per layout, the
   measured host skew kappa = max/mean slots per expert host, and the
   selector's pick -- select_strategy(..., expert_load=<measured counts>) on
   the box's calibrated links (paper_2601_08800_b200.calibration.measure) --
   next to the measured-best layout.
CUDA events on the launching stream, max over ranks, L2 flushed per step.
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
from paper_2601_08800_b200 import FP8SwiGLUExperts, SwiGLUExperts  # noqa: E402
from paper_2601_08800_b200.layer import MoELayer  # noqa: E402
from paper_2601_08800_b200.plan import GateSpec  # noqa: E402
from paper_2601_08800_b200.skew import host_skew, zipf_logits  # noqa: E402


def timed(run, layer, iters, flush):
    stream = torch.cuda.current_stream()
    for _ in range(3):
        run()
    ev = []
    for _ in range(iters):
        flush.fill_(1)
        layer.plan.barrier()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        run()
        b.record(stream)
        ev.append((a, b))
    torch.cuda.synchronize()
    t = torch.tensor([sum(a.elapsed_time(b) for a, b in ev) / iters], device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def layouts(world, min_tp=1, inter=None):
    """(n, m) of every TP degree the expert shapes allow (I/m % 128 == 0)."""
    return [(world // m, m) for m in (1, 2, 4, 8)
            if world % m == 0 and m >= min_tp and (inter is None or (inter // m) % 128 == 0)]


def config_c(args, rank, world, flush):
    H, I, E, K, IS = 7168, 2048, 256, 8, 2048
    out = []
    ex = FP8SwiGLUExperts.random(E, H, I, shared_inter=IS, seed=0)
    for n, m in layouts(world, min_tp=2 if world > 1 else 1, inter=I):
        T = args.tokens // n
        g = rank // m
        gen = torch.Generator(device="cuda").manual_seed(100 + g)
        x = torch.randn(T, H, device="cuda", generator=gen).to(torch.bfloat16)
        logits = torch.randn(T, E, device="cuda", generator=gen)
        wire = "token" if world > 1 else "slot"
        # DeepSeek-V3 gate: sigmoid scores + correction bias, 8 groups keep 4,
        # routed scaling 2.5 (transformers deepseek_v3 configuration)
        bias = 0.05 * torch.randn(E, generator=torch.Generator().manual_seed(5))
        layer = MoELayer(n, m, T, H, E, K, I, ex, rank=rank, wire=wire,
                         gate=GateSpec.deepseek_v3(bias))
        run = layer.capture(x, logits)
        ms = timed(run, layer, args.iters, flush)
        cnt = torch.bincount(layer.plan.rank_views(rank)["ids"].reshape(-1).long(), minlength=E)
        if m > 1:  # TP ranks of a group route the same tokens: count each group once
            cnt = cnt * (rank % m == 0)
        dist.all_reduce(cnt)
        slots = int(cnt.sum())
        # per-GPU expert flops (routed GEMM1+GEMM2 on the TP shard + shared expert)
        per_gpu = max(int(cnt[d * E // n:(d + 1) * E // n].sum()) for d in range(n))
        flops = 6 * per_gpu * H * I // m + 6 * T * H * IS // m
        res = {"config": "C", "n_gpus": world, "layout": f"TP{m}xEP{n}", "wire": wire,
               "global_tokens": args.tokens, "hidden": H, "moe_intermediate": I, "experts": E,
               "top_k": K, "shared_inter": IS, "dtype": "fp8 e4m3 experts, bf16 tokens",
               "gate": "DeepSeek-V3 group-limited (8 groups, top-4, scaling 2.5)",
               "ms_per_step": ms, "tokens_per_s": args.tokens / (ms / 1e3),
               "expert_tflops_per_gpu_incl_comm": flops / (ms / 1e3) / 1e12,
               "slots": slots}
        out.append(res)
        if rank == 0:
            print(json.dumps(res), flush=True)
        del run
        layer.close()
    return out


def config_e(args, rank, world, flush):
    from paper_2601_08800_b200.analyzer import calibrate, select_strategy
    from paper_2601_08800_b200.calibration import b200_cluster, measure
    from paper_2601_08800_b200.config import ModelHyperparams, WorkloadSpec
    from paper_2601_08800_b200.layer_model import select_layout
    from paper_2601_08800_b200.strategy import format_strategy

    H, I, E, K = 2048, 768, 128, 8
    ex = SwiGLUExperts.random(E, H, I, seed=0)
    obs = measure(sizes=(1 << 20, 1 << 24, 1 << 26), gemm=True)
    cal = calibrate(obs, ar_literal=False)
    model = ModelHyperparams(hidden_dim=H, num_layers=48, top_k=K, num_routed_experts=E,
                             num_shared_experts=0, psi_attn=1.5e9, psi_moe=2.9e10,
                             psi_active=3.3e9)
    wl = WorkloadSpec(1, args.tokens, args.tokens, 1, 1.0)
    out = []
    for s in (0.0, 0.8, 1.0, 1.2):
        res = {"config": "E", "zipf_s": s, "n_gpus": world, "global_tokens": args.tokens,
               "layouts": {}}
        counts = None
        for n, m in layouts(world, inter=I):
            T = args.tokens // n
            g = rank // m
            gen = torch.Generator(device="cuda").manual_seed(100 + g)
            x = torch.randn(T, H, device="cuda", generator=gen).to(torch.bfloat16)
            logits = zipf_logits(T, E, s, seed=1, device="cuda", generator=gen)
            w13, w2 = ex.rank_shard(n, m, rank)
            wire = "token" if world > 1 else "slot"
            layer = MoELayer(n, m, T, H, E, K, I, w13=w13, w2=w2, rank=rank, wire=wire)
            run = layer.capture(x, logits)
            ms = timed(run, layer, args.iters, flush)
            ids = torch.topk(logits, K, dim=1).indices.reshape(-1)
            c = torch.bincount(ids, minlength=E)
            if m > 1:  # TP ranks hold the same tokens: count each group once
                c = c * (rank % m == 0)
            dist.all_reduce(c)
            c = c.double().cpu().numpy()
            counts = c
            res["layouts"][f"TP{m}xEP{n}"] = {"ms_per_step": ms,
                                               "tokens_per_s": args.tokens / (ms / 1e3),
                                               "host_skew": host_skew(c, n), "wire": wire}
            del run
            layer.close()
            del w13, w2
        best_meas = min(res["layouts"], key=lambda k: res["layouts"][k]["ms_per_step"])
        # the fused-layer cost model on the EP-only layout's global routing
        # (regenerated group by group exactly as that run drew it)
        n_ep = world
        T_ep = args.tokens // n_ep
        ids_all = []
        for g in range(n_ep):
            gen = torch.Generator(device="cuda").manual_seed(100 + g)
            torch.randn(T_ep, H, device="cuda", generator=gen)
            lg_g = zipf_logits(T_ep, E, s, seed=1, device="cuda", generator=gen)
            ids_all.append(torch.topk(lg_g, K, dim=1).indices.cpu().numpy())
        ranked_fused = select_layout(np.concatenate(ids_all), world, E, H, I)
        res["fused_model_pick"] = ranked_fused[0]["layout"]
        res["fused_model_ms"] = {r["layout"]: r["seconds"] * 1e3 for r in ranked_fused}
        cl = b200_cluster(cal, 1, world)
        ranked = select_strategy(model, cl, wl, cal, expert_load=counts)
        moe = {}
        for e in ranked.entries:
            st = e.strategy
            if st.d_pp != 1:
                continue
            key = f"TP{st.moe_tp}xEP{st.moe_ep}"
            if key in res["layouts"] and key not in moe:
                moe[key] = e.estimate.ttft
        pick = min(moe, key=moe.get) if moe else None
        res.update({"measured_best": best_meas, "selector_pick": pick,
                    "selector_ttft_s": moe, "selector_best_overall": format_strategy(ranked.best.strategy),
                    "calibration": {"beta_GBps": cal.intra_beta / 1e9, "alpha_s": cal.intra_alpha,
                                    "compute_s_per_mac": cal.compute_coeff}})
        out.append(res)
        if rank == 0:
            print(json.dumps(res), flush=True)
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", choices=["C", "E"], required=True)
    ap.add_argument("--tokens", type=int, default=8192)
    ap.add_argument("--iters", type=int, default=20)
    ap.add_argument("--out", default=None)
    args = ap.parse_args()
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    rank, world = dist.get_rank(), dist.get_world_size()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    lines = (config_c if args.config == "C" else config_e)(args, rank, world, flush)
    if rank == 0 and args.out:
        Path(args.out).write_text("".join(json.dumps(r) + "\n" for r in lines))
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
