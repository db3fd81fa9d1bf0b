"""Multi-GPU parity of the SPMD layer (one rank per GPU, NVLink peer heaps).

    torchrun --nproc-per-node N --master-addr 127.0.0.1 tests/spmd_check.py [--tp M]

Checks, for the n x m cluster of the world size:
  * f64 affine experts, explicit RouterSpec routing: fused output bit-exact
    with the oracle's restatement of run_moe_block (sim:565-592);
  * bf16 SwiGLU experts with the fused gate: within 2e-2 of the oracle;
  * the NCCL AR+A2A baseline (sim:598-680) agrees with the oracle;
  * repeated forwards are deterministic (device barrier epochs advance).
Exit code 0 on success.
"""
import argparse
import os
import sys
from pathlib import Path

import numpy as np
import torch
import torch.distributed as dist

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

from oracle import mixserve_oracle as orc  # noqa: E402
from paper_2601_08800_b200 import RouterSpec, SwiGLUExperts  # noqa: E402
from paper_2601_08800_b200.layer import MoELayer, layout_for  # noqa: E402


SAME_DEVICE = False  # every rank on cuda:0 (gloo bootstrap, CUDA IPC on one device)


def fwd(layer, x, logits=None, ids=None, weights=None):
    """One layer forward: the fused forward with device barriers, or -- ranks
    sharing one GPU -- the same phases with non-spinning barrier halves and a
    host barrier between them (forward_stepped): kernels of different
    processes on one GPU are not guaranteed to run side by side, so no rank
    may spin on another's flag there."""
    if SAME_DEVICE:
        return layer.forward_stepped(x, logits, ids=ids, weights=weights,
                                     host_barrier=dist.barrier)
    return layer.forward(x, logits, ids=ids, weights=weights)


def gather_rows(y, world):
    """All ranks' [T, h] outputs (device tensors under NCCL, host under gloo)."""
    if SAME_DEVICE:
        y = y.cpu()
    out = [torch.empty_like(y) for _ in range(world)]
    dist.all_gather(out, y.contiguous())
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--tp", type=int, default=None)
    ap.add_argument("--bench-shape", action="store_true",
                    help="also run config B at bench.py's dimensions (8192 tokens, h=2048, "
                         "I=768, 128 experts top-8, token wire) in this layout and check a "
                         "token sample against the CPU oracle")
    ap.add_argument("--same-device", action="store_true",
                    help="every rank on cuda:0 as a separate process: gloo for the "
                         "bootstrap, the layer's CUDA IPC heaps, device barriers and "
                         "graph replay exercised on one GPU (no NCCL arm)")
    args = ap.parse_args()
    global SAME_DEVICE
    SAME_DEVICE = args.same_device
    local = 0 if SAME_DEVICE else int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if SAME_DEVICE:
        dist.init_process_group("gloo")
    else:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    rank, world = dist.get_rank(), dist.get_world_size()
    n, m = layout_for(world, args.tp)
    g, t = divmod(rank, m)
    failures = []

    # ---------------- f64 affine, explicit routing: bit-exact
    T, h, E, k = 96, 72, 16, 4
    rng = np.random.default_rng(7)
    x = rng.standard_normal((n * T, h))
    router = RouterSpec.random(n * T, E, k, seed=8)
    ids, w = router.arrays()
    scales = np.arange(1, E + 1, dtype=np.float64)
    biases = np.arange(E, dtype=np.float64)
    layer = MoELayer(n, m, T, h, E, k, 0, rank=rank, dtype=torch.float64,
                     expert_kind="affine", scales=scales, biases=biases)
    xs = torch.as_tensor(x[g * T:(g + 1) * T], device="cuda")
    ids_d = torch.as_tensor(ids[g * T:(g + 1) * T], device="cuda").contiguous()
    w_d = torch.as_tensor(w[g * T:(g + 1) * T], device="cuda").contiguous()
    y1 = fwd(layer, xs, ids=ids_d, weights=w_d).clone()
    y2 = fwd(layer, xs, ids=ids_d, weights=w_d).clone()
    if not torch.equal(y1, y2):
        failures.append("f64 affine: repeated forward differs")
    ys = gather_rows(y1, world)
    if rank == 0:
        y_ref, _ = orc.run_fused_affine(n, m, x, ids, w, E, scales, biases)
        for r in range(world):
            gg = r // m
            got = ys[r].cpu().numpy()
            if not np.array_equal(got, y_ref[gg * T:(gg + 1) * T]):
                err = np.abs(got - y_ref[gg * T:(gg + 1) * T]).max()
                failures.append(f"f64 affine rank {r}: not bit-exact (max err {err:.3e})")
    layer.close()

    # ---------------- bf16 SwiGLU, fused gate
    T, h, E, k, I = 128, 256, 32, 4, 512
    ex = SwiGLUExperts.random(E, h, I, seed=3)
    gen = torch.Generator(device="cuda").manual_seed(11)
    x_all = torch.randn(n * T, h, device="cuda", generator=gen).to(torch.bfloat16)
    l_all = torch.randn(n * T, E, device="cuda", generator=gen)
    layer = MoELayer(n, m, T, h, E, k, I, experts=ex, rank=rank)
    xs, ls = x_all[g * T:(g + 1) * T].contiguous(), l_all[g * T:(g + 1) * T].contiguous()
    for _ in range(3):
        y = fwd(layer, xs, ls).clone()
    y_bl = None if SAME_DEVICE else layer.forward_baseline(xs, ls).clone()
    ys = gather_rows(y, world)
    ybs = None if y_bl is None else gather_rows(y_bl, world)
    layer.close()
    # wire TOKEN (dedup dispatch + pre-reduced combine), eager and graph replay
    layer = MoELayer(n, m, T, h, E, k, I, experts=ex, rank=rank, wire="token")
    y_tok = fwd(layer, xs, ls).clone()
    if not SAME_DEVICE:
        run = layer.capture(xs, ls)
        y_tok_g = run().clone()
        torch.cuda.synchronize()
        if not torch.equal(y_tok, y_tok_g):
            failures.append("wire token: graph replay differs from eager")
        # the opt-in overlapped forward (NVLink phases on a side stream under
        # the GEMMs, n > 1) computes every row exactly as the sequential one
        os.environ["MX_OVERLAP"] = "1"
        y_ovl = layer.forward(xs, ls).clone()
        run_ovl = layer.capture(xs, ls)
        y_ovl_g = run_ovl().clone()
        del os.environ["MX_OVERLAP"]
        torch.cuda.synchronize()
        if not (torch.equal(y_ovl, y_tok) and torch.equal(y_ovl_g, y_tok)):
            failures.append("wire token: overlapped and sequential forwards differ")
    elif not torch.equal(y_tok, fwd(layer, xs, ls)):
        failures.append("wire token: repeated stepped forward differs")
    # larger token-wire batch (>= 32 pairs per SM): the combine side as one
    # persistent kernel (opt-in k_reduce_combine) gives the bits of the
    # three separate launches, eager and in a graph
    if not SAME_DEVICE:
        Tb = 2560
        xb = torch.randn(n * Tb, h, device="cuda", generator=gen).to(torch.bfloat16)
        lb = torch.randn(n * Tb, E, device="cuda", generator=gen)
        xbs, lbs = xb[g * Tb:(g + 1) * Tb].contiguous(), lb[g * Tb:(g + 1) * Tb].contiguous()
        big = MoELayer(n, m, Tb, h, E, k, I, experts=ex, rank=rank, wire="token")
        os.environ["MX_FUSED_COMBINE"] = "1"
        yf = big.forward(xbs, lbs).clone()
        yfg = big.capture(xbs, lbs)().clone()
        del os.environ["MX_FUSED_COMBINE"]
        ys3 = big.forward(xbs, lbs).clone()
        torch.cuda.synchronize()
        if not (torch.equal(yf, ys3) and torch.equal(yfg, ys3)):
            failures.append("fused combine kernel differs from the separate launches")
        ybig = gather_rows(yf, world)
        big.close()
        if rank == 0:
            oexb = orc.SwiGLUOracle(ex.w_gate.float().cpu().numpy(), ex.w_up.float().cpu().numpy(),
                                    ex.w_down.float().cpu().numpy())
            idsb, wb = orc.router_topk(lb.cpu().numpy(), k)
            samp = np.arange(0, n * Tb, 7)
            y_refb = orc.moe_layer_swiglu(xb.float().cpu().numpy()[samp], idsb[samp], wb[samp], oexb)
            got = torch.cat([ybig[r * m] for r in range(n)]).float().cpu().numpy()[samp]
            eb = orc.verify_metric(got, y_refb)
            print(f"fused-combine batch ({Tb} tokens/group): err {eb:.3e}", flush=True)
            if eb > 2e-2:
                failures.append(f"fused combine: err {eb:.3e}")
    yts = gather_rows(y_tok, world)
    if rank == 0:
        oex = orc.SwiGLUOracle(ex.w_gate.float().cpu().numpy(), ex.w_up.float().cpu().numpy(),
                               ex.w_down.float().cpu().numpy())
        ids, w = orc.router_topk(l_all.cpu().numpy(), k)
        y_ref = orc.moe_layer_swiglu(x_all.float().cpu().numpy(), ids, w, oex)
        for r in range(world):
            gg = r // m
            ref = y_ref[gg * T:(gg + 1) * T]
            e1 = orc.verify_metric(ys[r].float().cpu().numpy(), ref)
            e2 = orc.verify_metric(ybs[r].float().cpu().numpy(), ref) if ybs else 0.0
            e3 = orc.verify_metric(yts[r].float().cpu().numpy(), ref)
            bl = f"{e2:.3e}" if ybs else "skipped (one device)"
            print(f"rank {r}: fused err {e1:.3e}, nccl-baseline err {bl}, "
                  f"token-wire err {e3:.3e}", flush=True)
            if e1 > 2e-2:
                failures.append(f"swiglu fused rank {r}: err {e1:.3e}")
            if e3 > 2e-2:
                failures.append(f"swiglu token wire rank {r}: err {e3:.3e}")
            if e2 > 2e-2:
                failures.append(f"swiglu baseline rank {r}: err {e2:.3e}")
    layer.close()

    # ---------------- fp8 experts + shared expert (config C path), both wires
    from paper_2601_08800_b200 import FP8SwiGLUExperts
    T, h, E, k, I, Is = 64, 512, 16, 4, 512, 512
    fex = FP8SwiGLUExperts.random(E, h, I, shared_inter=Is, seed=21)
    x8 = torch.randn(n * T, h, device="cuda", generator=gen).to(torch.bfloat16)
    l8 = torch.randn(n * T, E, device="cuda", generator=gen)
    xs8, ls8 = x8[g * T:(g + 1) * T].contiguous(), l8[g * T:(g + 1) * T].contiguous()
    outs = {}
    for wire in ("slot", "token"):
        layer = MoELayer(n, m, T, h, E, k, I, experts=fex, rank=rank, wire=wire)
        outs[wire] = gather_rows(fwd(layer, xs8, ls8).clone(), world)
        layer.close()
    if rank == 0:
        gate, up, down, shared = fex.oracle_arrays(n, m)
        ids, w = orc.router_topk(l8.cpu().numpy(), k)
        y_ref = orc.moe_layer_fp8(x8.float().cpu().numpy(), ids, w, gate, up, down, shared)
        for wire, ys8 in outs.items():
            for r in range(world):
                gg = r // m
                ref = y_ref[gg * T:(gg + 1) * T]
                got = ys8[r].double().cpu().numpy()
                fro = float(np.linalg.norm(got - ref) / np.linalg.norm(ref))
                mx = orc.verify_metric(got, ref)
                if fro > 1e-2 or mx > 5e-2:
                    failures.append(f"fp8 {wire} rank {r}: fro {fro:.3e} max {mx:.3e}")
        print(f"fp8 layer checked over slot/token wires", flush=True)

    # ---------------- config B at the bench's dimensions in this layout
    if args.bench_shape:
        Tg, hb, Eb, kb, Ib = 8192, 2048, 128, 8, 768
        Tb = Tg // n
        exb = SwiGLUExperts.random(Eb, hb, Ib, seed=0)
        w13, w2 = exb.rank_shard(n, m, rank)
        genb = torch.Generator(device="cuda").manual_seed(77)
        xb = torch.randn(Tg, hb, device="cuda", generator=genb).to(torch.bfloat16)
        lb = torch.randn(Tg, Eb, device="cuda", generator=genb)
        big = MoELayer(n, m, Tb, hb, Eb, kb, Ib, w13=w13, w2=w2, rank=rank, wire="token")
        yb = fwd(big, xb[g * Tb:(g + 1) * Tb].contiguous(), lb[g * Tb:(g + 1) * Tb].contiguous())
        ybs = gather_rows(yb.clone(), world)
        big.close()
        del w13, w2
        if rank == 0:
            oexb = orc.SwiGLUOracle(exb.w_gate.float().cpu().numpy(), exb.w_up.float().cpu().numpy(),
                                    exb.w_down.float().cpu().numpy())
            samp = np.sort(np.random.default_rng(3).choice(Tg, 512, replace=False))
            idsb, wb = orc.router_topk(lb.cpu().numpy()[samp], kb)
            y_refb = orc.moe_layer_swiglu(xb.float().cpu().numpy()[samp], idsb, wb, oexb)
            got = torch.cat([ybs[j * m] for j in range(n)]).float().cpu().numpy()[samp]
            eb = orc.verify_metric(got, y_refb)
            print(f"config B bench shape ({n}x{m}, 8192 tokens): err {eb:.3e} on 512 sampled tokens",
                  flush=True)
            if eb > 2e-2:
                failures.append(f"config B bench shape: err {eb:.3e}")
        del exb
        torch.cuda.empty_cache()

    # ---------------- decode regime at config B's dimensions: the weight-
    # streaming GEMMs (128-column tiles, early start), the phase kernels'
    # early PDL triggers and the column-split warp kernels, eager and (one
    # rank per GPU) graph replay, every token against the CPU oracle
    Hd, Ed, Kd, Id = 2048, 128, 8, 768
    if (Id // m) % 128:  # config B has no TP4 layout (I/4 = 192)
        Id = 1024
    exd = SwiGLUExperts.random(Ed, Hd, Id, seed=11)
    w13d, w2d = exd.rank_shard(n, m, rank)
    oexd = None
    if rank == 0:
        oexd = orc.SwiGLUOracle(exd.w_gate.float().cpu().numpy(), exd.w_up.float().cpu().numpy(),
                                exd.w_down.float().cpu().numpy())
    for Td in (1, 16):
        Tgd = Td * n
        gend = torch.Generator(device="cuda").manual_seed(500 + Td)
        xd = torch.randn(Tgd, Hd, device="cuda", generator=gend).to(torch.bfloat16)
        ld = torch.randn(Tgd, Ed, device="cuda", generator=gend)
        dec = MoELayer(n, m, Td, Hd, Ed, Kd, Id, w13=w13d, w2=w2d, rank=rank, wire="token")
        xs_d, ls_d = xd[g * Td:(g + 1) * Td].contiguous(), ld[g * Td:(g + 1) * Td].contiguous()
        yd = fwd(dec, xs_d, ls_d).clone()
        if not SAME_DEVICE:
            yd_g = dec.capture(xs_d, ls_d)().clone()
            torch.cuda.synchronize()
            if not torch.equal(yd, yd_g):
                failures.append(f"decode T={Td}: graph replay differs from eager")
        yds = gather_rows(yd, world)
        dec.close()
        if rank == 0:
            idsd, wd = orc.router_topk(ld.cpu().numpy(), Kd)
            y_refd = orc.moe_layer_swiglu(xd.float().cpu().numpy(), idsd, wd, oexd)
            got = torch.cat([yds[j * m] for j in range(n)]).float().cpu().numpy()
            ed = orc.verify_metric(got, y_refd)
            print(f"decode regime ({n}x{m}, {Tgd} tokens, config B dims): err {ed:.3e}", flush=True)
            if ed > 2e-2:
                failures.append(f"decode T_g={Tgd}: err {ed:.3e}")
    del exd, w13d, w2d, oexd
    torch.cuda.empty_cache()

    # ---------------- capacity below the routed rows: every rank raises
    from paper_2601_08800_b200 import CapacityError
    T, h, E, k, I = 64, 256, 16, 4, 512
    layer = MoELayer(n, m, T, h, E, k, I, experts=SwiGLUExperts.random(E, h, I, seed=5),
                     rank=rank, wire="token", capacity=T // 2)
    xc = torch.randn(T, h, device="cuda", generator=gen).to(torch.bfloat16)
    lc = torch.randn(T, E, device="cuda", generator=gen)
    try:
        fwd(layer, xc, lc)
        failures.append(f"rank {rank}: capacity {T // 2} overflow not raised")
    except CapacityError as e:
        if "routed slots, capacity" not in str(e):
            failures.append(f"rank {rank}: capacity message {e}")
    layer.close()

    flag = torch.tensor([len(failures)], device="cpu" if SAME_DEVICE else "cuda")
    dist.all_reduce(flag)
    if rank == 0:
        for f in failures:
            print("FAIL:", f, flush=True)
        print(f"spmd_check world={world} n={n} m={m}: "
              f"{'OK' if flag.item() == 0 else 'FAILED'}", flush=True)
    dist.barrier()
    dist.destroy_process_group()
    sys.exit(0 if flag.item() == 0 else 1)


if __name__ == "__main__":
    main()
