"""Measure the B200 box and recalibrate the selector (north star item 4).

Produces ``ProfilingObservation`` rows (an:32-51, CSV an:54-73) from
collectives timed on the GPUs -- NCCL reduce-scatter / all-gather /
all-reduce / all-to-all and a peer copy over NVLink -- plus the grouped GEMM
(``MoE_compute``: multiply-accumulates, the unit of the compute law cm:94),
then fits them with :func:`analyzer.calibrate`.  On one NVSwitch box the
"intra" and "inter" link classes of the two-tier model are the same fabric,
so every collective row is recorded under both scopes; the fit then gives
``intra ~= inter`` (``validate_bundle`` accepts equality, cfg:248-252).

    torchrun --nproc-per-node N -m paper_2601_08800_b200.calibration \
        --out profiles/b200_links.csv

:func:`b200_cluster` turns a fit into the ``ClusterConfig`` of an
``n_node x n_proc`` layout of the box for :func:`analyzer.select_strategy`;
the winner's ``(moe_tp, moe_ep)`` is the ``(tp, n_group)`` of ``MoELayer``.
"""
from __future__ import annotations

import argparse
import os

from .analyzer import ProfilingObservation, calibrate, save_observations
from .config import ClusterConfig

B200_HBM_BYTES = 180e9
B200_BF16_MACS = 2.25e15 / 2     # nominal dense bf16, MAC/s


def b200_cluster(calib, n_node: int, n_proc: int, mem_per_device=B200_HBM_BYTES,
                 compute_rate=None) -> ClusterConfig:
    """ClusterConfig of one B200 box split into n_node groups of n_proc."""
    rate = compute_rate or (1.0 / calib.compute_coeff if calib.compute_coeff else B200_BF16_MACS)
    return ClusterConfig(n_node, n_proc,
                         calib.intra_alpha or 0.0, calib.intra_beta,
                         calib.inter_alpha or 0.0, calib.inter_beta,
                         mem_per_device, rate)


def _time(fn, iters=20, warmup=3):
    import torch
    import torch.distributed as dist
    for _ in range(warmup):
        fn()
    torch.cuda.synchronize()
    dist.barrier()
    a = torch.cuda.Event(enable_timing=True)
    b = torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(iters):
        fn()
    b.record()
    torch.cuda.synchronize()
    t = torch.tensor([a.elapsed_time(b) / iters / 1e3], device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def measure(sizes=(1 << 16, 1 << 20, 1 << 24, 1 << 26), gemm=True):
    """Collective + GEMM observations on the current process group."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size()
    obs = []

    def add(kind, size, deg, sec):
        for scope in ("intra", "inter"):
            obs.append(ProfilingObservation(kind, float(size), deg, scope, sec))

    for size in sizes:
        n = size // 2  # bf16 elements
        x = torch.randn(n, device="cuda").to(torch.bfloat16)
        out = torch.empty(n // world, device="cuda", dtype=torch.bfloat16)
        full = torch.empty(n, device="cuda", dtype=torch.bfloat16)
        add("RS", size, world, _time(lambda: dist.reduce_scatter_tensor(out, x)))
        add("AG", size, world, _time(lambda: dist.all_gather_into_tensor(full, out)))
        add("AR", size, world, _time(lambda: dist.all_reduce(x)))
        y = torch.empty_like(x)
        add("A2A", size, world, _time(lambda: dist.all_to_all_single(y, x)))
        if world >= 2:
            rank = dist.get_rank()
            peer = rank ^ 1
            buf = torch.empty_like(x)

            def p2p():
                ops = [dist.P2POp(dist.isend, x, peer), dist.P2POp(dist.irecv, buf, peer)]
                for r in dist.batch_isend_irecv(ops):
                    r.wait()
            add("P2P", size, 2, _time(p2p))
    if gemm:
        from . import _native as N
        for M in (1024, 4096, 16384):
            K, Nn, G = 2048, 1536, 8
            A = torch.randn(M, K, device="cuda").to(torch.bfloat16)
            B = torch.randn(G, Nn, K, device="cuda").to(torch.bfloat16)
            D = torch.empty(M, Nn, device="cuda", dtype=torch.bfloat16)
            cnt = torch.full((G,), M // G, dtype=torch.int32, device="cuda")
            off = torch.arange(G, dtype=torch.int32, device="cuda") * (M // G)
            s = torch.cuda.current_stream().cuda_stream
            sec = _time(lambda: N.call("mx_grouped_gemm", A.data_ptr(), B.data_ptr(),
                                       D.data_ptr(), N.MX_BF16, off.data_ptr(),
                                       cnt.data_ptr(), G, M, Nn, K, 0, s))
            obs.append(ProfilingObservation("MoE_compute", float(M) * Nn * K, 1, "intra", sec))
    return obs


def main():
    import torch
    import torch.distributed as dist
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default="profiles/b200_links.csv")
    args = ap.parse_args()
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    obs = measure()
    if dist.get_rank() == 0:
        save_observations(obs, args.out)
        cal = calibrate(obs, ar_literal=False)
        print(f"calibrated on {dist.get_world_size()} x B200: intra alpha {cal.intra_alpha:.3e} s, "
              f"beta {cal.intra_beta / 1e9:.1f} GB/s; compute {cal.compute_coeff:.3e} s/MAC")
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
