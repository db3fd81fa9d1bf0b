"""NVLink peer store / load ceiling for the token wire's access patterns.

Diagnostic, not product code: one process drives every visible GPU with
peer access enabled and runs ``tools/nvlink_push.cu`` (built here with nvcc)
on all of them at once -- each GPU moves 4 KB rows to / from its peers with
16-byte vector accesses, the pattern of the dispatch (broadcast to a host's
TP ranks), the pre-reduction push and the combine's y push.  Reports the
per-GPU NVLink GB/s (max-over-GPUs time) for grid sizes and bytes in flight,
so the phases' roofline fractions can be read against what SM-issued peer
accesses reach, not only the copy-engine figure (770 GB/s).

    python tools/nvlink_bench.py --out gpurun_out/nvlink.jsonl
"""
from __future__ import annotations

import argparse
import ctypes
import json
import os
import subprocess
import sys

import torch

HERE = os.path.dirname(os.path.abspath(__file__))
ROW = 4096
MODES = {"push": 0, "pull": 1, "bcast": 2, "local": 3, "mixed": 4, "split": 5, "reduce": 6, "scatter": 7}


def build(out_dir: str) -> ctypes.CDLL:
    so = os.path.join(out_dir, "nvlink_push.so")
    subprocess.run(["nvcc", "-O3", "-gencode", "arch=compute_100a,code=sm_100a", "-shared",
                    "-Xcompiler", "-fPIC", os.path.join(HERE, "nvlink_push.cu"), "-o", so],
                   check=True)
    return build_load(out_dir)


def main_ipc(a) -> int:
    """One process per GPU (torchrun): peer pointers are the layer's own
    symmetric heaps opened through CUDA IPC, aligned by its device barrier --
    the mapping and launch setting of the fused layer itself."""
    import torch.distributed as dist
    sys.path.insert(0, os.path.dirname(HERE))
    from paper_2601_08800_b200 import _native as N
    from paper_2601_08800_b200.plan import LayerPlan

    rank, W = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", rank)))
    dist.init_process_group("nccl")
    plan = LayerPlan(W, 1, 8192, 2048, 128, 8, dtype=torch.bfloat16, expert_kind="swiglu",
                     inter=768, emulate=False, rank=rank, wire="token")
    lib = build(os.path.dirname(a.out) or ".") if rank == 0 else None
    dist.barrier()
    if rank:
        lib = build_load(os.path.dirname(a.out) or ".")
    base = []
    for r in range(W):
        b, n = ctypes.c_void_p(), ctypes.c_size_t()
        N.check(N.load().mx_comm_heap(plan._comm, r, ctypes.byref(b), ctypes.byref(n)), "heap")
        base.append((b.value, n.value))
    nbytes = a.mib * (1 << 20)
    rows = nbytes // ROW
    need = nbytes * (1 + W)
    if base[rank][1] < need:
        raise SystemExit(f"heap {base[rank][1]} < {need}: lower --mib")
    src = base[rank][0]
    loc = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
    s = torch.cuda.current_stream()
    peers = [q for q in range(W) if q != rank]
    out = []
    for mode in [m for m in a.modes.split(",") if m in ("push", "bcast", "scatter", "reduce", "mixed")]:
        for blocks in [int(b) for b in a.blocks.split(",")]:
            pp = [base[q][0] + nbytes * (1 + rank) for q in peers]
            arr = (ctypes.c_void_p * 8)(*pp, *([pp[0]] * (8 - len(pp))))
            ts = []
            for it in range(4):
                plan.barrier(stream=s)
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(s)
                for _ in range(a.reps):
                    rc = lib.nb_launch(torch.cuda.current_device(), MODES[mode], arr, len(peers),
                                       ctypes.c_void_p(src), ctypes.c_void_p(loc.data_ptr()),
                                       rows, blocks, 0, ctypes.c_void_p(s.cuda_stream))
                    if rc:
                        raise RuntimeError(f"launch rc={rc}")
                e1.record(s)
                s.synchronize()
                t = torch.tensor([e0.elapsed_time(e1) / 1e3 / a.reps], device="cuda")
                dist.all_reduce(t, op=dist.ReduceOp.MAX)
                if it:
                    ts.append(t.item())
            t = min(ts)
            moved = nbytes * (len(peers) if mode == "bcast" else 1)
            r = {"ipc": True, "mode": mode, "peers": len(peers), "gpus": W, "blocks": blocks,
                 "bytes_per_gpu": moved, "us": t * 1e6, "gbs": moved / t / 1e9}
            out.append(r)
            if rank == 0:
                print(json.dumps(r), flush=True)
    if rank == 0:
        with open(a.out, "w") as f:
            f.writelines(json.dumps(r) + "\n" for r in out)
    plan.close()
    dist.destroy_process_group()
    return 0


def build_load(out_dir: str) -> ctypes.CDLL:
    lib = ctypes.CDLL(os.path.join(out_dir, "nvlink_push.so"))
    lib.nb_launch.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.POINTER(ctypes.c_void_p),
                              ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_longlong,
                              ctypes.c_int, ctypes.c_int, ctypes.c_void_p]
    return lib


def main() -> int:
    ap = argparse.ArgumentParser()
    ap.add_argument("--mib", type=int, default=256, help="MiB each GPU sends per launch")
    ap.add_argument("--reps", type=int, default=3, help="back-to-back launches per timing")
    ap.add_argument("--out", default="gpurun_out/nvlink.jsonl")
    ap.add_argument("--modes", default="local,push,pull,bcast,mixed,split")
    ap.add_argument("--blocks", default="148,296,592,1184,2368")
    a = ap.parse_args()
    if int(os.environ.get("WORLD_SIZE", "1")) > 1:
        return main_ipc(a)
    P = torch.cuda.device_count()
    if P < 2:
        print("needs >= 2 GPUs", file=sys.stderr)
        return 1
    os.makedirs(os.path.dirname(a.out) or ".", exist_ok=True)
    lib = build(os.path.dirname(a.out) or ".")
    if lib.nb_enable_peers(P):
        print("peer access unavailable", file=sys.stderr)
        return 1
    rows = a.mib * (1 << 20) // ROW
    nbytes = rows * ROW
    src = [torch.full((nbytes,), d + 1, dtype=torch.uint8, device=f"cuda:{d}") for d in range(P)]
    loc = [torch.empty(nbytes, dtype=torch.uint8, device=f"cuda:{d}") for d in range(P)]
    # inbox[d]: one region per sender, sized for the broadcast (every row)
    inbox = [torch.empty(P * nbytes, dtype=torch.uint8, device=f"cuda:{d}") for d in range(P)]
    streams = [torch.cuda.Stream(device=d) for d in range(P)]

    def peers_of(d, which):
        if which == "one":
            return [d ^ 1]
        return [q for q in range(P) if q != d]

    def run(mode, which, blocks, half):
        ptrs = []
        for d in range(P):
            pe = peers_of(d, which)
            if mode == "pull":
                pp = [src[q].data_ptr() for q in pe]
            elif mode == "local":
                pp = [loc[d].data_ptr()]
            else:
                pp = [inbox[q].data_ptr() + d * nbytes for q in pe]
            ptrs.append((ctypes.c_void_p * 8)(*pp, *([pp[0]] * (8 - len(pp)))))
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
              for _ in range(P)]
        times = []
        for it in range(3):
            for d in range(P):
                torch.cuda.synchronize(d)
            for d in range(P):
                with torch.cuda.device(d):
                    ev[d][0].record(streams[d])
            for _ in range(a.reps):
                for d in range(P):
                    rc = lib.nb_launch(d, MODES[mode], ptrs[d], len(peers_of(d, which)),
                                       ctypes.c_void_p(src[d].data_ptr()),
                                       ctypes.c_void_p(loc[d].data_ptr()), rows, blocks, half,
                                       ctypes.c_void_p(streams[d].cuda_stream))
                    if rc:
                        raise RuntimeError(f"launch failed rc={rc}")
            for d in range(P):
                with torch.cuda.device(d):
                    ev[d][1].record(streams[d])
            for d in range(P):
                torch.cuda.synchronize(d)
            t = max(ev[d][0].elapsed_time(ev[d][1]) for d in range(P)) / 1e3 / a.reps
            if it:
                times.append(t)
        t = min(times)
        npe = len(peers_of(0, which))
        moved = nbytes * (npe if mode == "bcast" else 1)   # NVLink bytes per GPU
        if mode == "local":
            moved = 2 * nbytes                              # HBM read + write
        if mode in ("mixed", "split", "reduce"):            # NVLink bytes; HBM 5x / 4x
            moved = nbytes
        return {"mode": mode, "peers": npe, "gpus": P, "blocks": blocks, "half": half,
                "bytes_per_gpu": moved, "us": t * 1e6, "gbs": moved / t / 1e9}

    with open(a.out, "w") as f:
        for mode in a.modes.split(","):
            for which in (("all",) if mode == "local" else ("one", "all")):
                for blocks in [int(b) for b in a.blocks.split(",")]:
                    for half in (0, 1):
                        r = run(mode, which, blocks, half)
                        print(json.dumps(r), flush=True)
                        f.write(json.dumps(r) + "\n")
    return 0


if __name__ == "__main__":
    sys.exit(main())
