"""Copy-engine peer bandwidth vs the SM-issued peer stores the layer uses.

    python tools/ce_probe.py [--mb 32]

One process, every visible GPU: each GPU copies --mb MB to every peer with
cudaMemcpyPeerAsync (torch .copy_ across devices, one stream per source
GPU), all copies at once, the all-to-all pattern of the dispatch.  Prints
per-GPU egress GB/s; compare with the layer's same-run `mx_nvlink_probe`
(SM stores through the IPC heaps, 585 GB/s at 2 GPUs, 640-651 at 4).
"""
import argparse
import json
import time

import torch


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--mb", type=int, default=32)
    ap.add_argument("--iters", type=int, default=20)
    a = ap.parse_args()
    n = torch.cuda.device_count()
    nbytes = a.mb << 20
    src = [torch.empty(nbytes, dtype=torch.uint8, device=f"cuda:{i}").fill_(i) for i in range(n)]
    dst = [[torch.empty(nbytes, dtype=torch.uint8, device=f"cuda:{j}") for _ in range(n)] for j in range(n)]
    streams = [torch.cuda.Stream(device=i) for i in range(n)]

    def once():
        for i in range(n):
            with torch.cuda.stream(streams[i]):
                for d in range(1, n):
                    j = (i + d) % n
                    dst[j][i].copy_(src[i], non_blocking=True)

    for _ in range(3):
        once()
    for i in range(n):
        torch.cuda.synchronize(i)
    t0 = time.perf_counter()
    for _ in range(a.iters):
        once()
    for i in range(n):
        torch.cuda.synchronize(i)
    dt = (time.perf_counter() - t0) / a.iters
    per_gpu = nbytes * (n - 1) / dt / 1e9
    print(json.dumps({"gpus": n, "mb_per_peer": a.mb, "egress_gb_s_per_gpu": round(per_gpu, 1),
                      "ms_per_round": round(dt * 1e3, 3)}))


if __name__ == "__main__":
    main()
