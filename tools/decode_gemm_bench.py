"""Decode-regime grouped GEMM microbenchmark: weight streaming.

    python tools/decode_gemm_bench.py [--G 64] [--active 8] [--rows 2] [--N 1536] [--K 2048] [--swiglu]

One rank's expert set (G experts' weights resident, 2*I x h for GEMM1 or
h x I for GEMM2), of which --active experts hold --rows rows each, a
different random active set every launch (R sets cycled, weights of the
active set therefore cold in L2 as in a real decode step whose other layers
evict them).  Reports µs per launch and the weight bytes streamed per
second (the decode roofline: every active expert's full weight matrix is
read once).
"""
import argparse
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2601_08800_b200 import _native as N  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--G", type=int, default=64)
    ap.add_argument("--active", type=int, default=8)
    ap.add_argument("--rows", type=int, default=2)
    ap.add_argument("--N", type=int, default=1536)
    ap.add_argument("--K", type=int, default=2048)
    ap.add_argument("--swiglu", action="store_true")
    ap.add_argument("--sets", type=int, default=16)
    ap.add_argument("--cap", type=int, default=0, help="A/D rows allocated (default max(rows, 128))")
    ap.add_argument("--iters", type=int, default=64)
    ap.add_argument("--trace", action="store_true",
                    help="per-CTA phase timeline of one more launch (MX_GEMM_TRACE)")
    a = ap.parse_args()
    if a.trace:
        import os
        os.environ["MX_GEMM_TRACE"] = "1"
    gen = torch.Generator().manual_seed(0)
    M = a.active * a.rows
    cap = max(M, a.cap or 128)
    A = torch.randn(cap, a.K, device="cuda").to(torch.bfloat16)
    B = (torch.randn(a.G, a.N, a.K, device="cuda") * 0.02).to(torch.bfloat16)
    D = torch.empty(cap, a.N // 2 if a.swiglu else a.N, device="cuda", dtype=torch.bfloat16)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    sets = []
    for _ in range(a.sets):
        act = torch.randperm(a.G, generator=gen)[:a.active].sort().values
        cnts = torch.zeros(a.G, dtype=torch.int32)
        cnts[act] = a.rows
        offs = torch.zeros(a.G, dtype=torch.int32)
        offs[1:] = torch.cumsum(cnts, 0)[:-1]
        sets.append((offs.cuda(), cnts.cuda()))
    s = torch.cuda.current_stream().cuda_stream

    def run(i):
        od, cd = sets[i % a.sets]
        N.call("mx_grouped_gemm", A.data_ptr(), B.data_ptr(), D.data_ptr(), N.MX_BF16,
               od.data_ptr(), cd.data_ptr(), a.G, cap, a.N, a.K, int(a.swiglu), s)

    for i in range(4):
        run(i)
    torch.cuda.synchronize()
    ts = []
    for i in range(a.iters):
        flush.fill_(i & 255)  # evict the previous set's weights from L2
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        run(i)
        e1.record()
        ts.append((e0, e1))
    torch.cuda.synchronize()
    us = sorted(e0.elapsed_time(e1) * 1e3 for e0, e1 in ts)
    med = us[len(us) // 2]
    wbytes = a.active * a.N * a.K * 2
    print(f"G={a.G} active={a.active} rows={a.rows} N={a.N} K={a.K} swiglu={a.swiglu}: "
          f"median {med:7.2f} us (min {us[0]:.2f})  weights {wbytes / 1e6:.1f} MB -> "
          f"{wbytes / med / 1e3:7.1f} GB/s")
    if a.trace:
        import ctypes
        import numpy as np
        lib = N.load()
        buf = np.zeros((1024, 16), dtype=np.uint64)
        lib.mx_debug_gemm_trace(buf.ctypes.data_as(ctypes.c_void_p), 1024)  # reset
        flush.fill_(7)
        run(0)
        torch.cuda.synchronize()
        lib.mx_debug_gemm_trace(buf.ctypes.data_as(ctypes.c_void_p), 1024)
        used = buf[:, 0] > 0
        t = buf[used].astype(np.int64)
        t0 = t[:, 0].min()
        work = t[:, 4] > 0
        names = ["entry", "setup", "-", "mma_issued", "epilogue_done", "exit"]
        rel = (t[:, :6] - t[:, :1]) / 1.9e3  # SM cycles -> ~us, per CTA from its entry
        print(f"  trace: {int(used.sum())} CTAs, {int(work.sum())} with tiles; us from first entry "
              "(median / max over CTAs with tiles):")
        for i, nme in enumerate(names):
            if nme == "-":
                continue
            col = rel[work, i]
            print(f"    {nme:14s} {np.median(col):7.2f} {col.max():7.2f}")


if __name__ == "__main__":
    main()
