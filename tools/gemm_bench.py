"""Grouped-GEMM microbenchmark (one process per kernel mode).

    MX_GEMM_PAIR=0|1 python tools/gemm_bench.py --G 128 --rows 512 --N 1536 --K 2048 [--swiglu]

Groups of exactly --rows rows (or --jitter random sizes), bf16, CUDA events
over --iters launches after warm-up; reports TFLOP/s of useful work.
"""
import argparse
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2601_08800_b200 import _native as N  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--G", type=int, default=128)
    ap.add_argument("--rows", type=int, default=512)
    ap.add_argument("--jitter", type=int, default=0)
    ap.add_argument("--N", type=int, default=1536)
    ap.add_argument("--K", type=int, default=2048)
    ap.add_argument("--swiglu", action="store_true")
    ap.add_argument("--iters", type=int, default=20)
    ap.add_argument("--reps", type=int, default=1)
    ap.add_argument("--trace", action="store_true",
                    help="per-CTA timeline + wait cycles of one more launch (MX_GEMM_TRACE; wait "
                         "cycles need a -DMX_GEMM_WAITSTATS build via MIXSERVE_B200_LIB)")
    a = ap.parse_args()
    if a.trace:
        import os
        os.environ["MX_GEMM_TRACE"] = "1"
    gen = torch.Generator().manual_seed(0)
    cnts = torch.full((a.G,), a.rows, dtype=torch.int32)
    if a.jitter:
        cnts += torch.randint(-a.jitter, a.jitter + 1, (a.G,), generator=gen, dtype=torch.int32)
    offs = torch.zeros(a.G, dtype=torch.int32)
    offs[1:] = torch.cumsum(cnts, 0)[:-1]
    M = int(cnts.sum())
    A = torch.randn(M, a.K, device="cuda").to(torch.bfloat16)
    B = torch.randn(a.G, a.N, a.K, device="cuda").to(torch.bfloat16) * 0.02
    D = torch.empty(M, a.N // 2 if a.swiglu else a.N, device="cuda", dtype=torch.bfloat16)
    od, cd = offs.cuda(), cnts.cuda()
    s = torch.cuda.current_stream().cuda_stream
    run = lambda: N.call("mx_grouped_gemm", A.data_ptr(), B.data_ptr(), D.data_ptr(), N.MX_BF16,
                         od.data_ptr(), cd.data_ptr(), a.G, M, a.N, a.K, int(a.swiglu), s)
    for _ in range(3):
        run()
    torch.cuda.synchronize()
    for _ in range(a.reps - 1):
        run()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(a.iters):
        run()
    e1.record()
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) / a.iters * 1e3
    try:
        import subprocess
        clk = subprocess.run(["nvidia-smi", "--query-gpu=clocks.sm,power.draw,temperature.gpu",
                              "--format=csv,noheader"], capture_output=True, text=True).stdout.strip()
    except OSError:
        clk = "?"
    if a.trace:
        import ctypes
        import numpy as np
        lib = N.load()
        buf = np.zeros((1024, 16), dtype=np.uint64)
        lib.mx_debug_gemm_trace(buf.ctypes.data_as(ctypes.c_void_p), 1024)  # reset
        run()
        torch.cuda.synchronize()
        lib.mx_debug_gemm_trace(buf.ctypes.data_as(ctypes.c_void_p), 1024)
        t = buf[buf[:, 0] > 0].astype(np.int64)
        if len(t) == 0:
            print("  trace: no CTA recorded (the CTA-pair kernel is not instrumented)")
            t = None
    if a.trace and t is not None:
        mhz = np.median((t[:, 5] - t[:, 0]) / np.maximum(t[:, 9] - t[:, 8], 1) * 1e3)
        span = (t[:, 9] - t[:, 8]) / 1e3
        f = lambda col: f"{np.median(col):8.1f} {col.max():8.1f}"
        print(f"  trace ({len(t)} CTAs, SM clock {mhz:.0f} MHz; us, median / max): CTA span {f(span)}")
        t = t.astype(np.float64)
        t[:, [2, 6, 7]] *= 1.9e3 / mhz  # wait cycles -> us below via the /1.9e3
        print(f"    mma issuer waiting for stages   {f(t[:, 2] / 1.9e3)}")
        print(f"    mma issuer waiting for TMEM buf {f(t[:, 7] / 1.9e3)}")
        print(f"    producer waiting for free stage {f(t[:, 6] / 1.9e3)}")
    tf = 2.0 * M * a.N * a.K / (us * 1e-6) / 1e12
    print(f"G={a.G} rows={a.rows}+-{a.jitter} N={a.N} K={a.K} swiglu={a.swiglu}: {us:8.1f} us  {tf:7.1f} TFLOP/s  [{clk}]")


if __name__ == "__main__":
    main()
