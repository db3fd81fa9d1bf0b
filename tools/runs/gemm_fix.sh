#!/bin/bash
bash tools/runs/gemm_trace.sh
timeout 120 python tools/gemm_bench.py --G 128 --rows 512 --jitter 56 --N 1536 --K 2048 --swiglu --iters 20
timeout 120 python tools/gemm_bench.py --G 128 --rows 512 --jitter 56 --N 2048 --K 768 --iters 20
MX_GEMM_PAIR=2 timeout 120 python tools/gemm_bench.py --G 1 --rows 8192 --N 4096 --K 4096 --iters 20
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
