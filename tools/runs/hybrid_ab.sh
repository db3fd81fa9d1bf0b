#!/bin/bash
# hybrid (pair over full 256-row blocks + single over tails) vs single-CTA grouped GEMM
for r in 1 2; do
for H in 0 1; do
  echo "== MX_GEMM_HYBRID=$H"
  for J in 0 56; do
    MX_GEMM_HYBRID=$H timeout 120 python tools/gemm_bench.py --G 128 --rows 512 --jitter $J --N 1536 --K 2048 --swiglu --iters 20
    MX_GEMM_HYBRID=$H timeout 120 python tools/gemm_bench.py --G 128 --rows 512 --jitter $J --N 2048 --K 768 --iters 20
  done
  MX_GEMM_HYBRID=$H timeout 120 python tools/gemm_bench.py --G 64 --rows 512 --jitter 56 --N 768 --K 2048 --swiglu --iters 20
  MX_GEMM_HYBRID=$H timeout 120 python tools/gemm_bench.py --G 64 --rows 512 --jitter 56 --N 2048 --K 384 --iters 20
done
done
MX_GEMM_HYBRID=1 timeout 900 python -m pytest tests -m gpu -x -q -k "gemm or config or swiglu or parity" 2>&1 | tail -2
MX_GEMM_HYBRID=1 timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/hy_n1.json 2> gpurun_out/hy_n1.err; echo "bench hybrid rc=$?"
python tools/summarize_line.py gpurun_out/hy_n1.json | cut -c1-200
