#!/bin/bash
# CTA-pair vs single-CTA grouped GEMM after the SiLU epilogue fix
for P in 0 2; do
  echo "== MX_GEMM_PAIR=$P"
  for J in 0 56; do
    MX_GEMM_PAIR=$P timeout 120 python tools/gemm_bench.py --G 128 --rows 512 --jitter $J --N 1536 --K 2048 --swiglu --iters 20
    MX_GEMM_PAIR=$P timeout 120 python tools/gemm_bench.py --G 128 --rows 512 --jitter $J --N 2048 --K 768 --iters 20
  done
  MX_GEMM_PAIR=$P timeout 120 python tools/gemm_bench.py --G 64 --rows 512 --jitter 56 --N 768 --K 2048 --swiglu --iters 20
  MX_GEMM_PAIR=$P timeout 120 python tools/gemm_bench.py --G 64 --rows 512 --jitter 56 --N 2048 --K 384 --iters 20
  MX_GEMM_PAIR=$P timeout 120 python tools/gemm_bench.py --G 1 --rows 16384 --N 4096 --K 4096 --iters 20
done
