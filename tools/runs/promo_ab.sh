#!/bin/bash
# (experiment) TMA L2 promotion of the grouped GEMM's tensor maps
for r in 1 2; do
for pr in 256 128 0; do
  echo "== MX_GEMM_PROMO=$pr"
  MX_GEMM_PROMO=$pr timeout 120 python tools/gemm_bench.py --G 128 --rows 512 --jitter 56 --N 1536 --K 2048 --swiglu --iters 20
  MX_GEMM_PROMO=$pr timeout 120 python tools/gemm_bench.py --G 128 --rows 512 --jitter 56 --N 2048 --K 768 --iters 20
  MX_GEMM_PROMO=$pr timeout 120 python tools/gemm_bench.py --G 64 --rows 512 --jitter 56 --N 2048 --K 384 --iters 20
done
done
