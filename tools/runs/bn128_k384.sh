#!/bin/bash
# (experiment: the code it toggles was reverted after this A/B; the numbers are in DESIGN.md §5/§8)
# GEMM2 at the TP2 shape (K = 384): BN=128 with six stages vs BN=256 with four
for r in 1 2; do
for b in 0 128; do
  MX_GEMM_BN=$b timeout 120 python tools/gemm_bench.py --G 64 --rows 512 --jitter 56 --N 2048 --K 384 --iters 20
  MX_GEMM_BN=$b timeout 120 python tools/gemm_bench.py --G 32 --rows 512 --jitter 56 --N 2048 --K 384 --iters 20
  MX_GEMM_BN=$b timeout 120 python tools/gemm_bench.py --G 128 --rows 512 --jitter 56 --N 2048 --K 768 --iters 20
done
done
