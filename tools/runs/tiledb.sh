#!/bin/bash
# (experiment: the code it toggles was reverted after this A/B; the numbers are in DESIGN.md §5/§8)
# experiment: B boxes contiguous in HBM (MX_GEMM_TILEDB=1, numerics garbage) vs row-major weights
for t in 0 1; do
  echo "== MX_GEMM_TILEDB=$t"
  for args in "--active 8 --rows 2 --N 1536 --K 2048 --swiglu" "--active 8 --rows 2 --N 2048 --K 768" \
              "--active 40 --rows 4 --N 1536 --K 2048 --swiglu" "--active 64 --rows 16 --N 1536 --K 2048 --swiglu" \
              "--active 64 --rows 16 --N 2048 --K 768"; do
    MX_GEMM_TILEDB=$t timeout 120 python tools/decode_gemm_bench.py $args
  done
  MX_GEMM_TILEDB=$t timeout 120 python tools/gemm_bench.py --G 128 --rows 512 --jitter 56 --N 1536 --K 2048 --swiglu --iters 20
  MX_GEMM_TILEDB=$t timeout 120 python tools/gemm_bench.py --G 128 --rows 512 --jitter 56 --N 2048 --K 768 --iters 20
done
