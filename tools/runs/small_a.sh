#!/bin/bash
# (experiment: the code it toggles was reverted after this A/B; the numbers are in DESIGN.md §5/§8)
# small A boxes for short tiles: A/B on the decode GEMM shapes, then GEMM parity tests
for t in 0 1; do
  echo "== MX_GEMM_SMALL_A=$t"
  for args in "--active 8 --rows 2 --N 1536 --K 2048 --swiglu" "--active 8 --rows 2 --N 2048 --K 768" \
              "--active 16 --rows 2 --N 1536 --K 2048 --swiglu" "--active 40 --rows 4 --N 1536 --K 2048 --swiglu" \
              "--active 64 --rows 16 --N 1536 --K 2048 --swiglu" "--active 64 --rows 16 --N 2048 --K 768" \
              "--active 64 --rows 32 --N 1536 --K 2048 --swiglu" "--active 64 --rows 60 --N 1536 --K 2048 --swiglu"; do
    MX_GEMM_SMALL_A=$t timeout 120 python tools/decode_gemm_bench.py $args
  done
done
timeout 900 python -m pytest tests -m gpu -x -q -k "gemm or decode or fp8" 2>&1 | tail -3
