#!/bin/bash
for args in "--active 8 --rows 2 --N 1536 --K 2048 --swiglu" "--active 8 --rows 2 --N 2048 --K 768" \
            "--active 64 --rows 4 --N 1536 --K 2048 --swiglu"; do
  timeout 120 python tools/decode_gemm_bench.py --trace $args
done
