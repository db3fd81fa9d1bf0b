#!/bin/bash
# decode-regime grouped GEMM: weight-streaming rate at small row counts
for args in "--active 8 --rows 2 --N 1536 --K 2048 --swiglu" "--active 8 --rows 2 --N 2048 --K 768" \
            "--active 16 --rows 2 --N 1536 --K 2048 --swiglu" "--active 16 --rows 2 --N 2048 --K 768" \
            "--active 40 --rows 4 --N 1536 --K 2048 --swiglu" "--active 40 --rows 4 --N 2048 --K 768" \
            "--active 64 --rows 16 --N 1536 --K 2048 --swiglu" "--active 64 --rows 16 --N 2048 --K 768"; do
  timeout 120 python tools/decode_gemm_bench.py $args
done
