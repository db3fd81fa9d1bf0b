#!/bin/bash
for c in 16 128 1024 8192; do
  timeout 120 python tools/decode_gemm_bench.py --N 1536 --swiglu --active 8 --rows 2 --cap $c
done
for c in 128 8192; do
  timeout 120 python tools/decode_gemm_bench.py --N 2048 --K 768 --active 8 --rows 2 --cap $c
  timeout 120 python tools/decode_gemm_bench.py --N 1536 --swiglu --active 64 --rows 16 --cap $c
done
