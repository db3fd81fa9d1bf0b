#!/bin/bash
mkdir -p gpurun_out/ncu
timeout 300 ncu --set full --clock-control none --import-source on -k regex:k_grouped_gemm -s 8 -c 1 \
  -o gpurun_out/ncu/decode_gemm1_a8 python tools/decode_gemm_bench.py --active 8 --rows 2 --N 1536 --K 2048 --swiglu --iters 8 > gpurun_out/dg1.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:k_grouped_gemm -s 8 -c 1 \
  -o gpurun_out/ncu/decode_gemm1_a64 python tools/decode_gemm_bench.py --active 64 --rows 16 --N 1536 --K 2048 --swiglu --iters 8 > gpurun_out/dg2.log 2>&1
ls -la gpurun_out/ncu
