#!/bin/bash
mkdir -p gpurun_out/ncu
timeout 300 ncu --set full --clock-control none --import-source on -k regex:k_grouped_gemm -s 8 -c 1 \
  -o gpurun_out/ncu/decode_gemm1_a4k8 python tools/decode_gemm_bench.py --active 4 --rows 2 --N 1536 --K 8192 --swiglu --iters 8 > gpurun_out/dg3.log 2>&1
ls -la gpurun_out/ncu
