#!/bin/bash
for L in paper_2601_08800_b200/lib/libmixserve_b200.so paper_2601_08800_b200/lib/variants/libmx_silu_IEEE.so; do
  echo "== $L"
  MIXSERVE_B200_LIB=$L timeout 120 python tools/decode_gemm_bench.py --trace --active 8 --rows 2 --N 1536 --K 2048 --swiglu | grep -E "median|epi_|mma_issued"
  MIXSERVE_B200_LIB=$L timeout 120 python tools/gemm_bench.py --G 128 --rows 512 --jitter 56 --N 1536 --K 2048 --swiglu --iters 20
done
