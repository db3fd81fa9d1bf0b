#!/bin/bash
# A/B: HEAD grouped GEMM (lib/variants/libmx_head.so) vs working tree, interleaved
for r in 1 2; do
 for L in paper_2601_08800_b200/lib/variants/libmx_head.so paper_2601_08800_b200/lib/libmixserve_b200.so; do
  echo "== $L"
  MIXSERVE_B200_LIB=$L timeout 120 python tools/gemm_bench.py --G 128 --rows 512 --jitter 56 --N 1536 --K 2048 --swiglu --iters 20
  MIXSERVE_B200_LIB=$L timeout 120 python tools/gemm_bench.py --G 128 --rows 512 --jitter 56 --N 2048 --K 768 --iters 20
  MIXSERVE_B200_LIB=$L timeout 120 python tools/decode_gemm_bench.py --active 8 --rows 2 --N 1536 --K 2048 --swiglu
 done
done
