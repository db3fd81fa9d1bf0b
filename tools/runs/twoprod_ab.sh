#!/bin/bash
# (experiment: the code it toggles was reverted after this A/B; the numbers are in DESIGN.md §5/§8)
# two TMA producer threads (A / B) vs one, grouped GEMM shapes, then tests and the N=1 bench
for r in 1 2; do
 for L in paper_2601_08800_b200/lib/variants/libmx_head.so paper_2601_08800_b200/lib/libmixserve_b200.so; do
  echo "== $L"
  export MIXSERVE_B200_LIB=$L
  timeout 120 python tools/gemm_bench.py --G 128 --rows 512 --jitter 56 --N 1536 --K 2048 --swiglu --iters 20
  timeout 120 python tools/gemm_bench.py --G 128 --rows 512 --jitter 56 --N 2048 --K 768 --iters 20
  timeout 120 python tools/gemm_bench.py --G 64 --rows 512 --jitter 56 --N 768 --K 2048 --swiglu --iters 20
  timeout 120 python tools/gemm_bench.py --G 64 --rows 512 --jitter 56 --N 2048 --K 384 --iters 20
  timeout 120 python tools/decode_gemm_bench.py --active 8 --rows 2 --N 1536 --K 2048 --swiglu
  timeout 120 python tools/decode_gemm_bench.py --active 64 --rows 4 --N 1536 --K 2048 --swiglu
 done
done
unset MIXSERVE_B200_LIB
timeout 900 python -m pytest tests -m gpu -x -q -k "gemm or config or swiglu or parity or fp8" 2>&1 | tail -2
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/tp_n1.json 2> gpurun_out/tp_n1.err; echo "bench rc=$?"
python tools/summarize_line.py gpurun_out/tp_n1.json | cut -c1-420
