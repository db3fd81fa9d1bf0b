#!/bin/bash
for args in "--active 8 --rows 2 --K 1024" "--active 8 --rows 2 --K 2048" "--active 8 --rows 2 --K 4096" "--active 8 --rows 2 --K 8192" \
            "--active 8 --rows 128 --K 2048" "--active 16 --rows 2 --K 4096" "--active 4 --rows 2 --K 8192"; do
  timeout 120 python tools/decode_gemm_bench.py --N 1536 --swiglu $args
done
