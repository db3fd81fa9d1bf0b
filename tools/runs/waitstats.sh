#!/bin/bash
# where the grouped GEMM's issuer and producer wait (MX_GEMM_WAITSTATS variant build)
export MIXSERVE_B200_LIB=paper_2601_08800_b200/lib/variants/libmx_waitstats.so
timeout 120 python tools/gemm_bench.py --trace --G 128 --rows 512 --jitter 56 --N 1536 --K 2048 --swiglu --iters 20
timeout 120 python tools/gemm_bench.py --trace --G 128 --rows 512 --jitter 56 --N 2048 --K 768 --iters 20
timeout 120 python tools/gemm_bench.py --trace --G 64 --rows 512 --jitter 56 --N 768 --K 2048 --swiglu --iters 20
timeout 120 python tools/gemm_bench.py --trace --G 64 --rows 512 --jitter 56 --N 2048 --K 384 --iters 20
timeout 120 python tools/gemm_bench.py --trace --G 1 --rows 16384 --N 4096 --K 4096 --iters 20
unset MIXSERVE_B200_LIB
timeout 120 python tools/gemm_bench.py --G 128 --rows 512 --jitter 56 --N 1536 --K 2048 --swiglu --iters 20
