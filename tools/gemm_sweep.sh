set -x
for P in 0 2; do
 for J in 0 56; do
  MX_GEMM_PAIR=$P python tools/gemm_bench.py --G 128 --rows 512 --jitter $J --N 1536 --K 2048 --swiglu
  MX_GEMM_PAIR=$P python tools/gemm_bench.py --G 128 --rows 512 --jitter $J --N 2048 --K 768
 done
 MX_GEMM_PAIR=$P python tools/gemm_bench.py --G 64 --rows 1024 --N 1536 --K 2048 --swiglu
 MX_GEMM_PAIR=$P python tools/gemm_bench.py --G 1 --rows 16384 --N 4096 --K 4096
 MX_GEMM_PAIR=$P python tools/gemm_bench.py --G 64 --rows 512 --jitter 56 --N 768 --K 2048 --swiglu
 MX_GEMM_PAIR=$P python tools/gemm_bench.py --G 64 --rows 512 --jitter 56 --N 2048 --K 384
done
