# dense single group of the same total M as config B's GEMM1/GEMM2 (B stays in L2)
for P in 0 2; do
  MX_GEMM_PAIR=$P python tools/gemm_bench.py --G 1 --rows 65536 --N 1536 --K 2048 --swiglu
  MX_GEMM_PAIR=$P python tools/gemm_bench.py --G 1 --rows 65536 --N 2048 --K 768
  MX_GEMM_PAIR=$P python tools/gemm_bench.py --G 8 --rows 8192 --N 1536 --K 2048 --swiglu
  MX_GEMM_PAIR=$P python tools/gemm_bench.py --G 32 --rows 2048 --N 1536 --K 2048 --swiglu
done
