for rep in 1 2; do
for v in 1 0; do
  echo "== MX_GEMM_ASTAT=$v"
  MX_GEMM_ASTAT=$v python tools/gemm_bench.py --G 64 --rows 512 --jitter 56 --N 2048 --K 384 --reps 5 | cut -c1-80
  MX_GEMM_ASTAT=$v python tools/gemm_bench.py --G 64 --rows 512 --N 2048 --K 384 --reps 5 | cut -c1-80
  MX_GEMM_ASTAT=$v python tools/gemm_bench.py --G 64 --rows 8 --jitter 4 --N 2048 --K 384 --reps 5 | cut -c1-80
  MX_GEMM_ASTAT=$v python tools/gemm_bench.py --G 16 --rows 4096 --N 2048 --K 384 --reps 5 | cut -c1-80
done
done
