# ncu --set full of the grouped GEMM (config-B GEMM1 shape, 128 experts x 512+-56 rows):
# single-CTA vs CTA-pair kernel, source-level stall sampling
mkdir -p gpurun_out
for P in 0 2; do
  MX_GEMM_PAIR=$P timeout 600 ncu --set full --import-source on --clock-control none \
    -k regex:k_grouped_gemm -s 3 -c 1 -o gpurun_out/gemm_p$P -f \
    python tools/gemm_bench.py --G 128 --rows 512 --jitter 56 --N 1536 --K 2048 --swiglu --iters 2 > gpurun_out/ncu_p$P.log 2>&1
  echo "P=$P rc=$?"
done
