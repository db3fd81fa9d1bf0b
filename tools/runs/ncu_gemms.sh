# ncu --set full: config C's fp8 GEMMs (layer at N=1) and config B's bf16 GEMM2 shape
mkdir -p gpurun_out
bash tools/runs/ncu_fp8.sh
timeout 300 python tools/gemm_bench.py --G 128 --rows 512 --jitter 56 --N 2048 --K 768 --iters 2 > gpurun_out/g2_plain.log 2>&1 && \
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_grouped_gemm -s 3 -c 1 \
  -o gpurun_out/gemm2_b -f python tools/gemm_bench.py --G 128 --rows 512 --jitter 56 --N 2048 --K 768 --iters 2 > gpurun_out/g2_ncu.log 2>&1
echo "gemm2 rc=$?"
ls -la gpurun_out/*.ncu-rep
