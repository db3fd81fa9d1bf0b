# ncu --set full of config C's routed fp8 GEMM1 (3rd forward), after a plain run
mkdir -p gpurun_out
timeout 600 python tools/fp8_layer_profile.py > gpurun_out/fp8_plain.log 2>&1 && \
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:k_grouped_gemm -s 8 -c 2 \
  -o gpurun_out/fp8_gemm -f python tools/fp8_layer_profile.py > gpurun_out/fp8_ncu.log 2>&1
echo "rc=$?"; tail -3 gpurun_out/fp8_ncu.log
