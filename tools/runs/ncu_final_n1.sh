#!/bin/bash
# final-code N=1 ncu: the launch list of the bench command and --set full captures of the layer's
# kernels in the bench (the bench's roofline.traffic source)
mkdir -p gpurun_out/ncu
timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu > gpurun_out/nf_plain.json 2>&1; echo "plain rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/r02_final_n1_launches.csv python bench.py --steps 3 --warmup 3 --no-cpu > gpurun_out/nf_l.log 2>&1; echo "launches rc=$?"
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"k_grouped_gemm|k_dispatch_rows|k_combine_local|k_gate|k_route|k_layout" -s 30 -c 8 \
  -o gpurun_out/ncu/r02_final_n1_layer python bench.py --steps 3 --warmup 3 --no-cpu > gpurun_out/nf_full.log 2>&1; echo "full rc=$?"
ls -la gpurun_out/ncu/ | tail -3
