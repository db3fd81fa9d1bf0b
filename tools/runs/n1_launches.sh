# N=1 ncu launch list of the bench command (cold-cache, serialised: compare shares)
mkdir -p gpurun_out
timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu > gpurun_out/l_plain.json 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/r02_n1_launches.csv python bench.py --steps 3 --warmup 3 --no-cpu > gpurun_out/l_ncu.log 2>&1
echo "rc=$?"; grep -c "" gpurun_out/r02_n1_launches.csv
