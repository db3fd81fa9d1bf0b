# ncu --set full of one rank's token-wire dispatch and pair pre-reduction (2 GPUs, config B EP2)
mkdir -p gpurun_out
export MASTER_ADDR=127.0.0.1 WORLD_SIZE=2 FORWARDS=4
(for i in 1 2; do MASTER_PORT=29811 RANK=1 LOCAL_RANK=1 timeout 600 python tools/nvlink_rank.py >> gpurun_out/nvf_r1.log 2>&1; done) &
P=$!
MASTER_PORT=29811 RANK=0 LOCAL_RANK=0 timeout 1200 ncu --set full --import-source on --clock-control none \
  -k regex:"k_dispatch_token|k_pair_reduce" -s 6 -c 2 -o gpurun_out/nvl_full -f \
  python tools/nvlink_rank.py > gpurun_out/nvf_r0.log 2>&1
echo "rc0=$?"; wait $P; echo "rc1=$?"
tail -2 gpurun_out/nvf_r0.log
