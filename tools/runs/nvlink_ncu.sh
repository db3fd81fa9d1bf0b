# NVLink counters of one rank's communicator kernels (2 GPUs, config B EP2):
# rank 1 runs plain, rank 0 runs under ncu (no multi-rank command is wrapped)
mkdir -p gpurun_out
export MASTER_ADDR=127.0.0.1 WORLD_SIZE=2
pair() {  # $1 port, $2 prefix for rank 0 (e.g. ncu ...), $3 rank-1 runs
  # (the box runs an ncu target once without ncu first: rank 1 then runs twice)
  (for i in $(seq ${3:-1}); do MASTER_PORT=$1 RANK=1 LOCAL_RANK=1 timeout 600 python tools/nvlink_rank.py >> gpurun_out/nv_r1_$1.log 2>&1; done) &
  P=$!
  MASTER_PORT=$1 RANK=0 LOCAL_RANK=0 timeout 900 $2 python tools/nvlink_rank.py > gpurun_out/nv_r0_$1.log 2>&1
  rc0=$?
  wait $P; rc1=$?
  echo "port $1 rc0=$rc0 rc1=$rc1"
  [ $rc0 -eq 0 ] && [ $rc1 -eq 0 ]
}
pair 29801 "" && \
pair 29802 "ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,nvltx__bytes.sum,nvlrx__bytes.sum,nvltx__bytes_data_user.sum,nvlrx__bytes_data_user.sum --clock-control none -k regex:k_dispatch_token|k_expand|k_pair_reduce|k_combine_token -s 12 -c 8 --csv --log-file gpurun_out/nvlink_ncu.csv" 2
tail -3 gpurun_out/nv_r0_29802.log
grep -c "" gpurun_out/nvlink_ncu.csv
