#!/usr/bin/env bash
# Round profile pass on a GPU box (run through gpurun from the repo root):
#   gpurun --gpus 4 -- bash tools/profile_round.sh r01
# Writes everything under gpurun_out/<tag>_*: bench lines at 1/2/4 GPUs, the
# reference arm, the N=1 ncu launch list, ncu --set full captures of the
# grouped GEMMs and the N=1 memory kernels, the N=4/N=2 GEMM shapes under
# ncu (DRAM traffic per launch), the token-wire memory kernels of one rank on
# the emulated cluster under ncu, the SM-issued NVLink ceiling, config C/E
# sweeps, decode sweeps and the measured trace.  Every ncu command runs only after the same command has
# exited 0 without ncu; multi-rank commands are never run under ncu.
set -u
TAG=${1:-r01}
OUT=gpurun_out
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
mkdir -p $OUT

timeout 400 python bench.py --steps 30 --warmup 5 > $OUT/${TAG}_n1_bench.json 2> $OUT/${TAG}_n1.err
echo "bench n1 rc=$?"
timeout 300 python bench.py --impl reference --steps 3 --warmup 1 > $OUT/${TAG}_ref.json 2>&1
echo "reference rc=$?"
for N in 2 4; do
  timeout 500 $TR --nproc-per-node $N --master-port 2967$N bench.py --gpus $N --steps 30 --warmup 5 \
    > $OUT/${TAG}_n${N}_bench.json 2> $OUT/${TAG}_n$N.err
  echo "bench n$N rc=$?"
done

# N=1 launch list (cold-cache, serialised) and full captures
if timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu > /dev/null 2>&1; then
  timeout 500 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file $OUT/${TAG}_n1_launches.csv python bench.py --steps 3 --warmup 3 --no-cpu > /dev/null 2>&1
  echo "ncu launches rc=$?"
  timeout 500 ncu --set full --clock-control none --import-source on -k regex:k_grouped_gemm -s 4 -c 2 \
    -o $OUT/${TAG}_gemm_n1 python bench.py --steps 3 --warmup 3 --no-cpu > /dev/null 2>&1
  echo "ncu gemm rc=$?"
  timeout 500 ncu --set full --clock-control none --import-source on \
    -k "regex:k_gate|k_route|k_layout|k_dispatch|k_combine" -s 12 -c 6 \
    -o $OUT/${TAG}_misc_n1 python bench.py --steps 3 --warmup 3 --no-cpu > /dev/null 2>&1
  echo "ncu misc rc=$?"
fi
# the per-rank GEMM shapes of the 2- and 4-GPU layouts (same kernel, same
# shape as inside the layer) for their DRAM traffic
for shape in "n4 64 768 2048 --swiglu" "n4 64 2048 384" "n2 128 768 2048 --swiglu" "n2 128 2048 384"; do
  set -- $shape
  key=$1; G=$2; NN=$3; KK=$4; SW=${5:-}
  if timeout 120 python tools/gemm_bench.py --G $G --rows 512 --jitter 56 --N $NN --K $KK $SW > /dev/null 2>&1; then
    timeout 300 ncu --set full --clock-control none -k regex:k_grouped_gemm -s 3 -c 1 \
      -o $OUT/${TAG}_gemm_${key}_N${NN}_K${KK} python tools/gemm_bench.py --G $G --rows 512 --jitter 56 \
      --N $NN --K $KK $SW --iters 1 > /dev/null 2>&1
    echo "ncu gemm $key N=$NN K=$KK rc=$?"
  fi
done

# token-wire memory kernels of one config-B rank (emulated cluster, one GPU)
if CUDA_VISIBLE_DEVICES=0 timeout 120 python tools/emu_layer.py > /dev/null 2>&1; then
  CUDA_VISIBLE_DEVICES=0 timeout 300 ncu --set full --clock-control none --import-source on \
    -k "regex:k_pair_reduce|k_expand|k_dispatch_token|k_combine_token" -s 16 -c 8 \
    -o $OUT/${TAG}_emu_token python tools/emu_layer.py > /dev/null 2>&1
  echo "ncu emu token rc=$?"
fi
# what SM-issued peer stores / loads reach (all GPUs of the box at once)
timeout 200 python tools/nvlink_bench.py --out $OUT/${TAG}_nvlink_ceiling.jsonl > /dev/null 2>&1
echo "nvlink ceiling rc=$?"

timeout 600 $TR --nproc-per-node 4 --master-port 29681 tools/config_sweep.py --config C \
  --out $OUT/${TAG}_configC_n4.jsonl > $OUT/${TAG}_configC.log 2>&1
echo "config C rc=$?"
timeout 900 $TR --nproc-per-node 4 --master-port 29682 tools/config_sweep.py --config E \
  --out $OUT/${TAG}_configE_n4.jsonl > $OUT/${TAG}_configE.log 2>&1
echo "config E rc=$?"
for N in 2 4; do
  timeout 500 $TR --nproc-per-node $N --master-port 2968$((N+2)) tools/decode_sweep.py \
    --out $OUT/${TAG}_decode_n$N.jsonl > $OUT/${TAG}_decode_n$N.log 2>&1
  echo "decode n$N rc=$?"
done
timeout 300 $TR --nproc-per-node 4 --master-port 29689 tools/measured_trace.py \
  --out $OUT/${TAG}_mt_n4 > $OUT/${TAG}_mt.log 2>&1
echo "measured trace rc=$?"
