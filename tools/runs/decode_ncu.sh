#!/bin/bash
# per-kernel durations of the decode-regime token wire (emulated 2-rank EP2
# cluster on one GPU) and of the N=1 slot wire, ncu launch lists
set -x
mkdir -p gpurun_out
for T in 2 64; do
  timeout 300 python tools/emu_layer.py --n 2 --m 1 --tokens $T --iters 3 || exit 1
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/decode_emu_T$T.csv python tools/emu_layer.py --n 2 --m 1 --tokens $T --iters 3 > /dev/null 2>&1
done
for T in 2 64; do
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/decode_emu_n1_T$T.csv python tools/emu_layer.py --n 1 --m 1 --tokens $T --iters 3 > /dev/null 2>&1
done
ls -la gpurun_out
