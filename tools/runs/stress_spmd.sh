#!/bin/bash
# repeat the SPMD parity checks (early triggers, lean barriers, graph replay) to catch intermittent races
R4="python -m torch.distributed.run --nnodes=1 --nproc-per-node=4 --master-addr=127.0.0.1"
fails=0
for rep in 1 2 3; do
  for tp in 1 2 4; do
    timeout 900 $R4 --master-port=$((33000 + 10*rep + tp)) tests/spmd_check.py --tp $tp > gpurun_out/st_${rep}_$tp.log 2>&1
    rc=$?; ok=$(grep -c "OK" gpurun_out/st_${rep}_$tp.log)
    echo "rep $rep tp $tp rc=$rc ok=$ok"; [ $rc -ne 0 ] && fails=$((fails+1)) && grep -E "FAIL" gpurun_out/st_${rep}_$tp.log | head -3
  done
done
echo "failures: $fails"
