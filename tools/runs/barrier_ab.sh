#!/bin/bash
for b in 0 1 2; do
  MX_BARRIER=$b timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 2961$b tools/barrier_probe.py 2>&1 | grep n_gpus | sed "s/^/MX_BARRIER=$b /"
done
