#!/bin/bash
# remap stress (S1/S2) per push-kernel variant; run under gpurun --gpus N
N=${1:-2}
for lib in build/variants/*.so; do
  echo "== $lib"
  ZP_LIB_PATH=$PWD/$lib timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29512 tools/remap_stress.py 2>&1 | grep -v Warn | tail -4
done
