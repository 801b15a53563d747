#!/usr/bin/env bash
# N > 1 functional check of bench.py with the po2 + random trees (two
# replicas share the 1-GPU box over gloo).
set -u
O=gpurun_out
mkdir -p $O
AG_DIST_BACKEND=gloo timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
  --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 4 --warmup 3 --no-cpu-baseline \
  > $O/bench_n2.json 2> $O/bench_n2.err; echo "rc=$?" >> $O/bench_n2.err
echo done
