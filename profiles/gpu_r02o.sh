#!/usr/bin/env bash
# N > 1 functional check of bench.py on the 1-GPU box (two replicas share
# the GPU over gloo), plus the ncu capture of the new dominant tf32x3 launch.
set -u
O=gpurun_out
mkdir -p $O
AG_DIST_BACKEND=gloo timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
  --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 4 --warmup 3 --no-cpu-baseline \
  > $O/bench_n2.json 2> $O/bench_n2.err; echo "rc=$?" >> $O/bench_n2.err
timeout 600 ncu --set full --clock-control none --import-source on -f -k regex:tc_gemm -s 2 -c 1 \
  -o $O/prof_x3_r02b python profiles/one_gemm.py 5124x9124x2560 tf32x3:128-128-32-3-1-1 4 > $O/prof_x3_r02b.out 2>&1
echo done
