#!/usr/bin/env bash
# go2 with the seeded tune_random sampler (96 of 1114 configs, bench regime)
# and the tc random set re-swept in the bench regime with tf32x3 added.
set -u
O=gpurun_out
mkdir -p $O
LIMIT=3000 bash profiles/sweep_r02b.sh go2r_b200 random_tc_r02
echo done
