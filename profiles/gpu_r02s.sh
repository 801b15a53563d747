#!/usr/bin/env bash
# ncu --set full of the DT's split-K pick on 35x8457x2560: N = 8457 is not
# 16-byte aligned, so the family takes the packed path (pack A, pack-pad B,
# tiled core over 16 K slices, HBM slab reduction): all four launches of
# the second call.
set -u
O=gpurun_out
mkdir -p $O
timeout 900 ncu --set full --clock-control none --import-source on -f -k 'regex:pack|tiled_gemm|splitk_reduce' -s 4 -c 4 \
  -o $O/prof_splitk_35x8457x2560 python profiles/one_gemm.py 35x8457x2560 splitk:32-64-16-4-4-16 4 > $O/prof_splitk_35x8457x2560.out 2>&1
echo "rc=$?"
