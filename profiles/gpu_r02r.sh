#!/usr/bin/env bash
# ncu --set full of the split-K picks the po2 + random tree makes on the
# M = 35 DeepBench shapes (in-place split-K core, 16-slice cluster reduction).
set -u
O=gpurun_out
mkdir -p $O
P="ncu --set full --clock-control none --import-source on -f"
for job in "35x700x2560 splitk:16-32-32-2-4-16" "35x8457x2560 splitk:32-64-16-4-4-16"; do
  set -- $job
  timeout 600 $P -k regex:inplace -s 2 -c 1 -o $O/prof_splitk_$1 python profiles/one_gemm.py $1 $2 4 > $O/prof_splitk_$1.out 2>&1
  python profiles/one_gemm.py $1 $2 6 >> $O/prof_splitk_$1.out 2>&1
done
echo done
