#!/usr/bin/env bash
# Split-K with > 8 slices takes the slab reduction: GPU tests, then the
# 16-slice split-K configs re-timed on the DeepBench, po2 and random tables
# (bench regime) and merged into the shipped tables.
set -u
O=gpurun_out
mkdir -p $O/resweep16_tar
timeout 900 python -m pytest tests -m gpu -x -q > $O/pytest_gpu_u.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu_u.log
S16=splitk:16-16-16-2-2-16,splitk:16-16-32-2-2-16,splitk:32-16-16-4-2-16,splitk:32-16-32-4-2-16,splitk:16-32-16-2-4-16,splitk:16-32-32-2-4-16,splitk:32-32-16-4-4-16,splitk:32-32-32-4-4-16,splitk:64-16-16-4-2-16,splitk:64-16-32-4-2-16,splitk:16-64-16-2-4-16,splitk:16-64-32-2-4-16,splitk:64-32-16-4-4-16,splitk:64-32-32-4-4-16,splitk:32-64-16-4-4-16,splitk:32-64-32-4-4-16,splitk:64-64-16-8-4-16,splitk:64-64-32-8-4-16,splitk:64-64-16-4-8-16,splitk:64-64-32-4-8-16,splitk:128-64-16-8-4-16,splitk:128-64-32-8-4-16,splitk:64-128-16-4-8-16,splitk:64-128-32-4-8-16,splitk:128-64-16-8-8-16,splitk:128-64-32-8-8-16,splitk:64-128-16-8-8-16,splitk:64-128-32-8-8-16,splitk:128-128-16-8-8-16,splitk:128-128-32-8-8-16
for c in deepbench_b200:tables_b200_deepbench po2_b200:tables_b200_po2 lograndom_b200:tables_b200_lograndom; do
  cfg=${c%%:*}; b=${c##*:}
  python configs/resweep_family.py --unbundle paper_1806_07060_b200/data/$b.csv.gz /tmp/old_$cfg
  timeout 1200 python configs/resweep_family.py list:$S16 configs/$cfg.json /tmp/old_$cfg /tmp/new_$cfg > $O/resweep16_$cfg.log 2>&1
  echo "$cfg rc=$? $(ls /tmp/new_$cfg | wc -l)" >> $O/resweep16_times.txt
  tar -czf $O/resweep16_tar/$cfg.tgz -C /tmp new_$cfg
done
echo done
