#!/usr/bin/env bash
# In-place split-K core with element copies of B (odd N): GPU tests, a
# timing probe on 35x8457, and the split-K family re-timed on the odd-N
# shapes of the DeepBench and random tables (bench regime).
set -u
O=gpurun_out
mkdir -p $O/resweep_tar
timeout 900 python -m pytest tests -m gpu -x -q > $O/pytest_gpu_t.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu_t.log
for j in "35x8457x2560 splitk:32-64-16-4-4-16" "35x8457x2048 splitk:32-64-16-4-4-16" "35x8457x2560 skinny_m:40-256-32-1-2-16" \
         "35x8457x2560 splitk:64-64-16-8-4-16" "35x8457x2560 splitk:32-64-32-4-4-16"; do
  python profiles/one_gemm.py $j 8 | tail -3 >> $O/oddn_probe.txt 2>&1
done
for c in deepbench_b200:tables_b200_deepbench lograndom_b200:tables_b200_lograndom; do
  cfg=${c%%:*}; b=${c##*:}
  python configs/resweep_family.py --unbundle paper_1806_07060_b200/data/$b.csv.gz /tmp/old_$cfg
  timeout 900 python configs/resweep_family.py splitk configs/$cfg.json /tmp/old_$cfg /tmp/new_$cfg --odd-n-only > $O/resweep_$cfg.log 2>&1
  echo "$cfg rc=$? $(ls /tmp/new_$cfg | wc -l)" >> $O/resweep_times.txt
  tar -czf $O/resweep_tar/$cfg.tgz -C /tmp new_$cfg
done
echo done
