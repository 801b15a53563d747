#!/usr/bin/env bash
# re-time the split-K family over the shipped DeepBench / po2 tables (scratch/sweep_*/tables)
set -u
O=gpurun_out
mkdir -p $O/bundles
for pair in deepbench_b200:sweep_deepbench po2_b200:sweep_po2; do
  cfg=${pair%%:*}; d=${pair##*:}
  python configs/resweep_family.py splitk configs/$cfg.json scratch/$d/tables $O/re2_$d/tables > $O/re2_$d.log 2>&1
  echo "resweep $cfg rc=$?" >> $O/re2_times.txt
done
python configs/bundle_tables.py configs/deepbench_b200.json $O/re2_sweep_deepbench/tables $O/bundles/tables_b200_deepbench.csv.gz >> $O/re2_times.txt 2>&1
python configs/bundle_tables.py configs/po2_b200.json $O/re2_sweep_po2/tables $O/bundles/tables_b200_po2.csv.gz >> $O/re2_times.txt 2>&1
