#!/usr/bin/env bash
# Add the TMA family's rows to the shipped fp32 tables (scratch/v3/sweep_*/tables =
# the current per-shape tables) and bundle them into gpurun_out/bundles/.
set -u
O=gpurun_out
mkdir -p $O/bundles
for pair in deepbench_b200:sweep_deepbench po2_b200:sweep_po2; do
  cfg=${pair%%:*}; d=${pair##*:}
  t0=$(date +%s)
  python configs/resweep_family.py tma configs/$cfg.json scratch/v3/$d/tables $O/tma_$d/tables > $O/tma_$d.log 2>&1
  echo "tma $cfg rc=$? wall_s=$(( $(date +%s) - t0 ))" >> $O/tma_times.txt
done
python configs/bundle_tables.py configs/deepbench_b200.json $O/tma_sweep_deepbench/tables $O/bundles/tables_b200_deepbench.csv.gz >> $O/tma_times.txt 2>&1
python configs/bundle_tables.py configs/po2_b200.json $O/tma_sweep_po2/tables $O/bundles/tables_b200_po2.csv.gz >> $O/tma_times.txt 2>&1
echo done >> $O/tma_times.txt
