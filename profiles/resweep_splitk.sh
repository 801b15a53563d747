#!/usr/bin/env bash
# After a split-K-only kernel change: re-time the split-K family over the
# finished sweeps (copied to scratch/sweep_*/tables, which travels with the
# snapshot) and bundle the merged tables into gpurun_out/bundles/.
set -u
O=gpurun_out
mkdir -p $O/bundles
timeout 900 python -m pytest tests -m gpu -x -q > $O/resweep_pytest.log 2>&1 || { echo "gpu tests failed" >> $O/resweep_pytest.log; exit 1; }
for pair in deepbench_b200:sweep_deepbench po2_b200:sweep_po2 random_tc_b200:sweep_random_tc; do
  cfg=${pair%%:*}; d=${pair##*:}
  t0=$(date +%s)
  python configs/resweep_family.py splitk configs/$cfg.json scratch/$d/tables $O/re_$d/tables > $O/re_$d.log 2>&1
  echo "resweep $cfg rc=$? wall_s=$(( $(date +%s) - t0 ))" >> $O/resweep_times.txt
done
python configs/bundle_tables.py configs/deepbench_b200.json $O/re_sweep_deepbench/tables $O/bundles/tables_b200_deepbench.csv.gz >> $O/resweep_times.txt 2>&1
python configs/bundle_tables.py configs/po2_b200.json $O/re_sweep_po2/tables $O/bundles/tables_b200_po2.csv.gz >> $O/resweep_times.txt 2>&1
python configs/bundle_tables.py configs/random_tc_b200.json $O/re_sweep_random_tc/tables $O/bundles/tables_b200tc_random.csv.gz >> $O/resweep_times.txt 2>&1
echo done >> $O/resweep_times.txt
