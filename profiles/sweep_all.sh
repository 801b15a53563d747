#!/usr/bin/env bash
# Re-sweep the shipped tables on one B200 (configs[1], [2], [4]) and bundle them:
#   gpurun --timeout 7000 -- 'bash profiles/sweep_all.sh'
# Tables land in gpurun_out/sweep_*/tables; bundles in gpurun_out/bundles/ (copy them to
# paper_1806_07060_b200/data/).  `cli tune` resumes, so a cut-off run can be continued.
set -u
O=gpurun_out
mkdir -p $O/bundles
timeout 900 python -m pytest tests -m gpu -x -q > $O/sweep_pytest.log 2>&1 || { echo "gpu tests failed" >> $O/sweep_pytest.log; exit 1; }
for c in deepbench_b200 po2_b200 random_tc_b200; do
  t0=$(date +%s)
  python -m paper_1806_07060_b200.cli tune --config configs/$c.json --gpus 1 > $O/sweep_$c.log 2>&1
  echo "tune $c rc=$? wall_s=$(( $(date +%s) - t0 ))" >> $O/sweep_times.txt
done
python configs/bundle_tables.py configs/deepbench_b200.json $O/sweep_deepbench/tables $O/bundles/tables_b200_deepbench.csv.gz >> $O/sweep_times.txt 2>&1
python configs/bundle_tables.py configs/po2_b200.json $O/sweep_po2/tables $O/bundles/tables_b200_po2.csv.gz >> $O/sweep_times.txt 2>&1
python configs/bundle_tables.py configs/random_tc_b200.json $O/sweep_random_tc/tables $O/bundles/tables_b200tc_random.csv.gz >> $O/sweep_times.txt 2>&1
echo done >> $O/sweep_times.txt
