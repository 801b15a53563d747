#!/usr/bin/env bash
# continue a cut-off go2 sweep: tables already done travel in scratch/go2_tables
set -u
O=gpurun_out
mkdir -p $O/sweep_go2/tables $O/bundles
cp scratch/go2_tables/*.csv $O/sweep_go2/tables/ 2>/dev/null
t0=$(date +%s)
python -m paper_1806_07060_b200.cli tune --config configs/go2_b200.json --gpus 1 > $O/sweep_go2_resume.log 2>&1
echo "tune go2 (resume) rc=$? wall_s=$(( $(date +%s) - t0 ))" >> $O/go2_times.txt
python configs/bundle_tables.py configs/go2_b200.json $O/sweep_go2/tables $O/bundles/tables_b200_go2.csv.gz >> $O/go2_times.txt 2>&1
echo done >> $O/go2_times.txt
