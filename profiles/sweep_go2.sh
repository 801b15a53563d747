#!/usr/bin/env bash
# go2 (256..3840 step 256, 3375 shapes) over the 133-config fp32 shortlist
# (per-shape top-3 of the po2 + DeepBench tables): configs/go2_b200.json
set -u
O=gpurun_out
mkdir -p $O/bundles
t0=$(date +%s)
python -m paper_1806_07060_b200.cli tune --config configs/go2_b200.json --gpus 1 > $O/sweep_go2.log 2>&1
echo "tune go2 rc=$? wall_s=$(( $(date +%s) - t0 ))" >> $O/go2_times.txt
python configs/bundle_tables.py configs/go2_b200.json $O/sweep_go2/tables $O/bundles/tables_b200_go2.csv.gz >> $O/go2_times.txt 2>&1
echo done >> $O/go2_times.txt
