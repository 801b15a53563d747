#!/usr/bin/env bash
# Round-2 re-sweep on one B200, every label in bench.py's timing regime (L2
# flushed before every sample, trimmed mean of 5): DeepBench (configs[2]),
# po2 16..4096 (the headline model's training set, ⊃ configs[1]) and go2 with
# the seeded tune_random sampler (96 of 1114 configs per shape).
#   gpurun --timeout 7000 -- 'bash profiles/sweep_r02.sh'
set -u
O=gpurun_out
mkdir -p $O/bundles
# (the GPU tests run in their own call before the sweep)
for c in deepbench_b200 po2_b200 go2r_b200; do
  t0=$(date +%s)
  python -m paper_1806_07060_b200.cli tune --config configs/$c.json --gpus 1 > $O/sweep_$c.log 2>&1
  echo "tune $c rc=$? wall_s=$(( $(date +%s) - t0 ))" >> $O/sweep_times.txt
  case $c in
    deepbench_b200) python configs/bundle_tables.py configs/$c.json $O/sweep_deepbench/tables $O/bundles/tables_b200_deepbench.csv.gz >> $O/sweep_times.txt 2>&1 ;;
    po2_b200) python configs/bundle_tables.py configs/$c.json $O/sweep_po2/tables $O/bundles/tables_b200_po2.csv.gz >> $O/sweep_times.txt 2>&1 ;;
    go2r_b200) python configs/bundle_tables.py configs/$c.json $O/sweep_go2r/tables $O/bundles/tables_b200_go2.csv.gz >> $O/sweep_times.txt 2>&1 ;;
  esac
done
echo done >> $O/sweep_times.txt
