#!/usr/bin/env bash
# Round-2 re-sweep: every label in bench.py's timing regime (L2 flushed
# before every sample, trimmed mean of the samples).  Raw per-shape tables
# live in /tmp on the box; after each config (finished or cut by its time
# limit) they are tarred into gpurun_out/sweep_tar/ and come back with the
# call.  (gpurun does not ship gpurun_out/ to the box, so a cut sweep resumes
# only if its tarball is copied into the repo tree before the next call.)
#   gpurun --timeout 3000 -- 'LIMIT=2700 bash profiles/sweep_r02b.sh deepbench_b200 po2_b200'
set -u
O=gpurun_out
mkdir -p $O/sweep_tar
LIMIT=${LIMIT:-2700}
t_start=$(date +%s)
for c in "$@"; do
  d=/tmp/sweep_$c
  mkdir -p $d
  [ -f $O/sweep_tar/$c.tgz ] && tar -xzf $O/sweep_tar/$c.tgz -C $d
  left=$(( LIMIT - ($(date +%s) - t_start) ))
  [ $left -lt 60 ] && { echo "skip $c (time)" >> $O/sweep_times.txt; continue; }
  t0=$(date +%s)
  timeout $left python -m paper_1806_07060_b200.cli tune --config configs/$c.json --out $d --gpus 1 > $O/sweep_$c.log 2>&1
  rc=$?
  n=$(ls $d/tables 2>/dev/null | wc -l)
  echo "tune $c rc=$rc wall_s=$(( $(date +%s) - t0 )) tables=$n" >> $O/sweep_times.txt
  tar -czf $O/sweep_tar/$c.tgz -C $d tables
done
echo done >> $O/sweep_times.txt
