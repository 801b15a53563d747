#!/usr/bin/env bash
# compute-sanitizer over every family incl. tf32x3 / skinny and the staged host path
set -u
O=gpurun_out
mkdir -p $O/sanitizer
for t in memcheck racecheck synccheck; do
  timeout 1200 compute-sanitizer --tool $t python profiles/sanitize_probe.py > $O/sanitizer/r02_$t.log 2>&1; echo "rc=$?" >> $O/sanitizer/r02_$t.log
done
echo done
