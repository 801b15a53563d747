#!/usr/bin/env bash
# tf32x3 accuracy (separate small-product accumulator), tc tests, x3 timing,
# host copy rates, TMEM-alloc racecheck repro.
set -u
O=gpurun_out
mkdir -p $O
timeout 300 python profiles/tc_accuracy_probe.py > $O/tc_accuracy.jsonl 2> $O/tc_accuracy.err; echo "rc=$?" >> $O/tc_accuracy.err
timeout 900 python -m pytest tests/test_gpu_tc.py -x -q > $O/pytest_tc.log 2>&1; echo "pytest rc=$?" >> $O/pytest_tc.log
timeout 600 python profiles/x3_probe.py > $O/x3_probe2.jsonl 2> $O/x3_probe2.err; echo "rc=$?" >> $O/x3_probe2.err
timeout 300 python profiles/host_copy_probe.py > $O/host_copy.jsonl 2> $O/host_copy.err; echo "rc=$?" >> $O/host_copy.err
nvcc -gencode arch=compute_100a,code=sm_100a -lineinfo -o /tmp/tmem_race profiles/tmem_alloc_race.cu > $O/tmem_race.log 2>&1
timeout 300 compute-sanitizer --tool racecheck /tmp/tmem_race >> $O/tmem_race.log 2>&1; echo "rc=$?" >> $O/tmem_race.log
echo done
