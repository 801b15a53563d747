#!/usr/bin/env bash
# tf32x3 with chunked TMEM accumulation: accuracy, tests, timing; staged host
# path (8 x 4 MB slots, spinning copy workers): e2e probe; x3 re-sweep.
set -u
O=gpurun_out
mkdir -p $O
timeout 300 python profiles/tc_accuracy_probe.py > $O/tc_accuracy2.jsonl 2> $O/tc_accuracy2.err; echo "rc=$?" >> $O/tc_accuracy2.err
timeout 900 python -m pytest tests/test_gpu_tc.py tests/test_gpu_dispatch.py tests/test_gpu_binding.py -x -q > $O/pytest_e.log 2>&1; echo "pytest rc=$?" >> $O/pytest_e.log
timeout 600 python profiles/e2e_numpy_probe.py > $O/e2e_probe2.jsonl 2> $O/e2e_probe2.err; echo "rc=$?" >> $O/e2e_probe2.err
timeout 600 python profiles/x3_probe.py > $O/x3_probe3.jsonl 2> $O/x3_probe3.err; echo "rc=$?" >> $O/x3_probe3.err
rm -f $O/sweep_tar/deepbench_x3.tgz $O/sweep_tar/po2_x3.tgz
LIMIT=900 bash profiles/sweep_r02b.sh deepbench_x3 po2_x3
echo done
