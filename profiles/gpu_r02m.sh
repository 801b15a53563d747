#!/usr/bin/env bash
# tf32x3 with the lo parts made in shared memory (converter warps)
set -u
O=gpurun_out
mkdir -p $O
timeout 240 python profiles/one_gemm.py 512x512x1024 tf32x3:128-64-32-2-1-1 2 > $O/x3m_one.log 2>&1; echo "rc=$?" >> $O/x3m_one.log
timeout 240 python profiles/one_gemm.py 1024x1024x1024 tf32x3:256-128-32-3-1-1 2 >> $O/x3m_one.log 2>&1; echo "rc=$?" >> $O/x3m_one.log
timeout 600 python -m pytest tests/test_gpu_tc.py -x -q > $O/pytest_m.log 2>&1; echo "pytest rc=$?" >> $O/pytest_m.log
timeout 300 python profiles/tc_accuracy_probe.py > $O/tc_accuracy4.jsonl 2> $O/tc_accuracy4.err
timeout 600 python profiles/x3_probe.py > $O/x3_probe4.jsonl 2> $O/x3_probe4.err
echo done
