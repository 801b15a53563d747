#!/usr/bin/env bash
# pinned result cache: host-path tests, e2e probe, bench
set -u
O=gpurun_out
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_dispatch.py tests/test_gpu_binding.py -x -q > $O/pytest_i.log 2>&1; echo "pytest rc=$?" >> $O/pytest_i.log
timeout 600 python profiles/e2e_numpy_probe.py > $O/e2e_probe4.jsonl 2> $O/e2e_probe4.err; echo "rc=$?" >> $O/e2e_probe4.err
timeout 1500 python bench.py > $O/bench.json 2> $O/bench.err; echo "bench rc=$?" >> $O/bench.err
echo done
