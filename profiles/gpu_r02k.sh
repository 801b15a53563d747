#!/usr/bin/env bash
set -u
O=gpurun_out
mkdir -p $O
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
timeout 900 python -m pytest tests/test_gpu_binding.py tests/test_gpu_tc.py -x -q > $O/pytest_k.log 2>&1; echo "pytest rc=$?" >> $O/pytest_k.log
timeout 1500 python bench.py > $O/bench.json 2> $O/bench.err; echo "bench rc=$?" >> $O/bench.err
echo done
