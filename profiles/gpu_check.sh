#!/usr/bin/env bash
# One GPU check of the tree as it stands: gpu tests, smoke, default bench line.
#   gpurun --timeout 1800 -- 'bash profiles/gpu_check.sh'
set -u
O=gpurun_out
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,temperature.gpu,power.draw --format=csv > $O/smi.txt 2>&1
nproc > $O/nproc.txt
if [ "${SKIP_TESTS:-0}" != 1 ]; then
timeout 1200 python -m pytest tests -m gpu -x -q ${PYTEST_ARGS:-} > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
fi
if [ "${SKIP_BENCH:-0}" != 1 ]; then
timeout 1200 python bench.py ${BENCH_ARGS:-} > $O/bench.json 2> $O/bench.err; echo "bench rc=$?" >> $O/bench.err
fi
echo done
