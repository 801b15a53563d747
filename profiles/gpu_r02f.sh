#!/usr/bin/env bash
# Full check after the re-sweep: gpu tests, smoke, bench line, tc accuracy.
set -u
O=gpurun_out
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,temperature.gpu,power.draw --format=csv > $O/smi.txt 2>&1
timeout 300 python profiles/tc_accuracy_probe.py > $O/tc_accuracy3.jsonl 2> $O/tc_accuracy3.err; echo "rc=$?" >> $O/tc_accuracy3.err
timeout 1500 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
timeout 1500 python bench.py > $O/bench.json 2> $O/bench.err; echo "bench rc=$?" >> $O/bench.err
echo done
