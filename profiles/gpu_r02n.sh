#!/usr/bin/env bash
# tf32x3 (lo parts in shared memory) re-sweep of its rows, then the full check
set -u
O=gpurun_out
mkdir -p $O
rm -f $O/sweep_tar/deepbench_x3.tgz $O/sweep_tar/po2_x3.tgz
LIMIT=900 bash profiles/sweep_r02b.sh deepbench_x3 po2_x3
timeout 1500 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
echo done
