#!/usr/bin/env bash
# Round-2 GPU session: gpu tests, smoke, bench, and ncu --set full captures of
# the kernels the DT picks that had no committed capture in round 1:
# the in-place split-K core with its cluster (DSMEM) reduction, the direct
# family and the packed split-K path's splitk_reduce_kernel.
#   gpurun --timeout 2400 -- 'bash profiles/gpu_round2.sh'
set -u
mkdir -p gpurun_out
O=gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,temperature.gpu,power.draw --format=csv > $O/smi.txt 2>&1
nproc > $O/nproc.txt
if [ "${SKIP_TESTS:-0}" != 1 ]; then
timeout 1500 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
fi
if [ "${SKIP_BENCH:-0}" != 1 ]; then
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err; echo "bench rc=$?" >> $O/bench.err
fi
if [ "${SKIP_NCU:-0}" != 1 ]; then
P="ncu --set full --clock-control none --import-source on -s 2 -c 1 -f"
timeout 600 $P -k regex:inplace_gemm -o $O/prof_inplace python profiles/one_gemm.py 2048x16x2048 splitk:32-16-32-4-2-8 4 > $O/prof_inplace.out 2>&1
timeout 600 $P -k regex:inplace_gemm -o $O/prof_inplace35 python profiles/one_gemm.py 35x8457x2560 splitk:64-128-32-8-8-8 4 > $O/prof_inplace35.out 2>&1
timeout 600 $P -k regex:direct_gemm -o $O/prof_direct python profiles/one_gemm.py 512x256x64 direct:32-32-16-2-1-1 4 > $O/prof_direct.out 2>&1
timeout 600 $P -k regex:splitk_reduce -o $O/prof_reduce python profiles/one_gemm.py 35x700x2048 splitk:16-32-32-2-4-8 4 TN > $O/prof_reduce.out 2>&1
fi
echo done
