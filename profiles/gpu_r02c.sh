#!/usr/bin/env bash
# Round-2 GPU call: tc + host-path GPU tests (tf32x3, staged pageable path),
# e2e numpy probe, tf32x3 probe, streaming-read floor, ncu of the skinny
# kernels the DT picks and of the tf32x3 kernel.
#   gpurun --timeout 2400 -- 'bash profiles/gpu_r02c.sh'
set -u
O=gpurun_out
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_tc.py tests/test_gpu_dispatch.py tests/test_gpu_binding.py -x -q > $O/pytest_c.log 2>&1; echo "pytest rc=$?" >> $O/pytest_c.log
timeout 600 python profiles/e2e_numpy_probe.py > $O/e2e_probe.jsonl 2> $O/e2e_probe.err; echo "rc=$?" >> $O/e2e_probe.err
timeout 600 python profiles/x3_probe.py > $O/x3_probe.jsonl 2> $O/x3_probe.err; echo "rc=$?" >> $O/x3_probe.err
timeout 300 python profiles/read_floor.py > $O/read_floor.jsonl 2> $O/read_floor.err; echo "rc=$?" >> $O/read_floor.err
P="ncu --set full --clock-control none --import-source on -s 2 -c 1 -f"
timeout 300 $P -k regex:skinny_n -o $O/prof_skinny_n python profiles/one_gemm.py 2048x16x2048 skinny_n:64-16-32-2-4-4 4 > $O/prof_skinny_n.out 2>&1
timeout 300 $P -k regex:skinny_m -o $O/prof_skinny_m python profiles/one_gemm.py 35x8457x2560 skinny_m:40-256-32-1-2-16 4 > $O/prof_skinny_m.out 2>&1
timeout 300 $P -k regex:tc_gemm -o $O/prof_x3 python profiles/one_gemm.py 5124x9124x2560 tf32x3:256-256-32-3-1-1 4 > $O/prof_x3.out 2>&1
echo done
