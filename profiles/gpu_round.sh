#!/usr/bin/env bash
# One GPU session: gpu tests, smoke, bench (default + reference arm), ncu launch
# list of one bench step and one `--set full` capture of the dominant kernel.
#   gpurun --timeout 3000 -- 'bash profiles/gpu_round.sh'
# Outputs land in gpurun_out/ (scratch); copy the summaries worth keeping into profiles/.
set -u
mkdir -p gpurun_out
O=gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,temperature.gpu,power.draw --format=csv > $O/smi.txt 2>&1
nproc > $O/nproc.txt
timeout 1500 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err; echo "bench rc=$?" >> $O/bench.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > $O/bench_ref.json 2> $O/bench_ref.err
timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none \
    --csv --log-file $O/launches.csv python profiles/profile_step.py > $O/launches.out 2>&1
timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on \
    -k regex:tiled_gemm -c 1 -f -o $O/prof_top python profiles/profile_step.py --only ${TOP_SHAPE:-5124x9124x2560} \
    > $O/prof_top.out 2>&1
# the tensor-core DT's dominant kernel (configs[4] roofline traffic)
timeout 600 ncu --set full --clock-control none --import-source on -k regex:tc_gemm -s 1 -c 1 -f -o $O/prof_tc \
    python profiles/one_gemm.py ${TC_SHAPE:-7640x4746x6966} ${TC_CFG:-bf16:256-256-64-6-1-1} 2 > $O/prof_tc.out 2>&1
echo done
