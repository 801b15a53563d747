#!/usr/bin/env bash
# Round-2 ncu evidence: the DT step's launch list, the dominant fp32 launch
# (DT pick at 5124x9124x2560) and the dominant tf32x3 launch, --set full.
set -u
O=gpurun_out
mkdir -p $O
timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file $O/launches_r02.csv python profiles/profile_step.py > $O/launches_r02.out 2>&1
P="ncu --set full --clock-control none --import-source on -f"
timeout 900 $P --profile-from-start off -k regex:tiled_gemm -c 1 -o $O/prof_top_r02 python profiles/profile_step.py --only 5124x9124x2560 > $O/prof_top_r02.out 2>&1
timeout 600 $P -k regex:tc_gemm -s 2 -c 1 -o $O/prof_x3_r02 python profiles/one_gemm.py 5124x9124x2560 tf32x3:256-128-32-3-1-1 4 > $O/prof_x3_r02.out 2>&1
echo done
