#!/usr/bin/env bash
# tf32x3 rows for the octave-uniform random shapes (the headline training
# set's second half), then the DT step's launch list with the po2 + random tree.
set -u
O=gpurun_out
mkdir -p $O
LIMIT=900 bash profiles/sweep_r02b.sh lograndom_x3
timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file $O/launches_r02p.csv python profiles/profile_step.py > $O/launches_r02p.out 2>&1
echo done
