#!/usr/bin/env bash
# time the fp32 default tiles over the tc random shapes and merge them in
set -u
O=gpurun_out
mkdir -p $O/bundles
python configs/resweep_family.py list:direct:16-32-16-2-1-1,indirect:64-64-32-8-8-1 configs/random_tc_b200.json \
    scratch/v5/sweep_random_tc/tables $O/tcdef/tables > $O/tcdef.log 2>&1
echo "rc=$?" >> $O/tcdef.log
python configs/bundle_tables.py configs/random_tc_b200.json $O/tcdef/tables $O/bundles/tables_b200tc_random.csv.gz >> $O/tcdef.log 2>&1
