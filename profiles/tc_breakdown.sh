set -u
O=gpurun_out
for spec in "7640x4746x6966 bf16:256-256-64-6-1-1" "8192x8192x8192 bf16:256-256-64-6-1-1" "7640x4746x6966 tf32:256-256-32-4-1-1" "4096x4096x4096 bf16:256-256-64-6-1-1"; do
  set -- $spec
  timeout 120 python profiles/one_gemm.py $1 $2 4 >> $O/tc_times.txt 2>&1
  timeout 200 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv python profiles/one_gemm.py $1 $2 2 > $O/tc_ncu_$1_${2%%:*}.csv 2>&1
done
