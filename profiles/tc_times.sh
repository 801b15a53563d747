# tensor-core path timings (device events inside gemm_execute) on ragged and aligned shapes
for spec in "7640x4746x6966 bf16:256-256-64-6-1-1" "7640x4744x6968 bf16:256-256-64-6-1-1" "8192x8192x8192 bf16:256-256-64-6-1-1" "4096x4096x4096 bf16:256-256-64-6-1-1" "7640x4746x6966 tf32:256-256-32-4-1-1" "8192x8192x8192 tf32:256-256-32-4-1-1" "3000x5000x1000 bf16:256-128-64-6-1-1"; do
  set -- $spec
  timeout 120 python profiles/one_gemm.py $1 $2 4 | tail -1
done
