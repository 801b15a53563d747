set -u
O=gpurun_out; mkdir -p $O
for j in "35x8456x2560 splitk:32-64-16-4-4-16 8 NN" "35x8456x2560 splitk:32-64-16-4-4-16 8 TN" "35x8457x2560 splitk:32-64-16-4-4-16 8 NN" \
         "35x1500x2560 splitk:32-64-16-4-4-16 8 NN" "35x1500x2560 splitk:32-64-16-4-4-16 8 TN" \
         "35x1500x2560 splitk:16-32-32-2-4-4 8 NN" "35x1500x2560 splitk:16-32-32-2-4-4 8 TN" \
         "2560x64x2560 splitk:64-32-32-4-4-8 8 NN" "2560x64x2560 splitk:64-32-32-4-4-8 8 TN" \
         "3072x128x1024 splitk:64-128-16-8-8-8 8 NN" "3072x128x1024 splitk:64-128-16-8-8-8 8 TN"; do
  echo "== $j" >> $O/inplace_vs_packed.txt
  python profiles/one_gemm.py $j 2>&1 | tail -3 >> $O/inplace_vs_packed.txt
done
