# ncu --set full of the TMA-fed core and the packed core on the same tile / shape
O=gpurun_out
for cfg in tma:128-128-32-8-8-1 indirect:128-128-32-8-8-1; do
  n=${cfg%%:*}
  timeout 300 ncu --set full --clock-control none --import-source on -k regex:'tma_gemm|tiled_gemm' -s 2 -c 1 -f \
      -o $O/cmp_$n python profiles/one_gemm.py 4096x4096x4096 $cfg 3 > $O/cmp_$n.out 2>&1
done
