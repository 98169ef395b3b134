# GEMM: ours vs cuBLAS, full ncu sets, two shapes
mkdir -p gpurun_out
for shp in "8192 2048 2048" "8192 5632 2048"; do
  tag=$(echo $shp | tr ' ' x)
  timeout 300 ncu --set full --clock-control none --import-source on -k regex:tc2_kernel -s 2 -c 1 -o gpurun_out/g_ours_$tag python tools/gemmbench.py $shp 0 1 > /dev/null 2>&1
  set -- $shp
  timeout 300 ncu --set full --clock-control none -k regex:nvjet -s 2 -c 1 -o gpurun_out/g_cublas_$tag python -c "
import torch
a=torch.randn($1,$3,device='cuda').bfloat16(); b=torch.randn($3,$2,device='cuda').bfloat16()
for _ in range(3): c=a@b
torch.cuda.synchronize()" > /dev/null 2>&1
done
ls gpurun_out/*.ncu-rep
