mkdir -p gpurun_out
timeout 300 ncu --set full --clock-control none --import-source on -k regex:tc2_kernel -s 2 -c 1 -o gpurun_out/gemm_pair python tools/gemmbench.py 8192 5632 2048 0 1 > gpurun_out/ncu_gemm_pair.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:tc_kernel -s 2 -c 1 -o gpurun_out/gemm_1cta python tools/gemmbench.py 8192 5632 2048 0 0 > gpurun_out/ncu_gemm_1cta.log 2>&1
timeout 300 ncu --set full --clock-control none -k regex:nvjet -s 2 -c 1 -o gpurun_out/gemm_cublas python -c "
import torch
a=torch.randn(8192,2048,device='cuda').bfloat16(); b=torch.randn(2048,5632,device='cuda').bfloat16()
for _ in range(3): c=a@b
torch.cuda.synchronize()" > gpurun_out/ncu_gemm_cublas.log 2>&1
