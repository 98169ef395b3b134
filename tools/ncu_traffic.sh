mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none -k regex:tc2_kernel -o gpurun_out/gemm_shapes python tools/gemm_shapes.py > gpurun_out/ncu_gemm_shapes.log 2>&1
