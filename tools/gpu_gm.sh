mkdir -p gpurun_out
( for g in 1 2 4 8 1; do echo "GROUP_M=$g"; POETX_GEMM_GROUP_M=$g timeout 300 python tools/microbench.py gemm 2>&1 | grep -E "transB=0" | sed -E 's/ours\(1cta\).*cuBLAS/cuBLAS/'; done
) > gpurun_out/gm.txt 2>&1
