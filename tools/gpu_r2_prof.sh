# round-2 evidence: fused CNP ncu (full set), GEMM microbench, graph step breakdown
mkdir -p gpurun_out
timeout 300 ncu --set full --clock-control none --import-source on -k regex:cnp_fwd_fused -s 1 -c 1 \
  -o gpurun_out/cnp_fused_fwd python tools/cnpbench.py 1024 256 > gpurun_out/ncu_cnp_fwd.log 2>&1; echo ncu fwd $?
timeout 300 ncu --set full --clock-control none --import-source on -k regex:cnp_bwd_fused -s 1 -c 1 \
  -o gpurun_out/cnp_fused_bwd python tools/cnpbench.py 1024 256 > gpurun_out/ncu_cnp_bwd.log 2>&1; echo ncu bwd $?
timeout 300 python tools/microbench.py gemm > gpurun_out/microbench_gemm.txt 2>&1; echo mb $?
timeout 600 python tools/profile_step.py --graph --timeline > gpurun_out/step_breakdown_graph.txt 2>&1; echo prof $?
python tools/ncu_summary.py gpurun_out/cnp_fused_fwd.ncu-rep gpurun_out/cnp_fused_bwd.ncu-rep > gpurun_out/ncu_cnp_fused.txt 2>&1
cat gpurun_out/ncu_cnp_fused.txt gpurun_out/microbench_gemm.txt; head -30 gpurun_out/step_breakdown_graph.txt
