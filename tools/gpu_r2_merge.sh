# tensor-core merge: parity tests, timing at Llama-1B shapes; fused CNP ncu
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_merge_tc.py tests/test_gpu_bench_config.py -q -m gpu -k "merge" -rf > gpurun_out/merge_tests.log 2>&1; echo tests $?
timeout 300 python tools/mergebench.py > gpurun_out/mergebench.txt 2>&1; echo mb $?
timeout 300 ncu --set full --clock-control none --import-source on -k regex:cnp_fused_kernel -s 0 -c 1 \
  -o gpurun_out/cnp_fused_fwd python tools/cnpbench.py 1024 256 > gpurun_out/ncu_cnp_fwd.log 2>&1; echo ncu fwd $?
timeout 300 ncu --set full --clock-control none --import-source on -k regex:cnp_fused_kernel -s 11 -c 1 \
  -o gpurun_out/cnp_fused_bwd python tools/cnpbench.py 1024 256 > gpurun_out/ncu_cnp_bwd.log 2>&1; echo ncu bwd $?
timeout 300 ncu --set full --clock-control none --import-source on -k regex:merge_tc_kernel -s 1 -c 1 \
  -o gpurun_out/merge_tc python tools/mergebench.py 2048 5632 > gpurun_out/ncu_merge.log 2>&1; echo ncu merge $?
python tools/ncu_summary.py gpurun_out/cnp_fused_fwd.ncu-rep gpurun_out/cnp_fused_bwd.ncu-rep gpurun_out/merge_tc.ncu-rep > gpurun_out/ncu_r2_summary.txt 2>&1
tail -5 gpurun_out/merge_tests.log; cat gpurun_out/mergebench.txt gpurun_out/ncu_r2_summary.txt
