# fused CNP after the scatter / output rework: ncu (--set full) of both directions + phase traces (new vs round-2 start)
mkdir -p gpurun_out
timeout 300 ncu --set full --clock-control none --import-source on -k regex:cnp_fused_kernel -s 0 -c 1 \
  -o gpurun_out/cnp_fused_fwd2 python tools/cnpbench.py 1024 256 > gpurun_out/ncu_cnp_fwd2.log 2>&1; echo ncu fwd $?
timeout 300 ncu --set full --clock-control none --import-source on -k regex:cnp_fused_kernel -s 11 -c 1 \
  -o gpurun_out/cnp_fused_bwd2 python tools/cnpbench.py 1024 256 > gpurun_out/ncu_cnp_bwd2.log 2>&1; echo ncu bwd $?
python tools/ncu_summary.py gpurun_out/cnp_fused_fwd2.ncu-rep gpurun_out/cnp_fused_bwd2.ncu-rep > gpurun_out/ncu_cnp2_summary.txt 2>&1
( echo "#### current"; POETX_LIB_PATH=abtest/lib_ctrace.so timeout 300 python tools/cnptrace.py 3696 256
  echo "#### round-2 start (per-element scatter, front row copies, branchy output)"; POETX_LIB_PATH=abtest/lib_ctrace_old.so timeout 300 python tools/cnptrace.py 3696 256
  echo "#### cnpbench"; timeout 300 python tools/cnpbench.py; timeout 300 python tools/cnpbench.py 3696 128 ) > gpurun_out/cnp_phases.txt 2>&1
cat gpurun_out/ncu_cnp2_summary.txt
