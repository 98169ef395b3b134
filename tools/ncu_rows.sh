mkdir -p gpurun_out
for m in 0 1; do
timeout 300 ncu --set full --clock-control none -k regex:swiglu -s 2 -c 1 -o gpurun_out/sw_bwd_$m python tools/rowbench.py swiglu_bwd $m > gpurun_out/ncu_sw_$m.log 2>&1
done
