mkdir -p gpurun_out
( for v in ctrace ctrace_o2 ctrace_o3; do echo "## $v"; POETX_LIB_PATH=abtest/lib_$v.so timeout 300 python tools/cnptrace.py 3696 256 | grep "per-warp output\|packed output\|== backward"; done ) > gpurun_out/cnptrace_out.txt 2>&1
cat gpurun_out/cnptrace_out.txt
