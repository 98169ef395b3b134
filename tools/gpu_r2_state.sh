# round-2 re-entry: smoke, the whole -m gpu suite, CNP microbench, bench (fused and unfused CNP)
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke rc $?
timeout 1800 python -m pytest tests -q -m gpu --timeout 900 -rf > gpurun_out/gputest.log 2>&1; echo tests rc $?
timeout 300 python tools/cnpbench.py > gpurun_out/cnpbench.log 2>&1; echo cnpbench rc $?
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/bench.log 2>&1; echo bench rc $?
POETX_CNP_FUSED=0 timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_unfused.log 2>&1; echo bench0 rc $?
tail -15 gpurun_out/gputest.log; cat gpurun_out/cnpbench.log; tail -2 gpurun_out/bench.log gpurun_out/bench_unfused.log
