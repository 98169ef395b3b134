# fused CNP wired into the trainer and the bf16 layer API: parity + timing
set -x
timeout 900 python -m pytest tests -q -m gpu --timeout 600 -x -k "cnp_fused or bench_config or bf16 or trainer or dropin or tc" > gpurun_out/gputest_fused.log 2>&1; echo tests rc $?
python tools/cnpbench.py > gpurun_out/cnpbench.log 2>&1; echo cnpbench rc $?
POETX_CNP_FUSED=0 timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_unfused.log 2>&1; echo bench0 rc $?
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_fused.log 2>&1; echo bench1 rc $?
tail -5 gpurun_out/gputest_fused.log; cat gpurun_out/cnpbench.log
