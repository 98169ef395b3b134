mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo "rc=$?" >> gpurun_out/gpu_tests.log
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench.log 2>&1
timeout 2000 python tools/configs_bench.py --cases 1b-poetx-fast,1b-poetx-mem,8b-poetx-fast,8b-poetx-mem,350m-poetx,60m-poetx --out gpurun_out/configs_v2.jsonl > gpurun_out/configs.log 2>&1
