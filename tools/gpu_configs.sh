mkdir -p gpurun_out
timeout 2400 python tools/configs_bench.py --out gpurun_out/configs.jsonl > gpurun_out/configs.log 2>&1
