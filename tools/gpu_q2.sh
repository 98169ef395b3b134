mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_quant.py -x -q > gpurun_out/quant.log 2>&1; echo "rc=$?" >> gpurun_out/quant.log
timeout 1500 python tools/configs_bench.py --cases 1b-poetxq-mem,8b-poetxq-mem --out gpurun_out/configs_q.jsonl > gpurun_out/configs_q.log 2>&1
