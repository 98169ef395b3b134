mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo "rc=$?" >> gpurun_out/gpu_tests.log
timeout 1500 python tools/configs_bench.py --cases 1b-poetxq-mem,8b-poetxq-mem,1b-poetx-mem,8b-poetx-mem --out gpurun_out/configs_q.jsonl > gpurun_out/configs_q.log 2>&1
