# round-2 GPU check: smoke + the whole -m gpu suite (+ optional bench)
set -x
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke rc $?
timeout 1800 python -m pytest tests -q -m gpu --timeout 900 -rf > gpurun_out/gputest.log 2>&1; echo tests rc $?
if [ "${BENCH:-0}" = 1 ]; then timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/bench.log 2>&1; echo bench rc $?; fi
tail -15 gpurun_out/gputest.log
