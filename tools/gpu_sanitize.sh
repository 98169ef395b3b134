# compute-sanitizer over the small-shape GPU tests (profiles/r01/sanitizer.md)
mkdir -p gpurun_out
( timeout 1500 compute-sanitizer --tool memcheck --error-exitcode 9 --print-limit 20 \
    python -m pytest tests/test_gpu_parity.py tests/test_gpu_audit.py tests/test_gpu_tc.py tests/test_gpu_rowops.py \
      tests/test_gpu_quant.py tests/test_gpu_attention.py tests/test_gpu_trainer.py -q -m gpu -k "not 8192 and not 5632" 2>&1 | tail -6
  echo "memcheck rc=$?"
  timeout 1200 compute-sanitizer --tool racecheck --racecheck-report hazard --print-limit 200 \
    python -m pytest tests/test_gpu_tc.py -q -m gpu -k "not 8192 and not 5632" 2>&1 \
    | grep -E "Error|hazard|access at" | sed -E 's/\+0x[0-9a-f]+//' | sort | uniq -c | sort -rn | head -40
) > gpurun_out/sanitize.txt 2>&1
