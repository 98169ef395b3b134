mkdir -p gpurun_out
( timeout 1200 compute-sanitizer --tool racecheck --racecheck-report hazard --print-limit 200 \
    python -m pytest tests/test_gpu_tc.py -q -m gpu -k "not 8192 and not 5632" 2>&1 | grep -E "Error|hazard|access at" | sed -E 's/\+0x[0-9a-f]+//' | sort | uniq -c | sort -rn | head -40
) > gpurun_out/racecheck.txt 2>&1
