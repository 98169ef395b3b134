# compute-sanitizer memcheck over the round-2 kernels' tests (fused CNP, K9 merge, int8 GEMM, 512x256 pair GEMM)
mkdir -p gpurun_out
( timeout 1500 compute-sanitizer --tool memcheck --error-exitcode 9 --print-limit 20 \
    python -m pytest tests/test_gpu_cnp_fused.py tests/test_gpu_merge_tc.py tests/test_gpu_q8_gemm.py tests/test_gpu_tc.py \
      tests/test_gpu_parity.py tests/test_gpu_quant.py -q -m gpu -k "not 8192 and not 5632 and not trainer" 2>&1 | tail -6
  echo "memcheck rc=$?"
) > gpurun_out/sanitize_r2.txt 2>&1
cat gpurun_out/sanitize_r2.txt
