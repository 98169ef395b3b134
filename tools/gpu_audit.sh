mkdir -p gpurun_out
( timeout 600 python -m pytest tests/test_gpu_audit.py tests/test_gpu_parity.py tests/test_gpu_trainer.py -q -m gpu -x 2>&1 | tail -15 ) > gpurun_out/audit_test.txt 2>&1
