mkdir -p gpurun_out
( for i in 1 2 3 4 5; do date +%T; timeout 200 python tools/hangprobe.py llama-8b 1 mem 30 2>&1 | tail -30; echo "rc=$?"; done
) > gpurun_out/hang.txt 2>&1
