mkdir -p gpurun_out
for kb in 24 48 96 160; do POETX_ROW_TILE_KB=$kb timeout 300 python tools/microbench.py rows > gpurun_out/mb_rows_$kb.txt 2>&1; done
