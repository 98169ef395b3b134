mkdir -p gpurun_out
( timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
  timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
) > gpurun_out/attn_prof.txt 2>&1
