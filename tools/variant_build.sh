#!/bin/bash
# abtest/lib_$1.so: the current sources built with extra nvcc flags (build knobs,
# probes), for same-box A/B runs via POETX_LIB_PATH=abtest/lib_$1.so
#   bash tools/variant_build.sh trace -DPOETX_GEMM_TRACE
set -e
name=$1; shift
root=$(cd "$(dirname "$0")/.." && pwd)
mkdir -p "$root/abtest"
srcs=$(python -c "import sys; sys.path.insert(0, '$root'); from paper_2603_05500_b200.build import SOURCES; print(' '.join(SOURCES))")
files=""
for s in $srcs; do files="$files $root/paper_2603_05500_b200/csrc/$s"; done
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC \
  -Xcompiler -O3 --expt-relaxed-constexpr -shared -cudart static "$@" -o "$root/abtest/lib_$name.so" $files
echo "$root/abtest/lib_$name.so"
