#!/bin/bash
# Build libpoetx_b200.so from the csrc/ of git revision $1 into abtest/lib_$2.so
# (for same-box A/B: POETX_LIB_PATH=abtest/lib_$2.so python bench.py ...)
set -e
rev=$1; name=$2
root=$(cd "$(dirname "$0")/.." && pwd)
tmp=$(mktemp -d)
git -C "$root" archive "$rev" paper_2603_05500_b200/csrc include | tar -x -C "$tmp"
mkdir -p "$root/abtest"
srcs=$(python -c "import sys; sys.path.insert(0, '$root'); from paper_2603_05500_b200.build import SOURCES; print(' '.join(SOURCES))")
files=""
for s in $srcs; do [ -f "$tmp/paper_2603_05500_b200/csrc/$s" ] && files="$files $tmp/paper_2603_05500_b200/csrc/$s"; done
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC \
  -Xcompiler -O3 --expt-relaxed-constexpr -shared -cudart static -o "$root/abtest/lib_$name.so" $files
rm -rf "$tmp"
echo "$root/abtest/lib_$name.so"
