#!/bin/bash
# Build libsj.so variants with extra nvcc defines, in parallel:  tools/variants.sh NAME "-DX=1" NAME2 "-DY=2" ...
cd "$(dirname "$0")/.."
FLAGS=$(python -c "from paper_1803_04120_b200 import build as b; print(' '.join(b.NVCC_FLAGS))")
SRCS=$(python -c "import os; from paper_1803_04120_b200 import build as b; print(' '.join(os.path.join(b.CSRC, f) for f in b.SOURCES))")
mkdir -p build/variants
while [ $# -gt 1 ]; do
  name=$1; defs=$2; shift 2
  /usr/local/cuda/bin/nvcc $FLAGS $defs $SRCS -shared -cudart static -o build/variants/libsj_$name.so &
done
wait
ls -la build/variants
