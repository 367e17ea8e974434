#!/bin/bash
# Build an experiment variant of libising.so: tools/build_exp.sh NAME [-DFLAG=V ...]
# -> tools/exp_NAME.so (git-ignored; timed by tools/exp_variants.py on the GPU box).
set -e
ROOT=$(cd "$(dirname "$0")/.." && pwd)
NAME=$1; shift
ND=$(python -c "import paper_1906_06297_b200.build as b; print(b.nccl_dir())")
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 \
  -Xcompiler -fPIC -shared "$@" -I "$ND/include" -I "$ROOT/include" \
  "$ROOT"/paper_1906_06297_b200/csrc/ising_kernels.cu "$ROOT"/paper_1906_06297_b200/csrc/ising_basic.cu \
  "$ROOT"/paper_1906_06297_b200/csrc/ising_runtime.cu -L "$ND/lib" -l:libnccl.so.2 \
  -Xlinker -rpath="$ND/lib" -o "$ROOT/tools/exp_$NAME.so"
echo "$ROOT/tools/exp_$NAME.so"
