#!/bin/bash
# Build a variant of the product library for A/B runs: tools/build_variant.sh out.so [-DMACRO=...]
out=$1; shift
NCCL=$(python -c "import __graft_entry__ as g; print(' '.join(g._nccl_flags()))")
exec /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -fmad=false \
  -Xcompiler -fPIC -shared "$@" -o "$out" paper_2104_01284_b200/csrc/eco_api.cu $NCCL
