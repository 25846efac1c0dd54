#!/bin/bash
# Build a variant of liblagsb200.so with extra -D flags (kernel experiments):
#   tools/build_variant.sh NAME -DFOO=1 ...   ->  variants/libNAME.so  (use via LAGS_B200_LIB)
set -e
cd "$(dirname "$0")/.."
name=$1; shift
mkdir -p variants
/usr/local/cuda/bin/nvcc -O3 -std=c++17 -lineinfo -gencode arch=compute_100a,code=sm_100a -Xcompiler -fPIC -shared \
  -ftz=false -prec-div=true -prec-sqrt=true -fmad=false -I include -I paper_1911_08727_b200/csrc "$@" \
  -o variants/lib$name.so paper_1911_08727_b200/csrc/lags_kernels.cu paper_1911_08727_b200/csrc/lags_wire.cu paper_1911_08727_b200/csrc/lags_p2p.cu
