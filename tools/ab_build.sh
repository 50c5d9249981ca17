#!/bin/bash
# build an A/B variant of libchkpcg.so with extra -D flags: tools/ab_build.sh NAME "-DFOO=0 -DBAR=1"
mkdir -p tmp_libs
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -diag-suppress 177 \
  -Xcompiler -fPIC -shared -I include $2 -o tmp_libs/$1.so paper_2007_06524_b200/csrc/chk_capi.cu
