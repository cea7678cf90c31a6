#!/bin/bash
# Build an A/B variant of libbsra.so with extra -D flags into abtmp/ (git-ignored, travels with
# gpurun):  scripts/build_variant.sh NAME -DFOO=1 ...   -> abtmp/libbsra_NAME.so
set -e
name=$1; shift
mkdir -p abtmp/$name
NVCC=/usr/local/cuda/bin/nvcc
FL="-O3 -lineinfo -std=c++17 -gencode arch=compute_100a,code=sm_100a -Xcompiler -fPIC,-O3 --expt-relaxed-constexpr $@"
$NVCC $FL -c paper_2501_01005_b200/csrc/tc_kernels.cu -o abtmp/$name/tc_kernels.o
$NVCC -gencode arch=compute_100a,code=sm_100a -shared -cudart static -o abtmp/libbsra_$name.so \
  build/engine.o build/scheduler.o abtmp/$name/tc_kernels.o build/dist.o -ldl
echo built abtmp/libbsra_$name.so
