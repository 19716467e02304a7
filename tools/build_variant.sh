#!/bin/bash
# Build a tuning variant of the product library: tools/build_variant.sh <tag> <nvcc -D flags...>
# e.g. tools/build_variant.sh c3 -DTTGBF_CTAS_PER_SM=3  -> paper_2501_07942_b200/_lib/libttgbf_c3.so
set -e
tag=$1; shift
cd "$(dirname "$0")/../paper_2501_07942_b200/csrc"
lib=../_lib
nvcc -std=c++17 -O3 -gencode arch=compute_100a,code=sm_100a -lineinfo --extended-lambda -Xcompiler -fPIC -Xptxas -v "$@" -c -o $lib/api_$tag.o api.cu > $lib/ptxas_api_$tag.log 2>&1
nvcc -shared -gencode arch=compute_100a,code=sm_100a -o $lib/libttgbf_$tag.so $lib/api_$tag.o $lib/dense.o
echo built $lib/libttgbf_$tag.so
