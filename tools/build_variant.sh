#!/bin/bash
# Build a tuning variant of the product library: tools/build_variant.sh <tag> <nvcc -D flags...>
# e.g. tools/build_variant.sh c3 -DTTGBF_CTAS_PER_SM=3  -> paper_2501_07942_b200/_lib/libttgbf_c3.so
# (run with TTGBF_LIB_VARIANT=c3 to load it)
set -e
tag=$1; shift
cd "$(dirname "$0")/.."
TTGBF_LIB_VARIANT=$tag TTGBF_NVCC_FLAGS="$*" python -m paper_2501_07942_b200.build --force
