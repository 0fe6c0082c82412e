#!/bin/bash
# Build and run the attention microbenchmark variants (full / loads only / compute only).
set -e
cd "$(dirname "$0")"
NV="nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../include"
$NV attn_bench.cu -o /tmp/attn_full
$NV -DRV_ATTN_NO_MMA attn_bench.cu -o /tmp/attn_load
$NV -DRV_ATTN_NO_LOAD attn_bench.cu -o /tmp/attn_mma
for args in "1440 57" "1440 27" "360 257"; do
  echo "== $args"; /tmp/attn_full $args; /tmp/attn_load $args; /tmp/attn_mma $args
done
