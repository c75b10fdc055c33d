#!/bin/bash
# build an experimental libzp_b200 variant: tools/build_variant.sh NAME [nvcc -D flags...]
set -e
name=$1; shift
cd "$(dirname "$0")/../paper_2509_21841_b200/csrc"
mkdir -p ../../build/variants
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC \
  -Xcompiler -fvisibility=hidden --use_fast_math -I../../include -shared "$@" \
  zp_attn.cu zp_attn_bwd.cu zp_move.cu zp_comm.cu zp_host.cu zp_block.cu -lcudart -o ../../build/variants/$name.so
