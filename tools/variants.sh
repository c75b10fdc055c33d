#!/bin/bash
# run the attention perf probe against each variant library in build/variants,
# once per kernel variant in $KINDS (pair / single)
for lib in build/variants/*.so; do
  for kind in ${KINDS:-pair single}; do
    echo "== $lib $kind"
    ZP_ATTN_VARIANT=$kind ZP_LIB_PATH=$PWD/$lib timeout 120 python tools/probe_attn_perf.py 2>&1 | tail -3
  done
done
