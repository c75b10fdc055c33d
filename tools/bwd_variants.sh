#!/bin/bash
# backward probe against each variant library in build/variants
for lib in build/variants/*.so; do
  echo "== $lib"
  ZP_LIB_PATH=$PWD/$lib timeout 120 python tools/probe_bwd_perf.py 2>&1 | tail -3
done
